"""represent_grid at E_t = 64 (fused per-element kernel) vs E_t = 128 / 256 (general
path): values/s and kernel evaluations/s on a level-4 cube, NPTS points."""
import json, os, sys
import numpy as np
import torch
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import paper_2102_09811_b200 as hb

M = int(os.environ.get("NPTS", "4000"))
m = hb.unit_cube_mesh(4)
rng = np.random.default_rng(0)
X = rng.uniform(0.05, 0.95, (M, 3))
res = {}
for Et in (64, 128, 256):
    tg = hb.TimeGrid(1.0, Et); p = hb.KernelParams(1.0, tg.step, length_scale=m.diameter)
    q = rng.uniform(-1, 1, (Et, m.n_triangles)); g = rng.uniform(-1, 1, (Et, m.n_vertices))
    hb.represent_grid(q, g, X[:128], m, tg, p, return_device=True)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(); u = hb.represent_grid(q, g, X, m, tg, p, return_device=True); e.record(); torch.cuda.synchronize()
    t = s.elapsed_time(e) * 1e-3
    res[Et] = {"s": round(t, 4), "values_per_s": M * Et / t, "pair_gap_evals_per_s": M * Et * m.n_vertices / t}
print(json.dumps(res))
