"""Time represent_grid (u = V~q - Wg at M config-4 points x 64 times) through
the public call; NPTS points (default all 1e5)."""
import json, os, sys
import numpy as np
import torch
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import paper_2102_09811_b200 as hb

M = int(os.environ.get("NPTS", "100000"))
m = hb.unit_cube_mesh(4); tg = hb.TimeGrid(1.0, 64); p = hb.KernelParams(1.0, tg.step, length_scale=m.diameter)
rng = np.random.default_rng(0)
q = rng.uniform(-1, 1, (64, m.n_triangles)); g = rng.uniform(-1, 1, (64, m.n_vertices))
X = rng.uniform(0.05, 0.95, (100000, 3))[:M]
hb.represent_grid(q, g, X[:256], m, tg, p, return_device=True)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record(); u = hb.represent_grid(q, g, X, m, tg, p, return_device=True); e.record(); torch.cuda.synchronize()
t = s.elapsed_time(e) * 1e-3
print(json.dumps({"points": M, "s": t, "values_per_s": M * 64 / t, "full_c4_s": t * 100000 / M,
                  "checksum": float(u.abs().sum()), "lib": os.environ.get("HB_LIB_PATH", "default")}))
