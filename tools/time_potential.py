"""Time the config-4 representation formula on a subset of the 1e5 points."""
import os, sys, time, json, numpy as np, torch
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import paper_2102_09811_b200 as hb
from paper_2102_09811_b200.field import _eval_grouped
M = int(os.environ.get("NPTS", "2000"))
m = hb.unit_cube_mesh(4); tg = hb.TimeGrid(1.0, 64); p = hb.KernelParams(1.0, tg.step, length_scale=m.diameter)
rng = np.random.default_rng(0)
q = rng.uniform(-1, 1, (64, m.n_triangles)); g = rng.uniform(-1, 1, (64, m.n_vertices)); X = rng.uniform(0.05, 0.95, (100000, 3))
xs = X[:M]
ks = np.arange(1, 65)
XX = np.repeat(xs, 64, axis=0); K = np.tile(ks, M); eps = np.zeros(M * 64); cur = np.zeros(M * 64, bool)
res = {}
for kind, coef in ((0, q), (1, g)):
    _eval_grouped(kind, coef, XX[:64 * 8], K[:64 * 8], eps[:64 * 8], cur[:64 * 8], m, tg, p, hb.QuadratureConfig())
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(); v = _eval_grouped(kind, coef, XX, K, eps, cur, m, tg, p, hb.QuadratureConfig()); e.record(); torch.cuda.synchronize()
    res[kind] = s.elapsed_time(e)
vals = M * 64
print(json.dumps({"points": M, "values": vals, "ms_single": res[0], "ms_double": res[1],
                  "values_per_s": vals / ((res[0] + res[1]) * 1e-3),
                  "full_c4_s_extrapolated": (res[0] + res[1]) * 1e-3 * 100000 / M}))
