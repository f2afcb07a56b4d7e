"""Register-blocked potential kernel vs the tile kernel (HB_POT_TILES) on a
config-4 sample: max relative difference and timings of both forms."""
import json, os, sys
import numpy as np
import torch
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import paper_2102_09811_b200 as hb
from paper_2102_09811_b200.field import _eval_grouped

M = int(os.environ.get("NPTS", "2000"))
m = hb.unit_cube_mesh(4); tg = hb.TimeGrid(1.0, 64); p = hb.KernelParams(1.0, tg.step, length_scale=m.diameter)
rng = np.random.default_rng(0)
q = rng.uniform(-1, 1, (64, m.n_triangles)); g = rng.uniform(-1, 1, (64, m.n_vertices))
X = rng.uniform(0.05, 0.95, (100000, 3))[:M]
K = np.tile(np.arange(1, 65), M); XX = np.repeat(X, 64, axis=0)
eps = np.zeros(M * 64); cur = np.zeros(M * 64, bool)
out = {"points": M}
for mode in ("reg", "tiles"):
    if mode == "tiles":
        os.environ["HB_POT_TILES"] = "1"
    res = {}
    for kind, coef in ((0, q), (1, g)):
        _eval_grouped(kind, coef, XX[:64 * 64], K[:64 * 64], eps[:64 * 64], cur[:64 * 64], m, tg, p, hb.QuadratureConfig())
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); v = _eval_grouped(kind, coef, XX, K, eps, cur, m, tg, p, hb.QuadratureConfig()); e.record()
        torch.cuda.synchronize()
        res[kind] = (s.elapsed_time(e), v.cpu().numpy())
    out[mode] = res
for kind in (0, 1):
    a, b = out["reg"][kind][1], out["tiles"][kind][1]
    out[f"maxrel_{kind}"] = float(np.abs(a - b).max() / np.abs(b).max())
    out[f"ms_reg_{kind}"] = out["reg"][kind][0]
    out[f"ms_tiles_{kind}"] = out["tiles"][kind][0]
del out["reg"], out["tiles"]
out["full_c4_s_reg"] = (out["ms_reg_0"] + out["ms_reg_1"]) * 1e-3 * 100000 / M
print(json.dumps(out))
