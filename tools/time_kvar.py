"""K pair time at config 2, level 4 / E_t 64 and a config-5 chunk for the current env (HB_MOMENTS etc.)."""
import json, os, sys, torch
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import paper_2102_09811_b200 as hb
from paper_2102_09811_b200.assembly import _assemble_operator
from paper_2102_09811_b200._native import AssemblyStats
res = {"env": {k: os.environ.get(k) for k in ("HB_MOMENTS", "HB_K_FAR_BATCH")}}
for name, lvl, Et, dr in (("c2", 3, 32, None), ("l4", 4, 64, None), ("c5_30", 5, 256, (32, 62))):
    m = hb.unit_cube_mesh(lvl); tg = hb.TimeGrid(1.0, Et); p = hb.KernelParams(1.0, tg.step, length_scale=m.diameter)
    q = hb.QuadratureConfig()
    d0, d1 = dr or (0, Et)
    out = torch.empty((d1 - d0, m.n_triangles, m.n_vertices), dtype=torch.float64, device="cuda")
    f = lambda st=None: _assemble_operator(1, False, True, False, m, tg, p, q, None, d_range=(d0, d1), out=out, stats=st)
    f(); torch.cuda.synchronize()
    st = AssemblyStats(); f(st)
    res[name] = {"pair_ms": round(st.pair_ms, 3), "fin_ms": round(st.finalize_ms, 3)}
    del out; torch.cuda.empty_cache()
print(json.dumps(res))
