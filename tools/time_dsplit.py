"""Per-operator pair time on config-5 block ranges with the current HB_MOMENTS
(decides where a direct / moment switch at a block index pays)."""
import json, os, sys, torch
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import paper_2102_09811_b200 as hb
from paper_2102_09811_b200.assembly import _assemble_operator
from paper_2102_09811_b200._native import AssemblyStats
m = hb.unit_cube_mesh(int(os.environ.get("LVL", "5"))); Et = int(os.environ.get("ET", "256"))
tg = hb.TimeGrid(1.0, Et); p = hb.KernelParams(1.0, tg.step, length_scale=m.diameter); q = hb.QuadratureConfig()
E, N = m.n_triangles, m.n_vertices
res = {"HB_MOMENTS": os.environ.get("HB_MOMENTS")}
for op, code, C in (("V", (0, False, False, True), E), ("D2", (2, True, True, True), N), ("K", (1, False, True, False), N)):
    R = N if op == "D2" else E
    for d0, d1 in ((0, 32), (32, 62), (62, 92)):
        out = torch.empty((d1 - d0, R, C), dtype=torch.float64, device="cuda")
        st = AssemblyStats()
        _assemble_operator(*code, m, tg, p, q, None, d_range=(d0, d1), out=out)
        torch.cuda.synchronize()
        _assemble_operator(*code, m, tg, p, q, None, d_range=(d0, d1), out=out, stats=st)
        res[f"{op}_{d0}_{d1}"] = (round(st.pair_ms, 1), round(st.finalize_ms, 1))
        del out; torch.cuda.empty_cache()
print(json.dumps(res))
