"""D2 / V11 pair-kernel time at config 2 (stats)."""
import json, os, sys
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import paper_2102_09811_b200 as hb
from paper_2102_09811_b200.assembly import _assemble_operator
from paper_2102_09811_b200._native import AssemblyStats
m = hb.unit_cube_mesh(3); tg = hb.TimeGrid(1.0, 32); p = hb.KernelParams(1.0, tg.step, length_scale=m.diameter); q = hb.QuadratureConfig()
res = {}
for name, code in (("D2", (2, True, True, True)), ("V11", (0, True, True, True)), ("V", (0, False, False, True))):
    for _ in range(2): _assemble_operator(*code, m, tg, p, q, None)
    st = AssemblyStats()
    for _ in range(5): _assemble_operator(*code, m, tg, p, q, None, stats=st)
    res[name] = round(st.pair_ms / 5, 3)
print(json.dumps({"lib": os.environ.get("HB_LIB_PATH", "default"), **res}))
