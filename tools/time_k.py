"""K pair timing at c2 (two class launches), for A/B library variants (HB_LIB_PATH)."""
import os, sys, torch
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import paper_2102_09811_b200 as hb
from paper_2102_09811_b200.assembly import _assemble_operator
from paper_2102_09811_b200._native import AssemblyStats
m = hb.unit_cube_mesh(3); tg = hb.TimeGrid(1.0, 32); p = hb.KernelParams(1.0, tg.step, length_scale=m.diameter)
q = hb.QuadratureConfig()
op = os.environ.get("OPK", "K")
args = {"V": (0, False, False, True), "K": (1, False, True, False), "D2": (2, True, True, True)}[op]
for _ in range(2): _assemble_operator(*args, m, tg, p, q, None)
st = AssemblyStats()
for _ in range(3): _assemble_operator(*args, m, tg, p, q, None, stats=st)
print(os.environ.get("HB_LIB_PATH", "lib/default/x").split("/")[-2], op, "pair_ms", st.pair_ms / 3)
