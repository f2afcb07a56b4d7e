"""One pair-kernel launch per case for ncu: c2 V (all blocks) and one late
c5 V window (d in [128, 158): moment blocks for nearly every pair)."""
import os, sys
import torch
R = os.environ.get("GRAFT_REPO_ROOT", "/root/repo"); sys.path.insert(0, R)
import paper_2102_09811_b200 as hb
from paper_2102_09811_b200.assembly import _assemble_operator
case = os.environ.get("CASE", "c2V")
q = hb.QuadratureConfig()
if case.startswith("c2"):
    m, tg = hb.unit_cube_mesh(3), hb.TimeGrid(1.0, 32)
    dr = (0, 32)
else:
    m, tg = hb.unit_cube_mesh(5), hb.TimeGrid(1.0, 256)
    d0 = int(os.environ.get("D0", "128")); dr = (d0, d0 + 30)
p = hb.KernelParams(1.0, tg.step, length_scale=m.diameter)
op = {"V": (0, False, False, True), "K": (1, False, True, False), "D": (2, True, True, True)}[case[-1]]
out = torch.empty((dr[1] - dr[0], m.n_triangles if not op[1] else m.n_vertices,
                   m.n_vertices if op[2] else m.n_triangles), dtype=torch.float64, device="cuda")
for _ in range(2):
    _assemble_operator(*op, m, tg, p, q, None, d_range=dr, out=out)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record(); _assemble_operator(*op, m, tg, p, q, None, d_range=dr, out=out); e.record(); torch.cuda.synchronize()
print(case, dr, "ms", s.elapsed_time(e))
