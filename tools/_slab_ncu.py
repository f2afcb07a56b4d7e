import os, sys, torch
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import paper_2102_09811_b200 as hb
from paper_2102_09811_b200.assembly import _assemble_operator, _row_slabs
m = hb.unit_cube_mesh(3); tg = hb.TimeGrid(1.0, 32); p = hb.KernelParams(1.0, tg.step, length_scale=m.diameter)
q = hb.QuadratureConfig(); E = m.n_triangles
out = torch.empty((32, E, E), dtype=torch.float64, device="cuda")
for it in range(2):
    for r0, r1 in _row_slabs(E, True, 8):
        _assemble_operator(0, False, False, True, m, tg, p, q, None, row_range=(r0, r1), out=out)
    torch.cuda.synchronize()
