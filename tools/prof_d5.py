"""D2 on one config-5 chunk, twice: for an ncu launch list."""
import os, sys, torch
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import paper_2102_09811_b200 as hb
from paper_2102_09811_b200.assembly import _assemble_operator
m = hb.unit_cube_mesh(5); tg = hb.TimeGrid(1.0, 256); p = hb.KernelParams(1.0, tg.step, length_scale=m.diameter)
q = hb.QuadratureConfig()
d0, d1 = int(os.environ.get("D0", "0")), int(os.environ.get("D1", "64"))
out = torch.empty((d1 - d0, m.n_vertices, m.n_vertices), dtype=torch.float64, device="cuda")
for _ in range(2):
    _assemble_operator(2, True, True, True, m, tg, p, q, None, d_range=(d0, d1), out=out)
torch.cuda.synchronize()
print("ok")
