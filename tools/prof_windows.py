"""Pair-kernel cost of one NJ=2 window (30 blocks) vs one NJ=1 window
(14 blocks) at config 5, per operator."""
import json, os, sys
import torch
R = os.environ.get("GRAFT_REPO_ROOT", "/root/repo"); sys.path.insert(0, R)
import paper_2102_09811_b200 as hb
from paper_2102_09811_b200.assembly import _assemble_operator
from paper_2102_09811_b200._native import AssemblyStats
m = hb.unit_cube_mesh(int(os.environ.get("LEVEL", "5")))
tg = hb.TimeGrid(1.0, 256); p = hb.KernelParams(1.0, tg.step, length_scale=m.diameter); q = hb.QuadratureConfig()
E, N = m.n_triangles, m.n_vertices
ops = {"V": (0, False, False, True, (E, E)), "K": (1, False, True, False, (E, N)), "D2": (2, True, True, True, (N, N))}
res = {}
for name, (op, tp, sp, sym, shp) in ops.items():
    buf = torch.empty((30,) + shp, dtype=torch.float64, device="cuda")
    for rng in ((32, 62), (62, 76), (62, 64)):
        for it in range(2):
            st = AssemblyStats()
            _assemble_operator(op, tp, sp, sym, m, tg, p, q, None, d_range=rng, out=buf[: rng[1] - rng[0]], stats=st,
                               workspace_bytes=40 << 30)
        res[f"{name}_{rng[0]}_{rng[1]}"] = round(st.pair_ms, 2)
    del buf
print(json.dumps(res))
