"""Config-5 D phases for one 32-block chunk: V pair/finalize, D2 pair/finalize,
curl combine (CUDA events), at a given staging workspace."""
import json, os, sys
import torch
R = os.environ.get("GRAFT_REPO_ROOT", "/root/repo"); sys.path.insert(0, R)
import paper_2102_09811_b200 as hb
from paper_2102_09811_b200 import device as hbdev
from paper_2102_09811_b200.assembly import _assemble_operator, curl_combine_into
from paper_2102_09811_b200._native import AssemblyStats
m = hb.unit_cube_mesh(int(os.environ.get("LEVEL", "5")))
tg = hb.TimeGrid(1.0, 256); p = hb.KernelParams(1.0, tg.step, length_scale=m.diameter); q = hb.QuadratureConfig()
tabs = hbdev.device_tables(m, q)
CH = 32; E, N = m.n_triangles, m.n_vertices
ws = int(float(os.environ.get("WS_GB", "4")) * (1 << 30))
bufV = torch.empty((CH, E, E), dtype=torch.float64, device="cuda")
bufD = torch.empty((CH, N, N), dtype=torch.float64, device="cuda")
res = {}
for d0 in (32,):   # a regular window (no singular-in-time gaps)
    for it in range(2):
        stV, stD = AssemblyStats(), AssemblyStats()
        _assemble_operator(0, False, False, True, m, tg, p, q, None, d_range=(d0, d0 + CH), out=bufV, stats=stV, workspace_bytes=ws)
        _assemble_operator(2, True, True, True, m, tg, p, q, None, d_range=(d0, d0 + CH), out=bufD, stats=stD, workspace_bytes=ws)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); s.record()
        curl_combine_into(tabs, bufV, bufD, bufD, p.alpha, workspace_cap=int(float(os.environ.get("CURL_GB", "1")) * (1 << 30)))
        e.record(); torch.cuda.synchronize()
        res = {"V_pair": stV.pair_ms, "V_fin": stV.finalize_ms, "D2_pair": stD.pair_ms, "D2_fin": stD.finalize_ms,
               "D2_launches": stD.launches, "curl": s.elapsed_time(e)}
print(json.dumps(res))
