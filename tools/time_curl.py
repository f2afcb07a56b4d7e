"""Curl-combine device time at config 2 and on a 32-block config-5 chunk."""
import json, os, sys, torch
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import paper_2102_09811_b200 as hb
from paper_2102_09811_b200 import device as hbdev
from paper_2102_09811_b200.assembly import curl_combine_into
res = {}
for name, lvl, Et, nb in (("c2", 3, 32, 32), ("c5", 5, 256, 32)):
    m = hb.unit_cube_mesh(lvl); tg = hb.TimeGrid(1.0, Et); q = hb.QuadratureConfig()
    tabs = hbdev.device_tables(m, q)
    E, N = m.n_triangles, m.n_vertices
    g = torch.Generator(device="cuda"); g.manual_seed(0)
    V = torch.rand((nb, E, E), dtype=torch.float64, device="cuda", generator=g)
    D2 = torch.rand((nb, N, N), dtype=torch.float64, device="cuda", generator=g)
    out = torch.empty_like(D2)
    for _ in range(2): curl_combine_into(tabs, V, D2, out, 1.0)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); s.record(); curl_combine_into(tabs, V, D2, out, 1.0); e.record(); torch.cuda.synchronize()
    ms = s.elapsed_time(e)
    res[name] = {"ms": round(ms, 3), "V_GBps": round(V.numel() * 8 / ms / 1e6, 1)}
    del V, D2, out; torch.cuda.empty_cache()
print(json.dumps(res))
