"""Curl combine (k_curl_tile) device time at config 2 (32 blocks) and on a config-5 16-block chunk."""
import json, os, sys, torch
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import paper_2102_09811_b200 as hb
from paper_2102_09811_b200 import device as hbdev
from paper_2102_09811_b200.assembly import _assemble_operator, curl_combine_into
q = hb.QuadratureConfig(); res = {"lib": os.environ.get("HB_LIB_PATH", "default")}
for name, lvl, Et, nb in (("c2", 3, 32, 32), ("c5_16", 5, 256, 16)):
    m = hb.unit_cube_mesh(lvl); tg = hb.TimeGrid(1.0, Et); p = hb.KernelParams(1.0, tg.step, length_scale=m.diameter)
    tabs = hbdev.device_tables(m, q)
    V = _assemble_operator(0, False, False, True, m, tg, p, q, None, d_range=(32 if Et > 32 else 0, (32 if Et > 32 else 0) + nb))
    D2 = _assemble_operator(2, True, True, True, m, tg, p, q, None, d_range=(32 if Et > 32 else 0, (32 if Et > 32 else 0) + nb))
    out = torch.empty_like(D2)
    for _ in range(2): curl_combine_into(tabs, V, D2, out, p.alpha)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(3): curl_combine_into(tabs, V, D2, out, p.alpha)
    e.record(); torch.cuda.synchronize()
    res[name + "_ms"] = s.elapsed_time(e) / 3
    res[name + "_checksum"] = float(out.double().abs().sum())
    del V, D2, out; torch.cuda.empty_cache()
print(json.dumps(res))
