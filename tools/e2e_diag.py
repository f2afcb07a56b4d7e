"""e2e overhead breakdown at config 2: D2H bandwidth, and the public-API step
with / without the per-step table re-upload and host copies."""
import json, os, sys, torch
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import paper_2102_09811_b200 as hb
from paper_2102_09811_b200 import device as hbdev
m = hb.unit_cube_mesh(3); tg = hb.TimeGrid(1.0, 32); p = hb.KernelParams(1.0, tg.step, length_scale=m.diameter)
q = hb.QuadratureConfig()
res = {}
x = torch.empty(151 << 20, dtype=torch.uint8, device="cuda"); h = torch.empty(x.shape, dtype=torch.uint8).pin_memory()
for _ in range(3): h.copy_(x, non_blocking=True)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record(); h.copy_(x, non_blocking=True); e.record(); torch.cuda.synchronize()
res["d2h_GBps"] = x.numel() / (s.elapsed_time(e) * 1e6)
hbdev.pin_host_tables(hbdev.host_tables(m, q))
pins = {}
def step(drop, copy):
    if drop: hbdev.drop_device_tables(m)
    V = hb.assemble_single_layer(m, tg, p, q)
    evs = []
    if copy: evs.append(V.to_host_async(pins.setdefault("V", torch.empty(V.device_blocks.shape, dtype=torch.float64).pin_memory()))[1])
    K = hb.assemble_double_layer(m, tg, p, q)
    if copy: evs.append(K.to_host_async(pins.setdefault("K", torch.empty(K.device_blocks.shape, dtype=torch.float64).pin_memory()))[1])
    if copy:
        pd = pins.setdefault("D", torch.empty((32, m.n_vertices, m.n_vertices), dtype=torch.float64).pin_memory())
        D = hb.assemble_hypersingular(m, tg, p, q, single_layer=V, host_out=pd); evs.append(D.host_copy[1])
    else:
        D = hb.assemble_hypersingular(m, tg, p, q, single_layer=V)
    for ev in evs: torch.cuda.current_stream().wait_event(ev)
for name, drop, copy in (("api_only", False, False), ("api_drop", True, False), ("api_copy", False, True), ("api_drop_copy", True, True)):
    for _ in range(3): step(drop, copy)
    torch.cuda.synchronize()
    ts = []
    for _ in range(20):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); step(drop, copy); e.record(); e.synchronize(); ts.append(s.elapsed_time(e))
    res[name + "_ms"] = sorted(ts)[len(ts) // 2]
print(json.dumps(res))
