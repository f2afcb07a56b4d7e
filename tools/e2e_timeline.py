"""Timeline of bench.py's e2e step at config 2: when each operator's compute
ends and when each device->host copy starts / ends (events on the compute
and copy streams), plus the raw D2H bandwidth of one 265 MB copy."""
import json, os, sys, torch
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import paper_2102_09811_b200 as hb
from paper_2102_09811_b200 import device as hbdev
from paper_2102_09811_b200 import assembly as A
m = hb.unit_cube_mesh(3); tg = hb.TimeGrid(1.0, 32); p = hb.KernelParams(1.0, tg.step, length_scale=m.diameter)
q = hb.QuadratureConfig()
E, N = m.n_triangles, m.n_vertices
res = {}
x = torch.empty(265 << 20, dtype=torch.uint8, device="cuda"); h = torch.empty(x.shape, dtype=torch.uint8).pin_memory()
for _ in range(3): h.copy_(x, non_blocking=True)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record(); h.copy_(x, non_blocking=True); e.record(); torch.cuda.synchronize()
res["d2h_GBps_265MB"] = x.numel() / (s.elapsed_time(e) * 1e6)
del x, h
Hpin = hbdev.pin_host_tables(hbdev.host_tables(m, q))
pinV = torch.empty((32, E, E), dtype=torch.float64).pin_memory()
pinK = torch.empty((32, E, N), dtype=torch.float64).pin_memory()
pinD = torch.empty((32, N, N), dtype=torch.float64).pin_memory()
_sl = os.environ.get("HB_E2E_SLABS", "2")
slabs = [float(x) for x in _sl.split(",")] if "," in _sl else int(_sl)
def step(marks):
    cur = torch.cuda.current_stream()
    def mark(name):
        ev = torch.cuda.Event(enable_timing=True); ev.record(cur); marks.append((name, ev))
    mark("start")
    hbdev.drop_device_tables(m)
    V = hb.assemble_single_layer(m, tg, p, q, host_out=pinV, host_out_slabs=slabs)
    mark("V_done"); _, ev_v = V.host_copy
    K = hb.assemble_double_layer(m, tg, p, q, host_out=pinK)
    mark("K_done"); _, ev_k = K.host_copy
    D = hb.assemble_hypersingular(m, tg, p, q, single_layer=V, host_out=pinD)
    mark("D_done"); _, ev_d = D.host_copy
    for nm, ev in (("V_copied", ev_v), ("K_copied", ev_k), ("D_copied", ev_d)):
        e2 = torch.cuda.Event(enable_timing=True); cur.wait_event(ev); e2.record(cur); marks.append((nm, e2))
for _ in range(3): step([])
torch.cuda.synchronize()
runs = []
for _ in range(5):
    marks = []
    step(marks); torch.cuda.synchronize()
    t0 = marks[0][1]
    runs.append({nm: round(t0.elapsed_time(ev), 3) for nm, ev in marks[1:]})
res["timeline_ms"] = runs
print(json.dumps(res))
# ---- assemble_all(host_out=...) ----
def step_all(marks):
    cur = torch.cuda.current_stream()
    ev0 = torch.cuda.Event(enable_timing=True); ev0.record(cur); marks.append(("start", ev0))
    hbdev.drop_device_tables(m)
    ops = hb.assemble_all(m, tg, p, q, host_out={"V": pinV, "K": pinK, "D": pinD}, v_slabs=slabs)
    sD, sV, sK = A._op_streams(torch.device("cuda", 0))
    for nm, st in (("Vstream_done", sV), ("Kstream_done", sK), ("Dstream_done", sD)):
        e2 = torch.cuda.Event(enable_timing=True); e2.record(st); marks.append((nm, e2))
    for nm in ("V", "K", "D"):
        ev = ops[nm].host_copy[1]
        e2 = torch.cuda.Event(enable_timing=True); cur.wait_event(ev); e2.record(cur); marks.append((nm + "_copied", e2))
for _ in range(3): step_all([])
torch.cuda.synchronize()
runs = []
for _ in range(3):
    marks = []
    step_all(marks); torch.cuda.synchronize()
    t0 = marks[0][1]
    runs.append({nm: round(t0.elapsed_time(ev), 3) for nm, ev in marks[1:]})
print(json.dumps({"all_timeline_ms": runs}))
