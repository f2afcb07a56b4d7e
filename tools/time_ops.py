"""Per-operator device timing (CUDA events) at a BASELINE config + FP64 probe."""
import os, sys, json, numpy as np, torch
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import paper_2102_09811_b200 as hb
from paper_2102_09811_b200 import _native
from paper_2102_09811_b200.assembly import _assemble_operator
lvl = int(os.environ.get("LVL", "3")); Et = int(os.environ.get("ET", "32"))
mesh = hb.unit_cube_mesh(lvl); tg = hb.TimeGrid(1.0, Et); p = hb.KernelParams(1.0, tg.step, length_scale=mesh.diameter)
q = hb.QuadratureConfig()
ops = {"V": (0, False, False, True), "K": (1, False, True, False), "D2": (2, True, True, True)}
res = {}
for name, (op, tp, sp, sym) in ops.items():
    for _ in range(2): _assemble_operator(op, tp, sp, sym, mesh, tg, p, q, None)
    torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); B = _assemble_operator(op, tp, sp, sym, mesh, tg, p, q, None); e.record(); torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    res[name] = min(ts)
    from paper_2102_09811_b200._native import AssemblyStats
    st = AssemblyStats()
    _assemble_operator(op, tp, sp, sym, mesh, tg, p, q, None, stats=st)
    res[name + "_pair"] = round(st.pair_ms, 3)
    res[name + "_fin"] = round(st.finalize_ms, 3)
sink = torch.zeros(148*8, dtype=torch.float64, device="cuda")
grid, iters = 148*8, 20000
for _ in range(2): _native.call("hb_fp64_probe", grid, iters, _native.ptr(sink), _native.stream_handle())
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record(); _native.call("hb_fp64_probe", grid, iters, _native.ptr(sink), _native.stream_handle()); e.record(); torch.cuda.synchronize()
tf = grid*256*iters*8*2/(s.elapsed_time(e)*1e-3)/1e12
print(json.dumps({"lib": os.environ.get("HB_LIB_PATH", "default"), "ms": res, "fp64_tflops": round(tf, 2)}))
# curl combine (D = D2 + a^2 curl(V)) at this config
from paper_2102_09811_b200 import device as hbdev
from paper_2102_09811_b200.assembly import curl_combine_into
tabs = hbdev.device_tables(mesh, q)
Vb = _assemble_operator(0, False, False, True, mesh, tg, p, q, None)
D2b = _assemble_operator(2, True, True, True, mesh, tg, p, q, None)
out = torch.empty_like(D2b)
for _ in range(2): curl_combine_into(tabs, Vb, D2b, out, p.alpha)
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize(); s.record(); curl_combine_into(tabs, Vb, D2b, out, p.alpha); e.record(); torch.cuda.synchronize()
print(json.dumps({"curl_ms": s.elapsed_time(e)}))
