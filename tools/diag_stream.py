import sys, torch, numpy as np, json
sys.path.insert(0, "/root/repo")
import paper_2102_09811_b200 as hb
from paper_2102_09811_b200 import _native
m = hb.unit_cube_mesh(3); tg = hb.TimeGrid(1.0, 32); p = hb.KernelParams(1.0, tg.step, length_scale=m.diameter)
def ev(f, n=5):
    f(); torch.cuda.synchronize()
    ts=[]
    for _ in range(n):
        s,e=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
        s.record(); f(); e.record(); torch.cuda.synchronize(); ts.append(s.elapsed_time(e))
    return min(ts)
out = torch.empty((32,768,768), dtype=torch.float64, device="cuda")
pin = torch.empty((32,768,768), dtype=torch.float64).pin_memory()
r = {}
r["V_one_call"] = ev(lambda: hb.assemble_single_layer(m, tg, p, out=out))
from paper_2102_09811_b200.assembly import _row_slabs, _assemble_operator
def slabs():
    for a,b in _row_slabs(768, True, 4):
        _assemble_operator(0, False, False, True, m, tg, p, hb.QuadratureConfig(), None, row_range=(a,b), out=out)
r["V_4_slabs"] = ev(slabs)
r["copy_full_V"] = ev(lambda: pin.copy_(out, non_blocking=True))
def c2d():
    for a,b in _row_slabs(768, True, 4):
        _native.call("hb_copy_row_slab_d2h", _native.ptr(pin), _native.ptr(out), 32, 768, 768, a, b, _native.stream_handle())
r["copy_4_slabs_2d"] = ev(c2d)
r["V_streamed_total"] = ev(lambda: hb.assemble_single_layer(m, tg, p, out=out, host_out=pin).host_copy[1].synchronize())
print(json.dumps(r))
