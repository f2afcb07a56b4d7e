"""Per-rank work of bench.py --gpus N (config 2, --parallel rows), timed one
rank at a time on one B200: V and K pair work on the rank's balanced test-row
range over all blocks (stores into one buffer standing in for the d-owners'
shards), D2 on the rank's d-range, the curl of its d-range -- sequential on one
stream ("seq") and on three streams as bench.py runs them ("conc").  The max
over ranks projects the N-GPU step (the peer stores overlap the pair
kernels; the barrier is not timed)."""
import json, os, sys, torch
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import paper_2102_09811_b200 as hb
from paper_2102_09811_b200 import device as hbdev, distributed as D
from paper_2102_09811_b200.assembly import _assemble_operator, curl_combine_into, _op_streams
m = hb.unit_cube_mesh(3); tg = hb.TimeGrid(1.0, 32); p = hb.KernelParams(1.0, tg.step, length_scale=m.diameter)
q = hb.QuadratureConfig(); E, N = m.n_triangles, m.n_vertices; Et = 32
tabs = hbdev.device_tables(m, q)
V = torch.empty((Et, E, E), dtype=torch.float64, device="cuda"); K = torch.empty((Et, E, N), dtype=torch.float64, device="cuda")
Dd = torch.empty((Et, N, N), dtype=torch.float64, device="cuda")
tV = torch.as_tensor(D.block_pointer_table([(V.data_ptr(), 0, Et)], Et, E * E * 8), device="cuda")
tK = torch.as_tensor(D.block_pointer_table([(K.data_ptr(), 0, Et)], Et, E * N * 8), device="cuda")
dev = torch.device("cuda", 0)
from paper_2102_09811_b200 import _native
import numpy as np
MODE = os.environ.get("MODE", "parts")
parts = [torch.zeros((Et, N, N), dtype=torch.float64, device="cuda") for _ in range(8)]
ptrs = {w: torch.as_tensor(np.array([t.data_ptr() for t in parts[:w]], dtype=np.int64), device="cuda") for w in (1, 2, 4, 8)}
sD, sV, sK = _op_streams(dev)
def ev(fn, reps=5):
    fn(); torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / reps
res = {}
for world in (1, 2, 4, 8):
    rv = D.row_partition(D.row_weights_mesh(m, q, True), world); rk = D.row_partition(D.row_weights_mesh(m, q, False), world)
    seq, conc = [], []
    for r in range(world):
        d0, d1 = D.block_range(r, world, Et)
        opV = lambda: _assemble_operator(0, False, False, True, m, tg, p, q, None, d_range=(0, Et), row_range=rv[r], block_ptrs=tV)
        opK = lambda: _assemble_operator(1, False, True, False, m, tg, p, q, None, d_range=(0, Et), row_range=rk[r], block_ptrs=tK)
        if MODE == "dshard":
            opD = lambda: _assemble_operator(2, True, True, True, m, tg, p, q, None, d_range=(d0, d1), out=Dd[d0:d1])
            curl = lambda: curl_combine_into(tabs, V[d0:d1], Dd[d0:d1], Dd[d0:d1], p.alpha)
        else:   # element-row D2 partials, summed by the curl kernel over "peer" buffers
            rd = D.row_partition(D.row_weights_mesh(m, q, True, True), world)[r]
            opD = lambda: _assemble_operator(2, True, True, True, m, tg, p, q, None, d_range=(0, Et), row_range=rd, out=parts[0])
            def curl():
                if d1 > d0:
                    _native.call("hb_curl_combine_parts", tabs.desc(True), d1 - d0, 1.0, _native.ptr(tabs.t["curls"]),
                                 _native.ptr(V[d0:d1]), world, _native.ptr(ptrs[world]), d0, _native.ptr(Dd[d0:d1]),
                                 _native.stream_handle())
        def s_work():
            opV(); opK(); opD(); curl()
        def c_work():
            cur = torch.cuda.current_stream()
            for st in (sD, sV, sK): st.wait_stream(cur)
            with torch.cuda.stream(sD): opD()
            with torch.cuda.stream(sV): opV()
            with torch.cuda.stream(sK): opK()
            sD.wait_stream(sV)
            with torch.cuda.stream(sD): curl()
            for st in (sD, sV, sK): cur.wait_stream(st)
        seq.append(round(ev(s_work), 3)); conc.append(round(ev(c_work), 3))
    res[world] = {"seq_ms": seq, "conc_ms": conc, "max_seq": max(seq), "max_conc": max(conc)}
b = res[1]["max_conc"]
for w in res: res[w]["speedup_conc"] = round(b / res[w]["max_conc"], 2)
print(json.dumps(res))
