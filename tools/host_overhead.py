"""Host cost of one _assemble_operator call vs its device time (config 2, a
rank-of-8 row range): wall time of N back-to-back calls without syncs
(launch-bound if the host is slower than the GPU) vs CUDA-event device time."""
import json, os, sys, time, torch
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import paper_2102_09811_b200 as hb
from paper_2102_09811_b200 import distributed as D
from paper_2102_09811_b200.assembly import _assemble_operator
m = hb.unit_cube_mesh(3); tg = hb.TimeGrid(1.0, 32); p = hb.KernelParams(1.0, tg.step, length_scale=m.diameter)
q = hb.QuadratureConfig(); E, N = m.n_triangles, m.n_vertices
V = torch.empty((32, E, E), dtype=torch.float64, device="cuda")
tV = torch.as_tensor(D.block_pointer_table([(V.data_ptr(), 0, 32)], 32, E * E * 8), device="cuda")
rv = D.row_partition(D.row_weights_mesh(m, q, True), 8)[0]
f = lambda: _assemble_operator(0, False, False, True, m, tg, p, q, None, d_range=(0, 32), row_range=rv, block_ptrs=tV)
for _ in range(3): f()
torch.cuda.synchronize()
n = 30
t0 = time.perf_counter()
for _ in range(n): f()
t_host = (time.perf_counter() - t0) / n
torch.cuda.synchronize()
t_all = (time.perf_counter() - t0) / n
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(n): f()
e.record(); torch.cuda.synchronize()
import cProfile, pstats, io
pr = cProfile.Profile(); pr.enable()
for _ in range(10): f()
pr.disable(); torch.cuda.synchronize()
st = io.StringIO(); pstats.Stats(pr, stream=st).sort_stats("cumulative").print_stats(12)
print(json.dumps({"host_issue_ms": t_host * 1e3, "wall_per_call_ms": t_all * 1e3, "device_per_call_ms": s.elapsed_time(e) / n}))
print(st.getvalue()[:3000])
