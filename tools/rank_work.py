"""Per-rank work of the N-GPU config-2 step, timed one rank at a time on one
B200 (no rank waits on another; the projection ignores the one-element fence
and the NVLink peer stores, which overlap the pair kernels): rank r = V and K
pair work on its balanced test-row range over all blocks (stores into the
d-owners' shards, here one buffer), D2 partial of its element rows over all
blocks (summed across ranks by a reduce-scatter of E_t N^2 doubles, not
timed), curl of its d-range."""
import json, os, sys, torch
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import paper_2102_09811_b200 as hb
from paper_2102_09811_b200 import device as hbdev, distributed as D
from paper_2102_09811_b200.assembly import _assemble_operator, curl_combine_into
m = hb.unit_cube_mesh(3); tg = hb.TimeGrid(1.0, 32); p = hb.KernelParams(1.0, tg.step, length_scale=m.diameter)
q = hb.QuadratureConfig(); E, N = m.n_triangles, m.n_vertices; Et = 32
tabs = hbdev.device_tables(m, q)
V = torch.empty((Et, E, E), dtype=torch.float64, device="cuda"); K = torch.empty((Et, E, N), dtype=torch.float64, device="cuda")
Dd = torch.empty((Et, N, N), dtype=torch.float64, device="cuda")
P2 = torch.empty((Et, N, N), dtype=torch.float64, device="cuda")
tV = torch.as_tensor(D.block_pointer_table([(V.data_ptr(), 0, Et)], Et, E * E * 8), device="cuda")
tK = torch.as_tensor(D.block_pointer_table([(K.data_ptr(), 0, Et)], Et, E * N * 8), device="cuda")
def ev(fn, reps=5):
    fn(); torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / reps
res = {}
for world in (1, 2, 4, 8):
    rv = D.row_partition(D.row_weights_mesh(m, q, True), world); rk = D.row_partition(D.row_weights_mesh(m, q, False), world); rd = D.row_partition(D.row_weights_mesh(m, q, True, True), world)
    per = []
    for r in range(world):
        d0, d1 = D.block_range(r, world, Et)
        def work():
            _assemble_operator(0, False, False, True, m, tg, p, q, None, d_range=(0, Et), row_range=rv[r], block_ptrs=tV)
            _assemble_operator(1, False, True, False, m, tg, p, q, None, d_range=(0, Et), row_range=rk[r], block_ptrs=tK)
            if world == 1:
                _assemble_operator(2, True, True, True, m, tg, p, q, None, d_range=(d0, d1), out=Dd[d0:d1])
            else:   # row partial of D2 for all blocks (the reduce-scatter itself is not timed here)
                _assemble_operator(2, True, True, True, m, tg, p, q, None, d_range=(0, Et), row_range=rd[r], out=P2)
            curl_combine_into(tabs, V[d0:d1], Dd[d0:d1], Dd[d0:d1], p.alpha)
        per.append(round(ev(work), 3))
    res[world] = {"per_rank_ms": per, "max_ms": max(per), "speedup_vs_1": None}
base = res[1]["max_ms"]
for w in res: res[w]["speedup_vs_1"] = round(base / res[w]["max_ms"], 2)
print(json.dumps(res))
# per-call breakdown, one rank of 8
world, r = 8, 7
rv = D.row_partition(D.row_weights_mesh(m, q, True), world); rk = D.row_partition(D.row_weights_mesh(m, q, False), world); rd = D.row_partition(D.row_weights_mesh(m, q, True, True), world)
d0, d1 = D.block_range(r, world, Et)
from paper_2102_09811_b200._native import AssemblyStats
det = {}
for name, fn in (("V", lambda st=None: _assemble_operator(0, False, False, True, m, tg, p, q, None, d_range=(0, Et), row_range=rv[r], block_ptrs=tV, stats=st)),
                 ("K", lambda st=None: _assemble_operator(1, False, True, False, m, tg, p, q, None, d_range=(0, Et), row_range=rk[r], block_ptrs=tK, stats=st)),
                 ("D2", lambda st=None: _assemble_operator(2, True, True, True, m, tg, p, q, None, d_range=(0, Et), row_range=rd[r], out=P2, stats=st))):
    st = AssemblyStats()
    fn(st); st = AssemblyStats(); fn(st)
    det[name] = {"total_ms": ev(fn), "pair_ms": st.pair_ms, "fin_ms": st.finalize_ms, "launches": st.launches}
det["curl"] = ev(lambda: curl_combine_into(tabs, V[d0:d1], Dd[d0:d1], Dd[d0:d1], p.alpha))
print(json.dumps(det))
