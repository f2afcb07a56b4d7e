"""Per-op device time of rank RANK0 of WORLD in the config-2 rows-mode step (CUDA events)."""
import json, os, sys, torch, numpy as np
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import paper_2102_09811_b200 as hb
from paper_2102_09811_b200 import device as hbdev, distributed as D, _native
from paper_2102_09811_b200.assembly import _assemble_operator
m = hb.unit_cube_mesh(3); tg = hb.TimeGrid(1.0, 32); p = hb.KernelParams(1.0, tg.step, length_scale=m.diameter)
q = hb.QuadratureConfig(); E, N = m.n_triangles, m.n_vertices; Et = 32
world = int(os.environ.get("WORLD", "8"))
tabs = hbdev.device_tables(m, q)
V = torch.empty((Et, E, E), dtype=torch.float64, device="cuda"); K = torch.empty((Et, E, N), dtype=torch.float64, device="cuda")
P = torch.zeros((Et, N, N), dtype=torch.float64, device="cuda")
tV = torch.as_tensor(D.block_pointer_table([(V.data_ptr(), 0, Et)], Et, E * E * 8), device="cuda")
tK = torch.as_tensor(D.block_pointer_table([(K.data_ptr(), 0, Et)], Et, E * N * 8), device="cuda")
def ev(fn, reps=5):
    fn(); torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps): fn()
    e.record(); torch.cuda.synchronize()
    return round(s.elapsed_time(e) / reps, 3)
out = {}
for r in range(world):
    rv = D.row_partition(D.row_weights_mesh(m, q, True), world)[r]; rk = D.row_partition(D.row_weights_mesh(m, q, False), world)[r]
    rd = D.row_partition(D.row_weights_mesh(m, q, True, True), world)[r]
    out[r] = {"V": ev(lambda: _assemble_operator(0, False, False, True, m, tg, p, q, None, d_range=(0, Et), row_range=rv, block_ptrs=tV)),
              "K": ev(lambda: _assemble_operator(1, False, True, False, m, tg, p, q, None, d_range=(0, Et), row_range=rk, block_ptrs=tK)),
              "D2p": ev(lambda: _assemble_operator(2, True, True, True, m, tg, p, q, None, d_range=(0, Et), row_range=rd, out=P))}
print(json.dumps({"env": {k: os.environ.get(k) for k in ("HB_MIN_SEG", "HB_MIN_SEG_FAR")}, "ranks": out,
                  "max": {k: max(v[k] for v in out.values()) for k in ("V", "K", "D2p")}}))
