"""Rank 0 of 8 of the config-2 rows-mode step (V rows, K rows, D2 element-row
partial, peer-partial curl), run a few times -- for an ncu launch list."""
import os, sys, torch, numpy as np
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import paper_2102_09811_b200 as hb
from paper_2102_09811_b200 import device as hbdev, distributed as D, _native
from paper_2102_09811_b200.assembly import _assemble_operator
m = hb.unit_cube_mesh(3); tg = hb.TimeGrid(1.0, 32); p = hb.KernelParams(1.0, tg.step, length_scale=m.diameter)
q = hb.QuadratureConfig(); E, N = m.n_triangles, m.n_vertices; Et = 32
world, r = int(os.environ.get("WORLD", "8")), int(os.environ.get("RANK0", "0"))
tabs = hbdev.device_tables(m, q)
V = torch.empty((Et, E, E), dtype=torch.float64, device="cuda"); K = torch.empty((Et, E, N), dtype=torch.float64, device="cuda")
Dd = torch.empty((Et, N, N), dtype=torch.float64, device="cuda")
parts = [torch.zeros((Et, N, N), dtype=torch.float64, device="cuda") for _ in range(world)]
ptrs = torch.as_tensor(np.array([t.data_ptr() for t in parts], dtype=np.int64), device="cuda")
tV = torch.as_tensor(D.block_pointer_table([(V.data_ptr(), 0, Et)], Et, E * E * 8), device="cuda")
tK = torch.as_tensor(D.block_pointer_table([(K.data_ptr(), 0, Et)], Et, E * N * 8), device="cuda")
rv = D.row_partition(D.row_weights_mesh(m, q, True), world)[r]; rk = D.row_partition(D.row_weights_mesh(m, q, False), world)[r]
rd = D.row_partition(D.row_weights_mesh(m, q, True, True), world)[r]
d0, d1 = D.block_range(r, world, Et)
for _ in range(3):
    _assemble_operator(0, False, False, True, m, tg, p, q, None, d_range=(0, Et), row_range=rv, block_ptrs=tV)
    _assemble_operator(1, False, True, False, m, tg, p, q, None, d_range=(0, Et), row_range=rk, block_ptrs=tK)
    _assemble_operator(2, True, True, True, m, tg, p, q, None, d_range=(0, Et), row_range=rd, out=parts[0])
    _native.call("hb_curl_combine_parts", tabs.desc(True), d1 - d0, 1.0, _native.ptr(tabs.t["curls"]),
                 _native.ptr(V[d0:d1]), world, _native.ptr(ptrs), d0, _native.ptr(Dd[d0:d1]), _native.stream_handle())
    torch.cuda.synchronize()
print("ok")
