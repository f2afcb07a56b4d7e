"""N > 1 host logic on CPU: world_size-2 gloo process groups.

The d-sharded products are checked against dense expansions; the per-rank
CUDA partial product is replaced by a numpy stand-in (a test double -- the
package itself has no CPU path)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2102_09811_b200 import distributed as D


def test_block_ranges_cover_exactly_once():
    for n in (1, 5, 16, 32, 64, 256):
        for w in (1, 2, 3, 4, 8):
            if w > n:
                continue
            rs = [D.block_range(r, w, n) for r in range(w)]
            assert rs[0][0] == 0 and rs[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
            assert max(b - a for a, b in rs) - min(b - a for a, b in rs) <= 1


def test_cost_balanced_ranges_equalise_measured_cost():
    """Front-loaded block costs (the moment form's low blocks): the measured
    split gives contiguous, covering ranges of near-equal cost, where the
    equal-count split leaves rank 0 with the most work."""
    VD = [824, 395, 298, 297, 421, 297, 297, 351]   # B200, config 5, ms per 32-block chunk
    costs = [(32 * i, 32 * i + 32, c) for i, c in enumerate(VD)]
    dens = np.repeat(np.array(VD) / 32.0, 32)
    for world in (2, 4, 8):
        r = D.cost_balanced_ranges(costs, 256, world)
        assert r[0][0] == 0 and r[-1][1] == 256 and all(a < b for a, b in r)
        assert all(r[i][1] == r[i + 1][0] for i in range(world - 1))
        per = [dens[a:b].sum() for a, b in r]
        uni = [dens[a:b].sum() for a, b in (D.block_range(k, world, 256) for k in range(world))]
        assert max(per) < max(uni) and sum(per) / (world * max(per)) > 0.9
    edges = D.window_edges(256)
    r = D.cost_balanced_ranges(costs, 256, 8, edges)
    assert r[0][0] == 0 and r[-1][1] == 256 and all(a < b for a, b in r)


def test_gap_slots_halo_accounting():
    assert D.gap_slots(0, 32) == 32
    assert D.gap_slots(0, 16) + D.gap_slots(16, 32) == 34        # one extra halo pair
    assert D.gap_slots(0, 256) == 256 + 2 * 8            # 9 windows: [0,32) then 30 blocks each
    assert D.gap_slots(3, 5) == 4                          # gaps 2..5


def _numpy_partial(self, x, d_min=0):
    A = self.local.numpy()
    if self.transpose:
        A = A.transpose(0, 2, 1)
    E_t = x.shape[0]
    y = np.zeros((E_t, A.shape[1]))
    for k in range(E_t):
        for d in range(max(self.d0, d_min), min(self.d1, k + 1)):
            y[k] += A[d - self.d0] @ x[k - d].numpy()
    return torch.from_numpy(y)


def _worker(rank, world, port, B, x, rhs, out):
    os.environ["MASTER_ADDR"], os.environ["MASTER_PORT"] = "127.0.0.1", str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        D.ShardedToeplitz.local_partial = _numpy_partial
        n = B.shape[0]
        d0, d1 = D.block_range(rank, world, n)
        for tr in (False, True):
            S = D.ShardedToeplitz(torch.from_numpy(B[d0:d1].copy()), d0, d1, n, transpose_blocks=tr)
            xx = torch.from_numpy(x if not tr else x[:, : B.shape[1]].copy())
            y = S.apply(xx)
            xs = S.forward_solve(torch.from_numpy(rhs if not tr else rhs[:, : B.shape[2]].copy()))
            full = D.gather_blocks(S)
            if rank == 0:
                out[f"y{int(tr)}"] = y.numpy()
                out[f"x{int(tr)}"] = xs.numpy()
                out[f"full{int(tr)}"] = full.numpy()
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world", [2])
def test_sharded_apply_and_forward_solve_gloo(world):
    rng = np.random.default_rng(0)
    E_t, n = 9, 6
    B = 0.2 * rng.standard_normal((E_t, n, n))
    B[0] += 3 * np.eye(n)
    x = rng.standard_normal((E_t, n))
    rhs = rng.standard_normal((E_t, n))
    out = mp.Manager().dict()
    mp.spawn(_worker, args=(world, _free_port(), B, x, rhs, out), nprocs=world, join=True)
    for tr in (False, True):
        A = B.transpose(0, 2, 1) if tr else B
        dense = np.zeros((E_t * n, E_t * n))
        for k in range(E_t):
            for i in range(k + 1):
                dense[k * n:(k + 1) * n, i * n:(i + 1) * n] = A[k - i]
        assert np.allclose(out[f"y{int(tr)}"].ravel(), dense @ x.ravel(), rtol=1e-13, atol=1e-13)
        assert np.allclose(dense @ out[f"x{int(tr)}"].ravel(), rhs.ravel(), rtol=1e-12, atol=1e-12)
        assert np.array_equal(out[f"full{int(tr)}"], B)


# ---------------------------------------------------------------------------
# row-parallel assembly: host planning (the kernel path is tested on the GPU
# in tests/test_assembly_gpu.py::test_row_parallel_into_d_shards_bitwise)
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("symmetric", [True, False])
def test_row_partition_covers_and_balances(symmetric):
    for n in (1, 7, 192, 768, 12288):
        w = D.row_weights(n, symmetric)
        for world in (1, 2, 3, 4, 8):
            parts = D.row_partition(w, world)
            assert parts[0][0] == 0 and parts[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(parts, parts[1:]))
            loads = [w[a:b].sum() for a, b in parts]
            assert max(loads) <= w.sum() / world + w.max() + 1e-9


def test_block_pointer_table_owners():
    t = D.block_pointer_table([(1000, 0, 2), (9000, 2, 5)], 5, 16)
    assert list(t) == [1000, 1016, 9000, 9016, 9032]
    with pytest.raises(ValueError):
        D.block_pointer_table([(0, 0, 3), (64, 2, 4)], 4, 8)     # block 2 twice
    with pytest.raises(ValueError):
        D.block_pointer_table([(0, 0, 2)], 4, 8)                  # blocks 2, 3 unowned


def _plan_worker(rank, world, port, out):
    os.environ["MASTER_ADDR"], os.environ["MASTER_PORT"] = "127.0.0.1", str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        E_t, R, C = 32, 768, 386
        d0, d1 = D.block_range(rank, world, E_t)
        fake_handle = bytes([rank]) * 64                  # stands in for hb_ipc_export's handle
        metas = D.exchange_shard_meta((fake_handle, 128 * rank, d0, d1))
        bases = [(10 ** 9 * (r + 1) + o, a, b) for r, (h, o, a, b) in enumerate(metas)]
        table = D.block_pointer_table(bases, E_t, R * C * 8)
        rows = D.row_partition(D.row_weights(768, False), world)[rank]
        out[rank] = ([h for h, *_ in metas], list(table), rows)
    finally:
        dist.destroy_process_group()


def test_row_parallel_plan_exchange_gloo():
    world = 2
    out = mp.Manager().dict()
    mp.spawn(_plan_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    assert out[0][0] == out[1][0] == [bytes([0]) * 64, bytes([1]) * 64]
    assert out[0][1] == out[1][1]                          # every rank addresses every block alike
    t = out[0][1]
    assert t[0] == 10 ** 9 and t[16] == 2 * 10 ** 9 + 128   # rank 1 owns blocks 16..31
    assert out[0][2] == (0, 384) and out[1][2] == (384, 768)


# ---------------------------------------------------------------------------
# row-sharded solve operator: one all-gather per product / per time step
# ---------------------------------------------------------------------------
def _np_local_apply(self, x):
    A = self.local.numpy()
    E_t = x.shape[0]
    y = np.zeros((E_t, A.shape[1]))
    for k in range(E_t):
        for d in range(min(k + 1, A.shape[0])):
            y[k] += A[d] @ x[k - d].numpy()
    return torch.from_numpy(y)


def _np_local_history_far(self, x, k0, nk):
    A = self.local.numpy()
    H = np.zeros((nk, A.shape[1]))
    for i in range(nk):
        for d in range(i + 1, min(k0 + i, A.shape[0] - 1) + 1):   # k0 + i - d < k0
            H[i] += A[d] @ x[k0 + i - d].numpy()
    return torch.from_numpy(H)


def _np_local_history(self, x, k, k0=0, Hk=None):
    A = self.local.numpy()
    h = np.zeros(A.shape[1]) if Hk is None else Hk.numpy().copy()
    for d in range(1, min(k - k0, A.shape[0] - 1) + 1):
        h += A[d] @ x[k - d].numpy()
    return torch.from_numpy(h)


def _np_inv_apply(self, inv, rhs_k, h):
    v = rhs_k.numpy() - (h.numpy() if h is not None else 0.0)
    return torch.from_numpy(inv.numpy() @ v)


def _row_worker(rank, world, port, B, x, rhs, out):
    os.environ["MASTER_ADDR"], os.environ["MASTER_PORT"] = "127.0.0.1", str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        D.RowShardedToeplitz.local_apply = _np_local_apply
        D.RowShardedToeplitz.local_history = _np_local_history
        D.RowShardedToeplitz.local_history_far = _np_local_history_far
        D.RowShardedToeplitz.inv_apply = _np_inv_apply
        n_blocks, R, _ = B.shape
        d0, d1 = D.block_range(rank, world, n_blocks)
        S = D.ShardedToeplitz(torch.from_numpy(B[d0:d1].copy()), d0, d1, n_blocks)
        Rs = D.row_shards_from_d_shards(S)
        r0, r1 = D.block_range(rank, world, R)
        assert (Rs.r0, Rs.r1) == (r0, r1)
        assert np.array_equal(Rs.local.numpy(), B[:, r0:r1, :])
        y = Rs.apply(torch.from_numpy(x))
        xs = Rs.forward_solve(torch.from_numpy(rhs))
        out[f"y{rank}"] = y.numpy()
        out[f"x{rank}"] = xs.numpy()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n", [(2, 7), (3, 8)])
def test_row_sharded_apply_and_forward_solve_gloo(world, n):
    """Row shards from d shards (all-to-all), apply (all-gather of the row
    pieces) and forward substitution (one all-gather of h^k per step):
    identical on every rank and equal to the dense expansion; row ranges of
    unequal length (n = 7 over 2 ranks, 8 over 3)."""
    rng = np.random.default_rng(n)
    E_t = 19   # three step tiles of the blocked substitution (8, 8, 3)
    B = 0.2 * rng.standard_normal((E_t, n, n))
    B[0] += 3 * np.eye(n)
    x = rng.standard_normal((E_t, n))
    rhs = rng.standard_normal((E_t, n))
    out = mp.Manager().dict()
    mp.spawn(_row_worker, args=(world, _free_port(), B, x, rhs, out), nprocs=world, join=True)
    dense = np.zeros((E_t * n, E_t * n))
    for k in range(E_t):
        for i in range(k + 1):
            dense[k * n:(k + 1) * n, i * n:(i + 1) * n] = B[k - i]
    for r in range(world):
        assert np.array_equal(out[f"y{r}"], out["y0"]) and np.array_equal(out[f"x{r}"], out["x0"])
    assert np.allclose(out["y0"].ravel(), dense @ x.ravel(), rtol=1e-13, atol=1e-13)
    assert np.allclose(dense @ out["x0"].ravel(), rhs.ravel(), rtol=1e-12, atol=1e-12)


def test_point_ranges_partition_every_point():
    from paper_2102_09811_b200.distributed import block_range

    for M, world in ((100000, 8), (301, 2), (3, 4)):
        ranges = [block_range(r, world, M) for r in range(world)]
        assert ranges[0][0] == 0 and ranges[-1][1] == M
        assert all(ranges[i][1] == ranges[i + 1][0] for i in range(world - 1))
        assert max(b - a for a, b in ranges) <= -(-M // world)
