"""Multi-GPU layout: one process per GPU, operators sharded by time-difference
block d.

Block d of every operator depends only on the kernel at the three gaps
d-1, d, d+1, so rank r assembles the contiguous range [d0_r, d1_r) with no
communication (``hb_assemble`` with d_begin/d_end; blocks are bitwise equal
to a 1-GPU assembly, tests/test_assembly_gpu.py).  Products with a
d-sharded operator need one collective: every rank forms the partial sum
over its own blocks (``hb_toeplitz_apply_range``) and an all-reduce adds the
partials -- E_t x n_out doubles per product (25 MB at config 5), ~30 us
over NVLink 5.  Forward substitution all-reduces one n_out vector per time
step; A^0 lives on rank 0 and is broadcast once, every rank factorises it.

The collective goes through torch.distributed (NCCL on GPUs; gloo on CPU in
tests/test_distributed.py, where the local products are injected).
"""
from __future__ import annotations

import numpy as np

from . import _native


def block_range(rank: int, world: int, n_blocks: int):
    """Contiguous balanced split of [0, n_blocks): (d0, d1) for ``rank``."""
    if not 0 <= rank < world:
        raise ValueError("rank out of range")
    base, rem = divmod(n_blocks, world)
    d0 = rank * base + min(rank, rem)
    return d0, d0 + base + (1 if rank < rem else 0)


def window_slots(n_blocks: int) -> int:
    """Gap slots per assembly window (hb_assembly.cu choose_nj): 16 per
    lanes-x-slots group, two groups when the history is longer than 16."""
    return 16 * max(1, min(2, -(-n_blocks // 16)))


def window_edges(n_blocks: int):
    """Block boundaries of hb_assemble's windows over [0, n_blocks): the
    first window holds W blocks, every later one W - 2 (its two halo gaps)."""
    W = window_slots(n_blocks)
    edges, d = [0], 0
    while d < n_blocks:
        d = min(n_blocks, W if d <= 1 else d + W - 2)
        edges.append(d)
    return edges


def aligned_chunks(n_blocks: int, max_blocks: int):
    """Contiguous d-chunks of at most ``max_blocks`` blocks that start and
    end on window edges (so chunked assembly evaluates no extra gap slots);
    a window longer than ``max_blocks`` is split."""
    edges = window_edges(n_blocks)
    out, lo = [], 0
    for a, b in zip(edges[:-1], edges[1:]):
        if b - lo > max_blocks and a > lo:
            out.append((lo, a))
            lo = a
        while b - lo > max_blocks:
            out.append((lo, lo + max_blocks))
            lo += max_blocks
    if lo < n_blocks:
        out.append((lo, n_blocks))
    return out


def gap_slots(d0: int, d1: int, window: int = 32):
    """Time gaps i_t >= 1 a rank evaluates for blocks [d0, d1) (incl. halo
    slots at window edges): the redundant work of d-sharding."""
    n, dd = 0, d0
    while dd < d1:
        nd1 = min(d1, window if dd <= 1 else dd + window - 2)
        n += nd1 - max(1, dd - 1) + 1
        dd = nd1
    return n


class ShardedToeplitz:
    """Blocks [d0, d1) of a block lower-triangular Toeplitz operator held by
    this rank.  ``local`` is the (d1-d0, R, C) tensor (device or host)."""

    def __init__(self, local, d0: int, d1: int, n_blocks: int, group=None, transpose_blocks: bool = False):
        self.local, self.d0, self.d1, self.n_blocks = local, d0, d1, n_blocks
        self.group = group
        self.transpose = transpose_blocks
        self._lu = None

    @property
    def R(self):
        return self.local.shape[2] if self.transpose else self.local.shape[1]

    @property
    def C(self):
        return self.local.shape[1] if self.transpose else self.local.shape[2]

    # local partial products: CUDA kernel (tests on CPU inject a stand-in)
    def local_partial(self, x, d_min: int = 0):
        """sum_{d in [max(d0, d_min), d1), d <= k} A^d x^{k-d} for all k."""
        import torch

        E_t = x.shape[0]
        y = torch.zeros((E_t, self.R), dtype=torch.float64, device=x.device)
        lo = max(self.d0, d_min)
        if lo >= self.d1:
            return y
        blocks = self.local[lo - self.d0:]
        nb, Rb, Cb = blocks.shape
        _native.call("hb_toeplitz_apply_range", lo, nb, Rb, Cb, _native.ptr(blocks), int(self.transpose), E_t,
                     _native.ptr(x), _native.ptr(y), _native.stream_handle())
        return y

    def apply(self, x):
        """Full-operator product y = A x (every rank gets y)."""
        import torch.distributed as dist

        y = self.local_partial(x)
        if dist.is_initialized():
            dist.all_reduce(y, op=dist.ReduceOp.SUM, group=self.group)
        return y

    def _factor(self):
        import torch
        import torch.distributed as dist

        if self._lu is None:
            if self.d0 == 0:
                A0 = self.local[0]
                A0 = (A0.T if self.transpose else A0).contiguous()
            else:
                A0 = torch.empty((self.R, self.C), dtype=torch.float64, device=self.local.device)
            if dist.is_initialized():
                dist.broadcast(A0, src=0, group=self.group)   # rank 0 owns d = 0
            self._lu = torch.linalg.lu_factor(A0)
        return self._lu

    def forward_solve(self, rhs):
        """Causal time marching with one all-reduce of an n_out vector per step."""
        import torch
        import torch.distributed as dist

        LU, piv = self._factor()
        E_t = rhs.shape[0]
        x = torch.zeros((E_t, self.C), dtype=torch.float64, device=rhs.device)
        for k in range(E_t):
            h = self.history(x, k)
            if dist.is_initialized():
                dist.all_reduce(h, op=dist.ReduceOp.SUM, group=self.group)
            x[k] = torch.linalg.lu_solve(LU, piv, (rhs[k] - h)[:, None])[:, 0]
        return x

    def history(self, x, k: int):
        """sum_{d in [max(d0,1), d1), d <= k} A^d x^{k-d} for one k."""
        y = self.local_partial(x[: k + 1], d_min=1)
        return y[k].clone()


def gather_blocks(shard: ShardedToeplitz):
    """All blocks on every rank (small operators / tests)."""
    import torch
    import torch.distributed as dist

    if not dist.is_initialized():
        return shard.local
    world = dist.get_world_size(shard.group)
    parts = []
    for r in range(world):
        d0, d1 = block_range(r, world, shard.n_blocks)
        buf = shard.local if r == dist.get_rank(shard.group) else torch.empty(
            (d1 - d0,) + tuple(shard.local.shape[1:]), dtype=shard.local.dtype, device=shard.local.device)
        dist.broadcast(buf, src=r, group=shard.group)
        parts.append(buf)
    return torch.cat(parts)
