"""Multi-GPU layout: one process per GPU, operators sharded by time-difference
block d; pair work split by d (halo gaps) or by test rows
(``assemble_row_parallel``: peer stores into the d-owners' shards).

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

FORWARD_TILE = 8   # steps per tile of the blocked forward substitution (hb_solver.cu kFT)


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


def cost_balanced_ranges(costs, n_blocks: int, world: int, edges=None):
    """Contiguous d-ranges of near-equal measured cost, one per rank.

    ``costs``: (d0, d1, ms) pieces covering [0, n_blocks) (e.g. the chunk
    times of a first step on block_range's split, gathered from every rank);
    the cost of a piece is spread evenly over its blocks.  Boundaries snap to
    the nearest of ``edges`` (window edges: a range edge inside a window
    costs extra gap slots) when that keeps the range non-empty.  With the
    moment form the low blocks are the expensive ones (per-point gaps below
    each pair's moment block), so equal block counts leave rank 0 with the
    most work (config 5, N = 8: balance 0.60)."""
    dens = np.zeros(n_blocks)
    for d0, d1, ms in costs:
        if d1 > d0:
            dens[int(d0):int(d1)] += float(ms) / (int(d1) - int(d0))
    if not np.all(dens > 0):
        dens = np.where(dens > 0, dens, dens[dens > 0].mean() if np.any(dens > 0) else 1.0)
    cum = np.concatenate([[0.0], np.cumsum(dens)])
    cuts = [0]
    for r in range(1, world):
        c = int(np.searchsorted(cum, cum[-1] * r / world))
        c = min(max(c, cuts[-1] + 1), n_blocks - (world - r))
        if edges is not None:
            e = min(edges, key=lambda x: abs(x - c))
            if cuts[-1] < e < n_blocks - (world - r) + 1 and abs(e - c) <= 8:
                c = e
        cuts.append(c)
    cuts.append(n_blocks)
    return [(cuts[r], cuts[r + 1]) for r in range(world)]


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


def row_weights(n_rows: int, symmetric: bool):
    """Pair-kernel work per test row: symmetric operators evaluate the upper
    triangle (row e: n_rows - e trial elements), the others every pair."""
    e = np.arange(n_rows, dtype=np.float64)
    return (n_rows - e) if symmetric else np.full(n_rows, float(n_rows))


def row_weights_mesh(mesh, config, symmetric: bool, skip_perpendicular: bool = False):
    """Pair-kernel work per test row in quadrature points: n_reg^2 per
    separated pair plus the Duffy point count of each touching pair (identical
    / edge / vertex) -- the touching pairs dominate rows near the end of an
    upper triangle, which the plain pair count misses.  ``skip_perpendicular``
    (D2): pairs with n_e . n_f == 0 cost nothing."""
    from .device import host_tables

    H = host_tables(mesh, config)
    E = mesh.n_triangles
    indptr, idx, case = H.tn[0], H.tn[1], H.tn[2]
    off = H.duf[0]
    q_case = np.diff(off).astype(np.float64)
    rows = np.repeat(np.arange(E), np.diff(indptr))
    keep = idx >= rows if symmetric else np.ones(len(idx), dtype=bool)
    nrm = np.asarray(mesh.normals, dtype=np.float64)
    if skip_perpendicular:
        keep &= np.einsum("ij,ij->i", nrm[rows], nrm[idx]) != 0.0
    sing_pts = np.bincount(rows[keep], weights=q_case[case[keep]], minlength=E)
    n_sing = np.bincount(rows[keep], minlength=E)
    if skip_perpendicular:   # non-perpendicular trial elements per row (f >= e when symmetric)
        n_pairs = np.empty(E)
        for a in range(0, E, 2048):
            nz = (nrm[a:a + 2048] @ nrm.T) != 0.0
            if symmetric:
                nz &= np.arange(E)[None, :] >= np.arange(a, min(E, a + 2048))[:, None]
            n_pairs[a:a + 2048] = nz.sum(axis=1)
    else:
        n_pairs = (E - np.arange(E)) if symmetric else np.full(E, E)
    n_reg = float(len(H.reg[1])) ** 2
    return n_reg * (n_pairs - n_sing) + sing_pts


def row_partition(weights, world: int):
    """Contiguous test-row ranges of near-equal total weight, one per rank."""
    w = np.asarray(weights, dtype=np.float64)
    c = np.concatenate([[0.0], np.cumsum(w)])
    cuts = [0]
    for r in range(1, world):
        cuts.append(max(cuts[-1], int(np.searchsorted(c, c[-1] * r / world, side="left"))))
    cuts.append(len(w))
    return [(cuts[r], cuts[r + 1]) for r in range(world)]


def block_pointer_table(shards, n_blocks: int, block_bytes: int):
    """Address of every block d in [0, n_blocks) given, per rank, (base
    address, d0, d1) of its contiguous d-shard: base_r + (d - d0_r) bytes."""
    table = np.zeros(n_blocks, dtype=np.int64)
    seen = np.zeros(n_blocks, dtype=bool)
    for base, d0, d1 in shards:
        for d in range(d0, d1):
            if seen[d]:
                raise ValueError(f"block {d} owned twice")
            seen[d] = True
            table[d] = int(base) + (d - d0) * block_bytes
    if not seen.all():
        raise ValueError("blocks without an owner")
    return table


def exchange_shard_meta(meta, group=None):
    """All ranks' (ipc handle, offset, d0, d1) -- one all_gather_object."""
    import torch.distributed as dist

    if not dist.is_initialized():
        return [meta]
    out = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, meta, group=group)
    return out


def map_peer_shards(local, extent, group=None):
    """Every rank's shard address in this process: each rank exports its
    shard (CUDA IPC, hb_ipc_export), the handles and ``extent`` (the shard's
    (lo, hi) range) are all-gathered, and peer shards are mapped
    (hb_ipc_import; peer access over NVLink).  Returns (addresses by rank --
    0 for an empty shard --, extents by rank, [(mapped address, offset)] to
    hand to hb_ipc_close).  Collective: every rank calls it, empty shards
    (more ranks than blocks or rows) included."""
    import ctypes

    import torch.distributed as dist

    rank = dist.get_rank(group) if dist.is_initialized() else 0
    if extent[1] > extent[0] and local.numel() > 0:
        h = (ctypes.c_char * 64)()
        off = ctypes.c_int64()
        _native.call("hb_ipc_export", local.data_ptr(), h, ctypes.byref(off))
        meta = (bytes(h), off.value) + tuple(extent)
    else:
        meta = (None, 0) + tuple(extent)
    metas = exchange_shard_meta(meta, group)
    addrs, opened = [], []
    for r, (hr, o, a, b) in enumerate(metas):
        if r == rank:
            addrs.append(local.data_ptr() if meta[0] is not None else 0)
        elif hr is None or b <= a:
            addrs.append(0)
        else:
            p = ctypes.c_void_p()
            _native.call("hb_ipc_import", hr, o, ctypes.byref(p))
            opened.append((p.value, o))
            addrs.append(p.value)
    return addrs, [(m[2], m[3]) for m in metas], opened


class PeerRowShards:
    """Row-sharded destination of an assembly (hb_assembly_desc.row_shard_*):
    rank k holds rows [bounds[k], bounds[k+1]) of every block; ``bounds`` and
    ``ptrs`` (int64 device tensors) are what the finalize kernels store
    through -- peer shards mapped by CUDA IPC.  ``close()`` unmaps."""

    def __init__(self, local, r0: int, r1: int, n_rows: int, group=None):
        import torch

        self._L = _native.load()
        addrs, ranges, self._opened = map_peer_shards(local, (r0, r1), group)
        bounds = [0]
        for a, b in ranges:
            if a != bounds[-1]:
                raise ValueError("row shards must be contiguous and in rank order")
            bounds.append(b)
        if bounds[-1] != n_rows:
            raise ValueError("row shards do not cover every row")
        self.bounds = torch.as_tensor(np.array(bounds, dtype=np.int64), device=local.device)
        self.ptrs = torch.as_tensor(np.array(addrs, dtype=np.int64), device=local.device)

    def close(self):
        for pv, o in self._opened:
            self._L.hb_ipc_close(pv, o)
        self._opened = []


class PeerShardTable:
    """Per-block addresses of a d-sharded operator across ranks: every rank
    exports its shard (CUDA IPC, hb_ipc_export), the metadata is all-gathered
    and peer shards are mapped (hb_ipc_import, peer access over NVLink).
    ``table`` (int64 device tensor, one address per block d) is what the
    row-parallel finalize kernels store through.  ``close()`` unmaps."""

    def __init__(self, local, d0: int, d1: int, n_blocks: int, group=None):
        import ctypes

        import torch
        import torch.distributed as dist

        self._L = _native.load()
        block_bytes = int(np.prod(tuple(local.shape[1:]))) * 8   # valid for an empty shard too
        addrs, ranges, self._opened = map_peer_shards(local, (d0, d1), group)
        bases = [(addr, a, b) for addr, (a, b) in zip(addrs, ranges)]
        self.table = torch.as_tensor(block_pointer_table(bases, n_blocks, block_bytes), device=local.device)

    def close(self):
        for pv, o in self._opened:
            self._L.hb_ipc_close(pv, o)
        self._opened = []


def assemble_row_parallel(op: int, test_p1: bool, trial_p1: bool, symmetric: bool, mesh, timegrid, params,
                          config, group=None, workspace_bytes=None):
    """Row-parallel assembly with d-sharded storage: rank r
    evaluates the pairs of a balanced test-row range for ALL blocks and the
    finalize kernels store each block straight into the memory of the rank
    that owns it (CUDA IPC peer pointers over NVLink; block_range split).
    No halo gaps and no collective on the data path; every entry is written
    by exactly one rank, so the shards are bitwise equal to the 1-GPU blocks.
    p0 x p0 and p0 x p1 only (p1 x p1 accumulates over rows: use d-sharding)."""
    import torch
    import torch.distributed as dist

    from .assembly import _assemble_operator

    if test_p1 and trial_p1:
        raise ValueError("row-parallel assembly needs p0 test functions (p1 x p1 accumulates over rows)")
    E_t = timegrid.n_steps
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    E_x, N_x = mesh.n_triangles, mesh.n_vertices
    R, C = (N_x if test_p1 else E_x), (N_x if trial_p1 else E_x)
    d0, d1 = block_range(rank, world, E_t)
    dev = torch.device("cuda", torch.cuda.current_device())
    local = torch.empty((d1 - d0, R, C), dtype=torch.float64, device=dev)
    if world == 1:
        _assemble_operator(op, test_p1, trial_p1, symmetric, mesh, timegrid, params, config, None,
                           d_range=(0, E_t), out=local, workspace_bytes=workspace_bytes)
        return ShardedToeplitz(local, d0, d1, E_t, group)
    peers = PeerShardTable(local, d0, d1, E_t, group)
    rows = row_partition(row_weights_mesh(mesh, config, symmetric), world)[rank]
    dist.barrier(group)                      # every shard allocated and mapped
    try:
        if rows[1] > rows[0]:
            _assemble_operator(op, test_p1, trial_p1, symmetric, mesh, timegrid, params, config, None,
                               d_range=(0, E_t), row_range=rows, block_ptrs=peers.table,
                               workspace_bytes=workspace_bytes)
        torch.cuda.synchronize(dev)
        dist.barrier(group)                  # every rank's stores into every shard are done
    finally:
        peers.close()
    return ShardedToeplitz(local, d0, d1, E_t, group)


def assemble_row_sharded(op: int, test_p1: bool, trial_p1: bool, symmetric: bool, mesh, timegrid, params,
                         config, group=None, workspace_bytes=None, d_range=None):
    """The solve operator's layout: rank r holds rows
    block_range(r, world, R) of every block, as a RowShardedToeplitz.  The
    pair work is split by balanced test-row ranges (upper-triangle weights for
    symmetric V) and the finalize kernels store every entry into the owner of
    its row -- V's mirrored entries into peer shards over NVLink (CUDA IPC):
    no halo, no data-path collective, and the shards are bitwise the rows of
    the 1-GPU blocks.  p0 test functions (V, K)."""
    import torch
    import torch.distributed as dist

    from .assembly import _assemble_operator

    if test_p1:
        raise ValueError("row-sharded assembly needs p0 test functions (p1 rows accumulate over elements)")
    E_t = timegrid.n_steps
    d0, d1 = (0, E_t) if d_range is None else (int(d_range[0]), int(d_range[1]))
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    E_x, N_x = mesh.n_triangles, mesh.n_vertices
    R, C = E_x, (N_x if trial_p1 else E_x)
    r0, r1 = block_range(rank, world, R)
    dev = torch.device("cuda", torch.cuda.current_device())
    local = torch.empty((d1 - d0, r1 - r0, C), dtype=torch.float64, device=dev)
    if world == 1:
        _assemble_operator(op, test_p1, trial_p1, symmetric, mesh, timegrid, params, config, None,
                           d_range=(d0, d1), out=local, workspace_bytes=workspace_bytes)
        return RowShardedToeplitz(local, 0, R, R, group)
    peers = PeerRowShards(local, r0, r1, R, group)
    work = (row_partition(row_weights_mesh(mesh, config, symmetric), world)[rank] if symmetric else (r0, r1))
    dist.barrier(group)                      # every shard allocated and mapped
    try:
        if work[1] > work[0]:
            _assemble_operator(op, test_p1, trial_p1, symmetric, mesh, timegrid, params, config, None,
                               d_range=(d0, d1), row_range=work, row_shards=(peers.bounds, peers.ptrs),
                               workspace_bytes=workspace_bytes)
        torch.cuda.synchronize(dev)
        dist.barrier(group)                  # every rank's stores into every shard are done
    finally:
        peers.close()
    return RowShardedToeplitz(local, r0, r1, R, group)


def reduce_scatter_blocks(partial, local, d0: int, d1: int, group=None):
    """Sum every rank's full-size partial (E_t, R, C) and leave block range
    [d0, d1) of the sum in ``local`` -- one NCCL reduce-scatter (block ranges
    of unequal length are padded to the longest)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    E_t = partial.shape[0]
    if dist.get_backend(group) == "gloo":   # no reduce-scatter in gloo (CPU tests, one-device emulation)
        dist.all_reduce(partial, group=group)
        local.copy_(partial[d0:d1])
        return local
    sizes = [b - a for a, b in (block_range(r, world, E_t) for r in range(world))]
    w = max(sizes)
    if all(n == w for n in sizes):
        dist.reduce_scatter_tensor(local, partial, group=group)
        return local
    padded = torch.zeros((world * w,) + tuple(partial.shape[1:]), dtype=partial.dtype, device=partial.device)
    for r in range(world):
        a, b = block_range(r, world, E_t)
        padded[r * w: r * w + (b - a)] = partial[a:b]
    out = torch.empty((w,) + tuple(partial.shape[1:]), dtype=partial.dtype, device=partial.device)
    dist.reduce_scatter_tensor(out, padded, group=group)
    local.copy_(out[: d1 - d0])
    return local


def assemble_p1p1_row_parallel(op: int, mesh, timegrid, params, config, group=None, workspace_bytes=None):
    """p1 x p1 operators (D2, V11) with the pair work split by element rows:
    each rank assembles its rows' symmetrised contribution to ALL blocks into a
    full-size partial (hb_assemble with a row range), one reduce-scatter sums
    the partials into the d-owners' shards.  Results equal the 1-GPU blocks to
    rounding (the cross-rank sum is NCCL's order).  Needs E_t N_x^2 doubles
    per rank (config 2: 38 MB; large configs keep d-sharding)."""
    import torch
    import torch.distributed as dist

    from .assembly import _assemble_operator

    E_t, E_x, N_x = timegrid.n_steps, mesh.n_triangles, mesh.n_vertices
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    d0, d1 = block_range(rank, world, E_t)
    dev = torch.device("cuda", torch.cuda.current_device())
    local = torch.empty((d1 - d0, N_x, N_x), dtype=torch.float64, device=dev)
    rows = row_partition(row_weights_mesh(mesh, config, True, skip_perpendicular=(op == 2)), world)[rank]
    partial = _assemble_operator(op, True, True, True, mesh, timegrid, params, config, None, d_range=(0, E_t),
                                 row_range=rows, workspace_bytes=workspace_bytes)
    if world == 1:
        local.copy_(partial)
    else:
        reduce_scatter_blocks(partial, local, d0, d1, group)
    return ShardedToeplitz(local, d0, d1, E_t, group)


class RowPartialD:
    """D = D2 + alpha^2 curl^T V curl on this rank's blocks [d0, d1) with the
    D2 pair work split by balanced element rows: every rank
    assembles its rows' (symmetrised) p1 x p1 contribution to ALL blocks into
    a full-size partial (``assemble_partial``), the partials are mapped into
    every rank over NVLink (CUDA IPC, once), and the curl kernel of each rank
    reads and sums them in rank order for its own blocks (``combine``,
    hb_curl_combine_parts) -- the cross-rank sum of D2 and the curl transform
    in one kernel: no collective, no halo gaps, and every rank touches only
    1/N of the pairs (the d split makes every rank evaluate every pair).
    Equal to the 1-GPU D to rounding (the partial sums associate
    differently).  Between ``assemble_partial`` and ``combine`` every rank's
    partial must be complete, after ``combine`` no rank may overwrite its
    partial before every rank's combine is done (host barriers)."""

    def __init__(self, mesh, timegrid, params, config, d0: int, d1: int, group=None, device=None):
        import torch
        import torch.distributed as dist

        self.mesh, self.timegrid, self.params, self.config = mesh, timegrid, params, config
        self.d0, self.d1, self.group = d0, d1, group
        E_t, N_x = timegrid.n_steps, mesh.n_vertices
        world = dist.get_world_size(group) if dist.is_initialized() else 1
        rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.world = world
        dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.rows = row_partition(row_weights_mesh(mesh, config, True, skip_perpendicular=True), world)[rank]
        self.partial = torch.zeros((E_t, N_x, N_x), dtype=torch.float64, device=dev)
        addrs, _, self._opened = map_peer_shards(self.partial, (0, E_t), group)
        self.ptrs = torch.as_tensor(np.array(addrs, dtype=np.int64), device=dev)
        self._L = _native.load()

    def assemble_partial(self, workspace_bytes=None, stream=None, stats=None):
        from .assembly import _assemble_operator

        if self.rows[1] > self.rows[0]:
            _assemble_operator(2, True, True, True, self.mesh, self.timegrid, self.params, self.config, None,
                               d_range=(0, self.timegrid.n_steps), row_range=self.rows, out=self.partial,
                               workspace_bytes=workspace_bytes, stream=stream, stats=stats)

    def combine(self, V_local, out, stream=None):
        from .device import device_tables

        if self.d1 <= self.d0:
            return out
        tabs = device_tables(self.mesh, self.config, V_local.device)
        _native.call("hb_curl_combine_parts", tabs.desc(True), self.d1 - self.d0, float(self.params.alpha),
                     _native.ptr(tabs.t["curls"]), _native.ptr(V_local), self.world, _native.ptr(self.ptrs),
                     self.d0, _native.ptr(out), _native.stream_handle(stream))
        return out

    def close(self):
        for pv, o in self._opened:
            self._L.hb_ipc_close(pv, o)
        self._opened = []


def hypersingular_rows_peer(mesh, timegrid, params, config, V_local, d0: int, d1: int, group=None, out=None,
                            workspace_bytes=None):
    """One-shot RowPartialD: D's blocks [d0, d1) on this rank.  ``V_local``:
    V's blocks [d0, d1), complete (after the V stores of every rank)."""
    import torch
    import torch.distributed as dist

    dev = V_local.device
    R = RowPartialD(mesh, timegrid, params, config, d0, d1, group, dev)
    D = out if out is not None else torch.empty((d1 - d0, mesh.n_vertices, mesh.n_vertices), dtype=torch.float64,
                                                device=dev)
    try:
        R.assemble_partial(workspace_bytes)
        torch.cuda.synchronize(dev)
        if R.world > 1:
            dist.barrier(group)                  # every rank's partial is complete
        R.combine(V_local, D)
        torch.cuda.synchronize(dev)
        if R.world > 1:
            dist.barrier(group)                  # no rank reads a partial any more
    finally:
        R.close()
    return D


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


class RowShardedToeplitz:
    """Rows [r0, r1) of every block A^d of a block lower-triangular Toeplitz
    operator on this rank (SURVEY 8(e), row-sharded solve operator):
    ``local`` (n_blocks, r1 - r0, C).  Vectors are replicated (E_t, n) time-
    major arrays, as in the 1-GPU solver, so ``fgmres`` runs unchanged on
    every rank.

    * ``apply``: the local rows of y = A x from the replicated x, then ONE
      all-gather of the row pieces -- the density all-gather of the solve.
    * ``forward_solve``: in tiles of 8 steps as hb_forward_solve_ws -- per tile
      the local rows of the far history (one pass over the local blocks), per
      step the near terms, one all-gather of h^k (R values) and
      x^k = (A^0)^{-1} (rhs^k - h^k) on every rank (the inverse is
      replicated: A^0's rows are gathered once).

    The per-rank kernels are the methods ``local_apply`` / ``local_history_far``
    / ``local_history`` / ``inv_apply`` (tests on CPU replace them by numpy stand-ins)."""

    def __init__(self, local, r0: int, r1: int, n_rows: int, group=None):
        if local.shape[1] != r1 - r0:
            raise ValueError("local must hold rows [r0, r1) of every block")
        self.local, self.r0, self.r1, self.n_rows, self.group = local, r0, r1, n_rows, group
        self._inv = None

    @property
    def n_blocks(self):
        return self.local.shape[0]

    @property
    def C(self):
        return self.local.shape[2]

    def _world(self):
        import torch.distributed as dist

        if not dist.is_initialized():
            return 1, 0
        return dist.get_world_size(self.group), dist.get_rank(self.group)

    def gather_rows(self, piece):
        """(..., r1 - r0) on every rank -> (..., n_rows): one all-gather
        (row ranges of unequal length are padded to the longest)."""
        import torch
        import torch.distributed as dist

        world, _ = self._world()
        if world == 1:
            return piece
        ranges = [block_range(r, world, self.n_rows) for r in range(world)]
        w = max(b - a for a, b in ranges)
        lead = tuple(piece.shape[:-1])
        send = torch.zeros((w,) + lead, dtype=piece.dtype, device=piece.device)
        send[: piece.shape[-1]] = piece.movedim(-1, 0)
        buf = torch.empty((world * w,) + lead, dtype=piece.dtype, device=piece.device)
        dist.all_gather_into_tensor(buf, send, group=self.group)
        rows = torch.cat([buf[r * w: r * w + (b - a)] for r, (a, b) in enumerate(ranges)])
        return rows.movedim(0, -1).contiguous()

    # ---- per-rank kernels ----
    def local_apply(self, x):
        import torch

        from .solver import _workspace

        E_t = x.shape[0]
        R = self.r1 - self.r0
        y = torch.empty((E_t, R), dtype=torch.float64, device=x.device)
        need = _native.load().hb_toeplitz_apply_workspace(self.n_blocks, R, self.C, 0, 0, E_t)
        ws = _workspace(x.device, need)
        _native.call("hb_toeplitz_apply_ws", self.n_blocks, R, self.C, _native.ptr(self.local), 0, 0, E_t,
                     _native.ptr(x), _native.ptr(y), _native.ptr(ws) if need else None, int(need),
                     _native.stream_handle())
        return y

    def local_history_far(self, x, k0: int, nk: int):
        """Local rows of the far history of the step tile [k0, k0 + nk): terms
        with k - d < k0, (nk, r1 - r0) (hb_forward_history_far)."""
        import torch

        H = torch.empty((nk, self.r1 - self.r0), dtype=torch.float64, device=x.device)
        _native.call("hb_forward_history_far", self.n_blocks, self.r1 - self.r0, self.C, _native.ptr(self.local), k0,
                     nk, _native.ptr(x), _native.ptr(H), _native.stream_handle())
        return H

    def local_history(self, x, k: int, k0: int = 0, Hk=None):
        """Local rows of h^k: Hk (the far terms, if given) + the near terms
        d = 1..k - k0 of step k of the tile starting at k0 (k - k0 < 8,
        hb_forward_history_near)."""
        import torch

        h = torch.empty(self.r1 - self.r0, dtype=torch.float64, device=x.device)
        _native.call("hb_forward_history_near", self.n_blocks, self.r1 - self.r0, self.C, _native.ptr(self.local), k,
                     k0, _native.ptr(x), _native.ptr(Hk) if Hk is not None else None, _native.ptr(h),
                     _native.stream_handle())
        return h

    def inv_apply(self, inv, rhs_k, h):
        import torch

        x = torch.empty(inv.shape[0], dtype=torch.float64, device=inv.device)
        _native.call("hb_inv_apply", inv.shape[0], _native.ptr(inv), _native.ptr(rhs_k), _native.ptr(h),
                     _native.ptr(x), _native.stream_handle())
        return x

    def inverse(self):
        """(A^0)^{-1}, replicated (A^0's rows gathered once, then inverted
        on every rank -- the reference factorises A^0, solver.py:176)."""
        import torch

        if self._inv is None:
            if self.n_rows != self.C:
                raise ValueError("forward substitution needs square blocks")
            A0 = self.gather_rows(self.local[0].T.contiguous()).T.contiguous()
            self._inv = torch.linalg.inv(A0).contiguous()
        return self._inv

    # ---- operator ----
    def apply(self, x):
        """y = A x for replicated x (E_t, C) (or flat) -> replicated y (E_t, n_rows)."""
        flat = x.dim() == 1
        x = x.reshape(-1, self.C)
        if x.shape[0] > self.n_blocks:
            raise ValueError("more time steps than stored blocks")
        y = self.gather_rows(self.local_apply(x.contiguous()))
        return y.reshape(-1) if flat else y

    def forward_solve(self, rhs):
        """Causal time marching, one all-gather of h^k per step k >= 1."""
        if rhs.dim() == 1:
            return self.forward_solve(rhs.reshape(-1, self.n_rows)).reshape(-1)
        import torch

        inv = self.inverse()
        E_t = rhs.shape[0]
        if E_t > self.n_blocks:
            raise ValueError("more time steps than stored blocks")
        rhs = rhs.contiguous()
        x = torch.zeros((E_t, self.C), dtype=torch.float64, device=rhs.device)
        for k0 in range(0, E_t, FORWARD_TILE):   # the tiles of hb_forward_solve_ws, same per-row sums
            nk = min(FORWARD_TILE, E_t - k0)
            H = self.local_history_far(x, k0, nk) if k0 > 0 else None
            for k in range(k0, k0 + nk):
                h = (self.gather_rows(self.local_history(x, k, k0, H[k - k0] if H is not None else None))
                     if k > 0 else None)
                x[k] = self.inv_apply(inv, rhs[k], h)
        return x

    def solve(self, rhs, rel_tol: float = 1e-10, max_iter: int = 500, restart: int = 50):
        """A x = rhs by FGMRES right-preconditioned with the forward
        substitution (the Dirichlet solve of study.py:133-136), replicated
        on every rank; returns (x, SolveReport)."""
        from .solver import LinearOperator, fgmres

        return fgmres(LinearOperator(self.apply), rhs, rel_tol=rel_tol, max_iter=max_iter, restart=restart,
                      right_precond=self.forward_solve)


def row_shards_from_d_shards(shard: ShardedToeplitz, group=None):
    """Re-distribute a d-sharded operator (blocks [d0, d1), all rows) into
    row shards (all blocks, rows block_range(rank, world, R)): one
    all-to-all (each rank sends every other rank that rank's rows of its
    blocks).  Non-transposed operators only."""
    import torch
    import torch.distributed as dist

    if shard.transpose:
        raise ValueError("row sharding of a transposed view: shard the stored operator instead")
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    nb_all, R, C = shard.n_blocks, shard.local.shape[1], shard.local.shape[2]
    if world == 1:
        return RowShardedToeplitz(shard.local, 0, R, R, group)
    rows = [block_range(r, world, R) for r in range(world)]
    dr = [block_range(r, world, nb_all) for r in range(world)]
    r0, r1 = rows[rank]
    send = torch.cat([shard.local[:, a:b, :].reshape(-1) for a, b in rows])
    in_splits = [(shard.d1 - shard.d0) * (b - a) * C for a, b in rows]
    out_splits = [(e - s) * (r1 - r0) * C for s, e in dr]
    recv = torch.empty(sum(out_splits), dtype=shard.local.dtype, device=shard.local.device)
    dist.all_to_all_single(recv, send, out_splits, in_splits, group=group)
    local = recv.reshape(nb_all, r1 - r0, C)   # senders in rank order = blocks in d order
    return RowShardedToeplitz(local, r0, r1, R, group)


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


# ---------------------------------------------------------------------------
# potentials: points are independent
# ---------------------------------------------------------------------------
def represent_grid_sharded(w, u, xs, mesh, timegrid, params, config=None, group=None, gather: bool = True):
    """``field.represent_grid`` with the evaluation points split across the
    ranks: rank r evaluates the contiguous point range block_range(r, world,
    M) (every rank holds the densities -- 2.4 MB at config 4 -- so there is
    no collective on the compute path) and, with ``gather``, one all-gather
    assembles the (M, n_times) result on every rank (rows in point order;
    over gloo the gather goes through host memory).  Returns the gathered
    device tensor, or (local rows, (p0, p1)) without ``gather``.  Each
    point's values are bitwise the 1-GPU ones (a point is evaluated by one
    rank with the same kernel)."""
    import torch
    import torch.distributed as dist

    from .field import represent_grid
    from .quadrature import QuadratureConfig

    config = config if config is not None else QuadratureConfig()
    xs = np.ascontiguousarray(np.asarray(xs, dtype=np.float64).reshape(-1, 3))
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    M = xs.shape[0]
    p0, p1 = block_range(rank, world, M)
    n_t = timegrid.n_steps
    if p1 > p0:
        local = represent_grid(w, u, xs[p0:p1], mesh, timegrid, params, config, return_device=True)
    else:
        local = torch.empty((0, n_t), dtype=torch.float64, device=torch.device("cuda", torch.cuda.current_device()))
    if not gather:
        return local, (p0, p1)
    if world == 1:
        return local
    width = -(-M // world)   # block_range sizes differ by at most one: pad to the largest
    host = dist.get_backend(group) == "gloo"
    buf = torch.zeros((width, local.shape[1]), dtype=torch.float64, device="cpu" if host else local.device)
    buf[: p1 - p0] = local.cpu() if host else local
    parts = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(parts, buf, group=group)
    rows = []
    for r in range(world):
        a, b = block_range(r, world, M)
        rows.append(parts[r][: b - a])
    return torch.cat(rows).to(local.device)


def dirichlet_solve_row_sharded(mesh, timegrid, params, config, datum, group=None, rel_tol: float = 1e-10,
                                workspace_bytes=None, timings=None):
    """The Dirichlet problem of BASELINE config 2/5 across the ranks of
    ``group`` (reference study.py:96-136, solver.py:47-73 / 165-184):

      1. V and K row-sharded (``assemble_row_sharded``: balanced pair work,
         finalize stores into the row owners' shards over NVLink);
      2. g = the X10 projection of ``datum`` (device, replicated: every rank
         projects the same data), rhs rows = 1/2 (M g)[rows] + K[rows] g,
         ONE all-gather of the rhs rows; K is dropped;
      3. FGMRES right-preconditioned by forward substitution on the row
         shards: one all-gather of the density rows per matvec and one of
         h^k (R values) per forward-substitution step -- the only
         collectives of the data path.

    Returns (x, SolveReport, V rows); ``timings`` (dict) receives the device
    times (ms, max over ranks is the caller's business) of the phases."""
    import torch

    from .assembly import assemble_mass
    from .field import project_to_space
    from .solver import apply_toeplitz

    ev = lambda: torch.cuda.Event(enable_timing=True)   # noqa: E731
    marks = [ev()]
    marks[0].record()
    V = assemble_row_sharded(0, False, False, True, mesh, timegrid, params, config, group, workspace_bytes)
    marks.append(ev()); marks[-1].record()
    K = assemble_row_sharded(1, False, True, False, mesh, timegrid, params, config, group, workspace_bytes)
    marks.append(ev()); marks[-1].record()
    g = project_to_space(datum, mesh, timegrid, "X10", return_device=True)
    Mg = apply_toeplitz(assemble_mass(mesh, timegrid), g)
    rhs_rows = 0.5 * Mg[:, K.r0:K.r1] + K.local_apply(g.contiguous())
    rhs = V.gather_rows(rhs_rows.contiguous())
    del K
    marks.append(ev()); marks[-1].record()
    x, rep = V.solve(rhs, rel_tol=rel_tol)
    marks.append(ev()); marks[-1].record()
    if timings is not None:
        torch.cuda.synchronize()
        for name, a, b in (("assemble_V", 0, 1), ("assemble_K", 1, 2), ("rhs", 2, 3), ("solve", 3, 4)):
            timings[name] = marks[a].elapsed_time(marks[b])
    return x, rep, V
