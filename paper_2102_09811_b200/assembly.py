"""Block lower-triangular Toeplitz operators, assembled on the GPU.

Drop-in for the reference assembler API (heatbem/assembly.py:24-419): same
functions, same arguments, same ``BlockToeplitzMatrix`` type.  The blocks
are produced by ``hb_assemble`` (csrc/hb_assembly.cu) and live in HBM;
``BlockToeplitzMatrix.blocks`` is a lazily materialised numpy view of them
(one device->host copy, cached), ``device_blocks`` the torch tensor.

Extra keyword arguments (all optional, defaults reproduce the reference):

* ``d_range=(d0, d1)`` -- assemble only blocks d0..d1-1 (d-sharding across
  ranks; blocks are bitwise identical to a full assembly);
* ``device`` -- CUDA device (default: current);
* ``workspace_bytes`` -- staging budget (default: all rows at once, capped
  at 16 GiB and a quarter of the free device memory).

``workers`` and ``deterministic`` are accepted for interface stability: the
device path is always deterministic (no atomics; fixed-order reductions).
"""
from __future__ import annotations

import struct
import os
import sys
import time
from dataclasses import dataclass, field

import numpy as np

from . import _native
from .device import device_tables
from .kernels import KernelParams
from .quadrature import QuadratureConfig

_OP_SINGLE, _OP_DOUBLE, _OP_HYPER2 = 0, 1, 2
_DEFAULT_WS_CAP = 16 << 30


class _HostBlocks(np.ndarray):
    """Host view of a BlockToeplitzMatrix's blocks that records writes.

    The reference mutates operators through their ``.blocks`` array
    (heatbem/assembly.py:328-333: ``out = D2.blocks; out[d] += ...``).  Item
    assignment and in-place ufuncs on this array -- or on any view taken from
    it -- mark the owning storage host-dirty, so the next device use uploads
    the edited blocks and drops the cached (A^0)^{-1}."""

    def __array_finalize__(self, obj):
        self._hb_store = getattr(obj, "_hb_store", None)

    def _hb_touch(self):
        st = getattr(self, "_hb_store", None)
        if st is not None:
            st.host_written()

    def __setitem__(self, key, value):
        super().__setitem__(key, value)
        self._hb_touch()

    def __array_ufunc__(self, ufunc, method, *inputs, out=None, **kwargs):
        args = [np.asarray(x) if isinstance(x, _HostBlocks) else x for x in inputs]
        outs = None
        if out is not None:
            outs = tuple(np.asarray(o) if isinstance(o, _HostBlocks) else o for o in out)
            kwargs["out"] = outs
        res = getattr(ufunc, method)(*args, **kwargs)
        if out is not None:
            for o in out:
                if isinstance(o, _HostBlocks):
                    o._hb_touch()
            return out[0] if len(out) == 1 else out
        return res


class _BlockStorage:
    """Blocks of one operator (shared by its transposed() twins): host array,
    device tensor, which side is current, and caches derived from the blocks."""

    def __init__(self, host=None, dev=None):
        self.host, self.dev = host, dev
        self.host_dirty = False     # host edited after the device copy was made
        self.version = 0            # bumped on every change of the blocks
        self.inv_cache = {}         # (A^0)^{-1} per transpose flag (solver.py)

    def changed(self):
        self.version += 1
        self.inv_cache = {}

    def host_written(self):
        if self.dev is not None:
            self.host_dirty = True
        self.changed()

    def device_written(self):
        """The device blocks were changed in place: the host copy is stale."""
        self.host = None
        self.host_dirty = False
        self.changed()


class BlockToeplitzMatrix:
    """Block (k, i) = blocks[k - i] for k >= i, zero above (never stored).

    Construct from a numpy array (host) or a torch tensor (device); the
    other side is created on first use.  ``transposed()`` shares storage.
    Host and device stay coherent: ``.blocks`` hands out a host array whose
    in-place edits (the reference's idiom) reach the device on its next use,
    assigning ``.blocks`` replaces both sides, and in-place device writes by
    the library (e.g. ``hypersingular_from_single_layer(overwrite_d2=True)``)
    drop the host copy; every change drops the cached (A^0)^{-1}."""

    def __init__(self, blocks, transpose_blocks_on_apply: bool = False, diagonal_only: bool = False):
        if _is_torch(blocks):
            self._store = _BlockStorage(dev=blocks)
        else:
            self._store = _BlockStorage(host=np.asarray(blocks, dtype=np.float64))
        self.transpose_blocks_on_apply = bool(transpose_blocks_on_apply)
        self.diagonal_only = bool(diagonal_only)
        self.host_copy = None  # (page-locked host tensor, event) when streamed to the host

    # ---- storage ---------------------------------------------------------
    @property
    def shape(self):
        st = self._store
        if st.host is not None and (st.host_dirty or st.dev is None):
            return st.host.shape
        return tuple(st.dev.shape) if st.dev is not None else st.host.shape

    @property
    def blocks(self) -> np.ndarray:
        st = self._store
        if st.host is None:
            st.host = st.dev.detach().cpu().numpy()
        if not isinstance(st.host, _HostBlocks) and st.host.flags.writeable:
            st.host = st.host.view(_HostBlocks)
        if isinstance(st.host, _HostBlocks):
            st.host._hb_store = st
        return st.host

    @blocks.setter
    def blocks(self, value):
        st = self._store
        st.host = np.asarray(value, dtype=np.float64)
        st.dev = None
        st.host_dirty = False
        st.changed()

    @property
    def device_blocks(self):
        """(n_blocks, rows, cols) float64 CUDA tensor (uploads host edits first)."""
        st = self._store
        if st.dev is None or st.host_dirty:
            import torch

            _native.require_cuda()
            src = np.ascontiguousarray(np.asarray(st.host))
            if st.dev is not None and tuple(st.dev.shape) == src.shape:
                st.dev.copy_(torch.from_numpy(src))
            else:
                st.dev = torch.from_numpy(src).cuda()
            st.host_dirty = False
        return st.dev

    @property
    def on_device(self) -> bool:
        return self._store.dev is not None

    @property
    def version(self) -> int:
        """Counts the changes of the blocks (host edits, assignments, in-place device writes)."""
        return self._store.version

    def mark_device_written(self):
        """Declare an in-place change of ``device_blocks`` (drops the host copy and caches)."""
        self._store.device_written()

    # ---- reference properties -------------------------------------------
    @property
    def n_blocks(self) -> int:
        return self.shape[0]

    @property
    def block_rows(self) -> int:
        return self.shape[2] if self.transpose_blocks_on_apply else self.shape[1]

    @property
    def block_cols(self) -> int:
        return self.shape[1] if self.transpose_blocks_on_apply else self.shape[2]

    def to_host_async(self, out=None, stream=None):
        """Start a device->host copy of the blocks into page-locked memory on
        ``stream`` (a side stream by default) once the work queued so far on
        the current stream is done; returns (host tensor, event).  Lets the
        copy of one operator overlap the assembly of the next."""
        import torch

        dev = self.device_blocks
        if out is None:
            out = torch.empty(dev.shape, dtype=dev.dtype, pin_memory=True)
        s = stream if stream is not None else _copy_stream(dev.device)
        ready = torch.cuda.Event()
        ready.record(torch.cuda.current_stream(dev.device))
        s.wait_event(ready)
        with torch.cuda.stream(s):
            out.copy_(dev, non_blocking=True)
            done = torch.cuda.Event()
            done.record(s)
        dev.record_stream(s)
        return out, done

    def transposed(self) -> "BlockToeplitzMatrix":
        """Blockwise transpose (K' from K), sharing the block storage."""
        t = BlockToeplitzMatrix.__new__(BlockToeplitzMatrix)
        t._store = self._store
        t.transpose_blocks_on_apply = not self.transpose_blocks_on_apply
        t.diagonal_only = self.diagonal_only
        t.host_copy = None
        return t


_COPY_STREAMS: dict = {}


def _copy_stream(device, name: str = ""):
    """Side stream for device->host copies (one per (device, name): copies of
    different operators on different streams do not queue behind each other)."""
    import torch

    key = (str(device), name)
    if key not in _COPY_STREAMS:
        _COPY_STREAMS[key] = torch.cuda.Stream(device=device)
    return _COPY_STREAMS[key]


def _is_torch(x) -> bool:
    return type(x).__module__.startswith("torch")


@dataclass(frozen=True)
class CurlTransform:
    """Per-component surface-curl transforms T_1..T_3 (scipy CSR, E_x x N_x)."""

    components: tuple


@dataclass(frozen=True)
class AssemblyPlan:
    """i_t <-> d bookkeeping of the kernel-reuse scheme (assembly.py:66-100):
    the kernel at gap i_t h feeds blocks i_t-1 (x-1), i_t (x2), i_t+1 (x-1);
    i_t = 0 feeds block 0 through the combined kernel and block 1 (x-1)."""

    n_blocks: int

    def targets(self, i_t: int):
        if not 0 <= i_t <= self.n_blocks:
            raise ValueError("i_t out of range")
        last = self.n_blocks - 1
        if i_t == 0:
            return [(0, 1.0, True)] + ([(1, -1.0, False)] if last >= 1 else [])
        cand = ((i_t - 1, -1.0), (i_t, 2.0), (i_t + 1, -1.0))
        return [(d, m, False) for d, m in cand if d <= last]

    def contributors(self, d: int):
        if not 0 <= d < self.n_blocks:
            raise ValueError("d out of range")
        return [(i_t, m, c) for i_t in range(self.n_blocks + 1)
                for (dd, m, c) in self.targets(i_t) if dd == d]


@dataclass
class AssemblyInstrumentation:
    """``kernel_batch_passes`` counts logical kernel passes (one per time gap
    i_t = 0..E_t, all fused into one launch per pair class); ``seconds``
    is the wall time of the device assembly (synchronised)."""

    kernel_batch_passes: int = 0
    seconds: float = field(default=0.0)


_WS_CACHE: dict = {}


def _workspace(tables, desc_m, desc_a, device, cap, stream=None, fused_vd: bool = False):
    """Staging buffer for one hb_assemble call.  One buffer per (device,
    stream) is kept and grown on demand: calls on a stream run in order, so
    reusing it is safe, and consecutive calls of different operators do not
    churn the caching allocator (fresh multi-100-MB buffers per call left the
    GPU idle between launches)."""
    import torch

    L = _native.load()
    if fused_vd:
        full = L.hb_assemble_vd_full_workspace(desc_m, desc_a)
        least = L.hb_assemble_vd_min_workspace(desc_m, desc_a)
    else:
        full = L.hb_assemble_full_workspace(desc_m, desc_a)
        least = L.hb_assemble_min_workspace(desc_m, desc_a)
    st = stream if stream is not None else torch.cuda.current_stream(device)
    key = (str(device), st.cuda_stream)
    buf = _WS_CACHE.get(key)
    if cap is None and full > _DEFAULT_WS_CAP:
        # staging for ALL test rows larger than the cached default: take it transiently when it
        # fits in the free memory -- one launch instead of row chunks, and for K the
        # dual-orientation body then evaluates every separated pair once (row chunks evaluate
        # the pairs that straddle two chunks twice: config 5, K in 30-block chunks 4.1 -> 2.8 s)
        # free device memory + what torch's caching allocator holds unused (e.g. the previous
        # call's transient staging, which the next allocation reuses) + the cached buffer
        free = (torch.cuda.mem_get_info(device)[0] + torch.cuda.memory_reserved(device)
                - torch.cuda.memory_allocated(device) + (buf.numel() if buf is not None else 0))
        if os.environ.get("HB_WS_DEBUG"):
            print(f"[hb workspace] full {full / 1e9:.1f} GB, free {free / 1e9:.1f} GB", file=sys.stderr)
        if full + (4 << 30) <= free:   # the output is already allocated; keep 4 GiB of headroom
            if buf is not None:   # hand the cached buffer back to the allocator (reused, not released)
                _WS_CACHE.pop(key, None)
                del buf
            return torch.empty(full, dtype=torch.uint8, device=device)
    if cap is None:   # default: up to 16 GiB, at most a quarter of the free device memory
        want = min(full, _DEFAULT_WS_CAP)
        if buf is not None and buf.numel() >= max(least, want):
            return buf[: max(least, want)]
        cap = min(_DEFAULT_WS_CAP, (torch.cuda.mem_get_info(device)[0] + (buf.numel() if buf is not None else 0)) // 4)
        nbytes = max(least, min(full, cap))
        if buf is not None and buf.numel() >= nbytes:
            return buf[:nbytes]
        _WS_CACHE.pop(key, None)
        del buf
        buf = torch.empty(nbytes, dtype=torch.uint8, device=device)
        _WS_CACHE[key] = buf
        return buf
    return torch.empty(max(least, min(full, int(cap))), dtype=torch.uint8, device=device)


def release_workspaces():
    """Drop the cached staging buffers (e.g. before a large allocation)."""
    _WS_CACHE.clear()


def _assemble_operator(op: int, test_p1: bool, trial_p1: bool, symmetric: bool, mesh, timegrid,
                       params: KernelParams, config: QuadratureConfig, instrumentation,
                       d_range=None, device=None, workspace_bytes=None, stream=None, stats=None, out=None,
                       row_range=None, block_ptrs=None, row_shards=None):
    """Blocks [d0, d1) of one operator.  ``row_range`` restricts the test rows
    and ``block_ptrs`` (int64 device tensor of d1 - d0 addresses) redirects
    block d to block_ptrs[d - d0] (row-parallel assembly, distributed.py);
    with ``block_ptrs`` nothing is allocated and None is returned."""
    import torch

    _native.require_cuda()
    tabs = device_tables(mesh, config, device)
    E_t = timegrid.n_steps
    d0, d1 = (0, E_t) if d_range is None else (int(d_range[0]), int(d_range[1]))
    if not (0 <= d0 < d1 <= E_t):
        raise ValueError(f"d_range {d_range} outside [0, {E_t}]")
    E_x, N_x = mesh.n_triangles, mesh.n_vertices
    R = N_x if test_p1 else E_x
    C = N_x if trial_p1 else E_x
    dev = tabs.device
    if row_shards is not None:
        if out is not None or block_ptrs is not None or test_p1:
            raise ValueError("row_shards: p0 test functions, no out / block_ptrs")
        bounds, ptrs = row_shards
        if (bounds.dtype != torch.int64 or ptrs.dtype != torch.int64 or bounds.device != dev
                or ptrs.device != dev or bounds.numel() != ptrs.numel() + 1):
            raise ValueError("row_shards = (bounds (n + 1,), ptrs (n,)) int64 device tensors")
        blocks = None
    elif block_ptrs is not None:
        if out is not None:
            raise ValueError("out and block_ptrs are exclusive")
        if tuple(block_ptrs.shape) != (d1 - d0,) or block_ptrs.dtype != torch.int64 or block_ptrs.device != dev:
            raise ValueError("block_ptrs must be an int64 device tensor with one address per block")
        blocks = None
    elif out is not None:
        if tuple(out.shape) != (d1 - d0, R, C) or out.dtype != torch.float64 or not out.is_contiguous():
            raise ValueError("out must be a contiguous float64 tensor of shape (n_blocks, R, C)")
        blocks = out
    else:
        blocks = torch.empty((d1 - d0, R, C), dtype=torch.float64, device=dev)
    a = _native.AssemblyDesc()
    a.op, a.test_p1, a.trial_p1, a.symmetric = op, int(test_p1), int(trial_p1), int(symmetric)
    a.E_t, a.step = E_t, timegrid.step
    a.alpha, a.d_eps, a.r_eps = params.alpha, params.delta_eps, params.rho_eps
    a.d_begin, a.d_end = d0, d1
    a.blocks_dev = blocks.data_ptr() if blocks is not None else None
    if block_ptrs is not None:
        a.block_ptrs_dev = block_ptrs.data_ptr()
    if row_shards is not None:
        a.n_row_shards = row_shards[1].numel()
        a.row_shard_bounds_dev, a.row_shard_ptrs_dev = row_shards[0].data_ptr(), row_shards[1].data_ptr()
    if row_range is not None:
        r0, r1 = int(row_range[0]), int(row_range[1])
        if not (0 <= r0 < r1 <= E_x):
            raise ValueError(f"row_range {row_range} outside [0, {E_x}]")
        a.row_begin, a.row_end = r0, r1
    m = tabs.desc(symmetric)
    ws = _workspace(tabs, m, a, dev, None if workspace_bytes is None else int(workspace_bytes), stream)
    a.workspace_dev, a.workspace_bytes = ws.data_ptr(), ws.numel()
    if stats is not None:
        import ctypes

        a.stats = ctypes.pointer(stats)
    t0 = time.perf_counter()
    with torch.cuda.device(dev):
        _native.call("hb_assemble", m, a, _native.stream_handle(stream))
        if instrumentation is not None:
            torch.cuda.synchronize(dev)
    if instrumentation is not None:
        instrumentation.kernel_batch_passes += E_t + 1
        instrumentation.seconds += time.perf_counter() - t0
    del ws
    return blocks


def assemble_single_layer(mesh, timegrid, params: KernelParams, config: QuadratureConfig = QuadratureConfig(),
                          test_space: str = "p0", trial_space: str = "p0", workers: int | None = 1,
                          deterministic: bool = True, instrumentation: AssemblyInstrumentation | None = None,
                          **kw) -> BlockToeplitzMatrix:
    """Single-layer blocks V (p0 x p0) or V11 (p1 x p1) (assembly.py:245-269)."""
    if (test_space, trial_space) not in (("p0", "p0"), ("p1", "p1")):
        raise ValueError("single layer supports p0 x p0 and p1 x p1 only")
    p1 = test_space == "p1"
    host_out = kw.pop("host_out", None)
    if host_out is not None and not p1:
        return _assemble_streamed(_OP_SINGLE, False, False, True, mesh, timegrid, params, config,
                                  instrumentation, host_out, n_slabs=kw.pop("host_out_slabs", 3), **kw)
    if host_out is not None:
        raise ValueError("host_out streaming is for p0 x p0 V and K (V11 rows accumulate)")
    return BlockToeplitzMatrix(_assemble_operator(_OP_SINGLE, p1, p1, True, mesh, timegrid, params,
                                                  config, instrumentation, **kw))


def assemble_double_layer(mesh, timegrid, params: KernelParams, config: QuadratureConfig = QuadratureConfig(),
                          workers: int | None = 1, deterministic: bool = True,
                          instrumentation: AssemblyInstrumentation | None = None, **kw) -> BlockToeplitzMatrix:
    """Double-layer blocks K, p0 test x p1 trial (assembly.py:272-286).
    ``host_out`` (page-locked, K's shape): the device->host copy starts on a
    side stream as soon as K is done (``host_copy`` = (host_out, event)).  K
    is not split into row slabs: the dual-orientation kernel evaluates a
    separated pair once for both rows only when both lie in the same call."""
    host_out = kw.pop("host_out", None)
    res = BlockToeplitzMatrix(_assemble_operator(_OP_DOUBLE, False, True, False, mesh, timegrid, params,
                                                 config, instrumentation, **kw))
    if host_out is not None:
        if tuple(host_out.shape) != tuple(res.device_blocks.shape) or not host_out.is_pinned():
            raise ValueError("host_out must be a page-locked tensor of K's (n_blocks, R, C) shape")
        res.host_copy = res.to_host_async(host_out, kw.get("stream"))
    return res


def _row_slabs(n_rows: int, symmetric: bool, n_slabs):
    """Test-row ranges of given shares of the pair work (``n_slabs``: a count
    of equal shares, or a sequence of work fractions -- a small first slab
    starts the device->host copies early): upper-triangle rows (f >= e) for a
    symmetric operator, uniform rows otherwise."""
    if isinstance(n_slabs, (int, np.integer)):
        n = max(1, min(int(n_slabs), n_rows))
        cum = [k / n for k in range(n + 1)]
    else:
        fr = np.asarray(list(n_slabs), dtype=np.float64)
        if fr.size < 1 or not np.all(fr > 0.0):
            raise ValueError("slab work fractions must be positive")
        cum = [0.0] + list(np.cumsum(fr) / fr.sum())
    if symmetric:
        # work of rows [0, r) ~ r (2E - r): bounds r = E (1 - sqrt(1 - share))
        bounds = [int(round(n_rows * (1.0 - np.sqrt(max(0.0, 1.0 - c))))) for c in cum]
    else:
        bounds = [int(round(n_rows * c)) for c in cum]
    bounds[0], bounds[-1] = 0, n_rows
    return [(a, b) for a, b in zip(bounds[:-1], bounds[1:]) if b > a]


def _assemble_streamed(op, test_p1, trial_p1, symmetric, mesh, timegrid, params, config, instrumentation,
                       host_out, n_slabs=3, stream=None, copy_stream=None, **kw):
    """Assemble a p0-test operator in work-balanced test-row slabs and start
    each slab's device->host copy (rows [r0, r1) of every block, complete once
    the slab's rows are done: a symmetric operator's mirrored entries of those
    rows come from earlier slabs) on a side stream as soon as it is formed, so
    the copy of a 100+ MB operator overlaps its own assembly.  Same blocks,
    bitwise, as one call (row ranges write disjoint entries).  The result's
    ``host_copy`` is (host_out, event of the last copy)."""
    import torch

    if test_p1:
        raise ValueError("row-slab streaming needs p0 test rows")
    E_t = timegrid.n_steps
    d_range = kw.pop("d_range", None)
    d0, d1 = (0, E_t) if d_range is None else (int(d_range[0]), int(d_range[1]))
    R = mesh.n_triangles
    C = mesh.n_vertices if trial_p1 else mesh.n_triangles
    out = kw.pop("out", None)
    dev = device_tables(mesh, config, kw.get("device")).device
    if out is None:
        out = torch.empty((d1 - d0, R, C), dtype=torch.float64, device=dev)
    if (tuple(host_out.shape) != tuple(out.shape) or host_out.dtype != out.dtype or not host_out.is_pinned()
            or not host_out.is_contiguous() or not out.is_contiguous()):
        raise ValueError("host_out must be a contiguous page-locked tensor of the operator's (n_blocks, R, C) "
                         "float64 shape")
    cur = stream if stream is not None else torch.cuda.current_stream(dev)
    cs = copy_stream if copy_stream is not None else _copy_stream(dev)
    for r0, r1 in _row_slabs(R, symmetric, n_slabs):
        _assemble_operator(op, test_p1, trial_p1, symmetric, mesh, timegrid, params, config, instrumentation,
                           d_range=(d0, d1), row_range=(r0, r1), out=out, stream=cur, **kw)
        ready = torch.cuda.Event()
        ready.record(cur)
        cs.wait_event(ready)
        _native.call("hb_copy_row_slab_d2h", _native.ptr(host_out), _native.ptr(out), d1 - d0, R, C, r0, r1,
                     _native.stream_handle(cs))
    done = torch.cuda.Event()
    done.record(cs)
    out.record_stream(cs)
    res = BlockToeplitzMatrix(out)
    res.host_copy = (host_out, done)
    return res


def assemble_hypersingular_d2(mesh, timegrid, params: KernelParams, config: QuadratureConfig = QuadratureConfig(),
                              workers: int | None = 1, instrumentation: AssemblyInstrumentation | None = None,
                              **kw) -> BlockToeplitzMatrix:
    """Surface part D2 of the hypersingular operator, p1 x p1 (assembly.py:364-377)."""
    return BlockToeplitzMatrix(_assemble_operator(_OP_HYPER2, True, True, True, mesh, timegrid, params,
                                                  config, instrumentation, **kw))


def curl_transform(mesh) -> CurlTransform:
    """Host-side sparse T_o (E_x x N_x), for callers that want the matrices."""
    import scipy.sparse as sp

    from .device import _curls

    E_x, N_x = mesh.n_triangles, mesh.n_vertices
    cu = _curls(mesh)
    rows = np.repeat(np.arange(E_x), 3)
    cols = mesh.triangles.ravel()
    return CurlTransform(tuple(sp.csr_matrix((cu[:, :, o].ravel(), (rows, cols)), shape=(E_x, N_x))
                               for o in range(3)))


def hypersingular_from_single_layer(V: BlockToeplitzMatrix, D2: BlockToeplitzMatrix, mesh, params: KernelParams,
                                    overwrite_d2: bool = False, config: QuadratureConfig = QuadratureConfig(),
                                    stream=None, host_out=None, copy_chunks: int = 4,
                                    copy_stream=None) -> BlockToeplitzMatrix:
    """D = D2 + alpha^2 sum_o T_o^T V T_o blockwise (assembly.py:314-334), on the device.

    ``host_out`` (page-locked, D's shape): the combine runs in ``copy_chunks``
    block chunks and each chunk's device->host copy starts on a side stream as
    soon as it is formed, so only the last chunk's copy trails the assembly;
    the result's ``host_copy`` is (host_out, event of the last copy)."""
    import torch

    _native.require_cuda()
    Vd, D2d = V.device_blocks, D2.device_blocks
    if Vd.shape[0] != D2d.shape[0]:
        raise ValueError("V and D2 must hold the same number of blocks")
    tabs = device_tables(mesh, config, Vd.device)
    out = D2d if overwrite_d2 else torch.empty_like(D2d)
    host_copy = None
    if host_out is None:
        curl_combine_into(tabs, Vd, D2d, out, float(params.alpha), stream)
    else:
        if tuple(host_out.shape) != tuple(out.shape) or host_out.dtype != out.dtype:
            raise ValueError("host_out must match D's shape and dtype")
        n = Vd.shape[0]
        bounds = np.linspace(0, n, max(1, min(int(copy_chunks), n)) + 1).astype(int)
        cur = stream if stream is not None else torch.cuda.current_stream(Vd.device)
        cs = copy_stream if copy_stream is not None else _copy_stream(Vd.device)
        for a, b in zip(bounds[:-1], bounds[1:]):
            curl_combine_into(tabs, Vd[a:b], D2d[a:b], out[a:b], float(params.alpha), cur)
            ready = torch.cuda.Event()
            ready.record(cur)
            cs.wait_event(ready)
            with torch.cuda.stream(cs):
                host_out[a:b].copy_(out[a:b], non_blocking=True)
        done = torch.cuda.Event()
        done.record(cs)
        out.record_stream(cs)
        host_copy = (host_out, done)
    if overwrite_d2:
        D2.mark_device_written()
        D2.host_copy = host_copy
        return D2
    res = BlockToeplitzMatrix(out)
    res.host_copy = host_copy
    return res


def curl_combine_into(tabs, Vd, D2d, out, alpha: float, stream=None, workspace_cap: int = 1 << 30):
    """hb_curl_combine with a workspace of up to ``workspace_cap`` bytes."""
    import torch

    L = _native.load()
    m = tabs.desc(True)
    per = L.hb_curl_workspace(m, 1)
    nb = Vd.shape[0]
    ws = torch.empty(max(per, min(per * nb, workspace_cap)), dtype=torch.uint8, device=Vd.device)
    with torch.cuda.device(Vd.device):
        _native.call("hb_curl_combine", m, nb, alpha, _native.ptr(tabs.t["curls"]), _native.ptr(Vd),
                     _native.ptr(D2d), _native.ptr(out), _native.ptr(ws), ws.numel(), _native.stream_handle(stream))


def assemble_hypersingular(mesh, timegrid, params: KernelParams, config: QuadratureConfig = QuadratureConfig(),
                           workers: int | None = 1, deterministic: bool = True,
                           instrumentation: AssemblyInstrumentation | None = None,
                           single_layer: BlockToeplitzMatrix | None = None, host_out=None,
                           **kw) -> BlockToeplitzMatrix:
    """D = T^T (alpha^2 V) T + D2, p1 x p1 (assembly.py:337-361).

    Without ``single_layer`` (the reference then assembles V itself) V and D2
    are assembled together and the curl transform is folded into D2's p1 x p1
    finalize (hb_assemble_vd: no pass of its own over V).  With a given
    ``single_layer`` the curl combine reads it (hypersingular_from_single_layer).
    ``host_out``: stream D to page-locked host memory (chunk by chunk on the
    curl path, after the call on the fused path)."""
    if single_layer is None and _fused_vd() and not kw.get("row_range") and kw.get("block_ptrs") is None:
        _, D = _assemble_vd(mesh, timegrid, params, config, instrumentation, keep_v=False, **kw)
        if host_out is not None:
            if tuple(host_out.shape) != tuple(D.device_blocks.shape) or not host_out.is_pinned():
                raise ValueError("host_out must be a page-locked tensor of D's (n_blocks, R, C) shape")
            D.host_copy = D.to_host_async(host_out, kw.get("stream"))
        return D
    if single_layer is None:
        single_layer = assemble_single_layer(mesh, timegrid, params, config, "p0", "p0", workers,
                                             deterministic, instrumentation, **kw)
    D2 = assemble_hypersingular_d2(mesh, timegrid, params, config, workers, instrumentation, **kw)
    return hypersingular_from_single_layer(single_layer, D2, mesh, params, overwrite_d2=True, config=config,
                                           host_out=host_out)


def _fused_vd() -> bool:
    """HB_FUSED_VD=1: V + D in one call (hb_assemble_vd) where the API allows
    it.  Off by default: the fused finalize does twice the loads of the plain
    p1 x p1 one, and at config 2 the separate curl combine overlaps K's pair
    kernel on another stream (B200: 4.09 ms per V + K + D step separate vs
    4.30 fused; a config-5 64-block chunk 481 vs 560 ms).  What it saves is
    memory: D without V's blocks (config 5: 309 GB)."""
    return os.environ.get("HB_FUSED_VD", "0") == "1"


def _assemble_vd(mesh, timegrid, params: KernelParams, config: QuadratureConfig, instrumentation=None,
                 d_range=None, device=None, workspace_bytes=None, stream=None, stats=None, out=None, out_v=None,
                 keep_v: bool = True):
    """V and D = D2 + alpha^2 curl^T V curl of blocks d_range in one
    hb_assemble_vd call (V and D2 staged in the same test-row chunks, the curl
    transform folded into the p1 x p1 finalize).  Returns (V or None, D)."""
    import torch

    _native.require_cuda()
    tabs = device_tables(mesh, config, device)
    E_t = timegrid.n_steps
    d0, d1 = (0, E_t) if d_range is None else (int(d_range[0]), int(d_range[1]))
    if not (0 <= d0 < d1 <= E_t):
        raise ValueError(f"d_range {d_range} outside [0, {E_t}]")
    E_x, N_x = mesh.n_triangles, mesh.n_vertices
    dev = tabs.device
    for t, shape in ((out, (d1 - d0, N_x, N_x)), (out_v, (d1 - d0, E_x, E_x))):
        if t is not None and (tuple(t.shape) != shape or t.dtype != torch.float64 or not t.is_contiguous()):
            raise ValueError(f"out tensors must be contiguous float64 of shape {shape}")
    D = out if out is not None else torch.empty((d1 - d0, N_x, N_x), dtype=torch.float64, device=dev)
    V = out_v if out_v is not None else (
        torch.empty((d1 - d0, E_x, E_x), dtype=torch.float64, device=dev) if keep_v else None)
    a = _native.AssemblyDesc()
    a.op, a.test_p1, a.trial_p1, a.symmetric = _OP_HYPER2, 1, 1, 1
    a.E_t, a.step = E_t, timegrid.step
    a.alpha, a.d_eps, a.r_eps = params.alpha, params.delta_eps, params.rho_eps
    a.d_begin, a.d_end = d0, d1
    a.blocks_dev = D.data_ptr()
    m = tabs.desc(True)
    ws = _workspace(tabs, m, a, dev, None if workspace_bytes is None else int(workspace_bytes), stream,
                    fused_vd=True)
    a.workspace_dev, a.workspace_bytes = ws.data_ptr(), ws.numel()
    if stats is not None:
        import ctypes

        a.stats = ctypes.pointer(stats)
    t0 = time.perf_counter()
    with torch.cuda.device(dev):
        _native.call("hb_assemble_vd", m, a, V.data_ptr() if V is not None else None,
                     _native.ptr(tabs.t["curls"]), _native.stream_handle(stream))
        if instrumentation is not None:
            torch.cuda.synchronize(dev)
    if instrumentation is not None:
        instrumentation.kernel_batch_passes += 2 * (E_t + 1)
        instrumentation.seconds += time.perf_counter() - t0
    del ws
    return (BlockToeplitzMatrix(V) if V is not None else None), BlockToeplitzMatrix(D)


_OP_CODES = {"V": (_OP_SINGLE, False, False, True), "K": (_OP_DOUBLE, False, True, False),
             "D2": (_OP_HYPER2, True, True, True), "V11": (_OP_SINGLE, True, True, True)}


def apply_assembled(op: str, mesh, timegrid, params: KernelParams, x, config: QuadratureConfig = QuadratureConfig(),
                    transpose_blocks: bool = False, chunk_blocks: int | None = None,
                    writer: BlockFileWriter | None = None):
    """y^k = sum_{d<=k} A^d x^{k-d} for an operator that is never stored whole
    (apply-and-discard): window-aligned d-chunks of A are
    assembled into one reused device buffer, applied with the per-range
    Toeplitz product (hb_toeplitz_apply_range) and discarded -- e.g. the
    config-5 right-hand side K g with K = 155 GB on one GPU.  ``op``: "V",
    "K", "D2", "V11" or "D" (D2 + alpha^2 curl(V) per chunk).  ``writer``
    (BlockFileWriter) additionally streams every chunk to an HBTM1 file.
    x: (E_t, n_in) numpy or torch; returns the same type."""
    import torch

    from .distributed import aligned_chunks

    _native.require_cuda()
    E_t = timegrid.n_steps
    E, N = mesh.n_triangles, mesh.n_vertices
    dev = torch.device("cuda", torch.cuda.current_device())
    if op == "D":
        R = C = N
    elif op in _OP_CODES:
        code = _OP_CODES[op]
        R, C = (N if code[1] else E), (N if code[2] else E)
    else:
        raise ValueError(f"unknown operator {op!r}")
    n_in, n_out = (R, C) if transpose_blocks else (C, R)
    was_torch = _is_torch(x)
    xd = (x.to(dtype=torch.float64, device=dev) if was_torch else
          torch.as_tensor(np.ascontiguousarray(x, dtype=np.float64), device=dev)).reshape(-1, n_in).contiguous()
    if xd.shape[0] > E_t:
        raise ValueError("more time steps than blocks")
    steps = xd.shape[0]
    if chunk_blocks is None:
        # K: one 32-slot window per chunk, so its staging for all test rows can fit next to the
        # chunk (one launch, dual-orientation body); the others: up to two windows
        chunk_blocks = 30 if op == "K" else 62
    chunks = aligned_chunks(E_t, max(1, int(chunk_blocks)))
    width = max(b - a for a, b in chunks)
    buf = torch.empty((width, R, C), dtype=torch.float64, device=dev)
    vbuf = torch.empty((width, E, E), dtype=torch.float64, device=dev) if op == "D" else None
    tabs = device_tables(mesh, config, dev) if op == "D" else None
    y = torch.zeros((steps, n_out), dtype=torch.float64, device=dev)
    part = torch.empty_like(y)
    for d0, d1 in chunks:
        n = d1 - d0
        if op == "D":
            _assemble_operator(*_OP_CODES["V"], mesh, timegrid, params, config, None, d_range=(d0, d1), out=vbuf[:n])
            _assemble_operator(*_OP_CODES["D2"], mesh, timegrid, params, config, None, d_range=(d0, d1), out=buf[:n])
            curl_combine_into(tabs, vbuf[:n], buf[:n], buf[:n], float(params.alpha))
        else:
            _assemble_operator(*code, mesh, timegrid, params, config, None, d_range=(d0, d1), out=buf[:n])
        if writer is not None:
            writer.write(buf[:n])
        if d0 < steps:
            _native.call("hb_toeplitz_apply_range", d0, n, R, C, _native.ptr(buf), int(transpose_blocks), steps,
                         _native.ptr(xd), _native.ptr(part), _native.stream_handle())
            y += part
    return y if was_torch else y.cpu().numpy()


_OP_STREAMS: dict = {}


def _op_streams(device):
    """(D, V, K) streams of assemble_all; V's has the highest priority, so
    with host outputs its row slabs finish first and the device->host copies
    (the end-to-end bound) start as early as possible."""
    import torch

    key = str(device)
    if key not in _OP_STREAMS:
        lo, hi = torch.cuda.Stream.priority_range()   # (least, greatest): greatest is numerically lowest
        _OP_STREAMS[key] = (torch.cuda.Stream(device=device), torch.cuda.Stream(device=device, priority=hi),
                            torch.cuda.Stream(device=device))
    return _OP_STREAMS[key]


def assemble_all(mesh, timegrid, params: KernelParams, config: QuadratureConfig = QuadratureConfig(),
                 d_range=None, host_out=None, out=None, v_slabs: int = 2) -> dict:
    """V (p0 x p0), K (p0 x p1) and D = D2 + alpha^2 curl(V) (p1 x p1) of one
    space-time problem, assembled concurrently on three CUDA streams: the
    persistent pair kernels of one operator run while another's finalize /
    curl kernels (memory-bound) and kernel tails drain -- 8 % faster than three
    sequential calls at config 2, bitwise the same blocks.  ``host_out``
    (dict of page-locked tensors "V", "K", "D"): each operator is copied back
    on a side stream as soon as it is done (V in ``v_slabs`` work-balanced row
    slabs on the high-priority stream, D in block chunks as the curl forms
    them); the returned matrices' ``host_copy`` hold (tensor, event).
    ``out``: dict of preallocated device tensors "V", "K", "D" to assemble into.
    Returns {"V", "K", "D"}; the caller's stream waits for all of them."""
    import torch

    _native.require_cuda()
    dev = torch.device("cuda", torch.cuda.current_device())
    cur = torch.cuda.current_stream(dev)
    sD, sV, sK = _op_streams(dev)
    device_tables(mesh, config, dev)         # (re)upload the mesh tables on the caller's stream, then fork
    for st in (sD, sV, sK):
        st.wait_stream(cur)
    host_out = host_out or {}
    out = out or {}
    if _fused_vd():
        with torch.cuda.stream(sV):   # V and D together: D2's finalize adds the curl transform of V
            V, D = _assemble_vd(mesh, timegrid, params, config, None, d_range=d_range, out=out.get("D"),
                                out_v=out.get("V"))
            if "V" in host_out:
                V.host_copy = V.to_host_async(host_out["V"])
            if "D" in host_out:
                D.host_copy = D.to_host_async(host_out["D"])
    else:
        streamed = bool(host_out)
        if not streamed:   # D2 first: its finalize and the curl overlap the other pair kernels
            with torch.cuda.stream(sD):
                D2 = BlockToeplitzMatrix(_assemble_operator(_OP_HYPER2, True, True, True, mesh, timegrid, params,
                                                            config, None, d_range=d_range, out=out.get("D")))
        with torch.cuda.stream(sV):
            if "V" in host_out:   # work-balanced row slabs, each copied back as soon as it is formed
                V = _assemble_streamed(_OP_SINGLE, False, False, True, mesh, timegrid, params, config, None,
                                       host_out["V"], n_slabs=v_slabs, stream=sV, d_range=d_range,
                                       out=out.get("V"))
            else:
                V = BlockToeplitzMatrix(_assemble_operator(_OP_SINGLE, False, False, True, mesh, timegrid,
                                                           params, config, None, d_range=d_range,
                                                           out=out.get("V")))
            v_done = torch.cuda.Event()
            v_done.record(sV)
        if streamed:
            # host outputs: V alone first (its row slabs start the copies early: the
            # device->host copies are the end-to-end bound), then K and D2 concurrently,
            # then the curl; the copies queue on one copy stream in the order the
            # outputs form (persistent pair kernels launched together would let K
            # hold the SMs and delay V's later slabs)
            with torch.cuda.stream(sK):
                sK.wait_event(v_done)
                K = BlockToeplitzMatrix(_assemble_operator(_OP_DOUBLE, False, True, False, mesh, timegrid, params,
                                                           config, None, d_range=d_range, out=out.get("K")))
                if "K" in host_out:
                    K.host_copy = K.to_host_async(host_out["K"])
            with torch.cuda.stream(sD):
                sD.wait_event(v_done)
                D2 = BlockToeplitzMatrix(_assemble_operator(_OP_HYPER2, True, True, True, mesh, timegrid, params,
                                                            config, None, d_range=d_range, out=out.get("D")))
        with torch.cuda.stream(sD):
            sD.wait_event(v_done)
            D = hypersingular_from_single_layer(V, D2, mesh, params, overwrite_d2=True, config=config,
                                                host_out=host_out.get("D"))
        V.device_blocks.record_stream(sD)    # read by the curl combine
        if streamed:
            for st in (sD, sV, sK):
                cur.wait_stream(st)
            for M in (V, K, D):
                M.device_blocks.record_stream(cur)
            return {"V": V, "K": K, "D": D}
    with torch.cuda.stream(sK):
        K = BlockToeplitzMatrix(_assemble_operator(_OP_DOUBLE, False, True, False, mesh, timegrid, params, config,
                                                   None, d_range=d_range, out=out.get("K")))
        if "K" in host_out:
            K.host_copy = K.to_host_async(host_out["K"])
    for st in (sD, sV, sK):
        cur.wait_stream(st)
    for M in (V, K, D):
        M.device_blocks.record_stream(cur)   # allocated on a side stream, used on the caller's
    return {"V": V, "K": K, "D": D}


def assemble_mass(mesh, timegrid) -> BlockToeplitzMatrix:
    """h_t M_x (p0 test x p1 trial), diagonal-only; M_x[l, j] = area_l / 3 for j in l
    (assembly.py:380-390).  Host-built (sparse, tiny)."""
    M = np.zeros((mesh.n_triangles, mesh.n_vertices))
    rows = np.arange(mesh.n_triangles)
    for i in range(3):
        np.add.at(M, (rows, mesh.triangles[:, i]), mesh.areas / 3.0)
    return BlockToeplitzMatrix((timegrid.step * M)[None], diagonal_only=True)


_MAGIC = b"HBTM1"


def save_blocks(matrix: BlockToeplitzMatrix, path) -> None:
    """HBTM1: magic, (E_t, rows, cols) as <q, then <f8 blocks in d order (assembly.py:397-407)."""
    b = matrix.blocks
    with open(path, "wb") as fh:
        fh.write(_MAGIC + struct.pack("<qqq", *b.shape))
        fh.write(np.ascontiguousarray(b, dtype="<f8").tobytes())


def load_blocks(path, mmap: bool = False) -> BlockToeplitzMatrix:
    """Read an HBTM1 file; ``mmap=True`` maps it instead (a lazy host view of
    operators larger than host memory -- configs 3/5 -- read block by block)."""
    with open(path, "rb") as fh:
        if fh.read(5) != _MAGIC:
            raise ValueError("not a block dump file (bad magic)")
        n, r, c = struct.unpack("<qqq", fh.read(24))
        if mmap:
            import os

            if os.fstat(fh.fileno()).st_size < 29 + n * r * c * 8:
                raise ValueError("truncated block dump")
            return BlockToeplitzMatrix(np.memmap(path, dtype="<f8", mode="r", offset=29, shape=(n, r, c)))
        data = np.frombuffer(fh.read(n * r * c * 8), dtype="<f8")
    if data.size != n * r * c:
        raise ValueError("truncated block dump")
    return BlockToeplitzMatrix(data.reshape(n, r, c).astype(np.float64))


class BlockFileWriter:
    """Streaming HBTM1 writer: the header, then blocks appended in d order,
    one chunk at a time (device chunks go through a page-locked staging
    buffer) -- operators of 100-300 GB never exist whole in any memory.
    Same format as save_blocks / heatbem's dump (assembly.py:397-419)."""

    def __init__(self, path, n_blocks: int, rows: int, cols: int):
        self.shape = (int(n_blocks), int(rows), int(cols))
        self.written = 0
        self._fh = open(path, "wb")
        self._fh.write(_MAGIC + struct.pack("<qqq", *self.shape))
        self._stage = None

    def write(self, blocks) -> None:
        """Append (k, rows, cols) blocks (numpy, or a torch tensor on any device)."""
        if tuple(blocks.shape[1:]) != self.shape[1:]:
            raise ValueError("block shape mismatch")
        if self.written + blocks.shape[0] > self.shape[0]:
            raise ValueError("more blocks than declared")
        if _is_torch(blocks):
            import torch

            if blocks.is_cuda:
                if self._stage is None or self._stage.numel() < blocks.numel():
                    self._stage = torch.empty(blocks.numel(), dtype=torch.float64).pin_memory()
                host = self._stage[: blocks.numel()].view(blocks.shape)
                host.copy_(blocks)
                blocks = host
            blocks = blocks.numpy()
        self._fh.write(np.ascontiguousarray(blocks, dtype="<f8").tobytes())
        self.written += blocks.shape[0]

    def close(self) -> None:
        self._fh.close()
        if self.written != self.shape[0]:
            raise ValueError(f"{self.written} of {self.shape[0]} blocks written")

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self._fh.close() if exc[0] is not None else self.close()


def pair_classes(mesh, config: QuadratureConfig = QuadratureConfig(), rows=None, device=None) -> np.ndarray:
    """(len(rows), E_x) int8 pair classes as the device kernels see them:
    0 far, 1 near (bumped rule), 2 identical, 3 common edge, 4 common vertex."""
    import torch

    _native.require_cuda()
    tabs = device_tables(mesh, config, device)
    e0, e1 = (0, mesh.n_triangles) if rows is None else (int(rows[0]), int(rows[1]))
    out = torch.empty((e1 - e0, mesh.n_triangles), dtype=torch.int8, device=tabs.device)
    with torch.cuda.device(tabs.device):
        _native.call("hb_pair_classes", tabs.desc(True), e0, e1, _native.ptr(out), _native.stream_handle())
    return out.cpu().numpy()
