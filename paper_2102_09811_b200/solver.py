"""Block-Toeplitz operator application and the Dirichlet-solve iterations.

Drop-in for heatbem/solver.py.  Space-time vectors are (E_t, n_dof)
time-major arrays.  ``apply_toeplitz`` and the history sums of
``forward_block_solve`` run in csrc/hb_solver.cu on the device-resident
blocks; the A^0 factorisation (cuSOLVER getrf via torch.linalg) is cached on
the matrix instead of being redone on every call (solver.py:176 refactors
per call).  ``fgmres`` is the reference's restarted flexible GMRES with
Givens rotations; its vectors stay on the device, the small Hessenberg
system lives on the host.  numpy in -> numpy out, torch in -> torch out.
"""
from __future__ import annotations

import time
from dataclasses import dataclass

import numpy as np

from . import _native
from .assembly import BlockToeplitzMatrix


class LinearOperator:
    def __init__(self, apply_fn, shape=None):
        self._apply = apply_fn
        self.shape = shape

    def __call__(self, x):
        return self._apply(x)


def toeplitz_operator(matrix: BlockToeplitzMatrix, transpose_blocks: bool = False) -> LinearOperator:
    return LinearOperator(lambda x: apply_toeplitz(matrix, x, transpose_blocks))


@dataclass
class SolveReport:
    iterations: int
    residual: float
    converged: bool
    wall_time: float


def _to_device(x):
    import torch

    if isinstance(x, torch.Tensor):
        return x.to(dtype=torch.float64, device="cuda").contiguous(), True
    return torch.as_tensor(np.ascontiguousarray(x, dtype=np.float64), device="cuda"), False


def _effective_transpose(matrix, transpose_blocks):
    return bool(transpose_blocks) != bool(matrix.transpose_blocks_on_apply)


def apply_toeplitz(matrix: BlockToeplitzMatrix, x, transpose_blocks: bool = False):
    """y^k = sum_{i<=k} A^{k-i} x^i, A^d transposed when requested (solver.py:47-73)."""
    import torch

    _native.require_cuda()
    B = matrix.device_blocks
    nb, R, C = B.shape
    tr = _effective_transpose(matrix, transpose_blocks)
    n_in, n_out = (R, C) if tr else (C, R)
    xd, was_torch = _to_device(x)
    if xd.dim() == 1:
        xd = xd.reshape(-1, n_in)
    if xd.shape[1] != n_in:
        raise ValueError(f"dimension mismatch: operator expects {n_in} spatial dofs, got {xd.shape[1]}")
    E_t = xd.shape[0]
    if not matrix.diagonal_only and E_t > nb:
        raise ValueError("more time steps than stored blocks")
    y = torch.empty((E_t, n_out), dtype=torch.float64, device=xd.device)
    L = _native.load()
    need = L.hb_toeplitz_apply_workspace(nb, R, C, int(tr), int(matrix.diagonal_only), E_t)
    ws = _workspace(xd.device, need)
    _native.call("hb_toeplitz_apply_ws", nb, R, C, _native.ptr(B), int(tr), int(matrix.diagonal_only), E_t,
                 _native.ptr(xd), _native.ptr(y), _native.ptr(ws) if need else None, int(need),
                 _native.stream_handle())
    return y if was_torch else y.cpu().numpy()


_WS: dict = {}


def _workspace(device, nbytes: int):
    """Cached device scratch (grows on demand) for the split Toeplitz product."""
    import torch

    if nbytes <= 0:
        return None
    buf = _WS.get(device)
    if buf is None or buf.numel() < nbytes:
        buf = torch.empty(nbytes, dtype=torch.uint8, device=device)
        _WS[device] = buf
    return buf


def _inverse(matrix, tr):
    """(A^0)^{-1} (of A^0^T when transposed), cached with the matrix's block
    storage and dropped on any change of the blocks (host edits through
    ``.blocks``, assignment, in-place device writes): the reference refactors
    A^0 on every call (solver.py:176)."""
    import torch

    A0 = matrix.device_blocks[0]   # uploads pending host edits (and drops the cache) first
    store = getattr(matrix, "_store", None)
    cache = store.inv_cache if store is not None else {}
    if tr not in cache:
        cache[tr] = torch.linalg.inv(A0.T.contiguous() if tr else A0).contiguous()
    return cache[tr]


def forward_block_solve(matrix: BlockToeplitzMatrix, rhs, transpose_blocks: bool = False):
    """Causal time marching A^0 x^k = rhs^k - sum_{d>=1} A^d x^{k-d} (solver.py:165-184):
    one hb_forward_solve call (history and inverse-apply kernels per step)."""
    import torch

    _native.require_cuda()
    B = matrix.device_blocks
    nb, R, C = B.shape
    if R != C:
        raise ValueError("forward substitution needs square blocks")
    tr = _effective_transpose(matrix, transpose_blocks)
    r, was_torch = _to_device(rhs)
    squeeze = r.dim() == 1
    if squeeze:
        r = r.reshape(-1, R)
    E_t = r.shape[0]
    if not matrix.diagonal_only and E_t > nb:
        raise ValueError("more time steps than stored blocks")
    inv = _inverse(matrix, tr)
    x = torch.empty((E_t, R), dtype=torch.float64, device=r.device)
    h = torch.empty(R, dtype=torch.float64, device=r.device)
    _native.call("hb_forward_solve", nb, R, _native.ptr(B), int(tr), int(matrix.diagonal_only), E_t,
                 _native.ptr(inv), _native.ptr(r), _native.ptr(x), _native.ptr(h), _native.stream_handle())
    out = x.reshape(-1) if squeeze else x
    return out if was_torch else out.cpu().numpy()


def build_hypersingular_preconditioner(V11: BlockToeplitzMatrix) -> LinearOperator:
    return LinearOperator(lambda x: forward_block_solve(V11, x))


def fgmres(op, rhs, rel_tol: float = 1e-8, max_iter: int = 500, restart: int = 50, right_precond=None):
    """Restarted flexible GMRES with right preconditioning (solver.py:76-162);
    the reported residual is the true relative residual of the iterate."""
    import torch

    t0 = time.perf_counter()
    b, was_torch = _to_device(rhs)
    shape = b.shape
    b = b.reshape(-1)

    # user callables see the array type the caller passed (numpy in -> numpy)
    view = (lambda v: v.reshape(shape)) if was_torch else (lambda v: v.reshape(shape).cpu().numpy())

    def A(v):
        return torch.as_tensor(op(view(v)), dtype=torch.float64, device=b.device).reshape(-1).clone()

    def M(v):
        if right_precond is None:
            return v
        return torch.as_tensor(right_precond(view(v)), dtype=torch.float64, device=b.device).reshape(-1)

    def out(x):
        x = x.reshape(shape)
        return x if was_torch else x.cpu().numpy()

    norm_b = float(torch.linalg.vector_norm(b))
    if norm_b == 0.0:
        return out(torch.zeros_like(b)), SolveReport(0, 0.0, True, time.perf_counter() - t0)
    x = torch.zeros_like(b)
    iterations, converged, res = 0, False, float("inf")
    first = True
    while iterations < max_iter and not converged:
        r = b.clone() if first else b - A(x)   # A(0) = 0 exactly: the first residual is b
        first = False
        beta = float(torch.linalg.vector_norm(r))
        if beta <= rel_tol * norm_b:
            converged, res = True, beta / norm_b
            break
        m = min(restart, max_iter - iterations)
        V = torch.zeros((m + 1, b.numel()), dtype=torch.float64, device=b.device)
        Z = torch.zeros((m, b.numel()), dtype=torch.float64, device=b.device)
        H = np.zeros((m + 1, m))
        cs, sn, g = np.zeros(m), np.zeros(m), np.zeros(m + 1)
        g[0] = beta
        V[0] = r / beta
        j_used = 0
        for j in range(m):
            Z[j] = M(V[j])
            w = A(Z[j])
            for i in range(j + 1):
                H[i, j] = float(torch.dot(w, V[i]))
                w -= H[i, j] * V[i]
            H[j + 1, j] = float(torch.linalg.vector_norm(w))
            if H[j + 1, j] > 0:
                V[j + 1] = w / H[j + 1, j]
            for i in range(j):
                t = cs[i] * H[i, j] + sn[i] * H[i + 1, j]
                H[i + 1, j] = -sn[i] * H[i, j] + cs[i] * H[i + 1, j]
                H[i, j] = t
            denom = np.hypot(H[j, j], H[j + 1, j])
            cs[j] = H[j, j] / denom if denom > 0 else 1.0
            sn[j] = H[j + 1, j] / denom if denom > 0 else 0.0
            H[j, j], H[j + 1, j] = denom, 0.0
            g[j + 1] = -sn[j] * g[j]
            g[j] = cs[j] * g[j]
            iterations += 1
            j_used = j + 1
            if abs(g[j + 1]) <= rel_tol * norm_b or H[j, j] == 0.0:
                break
        import scipy.linalg

        y = scipy.linalg.solve_triangular(H[:j_used, :j_used], g[:j_used], lower=False)
        x = x + Z[:j_used].T @ torch.as_tensor(y, device=b.device)
        res = float(torch.linalg.vector_norm(b - A(x))) / norm_b
        if res <= rel_tol:
            converged = True
    return out(x), SolveReport(iterations, float(res), converged, time.perf_counter() - t0)
