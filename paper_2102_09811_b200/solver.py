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
    one hb_forward_solve_ws call (steps in tiles of 8: one history pass over
    the blocks per tile, then the near terms and the inverse apply per step)."""
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
    need = _native.load().hb_forward_solve_workspace(R)
    ws = _workspace(r.device, need)
    _native.call("hb_forward_solve_ws", nb, R, _native.ptr(B), int(tr), int(matrix.diagonal_only), E_t,
                 _native.ptr(inv), _native.ptr(r), _native.ptr(x), _native.ptr(ws), int(need), _native.stream_handle())
    out = x.reshape(-1) if squeeze else x
    return out if was_torch else out.cpu().numpy()


def build_hypersingular_preconditioner(V11: BlockToeplitzMatrix) -> LinearOperator:
    return LinearOperator(lambda x: forward_block_solve(V11, x))


class _KrylovCycle:
    """One restart cycle of flexible GMRES on the device.

    The Arnoldi vectors V and the preconditioned directions Z (flexible:
    the preconditioner may change from step to step) are rows of device
    matrices.  A new direction is orthogonalised by classical Gram-Schmidt
    with one re-orthogonalisation pass (two GEMVs against the stored basis,
    CGS2 -- as stable as modified Gram-Schmidt, one host round trip per step
    instead of one per basis vector).  Each Hessenberg column is reduced by
    the accumulated Givens rotations as it is formed; the least-squares
    residual is then |g[j + 1]| of the rotated right-hand side."""

    def __init__(self, r, beta: float, m: int):
        import torch

        n = r.numel()
        self.m, self.k = m, 0
        self.V = torch.zeros((m + 1, n), dtype=torch.float64, device=r.device)
        self.Z = torch.zeros((m, n), dtype=torch.float64, device=r.device)
        self.V[0] = r / beta
        self.R = np.zeros((m, m))            # the rotated (upper-triangular) Hessenberg
        self.rot = np.zeros((m, 2))          # (c, s) of each step's rotation
        self.g = np.zeros(m + 1)
        self.g[0] = beta

    def extend(self, apply_A, apply_M) -> bool:
        """One Arnoldi step; False on breakdown (the Krylov space is invariant)."""
        import torch

        k = self.k
        Vk = self.V[: k + 1]
        self.Z[k] = apply_M(self.V[k])
        w = apply_A(self.Z[k])
        h = torch.mv(Vk, w)
        w = w - torch.mv(Vk.T, h)
        h2 = torch.mv(Vk, w)
        w = w - torch.mv(Vk.T, h2)
        h = h + h2
        nrm = torch.linalg.vector_norm(w)
        col = torch.cat([h, nrm.reshape(1)]).cpu().numpy()   # the one host round trip of the step
        if col[k + 1] > 0.0:
            self.V[k + 1] = w / nrm
        for i in range(k):                  # earlier rotations act on rows (i, i + 1)
            c, s = self.rot[i]
            col[i], col[i + 1] = c * col[i] + s * col[i + 1], c * col[i + 1] - s * col[i]
        rho = float(np.hypot(col[k], col[k + 1]))
        c, s = (col[k] / rho, col[k + 1] / rho) if rho > 0.0 else (1.0, 0.0)
        self.rot[k] = (c, s)
        col[k], col[k + 1] = rho, 0.0
        self.R[: k + 1, k] = col[: k + 1]
        self.g[k], self.g[k + 1] = c * self.g[k], -s * self.g[k]
        self.k = k + 1
        return rho != 0.0

    @property
    def residual(self) -> float:
        return abs(self.g[self.k])

    def correction(self):
        """Z^T y with R y = g (the least-squares solution of the cycle)."""
        import scipy.linalg
        import torch

        k = self.k
        y = scipy.linalg.solve_triangular(self.R[:k, :k], self.g[:k], lower=False)
        return self.Z[:k].T @ torch.as_tensor(y, device=self.Z.device)


def fgmres(op, rhs, rel_tol: float = 1e-8, max_iter: int = 500, restart: int = 50, right_precond=None):
    """Restarted flexible GMRES with right preconditioning, the semantics of
    solver.py:76-162 (restart length, iteration budget, stopping on the
    rotated least-squares residual, the true relative residual of the
    returned iterate in the report); the cycles run on the device
    (``_KrylovCycle``)."""
    import torch

    t0 = time.perf_counter()
    b, was_torch = _to_device(rhs)
    shape = b.shape
    b = b.reshape(-1)

    # user callables see the array type the caller passed (numpy in -> numpy)
    view = (lambda v: v.reshape(shape)) if was_torch else (lambda v: v.reshape(shape).cpu().numpy())

    def apply_A(v):
        return torch.as_tensor(op(view(v)), dtype=torch.float64, device=b.device).reshape(-1).clone()

    def apply_M(v):
        if right_precond is None:
            return v
        return torch.as_tensor(right_precond(view(v)), dtype=torch.float64, device=b.device).reshape(-1)

    def result(x, its, res, ok):
        x = x.reshape(shape)
        return (x if was_torch else x.cpu().numpy()), SolveReport(its, float(res), ok, time.perf_counter() - t0)

    norm_b = float(torch.linalg.vector_norm(b))
    if norm_b == 0.0:
        return result(torch.zeros_like(b), 0, 0.0, True)
    tol = rel_tol * norm_b
    x = torch.zeros_like(b)
    its, res = 0, float("inf")
    r = b.clone()                            # A(0) = 0 exactly: the first residual is b
    while its < max_iter:
        beta = float(torch.linalg.vector_norm(r))
        if beta <= tol:
            return result(x, its, beta / norm_b, True)
        cyc = _KrylovCycle(r, beta, min(restart, max_iter - its))
        while cyc.k < cyc.m:
            alive = cyc.extend(apply_A, apply_M)
            its += 1
            if cyc.residual <= tol or not alive:
                break
        x = x + cyc.correction()
        r = b - apply_A(x)
        res = float(torch.linalg.vector_norm(r)) / norm_b
        if res <= rel_tol:
            return result(x, its, res, True)
    return result(x, its, res, False)
