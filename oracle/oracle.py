"""ctypes front-end of the CPU oracle -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` leg may import this module, and only as the checker or
the timed CPU baseline; the product package never does.

It drives oracle/libheatbem_oracle.so (heatbem_oracle.c, a plain-C
restatement of heatbem/_assembly_numba.py and heatbem/_field_numba.py) with
the same host tables the reference builds in heatbem/assembly.py:201-206.
Those tables come from the product's host module
(paper_2102_09811_b200.quadrature), which tests/test_tables_golden.py pins
bit-for-bit against tables dumped from the reference itself.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libheatbem_oracle.so")
_LIBQ_PATH = os.path.join(_HERE, "libheatbem_oracle_q.so")
_lib = None
_libq = None

_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_D = ctypes.c_double
_INT = ctypes.c_int

_PROBLEM = [_INT, _INT, _INT, _INT, _I64, _I64, _D, _D, _D, _D,
            _P, _P, _P, _P, _P, _P,
            _P, _P, _P, _I64, _P, _P, _P, _I64,
            _P, _P, _P, _P, _P,
            _P, _P, _P, _P]


def build(force: bool = False) -> str:
    src = os.path.getmtime(os.path.join(_HERE, "heatbem_oracle.c"))
    if force or any(not os.path.exists(p) or os.path.getmtime(p) < src for p in (_LIB_PATH, _LIBQ_PATH)):
        subprocess.check_call(["make", "-s", "-C", _HERE], stdout=subprocess.DEVNULL)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        L.hb_oracle_assemble.argtypes = _PROBLEM + [_I64, _D, _P, _INT]
        L.hb_oracle_rows.argtypes = _PROBLEM + [_I64, _D, _P, _I64, _P, _INT]
        L.hb_oracle_pass.argtypes = _PROBLEM + [_D, _INT, _P, _I64, _P, _P, _INT]
        L.hb_oracle_potential.argtypes = [_INT, _P, _P, _P, _P, _P, _P, _P, _P, _P,
                                          _I64, _I64, _I64, _I64, _D, _D, _D, _D, _P, _INT]
        for f in (L.hb_oracle_assemble, L.hb_oracle_rows, L.hb_oracle_pass, L.hb_oracle_potential):
            f.restype = _INT
        L.hb_oracle_max_threads.restype = _INT
        _lib = L
    return _lib


def libq():
    """Quad-precision build (heatbem_oracle_q.c): exact value of the same quadrature."""
    global _libq
    if _libq is None:
        if not os.path.exists(_LIBQ_PATH):
            build()
        L = ctypes.CDLL(_LIBQ_PATH)
        L.hb_oracle_assemble_q.argtypes = _PROBLEM + [_I64, _D, _P, _INT]
        L.hb_oracle_rows_q.argtypes = _PROBLEM + [_I64, _D, _P, _I64, _P, _INT]
        L.hb_oracle_potential_q.argtypes = [_INT, _P, _P, _P, _P, _P, _P, _P, _P, _P,
                                            _I64, _I64, _I64, _I64, _D, _D, _D, _D, _P, _INT]
        L.hb_oracle_curl_combine_q.argtypes = [_I64, _I64, _I64, _D, _P, _P, _P, _P, _P, _INT]
        for f in (L.hb_oracle_assemble_q, L.hb_oracle_rows_q, L.hb_oracle_potential_q,
                  L.hb_oracle_curl_combine_q):
            f.restype = _INT
        _libq = L
    return _libq


def max_threads() -> int:
    return int(lib().hb_oracle_max_threads())


def _ptr(a):
    return ctypes.c_void_p(a.ctypes.data) if a is not None else ctypes.c_void_p(0)


# operator codes of the reference (assembly.py:21)
OPS = {
    "V": (0, False, False, True),      # single layer p0 x p0
    "V11": (0, True, True, True),      # single layer p1 x p1
    "K": (1, False, True, False),      # double layer p0 x p1
    "D2": (2, True, True, True),       # hypersingular surface part p1 x p1
}


class OracleProblem:
    """Host tables for one (mesh, op) -- the inputs of _toeplitz_pass."""

    def __init__(self, mesh, params, config, op: str, step: float):
        from paper_2102_09811_b200 import quadrature as Q

        self.mesh, self.params, self.step = mesh, params, float(step)
        self.op, self.test_p1, self.trial_p1, self.symmetric = OPS[op]
        c = np.ascontiguousarray
        self.arrays = dict(
            tri_nodes=c(mesh.triangles, dtype=np.int64),
            verts_tri=c(mesh.triangle_vertices()),
            normals=c(mesh.normals), centroids=c(mesh.centroids),
            diameters=c(mesh.diameters), areas=c(mesh.areas),
        )
        rh, rw, rp = Q.rule_tables(mesh, config.regular_order)
        nh, nw, npt = Q.rule_tables(mesh, config.near_order)
        tn = Q.touching_csr(mesh)
        duf = Q.duffy_tables(config.singular_order)
        self.rule = [c(x) for x in (rh, rw, rp)]
        self.near = [c(x) for x in (nh, nw, npt)]
        self.tn = [c(x) for x in tn]
        self.duf = [c(x) for x in duf]

    def args(self):
        m, p, A = self.mesh, self.params, self.arrays
        return [self.op, int(self.test_p1), int(self.trial_p1), int(self.symmetric),
                m.n_triangles, m.n_vertices, p.alpha, self.step, p.delta_eps, p.rho_eps,
                _ptr(A["tri_nodes"]), _ptr(A["verts_tri"]), _ptr(A["normals"]),
                _ptr(A["centroids"]), _ptr(A["diameters"]), _ptr(A["areas"]),
                _ptr(self.rule[0]), _ptr(self.rule[1]), _ptr(self.rule[2]), len(self.rule[1]),
                _ptr(self.near[0]), _ptr(self.near[1]), _ptr(self.near[2]), len(self.near[1]),
                *[_ptr(x) for x in self.tn], *[_ptr(x) for x in self.duf]]

    @property
    def shape_rc(self):
        m = self.mesh
        return (m.n_vertices if self.test_p1 else m.n_triangles,
                m.n_vertices if self.trial_p1 else m.n_triangles)


def assemble(mesh, timegrid, params, config, op: str, n_threads: int = 0, exact: bool = False) -> np.ndarray:
    """Full (E_t, R, C) blocks, as heatbem.assembly._assemble_operator
    (exact=True: the same quadrature in 113-bit arithmetic, rounded once)."""
    P = OracleProblem(mesh, params, config, op, timegrid.step)
    R, C = P.shape_rc
    out = np.empty((timegrid.n_steps, R, C))
    fn = libq().hb_oracle_assemble_q if exact else lib().hb_oracle_assemble
    rc = fn(*P.args(), timegrid.n_steps, timegrid.step, _ptr(out), n_threads)
    if rc != 0:
        raise MemoryError("oracle assemble failed")
    return out


def assemble_rows(mesh, timegrid, params, config, op: str, rows, n_threads: int = 0,
                  exact: bool = False) -> np.ndarray:
    """Rows of all blocks of a p0-test operator (V or K): (E_t, len(rows), C)."""
    P = OracleProblem(mesh, params, config, op, timegrid.step)
    rows = np.ascontiguousarray(rows, dtype=np.int64)
    _, C = P.shape_rc
    out = np.empty((timegrid.n_steps, len(rows), C))
    fn = libq().hb_oracle_rows_q if exact else lib().hb_oracle_rows
    rc = fn(*P.args(), timegrid.n_steps, timegrid.step, _ptr(rows), len(rows), _ptr(out), n_threads)
    if rc != 0:
        raise RuntimeError(f"oracle rows failed ({rc})")
    return out


def single_pass(mesh, params, config, op: str, step: float, i_t: int, rows=None, n_threads: int = 0):
    """One _toeplitz_pass at delta = i_t * step: (loc, loc_comb)."""
    P = OracleProblem(mesh, params, config, op, step)
    m = mesh
    n_t = 3 if P.test_p1 else 1
    C = m.n_vertices if P.trial_p1 else m.n_triangles
    n = m.n_triangles if rows is None else len(rows)
    rows_a = None if rows is None else np.ascontiguousarray(rows, dtype=np.int64)
    loc = np.zeros((n, n_t, C))
    locc = np.zeros((n, n_t, C))
    lib().hb_oracle_pass(*P.args(), float(i_t) * step, int(i_t == 0), _ptr(rows_a),
                         0 if rows_a is None else len(rows_a), _ptr(loc), _ptr(locc), n_threads)
    return loc, locc


def curl_combine(V, D2, mesh, alpha):
    """D = D2 + alpha^2 sum_o T_o^T V T_o (heatbem/assembly.py:289-334),
    evaluated with scipy.sparse exactly as the reference does."""
    import scipy.sparse as sp

    E_x, N_x = mesh.n_triangles, mesh.n_vertices
    v = mesh.triangle_vertices()
    rows = np.repeat(np.arange(E_x), 3)
    cols = mesh.triangles.ravel()
    curls = np.empty((E_x, 3, 3))
    for i in range(3):
        curls[:, i, :] = (v[:, (i + 1) % 3, :] - v[:, (i + 2) % 3, :]) / (2.0 * mesh.areas[:, None])
    T = [sp.csr_matrix((curls[:, :, o].ravel(), (rows, cols)), shape=(E_x, N_x)) for o in range(3)]
    out = D2.copy()
    a2 = alpha ** 2
    for d in range(V.shape[0]):
        for To in T:
            out[d] += a2 * (To.T @ (V[d] @ To))
    return out


def curl_combine_exact(V, D2, mesh, alpha, n_threads: int = 0) -> np.ndarray:
    """Quad-precision D = D2 + alpha^2 sum (curl . curl) V (inputs double)."""
    from paper_2102_09811_b200.device import _curls

    c = np.ascontiguousarray
    V, D2 = c(V, dtype=np.float64), c(D2, dtype=np.float64)
    curls = c(_curls(mesh))
    tri = c(mesh.triangles, dtype=np.int64)
    out = np.empty_like(D2)
    rc = libq().hb_oracle_curl_combine_q(V.shape[0], mesh.n_triangles, mesh.n_vertices, float(alpha),
                                         _ptr(tri), _ptr(curls), _ptr(V), _ptr(D2), _ptr(out), n_threads)
    if rc != 0:
        raise MemoryError("oracle curl combine failed")
    return out


def potential(kind, points, k_arr, eps_arr, cur_arr, dens, qpts, qw, areas, normals,
              h_t, alpha, d_eps, r_eps, n_threads: int = 0, exact: bool = False) -> np.ndarray:
    c = np.ascontiguousarray
    points, dens, qpts, qw = c(points, dtype=np.float64), c(dens), c(qpts), c(qw)
    k_arr = c(k_arr, dtype=np.int64)
    eps_arr = c(eps_arr, dtype=np.float64)
    cur = c(cur_arr, dtype=np.uint8)
    areas, normals = c(areas), c(normals)
    out = np.empty(len(points))
    fn = libq().hb_oracle_potential_q if exact else lib().hb_oracle_potential
    fn(int(kind), _ptr(points), _ptr(k_arr), _ptr(eps_arr), _ptr(cur),
                              _ptr(dens), _ptr(qpts), _ptr(qw), _ptr(areas), _ptr(normals),
                              len(points), dens.shape[0], dens.shape[1], dens.shape[2],
                              h_t, alpha, d_eps, r_eps, _ptr(out), n_threads)
    return out


# ---------------------------------------------------------------------------
# solver restatements (numpy; the reference's solver is numpy too)
# ---------------------------------------------------------------------------
def apply_toeplitz(blocks: np.ndarray, x: np.ndarray) -> np.ndarray:
    """y^k = sum_{d <= k} A^d x^{k-d} -- heatbem/solver.py:47-73 (the
    non-transposed, non-diagonal case), same loop order."""
    E_t = x.shape[0]
    y = np.empty((E_t, blocks.shape[1]))
    for k in range(E_t):
        acc = blocks[0] @ x[k]
        for d in range(1, k + 1):
            acc += blocks[d] @ x[k - d]
        y[k] = acc
    return y


def forward_block_solve(blocks: np.ndarray, rhs: np.ndarray) -> np.ndarray:
    """A^0 x^k = rhs^k - sum_{d>=1} A^d x^{k-d} with one LU of A^0 --
    heatbem/solver.py:165-184, same loop order."""
    import scipy.linalg

    E_t = rhs.shape[0]
    lu = scipy.linalg.lu_factor(np.ascontiguousarray(blocks[0]))
    x = np.empty((E_t, blocks.shape[2]))
    for k in range(E_t):
        acc = rhs[k].copy()
        for d in range(1, k + 1):
            acc -= blocks[d] @ x[k - d]
        x[k] = scipy.linalg.lu_solve(lu, acc)
    return x
