"""Interior potentials (representation formula) on the GPU, plus the host-side
boundary-data utilities the solve needs.

Drop-in for heatbem/field.py: ``eval_single_layer_potential``,
``eval_double_layer_potential`` and ``represent`` keep the reference
signatures (a list of :class:`EvalPoint`), ``represent_grid`` is the array
form for "M points x all time-step ends" (BASELINE config 4).  Evaluation
points are grouped by (x, eps) so that one warp evaluates the kernel history
of a spatial point once for all its output times (csrc/hb_field.cu).

``project_to_space`` / ``relative_error_sigma`` / ``ManufacturedSolution``
are the reference's host utilities (field.py:20-221), kept in numpy: they
build the right-hand side of the Dirichlet solve and measure errors.
"""
from __future__ import annotations

import os
from dataclasses import dataclass

import numpy as np
import scipy.linalg
import scipy.sparse as sp

from . import _native
from .kernels import KernelParams, fundamental, grad_fundamental_normal
from .quadrature import QuadratureConfig, gauss01, rule_tables

_NORM_TRI_ORDER = 6
_NORM_TIME_POINTS = 4


@dataclass(frozen=True)
class ManufacturedSolution:
    """u(x, t) = G_alpha(x - source_point, t), source outside the domain."""

    source_point: np.ndarray
    alpha: float

    def __post_init__(self):
        object.__setattr__(self, "source_point", np.asarray(self.source_point, dtype=np.float64))

    def value(self, points, t, normals=None):
        return fundamental(np.asarray(points) - self.source_point, t, self.alpha)

    def dirichlet_trace(self, points, t, normals=None):
        return self.value(points, t)

    def neumann_trace(self, points, t, normals):
        return grad_fundamental_normal(np.asarray(points) - self.source_point, normals, t, self.alpha)


@dataclass(frozen=True)
class EvalPoint:
    """Interior point x at time t = k h_t + eps (heatbem/field.py:45-58)."""

    x: np.ndarray
    t: float

    def decompose(self, h_t: float):
        k, eps = _decompose(np.array([self.t]), h_t)
        return int(k[0]), float(eps[0])


def _decompose(t: np.ndarray, h: float):
    """Vectorised EvalPoint.decompose (same float operations)."""
    ratio = t / h
    k = np.floor(ratio + 1e-12).astype(np.int64)
    eps = t - k * h
    snap = (eps < 0.0) | (np.abs(ratio - k) <= 1e-12 * np.maximum(1.0, np.abs(ratio)))
    return k, np.where(snap, 0.0, eps)


def _p1_mass(mesh) -> sp.csr_matrix:
    local = (np.ones((3, 3)) + np.eye(3)) / 12.0
    rows = np.repeat(mesh.triangles, 3, axis=1).ravel()
    cols = np.tile(mesh.triangles, (1, 3)).ravel()
    vals = (mesh.areas[:, None, None] * local).ravel()
    return sp.csr_matrix((vals, (rows, cols)), shape=(mesh.n_vertices,) * 2)


def project_to_space(fn, mesh, timegrid, space: str) -> np.ndarray:
    """L2(Sigma) projection onto X00 (p0 x p0) or X10 (p1 x p0): (E_t, n_dof)
    (heatbem/field.py:84-119; triangle order 6, 4 Gauss points per step)."""
    if space not in ("X00", "X10"):
        raise ValueError("space must be 'X00' or 'X10'")
    hats, qw, qpts = rule_tables(mesh, _NORM_TRI_ORDER)
    tq, tw = gauss01(_NORM_TIME_POINTS)
    h, E_t, E_x = timegrid.step, timegrid.n_steps, mesh.n_triangles
    flat = qpts.reshape(-1, 3)
    normals = np.repeat(mesh.normals[:, None, :], qpts.shape[1], axis=1).reshape(-1, 3)
    if space == "X00":
        out = np.empty((E_t, E_x))
        for i in range(E_t):
            acc = np.zeros(E_x)
            for q, w in zip(tq, tw):
                acc += w * (fn(flat, timegrid.node(i) + q * h, normals).reshape(E_x, -1) @ qw)
            out[i] = 2.0 * acc
        return out
    cho = scipy.linalg.cho_factor(_p1_mass(mesh).toarray())
    out = np.empty((E_t, mesh.n_vertices))
    wh = qw[:, None] * hats
    for i in range(E_t):
        b = np.zeros(mesh.n_vertices)
        for q, w in zip(tq, tw):
            vals = fn(flat, timegrid.node(i) + q * h, normals).reshape(E_x, -1)
            np.add.at(b, mesh.triangles.ravel(), (w * (2.0 * mesh.areas[:, None] * (vals @ wh))).ravel())
        out[i] = scipy.linalg.cho_solve(cho, b)
    return out


def relative_error_sigma(coeffs, fn, mesh, timegrid) -> float:
    """Relative L2(Sigma_h) error of a coefficient function against fn."""
    hats, qw, qpts = rule_tables(mesh, _NORM_TRI_ORDER)
    tq, tw = gauss01(_NORM_TIME_POINTS)
    coeffs = np.asarray(coeffs)
    dens = _interp_density_np(coeffs, mesh, hats)
    normals = np.repeat(mesh.normals[:, None, :], qpts.shape[1], axis=1).reshape(-1, 3)
    h = timegrid.step
    area_w = 2.0 * mesh.areas[:, None] * qw[None, :]
    num = den = 0.0
    for i in range(timegrid.n_steps):
        for q, w in zip(tq, tw):
            vals = fn(qpts.reshape(-1, 3), timegrid.node(i) + q * h, normals).reshape(mesh.n_triangles, -1)
            num += w * h * np.sum(area_w * (vals - dens[i]) ** 2)
            den += w * h * np.sum(area_w * vals ** 2)
    if den == 0.0:
        raise ValueError("exact function has zero L2(Sigma) norm")
    return float(np.sqrt(num / den))


def eoc(errors) -> list:
    errors = list(errors)
    if any(e <= 0 for e in errors):
        raise ValueError("errors must be positive")
    return [float(np.log2(errors[k - 1] / errors[k])) for k in range(1, len(errors))]


def _interp_density_np(coeffs, mesh, hats):
    if coeffs.shape[1] == mesh.n_triangles:
        return np.repeat(coeffs[:, :, None], hats.shape[0], axis=2)
    return coeffs[:, mesh.triangles] @ hats.T


# ---------------------------------------------------------------------------
# device potentials
# ---------------------------------------------------------------------------

class _PotentialTables:
    def __init__(self, mesh, config, device):
        import torch

        hats, qw, qpts = rule_tables(mesh, config.regular_order + 2)
        up = lambda a, dt=torch.float64: torch.as_tensor(np.ascontiguousarray(a), dtype=dt, device=device)  # noqa
        self.hats = up(hats)
        self.qw = up(qw)
        self.qpts = up(qpts)
        self.areas = up(mesh.areas)
        self.normals = up(mesh.normals)
        self.centroids = up(mesh.centroids)
        self.tri = up(mesh.triangles, torch.int64)
        self.nq = len(qw)


_POT_CACHE: dict = {}


def _tables(mesh, config, device):
    key = (id(mesh), config.regular_order, str(device))
    hit = _POT_CACHE.get(key)
    if hit is None or hit[0]() is not mesh:
        import weakref

        hit = (weakref.ref(mesh), _PotentialTables(mesh, config, device))
        _POT_CACHE[key] = hit
    return hit[1]


def _density(coeffs, mesh, T):
    """(E_t, E_x, nq) density at quadrature nodes, on the device."""
    import torch

    c = torch.as_tensor(coeffs, dtype=torch.float64, device=T.qw.device)
    if c.shape[1] == mesh.n_triangles:
        return c[:, :, None].expand(-1, -1, T.nq).contiguous()
    if c.shape[1] != mesh.n_vertices:
        raise ValueError("density must have E_x (p0) or N_x (p1) columns")
    return torch.matmul(c[:, T.tri], T.hats.T).contiguous()


def _boundary_warnings(xs, mesh, T, chunk=8192):
    import torch

    thr = 1e-8 * mesh.diameter
    out = torch.empty(xs.shape[0], dtype=torch.bool, device=xs.device)
    for i in range(0, xs.shape[0], chunk):
        d = torch.cdist(xs[i:i + chunk], T.centroids)
        out[i:i + chunk] = d.min(dim=1).values < thr
    return out


def _eval_grouped(kind, coeffs, xs, k, eps, cur, mesh, timegrid, params, config, stream=None):
    """Core: points xs (n,3) with per-point (k, eps, cur) -> values (n,) on device."""
    n = xs.shape[0]
    if n == 0:
        return _launch_groups(kind, coeffs, None, mesh, timegrid, params, config, stream)
    # group by (x, eps): lexicographic sort on (x0, x1, x2, eps, k)
    key = np.column_stack([xs, eps])
    order = np.lexsort((k, key[:, 3], key[:, 2], key[:, 1], key[:, 0]))
    ks = key[order]
    new = np.ones(n, dtype=bool)
    new[1:] = np.any(ks[1:] != ks[:-1], axis=1)
    starts = np.flatnonzero(new)
    groups = dict(gx=ks[starts, :3], geps=ks[starts, 3], gptr=np.append(starts, n), k=k[order],
                  cur=cur[order], out_idx=order, kmax=int(k.max()))
    return _launch_groups(kind, coeffs, groups, mesh, timegrid, params, config, stream)


def _grid_groups(xs, ks):
    """Groups of represent_grid: point i owns outputs i*nt .. i*nt + nt - 1
    (times ks, ascending), eps = 0 -- no sort needed."""
    M, nt = xs.shape[0], len(ks)
    return dict(gx=xs, geps=np.zeros(M), gptr=np.arange(0, M * nt + 1, nt), k=np.tile(ks, M),
                cur=np.zeros(M * nt, dtype=bool), out_idx=np.arange(M * nt), kmax=int(ks.max()) if nt else 0)


def _launch_groups(kind, coeffs, groups, mesh, timegrid, params, config, stream=None):
    import torch

    _native.require_cuda()
    T = _tables(mesh, config, torch.device("cuda", torch.cuda.current_device()))
    dev = T.qw.device
    if groups is None or len(groups["k"]) == 0:
        return torch.empty(0, dtype=torch.float64, device=dev)
    dens = _density(coeffs, mesh, T).permute(1, 2, 0).contiguous()   # (E_x, nq, E_t): time fastest
    out = torch.empty(len(groups["k"]), dtype=torch.float64, device=dev)
    up = lambda a, dt: torch.as_tensor(np.ascontiguousarray(a), dtype=dt, device=dev)  # noqa: E731
    gx = up(groups["gx"], torch.float64)
    geps = up(groups["geps"], torch.float64)
    kk = up(groups["k"], torch.int64)
    cc = up(np.asarray(groups["cur"]).astype(np.uint8), torch.uint8)
    oi = up(groups["out_idx"], torch.int64)
    gp = up(groups["gptr"], torch.int64)
    _native.call("hb_potential", int(kind), len(groups["gx"]), timegrid.n_steps, mesh.n_triangles, T.nq,
                 _native.ptr(gx), _native.ptr(geps), _native.ptr(gp), _native.ptr(kk), _native.ptr(cc),
                 _native.ptr(oi), groups["kmax"], _native.ptr(dens), _native.ptr(T.qpts), _native.ptr(T.qw),
                 _native.ptr(T.areas), _native.ptr(T.normals), timegrid.step, params.alpha,
                 params.delta_eps, params.rho_eps, _native.ptr(out), _native.stream_handle(stream))
    return out


def _eval_potential(kind, coeffs, points, mesh, timegrid, params, config=QuadratureConfig()):
    import torch

    xs = np.array([np.asarray(p.x, dtype=np.float64) for p in points]).reshape(-1, 3)
    t = np.array([float(p.t) for p in points])
    k, eps = _decompose(t, timegrid.step)
    cur = (eps > 0.0) & (k < timegrid.n_steps)
    vals = _eval_grouped(kind, np.asarray(coeffs), xs, k, eps, cur, mesh, timegrid, params, config)
    T = _tables(mesh, config, vals.device)
    warn = _boundary_warnings(torch.as_tensor(xs, device=vals.device), mesh, T)
    return vals.cpu().numpy(), warn.cpu().numpy()


def eval_single_layer_potential(w, points, mesh, timegrid, params: KernelParams,
                                config: QuadratureConfig = QuadratureConfig()):
    """Single-layer potential of the p0 density w at EvalPoints (field.py:170-174)."""
    return _eval_potential(0, w, points, mesh, timegrid, params, config)


def eval_double_layer_potential(u, points, mesh, timegrid, params: KernelParams,
                                config: QuadratureConfig = QuadratureConfig()):
    """Double-layer potential of the p1 density u at EvalPoints (field.py:177-181)."""
    return _eval_potential(1, u, points, mesh, timegrid, params, config)


def represent(w, u, points, mesh, timegrid, params: KernelParams, config: QuadratureConfig = QuadratureConfig()):
    """Representation formula V~w - Wu at EvalPoints (field.py:184-190)."""
    sv, w1 = eval_single_layer_potential(w, points, mesh, timegrid, params, config)
    dv, w2 = eval_double_layer_potential(u, points, mesh, timegrid, params, config)
    return sv - dv, w1 | w2


def _represent_grid_fused(w, u, xs, ks, mesh, timegrid, params, config, stream=None):
    """u = V~w - W u at (x_i, k_j h) in one hb_represent_grid launch: the two
    potentials share the kernel-value evaluation (csrc/hb_field.cu)."""
    import torch

    _native.require_cuda()
    T = _tables(mesh, config, torch.device("cuda", torch.cuda.current_device()))
    dev = T.qw.device
    ds = _density(w, mesh, T).permute(1, 2, 0).contiguous()
    dd = _density(u, mesh, T).permute(1, 2, 0).contiguous()
    X = torch.as_tensor(np.ascontiguousarray(xs), dtype=torch.float64, device=dev)
    K = torch.as_tensor(np.ascontiguousarray(ks, dtype=np.int64), device=dev)
    out = torch.empty((xs.shape[0], len(ks)), dtype=torch.float64, device=dev)
    _native.call("hb_represent_grid", xs.shape[0], len(ks), timegrid.n_steps, mesh.n_triangles, T.nq,
                 _native.ptr(X), _native.ptr(K), int(ks.max()), _native.ptr(ds), _native.ptr(dd),
                 _native.ptr(T.qpts), _native.ptr(T.qw), _native.ptr(T.areas), _native.ptr(T.normals),
                 timegrid.step, params.alpha, params.delta_eps, params.rho_eps, _native.ptr(out),
                 _native.stream_handle(stream))
    return out


def represent_grid(w, u, xs, mesh, timegrid, params: KernelParams, config: QuadratureConfig = QuadratureConfig(),
                   time_steps=None, return_device: bool = False):
    """u(x_i, k h) for every point x_i (M, 3) and every k in time_steps
    (default 1..E_t): the representation formula on a space-time grid,
    returned as (M, n_times).  Equivalent to ``represent`` on the EvalPoints
    (x_i, k h) -- one group per point, the kernel history shared by all k."""
    import torch

    xs = np.ascontiguousarray(xs, dtype=np.float64).reshape(-1, 3)
    ks = np.arange(1, timegrid.n_steps + 1) if time_steps is None else np.asarray(time_steps, dtype=np.int64)
    M, nt = xs.shape[0], len(ks)
    if nt and (np.any(ks < 0) or np.any(ks > timegrid.n_steps)):
        raise ValueError("time_steps must lie in [0, n_steps]")
    if nt > 1 and np.any(np.diff(ks) < 0):
        raise ValueError("time_steps must be ascending")
    if nt and int(ks.max()) <= 64 and not os.environ.get("HB_REP_SEPARATE"):
        res = _represent_grid_fused(np.asarray(w), np.asarray(u), xs, ks, mesh, timegrid, params, config)
        return res if return_device else res.cpu().numpy()
    groups = _grid_groups(xs, ks)
    sv = _launch_groups(0, np.asarray(w), groups, mesh, timegrid, params, config)
    dv = _launch_groups(1, np.asarray(u), groups, mesh, timegrid, params, config)
    res = (sv - dv).reshape(M, nt)
    return res if return_device else res.cpu().numpy()


def interior_evaluation_points(n_points: int = 10_000, n_axis: int = 22, half_width: float = 0.5,
                               end_time: float = 1.0) -> list:
    """Deterministic lattice points with cycling times (field.py:224-243)."""
    axis = np.linspace(-half_width, half_width, n_axis)
    g = np.stack(np.meshgrid(axis, axis, axis, indexing="ij"), axis=-1).reshape(-1, 3)[:n_points]
    times = end_time * (0.25 + 0.5 * (np.arange(len(g)) % 10) / 9.0)
    return [EvalPoint(g[i].copy(), float(times[i])) for i in range(len(g))]
