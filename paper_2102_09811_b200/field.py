"""Interior potentials (representation formula) on the GPU, plus the host-side
boundary-data utilities the solve needs.

Drop-in for heatbem/field.py: ``eval_single_layer_potential``,
``eval_double_layer_potential`` and ``represent`` keep the reference
signatures (a list of :class:`EvalPoint`), ``represent_grid`` is the array
form for "M points x all time-step ends" (BASELINE config 4).  Evaluation
points are grouped by (x, eps) so that one warp evaluates the kernel history
of a spatial point once for all its output times (csrc/hb_field.cu).

``project_to_space`` / ``relative_error_sigma`` (field.py:84-119, 193-215)
run on the device (csrc/hb_data.cu) whenever the datum is one the GPU can
evaluate -- a :class:`HeatKernelDatum` or a trace method of
:class:`ManufacturedSolution` (the study driver's data); an arbitrary Python
callable can only be evaluated on the host, so for those the reference's
numpy algorithm runs as before.
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
class HeatKernelDatum:
    """Boundary datum the GPU evaluates: ``kind="value"`` is
    G_alpha(x - source_point, t + time_shift) (kernels.py:59-66),
    ``kind="normal_derivative"`` is alpha dG_alpha/dn_x at the same
    arguments (kernels.py:69-86).  Callable like the reference's data
    functions ``fn(points, t, normals)`` (numpy, host)."""

    source_point: tuple
    alpha: float
    time_shift: float = 0.0
    kind: str = "value"

    def __post_init__(self):
        if self.kind not in ("value", "normal_derivative"):
            raise ValueError("kind must be 'value' or 'normal_derivative'")
        object.__setattr__(self, "source_point", tuple(float(v) for v in np.ravel(self.source_point)))

    def __call__(self, points, t, normals=None):
        r = np.asarray(points) - np.asarray(self.source_point)
        if self.kind == "value":
            return fundamental(r, t + self.time_shift, self.alpha)
        return grad_fundamental_normal(r, normals, t + self.time_shift, self.alpha)


def device_datum(fn):
    """The :class:`HeatKernelDatum` equivalent of fn, or None when fn is an
    arbitrary callable (host-only)."""
    if isinstance(fn, HeatKernelDatum):
        return fn
    owner = getattr(fn, "__self__", None)
    if isinstance(owner, ManufacturedSolution):
        name = getattr(fn, "__name__", "")
        kind = {"value": "value", "dirichlet_trace": "value", "neumann_trace": "normal_derivative"}.get(name)
        if kind is not None and getattr(type(owner), name) is getattr(ManufacturedSolution, name):
            return HeatKernelDatum(tuple(owner.source_point), float(owner.alpha), 0.0, kind)
    return None


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


# ---------------------------------------------------------------------------
# boundary data on the device (csrc/hb_data.cu)
# ---------------------------------------------------------------------------

class _DataTables:
    """Order-6 triangle rule, 4-point time rule and node stars on the device."""

    def __init__(self, mesh, device):
        import torch

        hats, qw, qpts = rule_tables(mesh, _NORM_TRI_ORDER)
        tq, tw = gauss01(_NORM_TIME_POINTS)
        up = lambda a, dt=torch.float64: torch.as_tensor(np.ascontiguousarray(a), dtype=dt, device=device)  # noqa
        indptr, elem, local = mesh.node_star()
        self.t = {"qpts": up(qpts), "qw": up(qw), "hats": up(hats), "areas": up(mesh.areas),
                  "normals": up(mesh.normals), "tri": up(mesh.triangles, torch.int64),
                  "indptr": up(indptr, torch.int64), "elem": up(elem, torch.int64),
                  "local": up(local, torch.int64)}
        d = _native.DataDesc()
        d.E_x, d.N_x, d.nq = mesh.n_triangles, mesh.n_vertices, len(qw)
        P = _native.ptr
        d.qpts_dev, d.qw_dev, d.hats_dev = P(self.t["qpts"]), P(self.t["qw"]), P(self.t["hats"])
        d.areas_dev, d.normals_dev, d.tri_nodes_dev = P(self.t["areas"]), P(self.t["normals"]), P(self.t["tri"])
        d.star_indptr_dev, d.star_elem_dev = P(self.t["indptr"]), P(self.t["elem"])
        d.star_local_dev = P(self.t["local"])
        d.n_tq = len(tq)
        for i in range(len(tq)):
            d.tq[i], d.tw[i] = float(tq[i]), float(tw[i])
        self.desc = d
        self.device = device


_DATA_CACHE: dict = {}


def _data_tables(mesh, device=None):
    import torch
    import weakref

    _native.require_cuda()
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    key = (id(mesh), str(dev))
    hit = _DATA_CACHE.get(key)
    if hit is None or hit[0]() is not mesh:
        hit = (weakref.ref(mesh), _DataTables(mesh, dev))
        _DATA_CACHE[key] = hit
    return hit[1]


def _datum_struct(g: HeatKernelDatum) -> "_native.HeatDatum":
    h = _native.HeatDatum()
    h.kind = 0 if g.kind == "value" else 1
    for i in range(3):
        h.src[i] = g.source_point[i]
    h.alpha, h.time_shift = float(g.alpha), float(g.time_shift)
    return h


#: X10 mass solve: Jacobi-PCG per time step to ||r|| <= tol ||b||
MASS_CG_TOL = 1e-15
MASS_CG_MAX_ITER = 1000


def project_data_device(datum: HeatKernelDatum, mesh, timegrid, space: str, stream=None):
    """project_to_space of a device datum on the GPU; returns the (E_t, n_dof)
    float64 tensor and the largest CG iteration count (X10; 0 for X00)."""
    import ctypes

    import torch

    if space not in ("X00", "X10"):
        raise ValueError("space must be 'X00' or 'X10'")
    T = _data_tables(mesh)
    sp_id = 0 if space == "X00" else 1
    E_t = timegrid.n_steps
    n = mesh.n_triangles if sp_id == 0 else mesh.n_vertices
    out = torch.empty((E_t, n), dtype=torch.float64, device=T.device)
    L = _native.load()
    ws = int(L.hb_project_workspace(ctypes.byref(T.desc), sp_id, E_t))
    work = torch.empty(max(ws, 8), dtype=torch.uint8, device=T.device)
    iters = ctypes.c_int64(0)
    _native.call("hb_project_data", ctypes.byref(T.desc), ctypes.byref(_datum_struct(datum)), sp_id, E_t,
                 float(timegrid.step), _native.ptr(out), _native.ptr(work), ctypes.c_size_t(ws),
                 MASS_CG_TOL, MASS_CG_MAX_ITER, ctypes.byref(iters) if sp_id == 1 else None,
                 _native.stream_handle(stream))
    return out, int(iters.value)


def error_sigma_device(coeffs, datum: HeatKernelDatum, mesh, timegrid, stream=None):
    """(num, den) of relative_error_sigma on the GPU (fixed-order sums)."""
    import ctypes

    import torch

    T = _data_tables(mesh)
    c = torch.as_tensor(coeffs, dtype=torch.float64, device=T.device).contiguous()
    if c.ndim != 2 or c.shape[0] != timegrid.n_steps or c.shape[1] not in (mesh.n_triangles, mesh.n_vertices):
        raise ValueError("coefficients must be (E_t, E_x) or (E_t, N_x)")
    p1 = int(c.shape[1] == mesh.n_vertices and c.shape[1] != mesh.n_triangles)
    out2 = torch.empty(2, dtype=torch.float64, device=T.device)
    nb = 16 * timegrid.n_steps * mesh.n_triangles
    work = torch.empty(nb, dtype=torch.uint8, device=T.device)
    _native.call("hb_error_sigma", ctypes.byref(T.desc), ctypes.byref(_datum_struct(datum)), timegrid.n_steps,
                 float(timegrid.step), _native.ptr(c), p1, _native.ptr(out2), _native.ptr(work),
                 ctypes.c_size_t(nb), _native.stream_handle(stream))
    num, den = out2.cpu().tolist()
    return num, den


def project_to_space(fn, mesh, timegrid, space: str, return_device: bool = False):
    """L2(Sigma) projection onto X00 (p0 x p0) or X10 (p1 x p0): (E_t, n_dof)
    (heatbem/field.py:84-119; triangle order 6, 4 Gauss points per step).
    Device datum (HeatKernelDatum / ManufacturedSolution trace): computed on
    the GPU (X10 mass system by PCG instead of the reference's dense
    Cholesky; agrees to ~1e-15); any other callable: the reference's host
    algorithm (``return_device`` then uploads the result)."""
    if space not in ("X00", "X10"):
        raise ValueError("space must be 'X00' or 'X10'")
    g = device_datum(fn)
    if g is not None:
        out, _ = project_data_device(g, mesh, timegrid, space)
        return out if return_device else out.cpu().numpy()
    res = _project_host(fn, mesh, timegrid, space)
    if return_device:
        import torch

        return torch.as_tensor(res, device=torch.device("cuda", torch.cuda.current_device()))
    return res


def _project_host(fn, mesh, timegrid, space: str) -> np.ndarray:
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
    """Relative L2(Sigma_h) error of a coefficient function against fn
    (heatbem/field.py:193-215); on the GPU for a device datum."""
    g = device_datum(fn)
    if g is not None:
        num, den = error_sigma_device(coeffs, g, mesh, timegrid)
        if den == 0.0:
            raise ValueError("exact function has zero L2(Sigma) norm")
        return float(np.sqrt(num / den))
    if not isinstance(coeffs, np.ndarray) and hasattr(coeffs, "cpu"):
        coeffs = coeffs.cpu().numpy()
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
    coeffs = coeffs if isinstance(coeffs, torch.Tensor) else np.asarray(coeffs)
    vals = _eval_grouped(kind, coeffs, xs, k, eps, cur, mesh, timegrid, params, config)
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


_ELEM_MAX_STEPS = 512   # longest history of hb_represent_grid_elem at time-step ends (8 blocks of 64)


def represent(w, u, points, mesh, timegrid, params: KernelParams, config: QuadratureConfig = QuadratureConfig()):
    """Representation formula V~w - Wu at EvalPoints (field.py:184-190).
    Points at time-step ends (eps = 0, k <= 512) with a p0 w and a p1 u go
    through the fused per-element path of ``represent_grid`` (one history per
    distinct spatial point); the others through the two potential launches."""
    import torch

    w_np = w.cpu().numpy() if isinstance(w, torch.Tensor) else np.asarray(w)
    u_np = u.cpu().numpy() if isinstance(u, torch.Tensor) else np.asarray(u)
    n = len(points)
    xs = np.array([np.asarray(p.x, dtype=np.float64) for p in points]).reshape(-1, 3)
    k, eps = _decompose(np.array([float(p.t) for p in points]), timegrid.step)
    fused_ok = (n and w_np.shape[1] == mesh.n_triangles and u_np.shape[1] == mesh.n_vertices
                and not os.environ.get("HB_REP_SEPARATE"))
    # (points past the final time, k > n_steps, take the general path below)
    grid = ((eps == 0.0) & (k <= _ELEM_MAX_STEPS) & (k <= timegrid.n_steps)) if fused_ok else np.zeros(n, bool)
    done = grid.copy()
    vals = np.empty(n)
    if grid.any():
        xu, inv = np.unique(xs[grid], axis=0, return_inverse=True)
        kg = k[grid]
        hist = represent_grid(w_np, u_np, xu, mesh, timegrid, params, config,
                              time_steps=np.arange(0, int(kg.max()) + 1))
        vals[grid] = hist[inv.reshape(-1), kg]
    if fused_ok:
        # eps > 0 (inside a step): one per-element launch per distinct eps with >= 8 points
        off = (eps > 0.0) & (k >= 1) & (k <= 64) & (k <= timegrid.n_steps)
        ev, cnt = np.unique(eps[off], return_counts=True)
        for e_val in ev[cnt >= 8]:
            sel = off & (eps == e_val)
            xu, inv = np.unique(xs[sel], axis=0, return_inverse=True)
            ksel = k[sel]
            ks_all = np.arange(1, int(ksel.max()) + 1)
            hist = _represent_grid_fused(w_np, u_np, xu, ks_all, mesh, timegrid, params, config,
                                         eps=float(e_val)).cpu().numpy()
            vals[sel] = hist[inv.reshape(-1), ksel - 1]
            done |= sel
    if not done.any():
        sv, w1 = eval_single_layer_potential(w, points, mesh, timegrid, params, config)
        dv, w2 = eval_double_layer_potential(u, points, mesh, timegrid, params, config)
        return sv - dv, w1 | w2
    rest = np.flatnonzero(~done)
    if len(rest):
        pts = [points[i] for i in rest]
        sv, _ = eval_single_layer_potential(w, pts, mesh, timegrid, params, config)
        dv, _ = eval_double_layer_potential(u, pts, mesh, timegrid, params, config)
        vals[rest] = sv - dv
    T = _tables(mesh, config, torch.device("cuda", torch.cuda.current_device()))
    warn = _boundary_warnings(torch.as_tensor(xs, device=T.qw.device), mesh, T).cpu().numpy()
    return vals, warn


def _represent_grid_fused(w, u, xs, ks, mesh, timegrid, params, config, stream=None, eps: float = 0.0):
    """u = V~w - W u at (x_i, k_j h) in one hb_represent_grid launch: the two
    potentials share the kernel-value evaluation (csrc/hb_field.cu)."""
    import torch

    _native.require_cuda()
    T = _tables(mesh, config, torch.device("cuda", torch.cuda.current_device()))
    dev = T.qw.device
    if (w.shape[1] == mesh.n_triangles and u.shape[1] == mesh.n_vertices
            and not os.environ.get("HB_REP_NODES")):
        # p0 / p1 densities: the contraction runs once per element (hb_represent_grid_elem)
        de = torch.as_tensor(np.ascontiguousarray(np.asarray(w).T), dtype=torch.float64, device=dev)
        uu = torch.as_tensor(np.asarray(u), dtype=torch.float64, device=dev)
        dv = uu[:, T.tri].permute(1, 2, 0).contiguous()          # (E_x, 3, E_t)
        X = torch.as_tensor(np.ascontiguousarray(xs), dtype=torch.float64, device=dev)
        K = torch.as_tensor(np.ascontiguousarray(ks, dtype=np.int64), device=dev)
        out = torch.empty((xs.shape[0], len(ks)), dtype=torch.float64, device=dev)
        _native.call("hb_represent_grid_elem", xs.shape[0], len(ks), timegrid.n_steps, mesh.n_triangles, T.nq,
                     _native.ptr(X), _native.ptr(K), int(ks.max()), _native.ptr(de), _native.ptr(dv),
                     _native.ptr(T.hats), _native.ptr(T.qpts), _native.ptr(T.qw), _native.ptr(T.areas),
                     _native.ptr(T.normals), timegrid.step, params.alpha, params.delta_eps, params.rho_eps,
                     float(eps), _native.ptr(out), _native.stream_handle(stream))
        return out
    if eps:
        raise ValueError("eps > 0 needs a p0 single-layer and a p1 double-layer density")
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
    elem_ok = (np.asarray(w).shape[1] == mesh.n_triangles and np.asarray(u).shape[1] == mesh.n_vertices
               and not os.environ.get("HB_REP_NODES"))
    # histories up to 64 steps: the fused kernels; up to 512 with p0 / p1 densities: the
    # per-element kernel, one launch per 64 output steps (csrc/hb_field.cu k_represent_elem LONG)
    if nt and int(ks.max()) <= (_ELEM_MAX_STEPS if elem_ok else 64) and not os.environ.get("HB_REP_SEPARATE"):
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
