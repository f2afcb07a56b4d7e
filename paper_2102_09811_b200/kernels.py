"""Heat-kernel parameters and host-side (numpy) kernel evaluations.

``KernelParams`` carries alpha, the step width and the geometric length
scale that fix the two branch thresholds of the closed-form temporal
antiderivatives (heatbem/kernels.py:27-50):

    delta_eps = 1e-14 * h_t        rho_eps = 1e-12 * length_scale

The device kernels (csrc/hb_special.cuh, csrc/hb_assembly.cu) evaluate the same antiderivatives;
the numpy versions here serve host-side data (projection of boundary data,
manufactured solutions) and tests.  G^{dtau} and G^{dtau dt} denote the first
and second temporal antiderivatives of the heat kernel G_alpha.
"""
from __future__ import annotations

from dataclasses import dataclass
from enum import Enum

import numpy as np
from scipy.special import erf


class SingularEvaluationError(ValueError):
    """Kernel requested where no finite limit exists (rho = delta = 0)."""


@dataclass(frozen=True)
class KernelParams:
    alpha: float
    h_t: float
    length_scale: float = 1.0

    def __post_init__(self):
        if not self.alpha > 0:
            raise ValueError("alpha must be positive")
        if not self.h_t > 0:
            raise ValueError("h_t must be positive")

    @property
    def delta_eps(self) -> float:
        return 1e-14 * self.h_t

    @property
    def rho_eps(self) -> float:
        return 1e-12 * self.length_scale


class TemporalWeightKind(Enum):
    SingleLayer = "single_layer"
    DoubleLayer = "double_layer"
    HypersingularD2 = "hypersingular_d2"


def _norm(r):
    return np.sqrt(np.sum(r * r, axis=-1))


def fundamental(r, dt, alpha: float):
    """G_alpha(r, dt) = (4 pi alpha dt)^{-3/2} exp(-|r|^2 / (4 alpha dt)), 0 for dt <= 0."""
    r = np.asarray(r, dtype=np.float64)
    dt = np.asarray(dt, dtype=np.float64)
    pos = dt > 0
    t = np.where(pos, dt, 1.0)
    g = (4.0 * np.pi * alpha * t) ** -1.5 * np.exp(-np.sum(r * r, axis=-1) / (4.0 * alpha * t))
    return np.where(pos, g, 0.0)[()]


def grad_fundamental_normal(r, n_x, dt, alpha: float):
    """alpha * dG_alpha/dn_x(r, dt) (derivative in the first argument)."""
    r = np.asarray(r, dtype=np.float64)
    n_x = np.asarray(n_x, dtype=np.float64)
    dt = np.asarray(dt, dtype=np.float64)
    pos = dt > 0
    t = np.where(pos, dt, 1.0)
    rn = np.sum(r * n_x, axis=-1)
    g = -rn / (16.0 * (np.pi * alpha) ** 1.5 * t ** 2.5) * np.exp(-np.sum(r * r, axis=-1) / (4.0 * alpha * t))
    return np.where(pos, g, 0.0)[()]


def _split(rho, delta, params):
    small_d = delta <= params.delta_eps
    small_r = rho <= params.rho_eps
    return small_d, small_r, np.where(small_r, 1.0, rho), np.where(small_d, 1.0, delta)


def antideriv_tau(rho, delta, params: KernelParams, negate: bool = False):
    """G^{dtau}(rho, delta) = erf(rho / (2 sqrt(alpha delta))) / (4 pi alpha rho)."""
    a = params.alpha
    rho = np.asarray(rho, dtype=np.float64)
    delta = np.asarray(delta, dtype=np.float64)
    sd, sr, r, d = _split(rho, delta, params)
    if np.any(sd & sr):
        raise SingularEvaluationError("g_dtau has no finite limit at rho = delta = 0")
    gen = erf(r / (2.0 * np.sqrt(a * d))) / (4.0 * np.pi * a * r)
    out = np.where(sd, 1.0 / (4.0 * np.pi * a * r),
                   np.where(sr, 1.0 / (4.0 * np.sqrt(np.pi ** 3 * a ** 3 * d)), gen))
    return (-out if negate else out)[()]


def antideriv_tau_t(rho, delta, params: KernelParams):
    """G^{dtau dt}(rho, delta); 0 at the origin."""
    a = params.alpha
    rho = np.asarray(rho, dtype=np.float64)
    delta = np.asarray(delta, dtype=np.float64)
    sd, sr, r, d = _split(rho, delta, params)
    x = r / (2.0 * np.sqrt(a * d))
    gen = ((r / (2.0 * a * a) + d / (a * r)) * erf(x)
           + np.sqrt(d) / np.sqrt(np.pi * a ** 3) * np.exp(-x * x)) / (4.0 * np.pi)
    lim_d = rho / (8.0 * np.pi * a * a)
    lim_r = np.sqrt(np.where(sd, 0.0, delta)) / (2.0 * np.sqrt(np.pi ** 3 * a ** 3))
    return np.where(sd, lim_d, np.where(sr, lim_r, gen))[()]


def normal_deriv_antideriv_tau(r, n_y, delta, params: KernelParams):
    """alpha * dG^{dtau}/dn_y."""
    a = params.alpha
    r = np.asarray(r, dtype=np.float64)
    delta = np.asarray(delta, dtype=np.float64)
    rho = _norm(r)
    rn = np.sum(r * np.asarray(n_y, dtype=np.float64), axis=-1)
    sd, sr, rs, d = _split(rho, delta, params)
    if np.any(sd & sr):
        raise SingularEvaluationError("d(g_dtau)/dn_y undefined at rho = 0")
    x = rs / (2.0 * np.sqrt(a * d))
    gen = (rn / (rs * rs)) * (erf(x) / rs - np.exp(-x * x) / np.sqrt(np.pi * a * d)) / (4.0 * np.pi)
    return np.where(sr, 0.0, np.where(sd, rn / (4.0 * np.pi * rs ** 3), gen))[()]


def normal_deriv_antideriv_tau_t(r, n_y, delta, params: KernelParams):
    """alpha * dG^{dtau dt}/dn_y."""
    a = params.alpha
    r = np.asarray(r, dtype=np.float64)
    delta = np.asarray(delta, dtype=np.float64)
    rho = _norm(r)
    rn = np.sum(r * np.asarray(n_y, dtype=np.float64), axis=-1)
    sd, sr, rs, d = _split(rho, delta, params)
    if np.any(sd & sr):
        raise SingularEvaluationError("d(g_dtau_dt)/dn_y undefined at rho = delta = 0")
    x = rs / (2.0 * np.sqrt(a * d))
    gen = -(rn / rs) * ((1.0 / (2.0 * a) - d / (rs * rs)) * erf(x)
                        + np.sqrt(d) / (rs * np.sqrt(np.pi * a)) * np.exp(-x * x)) / (4.0 * np.pi)
    return np.where(sr, 0.0, np.where(sd, -rn / (8.0 * np.pi * a * rs), gen))[()]


def temporal_weight(kind: TemporalWeightKind, r, d: int, params: KernelParams, n_y=None):
    """Pointwise block weight V^d / K^d / D2^d: the second difference in time
    of the antiderivative (heatbem/kernels.py:197-251)."""
    if d < 0:
        raise ValueError("block index d must be non-negative")
    h, a = params.h_t, params.alpha
    r = np.asarray(r, dtype=np.float64)
    rho = _norm(r)
    if kind is TemporalWeightKind.SingleLayer:
        F = lambda t: antideriv_tau_t(rho, t, params)  # noqa: E731
        if d == 0:
            return h * antideriv_tau(rho, 0.0, params) - F(h) + F(0.0)
    elif kind is TemporalWeightKind.DoubleLayer:
        if n_y is None:
            raise ValueError("DoubleLayer weight requires the trial normal n_y")
        F = lambda t: normal_deriv_antideriv_tau_t(r, n_y, t, params)  # noqa: E731
        if d == 0:
            return h * normal_deriv_antideriv_tau(r, n_y, 0.0, params) - F(h) + F(0.0)
    elif kind is TemporalWeightKind.HypersingularD2:
        F = lambda t: a * antideriv_tau(rho, t, params)  # noqa: E731
        if d == 0:
            return F(0.0) - F(h)
    else:
        raise ValueError(f"unknown temporal weight kind {kind!r}")
    return 2.0 * F(d * h) - F((d + 1) * h) - F((d - 1) * h)
