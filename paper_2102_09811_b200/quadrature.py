"""Quadrature tables for the pair integrals (host side, numpy).

Same rules as the reference ``heatbem.quadrature``:

* symmetric positive triangle rules of orders 1-6 and collapsed-Gauss rules
  for orders 7-10 (quadrature.py:26-110);
* pair classification into identical / common edge / common vertex /
  separated with the vertex permutations the Sauter-Schwab maps assume
  (quadrature.py:117-153);
* Sauter-Schwab subdomain maps pulled back to a tensor Gauss rule on the
  unit 4-cube: 6 / 5 / 2 subdomains (quadrature.py:160-279).

The tables are device-kernel inputs; their node/weight arithmetic is kept
in the reference's evaluation order so the CPU oracle built on them
reproduces the reference bit-for-bit (tests/test_tables_golden.py).
"""
from __future__ import annotations

from dataclasses import dataclass
from functools import lru_cache

import numpy as np


@lru_cache(maxsize=None)
def gauss01(n_points: int):
    """Gauss-Legendre on [0, 1] (exact to degree 2n-1)."""
    if n_points < 1:
        raise ValueError("n_points must be >= 1")
    x, w = np.polynomial.legendre.leggauss(n_points)
    return 0.5 * (x + 1.0), 0.5 * w


@dataclass(frozen=True)
class TriangleRule:
    """Rule on {u, v >= 0, u + v <= 1}; weights sum to 1/2."""

    order: int
    nodes: np.ndarray
    weights: np.ndarray


def _centroid_orbit():
    return [(1.0 / 3.0, 1.0 / 3.0)]


def _three_orbit(a: float):
    b = 0.5 * (1.0 - a)
    return [(b, b), (a, b), (b, a)]


def _six_orbit(a: float, b: float, c: float):
    perms = ((a, b, c), (a, c, b), (b, a, c), (b, c, a), (c, a, b), (c, b, a))
    return [(p[1], p[2]) for p in perms]


# barycentric orbit generators and unit-area weights (Strang-Fix / Dunavant)
_ORBITS = {
    1: ((_centroid_orbit, (), 1.0),),
    2: ((_three_orbit, (2.0 / 3.0,), 1.0 / 3.0),),
    3: ((_six_orbit, (0.659027622374092, 0.231933368553031, 0.109039009072877), 1.0 / 6.0),),
    4: ((_three_orbit, (0.816847572980459,), 0.109951743655322),
        (_three_orbit, (0.108103018168070,), 0.223381589678011)),
    5: ((_centroid_orbit, (), 0.225),
        (_three_orbit, (0.79742698535308720,), 0.12593918054482717),
        (_three_orbit, (0.05971587178976981,), 0.13239415278850616)),
    6: ((_three_orbit, (0.873821971016996,), 0.050844906370207),
        (_three_orbit, (0.501426509658179,), 0.116786275726379),
        (_six_orbit, (0.636502499121399, 0.310352451033785, 0.053145049844816), 0.082851075618374)),
}


@lru_cache(maxsize=None)
def triangle_rule(order: int) -> TriangleRule:
    if order in _ORBITS:
        pts, wts = [], []
        for gen, args, w in _ORBITS[order]:
            orbit = gen(*args)
            pts += orbit
            wts += [w / 2.0] * len(orbit)
        return TriangleRule(order, np.array(pts), np.array(wts))
    if 7 <= order <= 10:
        m = (order + 3) // 2
        s, ws = gauss01(m)
        t, wt = gauss01(m)
        S, T = np.meshgrid(s, t, indexing="ij")
        WS, WT = np.meshgrid(ws, wt, indexing="ij")
        u = S.ravel()
        v = (T * (1.0 - S)).ravel()
        w = (WS * WT * (1.0 - S)).ravel()
        return TriangleRule(order, np.column_stack([u, v]), w)
    raise ValueError(f"unsupported triangle rule order {order}")


# ---------------------------------------------------------------------------
# pair classification
# ---------------------------------------------------------------------------

CASE_IDS = {"identical": 0, "common_edge": 1, "common_vertex": 2}
_IDENT = (0, 1, 2)


def _rot(k: int):
    return (k, (k + 1) % 3, (k + 2) % 3)


def classify_triangles(t, s, same: bool):
    """Classification of two vertex triples (see :func:`classify_pair`)."""
    if same:
        return "identical", _IDENT, _IDENT
    common = [g for g in t if g in s]
    if not common:
        return "separated", _IDENT, _IDENT
    if len(common) == 1:
        return "common_vertex", _rot(t.index(common[0])), _rot(s.index(common[0]))
    if len(common) == 2:
        # first local edge (k, k+1) of the test triangle lying on both
        k = next(k for k in range(3) if t[k] in common and t[(k + 1) % 3] in common)
        ia, ib = s.index(t[k]), s.index(t[(k + 1) % 3])
        return "common_edge", _rot(k), (ia, ib, 3 - ia - ib)
    return "identical", _IDENT, tuple(s.index(g) for g in t)


def classify_pair(mesh, i_test: int, i_trial: int):
    """(case, perm_test, perm_trial): shared vertices first, in the same
    global order on both triangles (heatbem.quadrature.classify_pair)."""
    return classify_triangles(mesh.triangles[i_test].tolist(),
                              mesh.triangles[i_trial].tolist(), i_test == i_trial)


def touching_csr(mesh):
    """Per test element, the sorted touching trial elements with case ids
    and alignment permutations (heatbem.assembly._touching_csr,
    assembly.py:119-144): (indptr, idx, case, perm_test, perm_trial)."""
    tris = mesh.triangles.tolist()
    incident: dict = {}
    for e, tri in enumerate(tris):
        for v in tri:
            incident.setdefault(v, []).append(e)
    indptr = [0]
    idx, case, pt, ps = [], [], [], []
    for e, tri in enumerate(tris):
        for f in sorted({g for v in tri for g in incident[v]}):
            c, p_t, p_s = classify_triangles(tri, tris[f], e == f)
            idx.append(f)
            case.append(CASE_IDS[c])
            pt.append(p_t)
            ps.append(p_s)
        indptr.append(len(idx))
    i64 = np.int64
    return (np.array(indptr, dtype=i64), np.array(idx, dtype=i64), np.array(case, dtype=i64),
            np.array(pt, dtype=i64).reshape(-1, 3), np.array(ps, dtype=i64).reshape(-1, 3))


# ---------------------------------------------------------------------------
# Sauter-Schwab maps: (xi, e1, e2, e3) in [0,1]^4 -> (x1, x2, y1, y2, jac) on
# the product of two simplices {0 <= x2 <= x1 <= 1}
# ---------------------------------------------------------------------------

def _ident_maps():
    def a(xi, e1, e2, e3):
        return (xi, xi * (1 - e1 + e1 * e2), xi * (1 - e1 * e2 * e3), xi * (1 - e1),
                xi ** 3 * e1 ** 2 * e2)

    def b(xi, e1, e2, e3):
        return (xi, xi * e1 * (1 - e2 + e2 * e3), xi * (1 - e1 * e2), xi * e1 * (1 - e2),
                xi ** 3 * e1 ** 2 * e2)

    def c(xi, e1, e2, e3):
        return (xi * (1 - e1 * e2 * e3), xi * e1 * (1 - e2 * e3), xi, xi * e1 * (1 - e2),
                xi ** 3 * e1 ** 2 * e2)

    def swapped(fn):
        def g(*args):
            x1, x2, y1, y2, jac = fn(*args)
            return y1, y2, x1, x2, jac
        return g

    return [a, swapped(a), b, swapped(b), c, swapped(c)]


def _edge_maps():
    return [
        lambda xi, e1, e2, e3: (xi, xi * e1 * e3, xi * (1 - e1 * e2), xi * e1 * (1 - e2),
                                xi ** 3 * e1 ** 2),
        lambda xi, e1, e2, e3: (xi, xi * e1, xi * (1 - e1 * e2 * e3), xi * e1 * e2 * (1 - e3),
                                xi ** 3 * e1 ** 2 * e2),
        lambda xi, e1, e2, e3: (xi * (1 - e1 * e2), xi * e1 * (1 - e2), xi, xi * e1 * e2 * e3,
                                xi ** 3 * e1 ** 2 * e2),
        lambda xi, e1, e2, e3: (xi * (1 - e1 * e2 * e3), xi * e1 * e2 * (1 - e3), xi, xi * e1,
                                xi ** 3 * e1 ** 2 * e2),
        lambda xi, e1, e2, e3: (xi * (1 - e1 * e2 * e3), xi * e1 * (1 - e2 * e3), xi, xi * e1 * e2,
                                xi ** 3 * e1 ** 2 * e2),
    ]


def _vertex_maps():
    return [
        lambda xi, e1, e2, e3: (xi, xi * e1, xi * e2, xi * e2 * e3, xi ** 3 * e2),
        lambda xi, e1, e2, e3: (xi * e2, xi * e2 * e3, xi, xi * e1, xi ** 3 * e2),
    ]


_MAPS = {"identical": _ident_maps, "common_edge": _edge_maps, "common_vertex": _vertex_maps}


@dataclass(frozen=True)
class DuffyRule:
    case: str
    n_subdomains: int
    nodes_test: np.ndarray
    nodes_trial: np.ndarray
    weights: np.ndarray


@lru_cache(maxsize=None)
def duffy_rule(case: str, singular_order: int) -> DuffyRule:
    """Mapped 4-cube Gauss rule for a touching pair; weights sum to 1/4."""
    if case not in _MAPS:
        raise ValueError(f"no Duffy rule for case {case!r}")
    if singular_order < 1:
        raise ValueError("singular_order must be >= 1")
    z, w = gauss01(singular_order)
    xi, e1, e2, e3 = (g.ravel() for g in np.meshgrid(z, z, z, z, indexing="ij"))
    wg = np.meshgrid(w, w, w, w, indexing="ij")
    w4 = (wg[0] * wg[1] * wg[2] * wg[3]).ravel()
    tn, sn, wt = [], [], []
    maps = _MAPS[case]()
    for fn in maps:
        x1, x2, y1, y2, jac = fn(xi, e1, e2, e3)
        tn.append(np.column_stack([x1 - x2, x2]))   # simplex -> reference chart
        sn.append(np.column_stack([y1 - y2, y2]))
        wt.append(w4 * jac)
    return DuffyRule(case, len(maps), np.concatenate(tn), np.concatenate(sn), np.concatenate(wt))


@dataclass(frozen=True)
class QuadratureConfig:
    """Regular triangle-rule order and Gauss points per 4-cube axis."""

    regular_order: int = 4
    singular_order: int = 4

    def __post_init__(self):
        if self.regular_order < 1 or self.singular_order < 1:
            raise ValueError("quadrature orders must be >= 1")

    @property
    def near_order(self) -> int:
        return min(self.regular_order + 2, 10)


# ---------------------------------------------------------------------------
# packed device tables
# ---------------------------------------------------------------------------

def rule_tables(mesh, order: int):
    """(hats (nq,3), weights (nq,), physical points (E_x,nq,3)) for the
    product rule; points evaluated as v0 + u (v1-v0) + v (v2-v0)."""
    rule = triangle_rule(order)
    u, v = rule.nodes[:, 0], rule.nodes[:, 1]
    hats = np.column_stack([1.0 - u - v, u, v])
    tv = mesh.triangle_vertices()
    base = tv[:, None, 0, :]
    pts = base + u[None, :, None] * (tv[:, None, 1, :] - base) + v[None, :, None] * (tv[:, None, 2, :] - base)
    return hats, rule.weights.copy(), np.ascontiguousarray(pts)


def duffy_tables(singular_order: int):
    """Concatenated identical / edge / vertex rules: offsets (4,), test and
    trial nodes (n,2), weights (n,)."""
    rules = [duffy_rule(c, singular_order) for c in ("identical", "common_edge", "common_vertex")]
    off = np.cumsum([0] + [len(r.weights) for r in rules]).astype(np.int64)
    return (off,
            np.ascontiguousarray(np.concatenate([r.nodes_test for r in rules])),
            np.ascontiguousarray(np.concatenate([r.nodes_trial for r in rules])),
            np.concatenate([r.weights for r in rules]))
