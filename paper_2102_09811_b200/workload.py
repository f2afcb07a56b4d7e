"""Algorithmic work of one assembly (the roofline numerator).

N_eval(op) = E_t * sum_class n_pairs(class) * q(class), with q = 1536 / 1280 /
512 (identical / common edge / common vertex, singular order 4), 144 (near,
order-6 product rule) and 36 (far, order-4 product rule); n_pairs counts the
upper triangle (f >= e) for the symmetric V, V11, D2 and all ordered pairs for
K -- the reference's own work (_assembly_numba.py:137).  The delta = 0 pass
(closed-form limits, no erf/exp) is excluded.  FLOPs per evaluation (SASS
census of the erf + exp + kernel body, DFMA = 2):
F_V = 118, F_K = 124, F_D2 = 98.
"""
from __future__ import annotations

import numpy as np

from .quadrature import QuadratureConfig, duffy_rule, touching_csr, triangle_rule

FLOPS_PER_EVAL = {"V": 118, "V11": 118, "K": 124, "D2": 98}


def pair_counts(mesh, symmetric: bool, config: QuadratureConfig = QuadratureConfig(), chunk: int = 2048):
    """dict class -> number of (e, f) pairs; also 'd2_zero' = separated and
    touching pairs with n_e . n_f == 0 exactly (skipped by the D2 kernel)."""
    E = mesh.n_triangles
    ip, idx, case = touching_csr(mesh)[:3]
    rows = np.repeat(np.arange(E), np.diff(ip))
    keep = idx >= rows if symmetric else np.ones(len(idx), dtype=bool)
    out = {"identical": int(np.sum(keep & (case == 0))), "common_edge": int(np.sum(keep & (case == 1))),
           "common_vertex": int(np.sum(keep & (case == 2))), "near": 0, "far": 0, "d2_zero": 0}
    touch = np.zeros(0, dtype=np.int64)
    c, dm, nrm = mesh.centroids, mesh.diameters, mesh.normals
    for e0 in range(0, E, chunk):
        e1 = min(E, e0 + chunk)
        dx = c[e0:e1, None, 0] - c[None, :, 0]
        dy = c[e0:e1, None, 1] - c[None, :, 1]
        dz = c[e0:e1, None, 2] - c[None, :, 2]
        near = np.sqrt(dx * dx + dy * dy + dz * dz) < 2.0 * np.maximum(dm[e0:e1, None], dm[None, :])
        valid = np.ones_like(near)
        if symmetric:
            valid &= np.arange(E)[None, :] >= np.arange(e0, e1)[:, None]
        tmask = np.zeros_like(near)
        sel = (rows >= e0) & (rows < e1)
        tmask[rows[sel] - e0, idx[sel]] = True
        sep = valid & ~tmask
        out["near"] += int(np.sum(sep & near))
        out["far"] += int(np.sum(sep & ~near))
        dot = (nrm[e0:e1, None, 0] * nrm[None, :, 0] + nrm[e0:e1, None, 1] * nrm[None, :, 1]) \
            + nrm[e0:e1, None, 2] * nrm[None, :, 2]
        out["d2_zero"] += int(np.sum(valid & (dot == 0.0)))
    del touch
    return out


def q_per_class(config: QuadratureConfig = QuadratureConfig()):
    so = config.singular_order
    return {"identical": len(duffy_rule("identical", so).weights),
            "common_edge": len(duffy_rule("common_edge", so).weights),
            "common_vertex": len(duffy_rule("common_vertex", so).weights),
            "near": len(triangle_rule(config.near_order).weights) ** 2,
            "far": len(triangle_rule(config.regular_order).weights) ** 2}


def operator_work(mesh, op: str, n_gaps: int, config: QuadratureConfig = QuadratureConfig()):
    """(N_eval, flops) for n_gaps time gaps (E_t for a full assembly)."""
    sym = op != "K"
    counts = pair_counts(mesh, sym, config)
    q = q_per_class(config)
    per_gap = sum(counts[k] * q[k] for k in q)
    n_eval = n_gaps * per_gap
    return {"pairs": counts, "evals_per_gap": per_gap, "n_eval": n_eval,
            "flops": n_eval * FLOPS_PER_EVAL[op]}


def entries(mesh, op: str, n_blocks: int) -> int:
    E, N = mesh.n_triangles, mesh.n_vertices
    R = N if op in ("D", "D2", "V11") else E
    C = E if op == "V" else N
    return n_blocks * R * C
