"""CPU prototype of the moment form of the time second difference (accuracy study).

For a pair whose points all satisfy t = x^2 = rho~^2 / i <= TM at gaps i >= i*,
the factor-free kernel value is a power series in t, so

    L(i) = jac S sum_k a_k Mk i^(s-k),   Mk = sum_p W_p rho~_p^(2k)
    B^d  = jac S sum_k a_k Mk D2[i^(s-k)](d)      (d - 1 >= i*)

with the second difference D2 of the powers taken exactly (mpmath).  Compares
B^d against the exact quadrature (tests/golden/exact.npz) on the c2 golden rows.
"""
import os
import sys

import mpmath as mp
import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2102_09811_b200 as hb  # noqa: E402
from paper_2102_09811_b200.device import host_tables  # noqa: E402

mp.mp.dps = 40
SQPI = mp.sqrt(mp.pi)
NK = int(os.environ.get("NK", "22"))
TM = float(os.environ.get("TM", "1.0"))


def coeffs(op):
    out = []
    for k in range(NK):
        if op == "V":   # x H
            c = (mp.mpf(-1) ** k) / (mp.factorial(k) * (2 * k + 1)) / SQPI + (mp.mpf(-1) ** k) / mp.factorial(k) / SQPI
            if k >= 1:
                c += 2 / SQPI * (mp.mpf(-1) ** (k - 1)) / (mp.factorial(k - 1) * (2 * k - 1))
        elif op == "K":  # F / x
            c = 2 / SQPI * (mp.mpf(-1) ** k) / (mp.factorial(k) * (2 * k + 1)) \
                - (mp.mpf(-1) ** (k + 1)) / (mp.factorial(k + 1) * (2 * k + 3)) / SQPI \
                + (mp.mpf(-1) ** (k + 1)) / mp.factorial(k + 1) / SQPI
        else:            # erf / x
            c = 2 / SQPI * (mp.mpf(-1) ** k) / (mp.factorial(k) * (2 * k + 1))
        out.append(c)
    return out


def main():
    op = os.environ.get("OP", "V")
    m = hb.unit_cube_mesh(3)
    Et, alpha = 32, 1.0
    h = 1.0 / Et
    g = np.load(os.path.join(ROOT, "tests/golden/c2.npz"))
    ex = np.load(os.path.join(ROOT, "tests/golden/exact.npz"))
    rows = g["rows_p0"]
    H = host_tables(m, hb.QuadratureConfig())
    reg_h, reg_w, reg_p = H.reg
    near_h, near_w, near_p = H.near
    ip, idx = H.tn[0], H.tn[1]
    u2 = 4 * alpha * h
    u = np.sqrt(u2)
    a = coeffs(op)
    s = mp.mpf(0.5) if op == "V" else mp.mpf(-0.5)
    S = (1 / (2 * alpha * alpha)) * u if op == "V" else 1.0 / u
    # T[k][d] = a_k * D2[i^(s-k)](d) (exact, rounded once), d = 2..Et-1
    T = np.zeros((NK, Et))
    Lt = np.zeros((NK, Et + 2))
    for k in range(NK):
        for d in range(2, Et):
            v = -(mp.mpf(d - 1) ** (s - k)) + 2 * mp.mpf(d) ** (s - k) - mp.mpf(d + 1) ** (s - k)
            T[k, d] = float(a[k] * v)
    bmax = g[f"{op}_maxabs"]
    exr = ex[f"c2_{op}_exact_rows"]
    refr = g[f"{op}_rows"]
    E = m.n_triangles
    C = E if op == "V" else m.n_vertices
    got = np.full((Et, len(rows), C), np.nan)
    for ri, e in enumerate(rows):
        touch = set(idx[ip[e]:ip[e + 1]].tolist())
        acc_rows = np.zeros((Et, C))
        valid = np.ones((Et, C), dtype=bool)
        for f in range(E):
            dist = np.sqrt(((m.centroids[e] - m.centroids[f]) ** 2).sum())
            near = dist < 2.0 * max(m.diameters[e], m.diameters[f])
            hats, w, P = (near_h, near_w, near_p) if near else (reg_h, reg_w, reg_p)
            x, y = P[e], P[f]
            r = x[:, None, :] - y[None, :, :]
            rho2 = (r * r).sum(-1)
            W = w[:, None] * w[None, :]
            jac = m.areas[e] * m.areas[f] / np.pi
            if op == "V":
                Wt = [W]
                cols = [f]
            else:
                rn = (r * m.normals[f][None, None, :]).sum(-1)
                Wt = [W * hats[None, :, j] * (-rn) / (2 * alpha) for j in range(3)]
                cols = [int(m.triangles[f, j]) for j in range(3)]
            rt2 = rho2 / u2
            istar = max(1, int(np.ceil(rt2.max() / TM)))
            pw = np.ones_like(rt2)
            M = np.zeros((len(Wt), NK))
            for k in range(NK):
                for j, Wj in enumerate(Wt):
                    M[j, k] = (Wj * pw).sum()
                pw = pw * rt2
            for d in range(Et):
                if f in touch or d < 2 or d - 1 < istar:
                    for c in cols:
                        valid[d, c] = False
                    continue
                for j, c in enumerate(cols):
                    acc_rows[d, c] += jac * S * (M[j] @ T[:, d])
        acc_rows[~valid] = np.nan
        got[:, ri, :] = acc_rows
    print(f"op {op} NK {NK} TM {TM}")
    print(" d  n_valid   moment-vs-exact  ref-vs-exact(same entries)  eps_ref(d)")
    for d in range(Et):
        ok = ~np.isnan(got[d])
        if not ok.any():
            continue
        em = np.abs(got[d][ok] - exr[d][ok]).max() / bmax[d]
        er = np.abs(refr[d][ok] - exr[d][ok]).max() / bmax[d]
        print(f"{d:2d} {ok.sum():7d}   {em:.2e}        {er:.2e}              {ex[f'c2_{op}_eps_ref'][d]:.2e}")


if __name__ == "__main__":
    main()
