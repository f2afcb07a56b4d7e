"""Generate paper_2102_09811_b200/csrc/hb_special_coeffs.h (run in the build
container; needs mpmath).  Deterministic: re-running reproduces the header.

The pair kernels evaluate, per (point pair, time gap), one univariate
function of x = rho / (2 sqrt(alpha delta)):

    erf(x)                                           (D2)
    F(x) = erf(x) (1 - 1/(2x^2)) + e^{-x^2} / (sqrt(pi) x)   (K, cancellation-free)
    H(x) = erf(x) (1 + 1/(2x^2)) + e^{-x^2} / (sqrt(pi) x)   (V)

* x < X0: polynomials in t = x^2 -- erf = x Pe(t), F = x Pf(t),
  H = 2/(sqrt(pi) x) + x Ph(t) -- Chebyshev interpolants on [0, X0^2]
  converted to monomials in t (well conditioned: the Taylor coefficients
  decay like 1/m!).
* X0 <= x < XL: the function values themselves, piecewise (21 pieces of
  width 1/4, degree 12 in u = (x - mid) / half; all four are analytic there).
* x >= XL = 6.25: the asymptotes erf = E = 1, H/F = 1 +- 1/(2x^2), which the
  exact values round to (e^{-x^2}(...) < 2^-53 relative; reported below).
* the direct pair kernels' factor-free kinds (x H as M, F/x, erf/x) also as
  uniform pieces of [0, XL): width 1/16, degree 7.
"""
import os
import sys

import mpmath as mp

mp.mp.dps = 50
X0 = mp.mpf(os.environ.get("HB_X0", "1.0"))
# per-function degrees: the lowest at which the double Horner evaluation is
# within ~2.5e-16 relative (lower degrees lose digits: see the report lines)
DEG_S = {k: int(os.environ.get(f"HB_DEGS_{k}", os.environ.get("HB_DEGS", d)))
         for k, d in (("Pe", "11"), ("Pf", "10"), ("Ph", "10"), ("Pg", "11"))}
SQPI = mp.sqrt(mp.pi)
MID_W = mp.mpf(os.environ.get("HB_MID_W", "0.25"))
MID_PIECES = int(os.environ.get("HB_MID_PIECES", "21"))
DEG_M = {k: int(os.environ.get(f"HB_DEGM_{k}", os.environ.get("HB_DEGM", d)))
         for k, d in (("H", "12"), ("F", "10"), ("erf", "10"), ("E", "11"), ("xH", "9"), ("Fx", "9"),
                      ("ex", "10"), ("Ex3", "11"))}


def F_H(x):
    return mp.erf(x) * (1 + 1 / (2 * x * x)) + mp.exp(-x * x) / (SQPI * x)


def F_F(x):
    return mp.erf(x) * (1 - 1 / (2 * x * x)) + mp.exp(-x * x) / (SQPI * x)


def F_E(x):
    return mp.erf(x) - 2 * x * mp.exp(-x * x) / SQPI


# assembly forms without a per-point factor (csrc/hb_special.cuh kinds 4-6):
#   V  = rho/(2a^2) H(x)   = [x H(x)]   * ic / (2a^2)      (ic = 1/cx per gap;
#        x H = 2/sqrt(pi) + t M(x): the series is M = Ph(t), the table holds M)
#   K  = -(rn/rho)/(2a) F  = [F(x) / x] * rho (-(rn/rho)/(2a)) * cx
#   D2 = erf(x) / rho      = [erf(x)/x] * cx
def F_xH(x):   # tabulated as M(x) = (x H(x) - 2/sqrt(pi)) / x^2, so that x H = 2/sqrt(pi) + t M in every region
    return (x * F_H(x) - 2 / SQPI) / (x * x)


def F_Fx(x):
    return F_F(x) / x


def F_ex(x):
    return mp.erf(x) / x


def F_Ex3(x):   # E(x) / x^3 (double-layer potential, factor-free: E rn / rho^3 = [E / x^3] rn cx^3)
    return F_E(x) / (x * x * x)


def S_e(t):
    if t == 0:
        return 2 / SQPI
    x = mp.sqrt(t)
    return mp.erf(x) / x


def S_f(t):
    if t == 0:
        return mp.mpf(4) / (3 * SQPI)
    x = mp.sqrt(t)
    return (mp.erf(x) * (1 - 1 / (2 * t)) + mp.exp(-t) / (SQPI * x)) / x


def S_h(t):
    if t == 0:
        return mp.mpf(2) / (3 * SQPI)
    x = mp.sqrt(t)
    return (mp.erf(x) * (1 + 1 / (2 * t)) + mp.exp(-t) / (SQPI * x) - 2 / (SQPI * x)) / x


def S_g(t):  # E(x) / x^3, E = erf(x) - 2x e^{-x^2}/sqrt(pi)  (double-layer potential kernel)
    if t == 0:
        return mp.mpf(4) / (3 * SQPI)
    x = mp.sqrt(t)
    return (mp.erf(x) - 2 * x * mp.exp(-t) / SQPI) / (x * t)


def cheb_interp_monomial(f, a, b, n):
    """Monomial coefficients (in the variable v = (2y - a - b)/(b - a) if
    `centered`, else in y itself) of the degree-n Chebyshev interpolant."""
    k = range(n + 1)
    nodes = [mp.cos(mp.pi * (j + mp.mpf(1) / 2) / (n + 1)) for j in k]
    vals = [f((b - a) / 2 * u + (a + b) / 2) for u in nodes]
    c = [2 * mp.fsum(vals[j] * mp.cos(mp.pi * i * (j + mp.mpf(1) / 2) / (n + 1)) for j in k) / (n + 1) for i in k]
    c[0] /= 2
    # Chebyshev -> monomial in u
    T = [[mp.mpf(1)], [mp.mpf(0), mp.mpf(1)]]
    for i in range(2, n + 1):
        nxt = [mp.mpf(0)] * (i + 1)
        for j, v in enumerate(T[i - 1]):
            nxt[j + 1] += 2 * v
        for j, v in enumerate(T[i - 2]):
            nxt[j] -= v
        T.append(nxt)
    mono_u = [mp.mpf(0)] * (n + 1)
    for i in k:
        for j, v in enumerate(T[i]):
            mono_u[j] += c[i] * v
    return mono_u


def u_to_y(mono_u, a, b):
    """monomial in u = (2y - a - b)/(b - a) -> monomial in y."""
    n = len(mono_u) - 1
    s, o = 2 / (b - a), -(a + b) / (b - a)     # u = s y + o
    out = [mp.mpf(0)] * (n + 1)
    for i, ci in enumerate(mono_u):            # ci (s y + o)^i
        for j in range(i + 1):
            out[j] += ci * mp.binomial(i, j) * s ** j * o ** (i - j)
    return out


def horner_double(coefs, y):
    """Double-precision Horner with exact fma (as the device does)."""
    acc = mp.mpf(float(coefs[-1]))
    for c in reversed(coefs[:-1]):
        acc = mp.mpf(float(acc * y + mp.mpf(float(c))))   # fma: one rounding
    return acc


def hexd(v):
    return float(v).hex()


def main():
    out = ["// Generated by tools/gen_special.py -- do not edit.  (mpmath, %d digits)" % mp.mp.dps,
           "#pragma once", "", "namespace hb {", "namespace special {", ""]
    T0 = X0 * X0
    out.append(f"constexpr double kX0 = {hexd(X0)};   // small-x / large-x switch")
    out.append(f"constexpr double kInvSqrtPi = {hexd(1 / SQPI)};")
    out.append(f"constexpr double kTwoInvSqrtPi = {hexd(2 / SQPI)};")
    report = []
    for name, f in (("Pe", S_e), ("Pf", S_f), ("Ph", S_h), ("Pg", S_g)):
        mono_t = u_to_y(cheb_interp_monomial(f, mp.mpf(0), T0, DEG_S[name]), mp.mpf(0), T0)
        worst = 0
        for i in range(2001):
            t = T0 * i / 2000
            worst = max(worst, abs(horner_double(mono_t, t) - f(t)) / abs(f(t)))
        report.append(f"{name}: degree {DEG_S[name]} on t in [0, {float(T0)}], max rel err (double Horner) {float(worst):.2e}")
        out.append(f"// {report[-1]}")
        out.append(f"static __device__ __constant__ double k{name}[{DEG_S[name] + 1}] = {{" + ", ".join(hexd(c) for c in mono_t) + "};")
    out.append("")
    # ---- middle region: the function values themselves, piecewise on [X0, XL) ----
    # (all four are analytic there; no exp needed).  Beyond XL every kind equals
    # its asymptote to within half an ulp: e^{-x^2}(...) < 2^-53 relative.
    XL = X0 + MID_W * MID_PIECES
    out.append(f"constexpr double kXL = {hexd(XL)};   // middle / asymptotic switch")
    out.append(f"constexpr int kMidPieces = {MID_PIECES};")
    names = ("H", "F", "erf", "E", "xH", "Fx", "ex", "Ex3")
    out.append("// degree of the middle-region pieces per kind (0 H, 1 F, 2 erf, 3 E, 4 xH, 5 F/x, 6 erf/x, 7 E/x^3)")
    out.append("constexpr int kMidDegK[8] = {" + ", ".join(str(DEG_M[n]) for n in names) + "};")
    out.append(f"constexpr int kMidDegMax = {max(DEG_M.values())};")
    out.append(f"constexpr double kMidInvW = {hexd(1 / MID_W)};")
    out.append(f"constexpr double kMidInvHalf = {hexd(2 / MID_W)};")
    for kind, (fname, f) in enumerate((("H", F_H), ("F", F_F), ("erf", mp.erf), ("E", F_E), ("xH", F_xH),
                                       ("Fx", F_Fx), ("ex", F_ex), ("Ex3", F_Ex3))):
        worst, tab = 0, []
        for pc in range(MID_PIECES):
            a = X0 + MID_W * pc
            b = a + MID_W
            mono_u = cheb_interp_monomial(f, a, b, DEG_M[fname])
            mid = (a + b) / 2
            for j in range(401):
                x = mp.mpf(float(a + (b - a) * j / 400))
                u = mp.mpf(float(mp.mpf(float(x - mid)) * (2 / MID_W)))
                worst = max(worst, abs(horner_double(mono_u, u) - f(x)) / abs(f(x)))
            tab.append(mono_u)
        asym = {"H": lambda x: 1 + 1 / (2 * x * x), "F": lambda x: 1 - 1 / (2 * x * x),
                "erf": lambda x: mp.mpf(1), "E": lambda x: mp.mpf(1),
                "xH": lambda x: (x + 1 / (2 * x) - 2 / SQPI) / (x * x), "Fx": lambda x: 1 / x - 1 / (2 * x * x * x),
                "ex": lambda x: 1 / x, "Ex3": lambda x: 1 / (x * x * x)}[fname]
        tail = max(abs(asym(XL + k / mp.mpf(8)) - f(XL + k / mp.mpf(8))) / abs(f(XL + k / mp.mpf(8))) for k in range(40))
        report.append(f"mid {fname}: {MID_PIECES} pieces x degree {DEG_M[fname]} on [{float(X0)}, {float(XL)}), "
                      f"max rel err (double Horner) {float(worst):.2e}; asymptote rel err for x >= XL {float(tail):.1e}")
        out.append(f"// {report[-1]}")
        out.append(f"static __device__ __constant__ double kMid{kind}[(kMidDegK[{kind}] + 1) * kMidPieces] = {{")
        for k in range(DEG_M[fname] + 1):
            out.append("    " + ", ".join(hexd(tab[pc][k]) for pc in range(MID_PIECES)) + ",")
        out.append("};")
    # ---- uniform pieces for the factor-free kinds (pair kernels: 4 xH, 5 F/x, 6 erf/x; potentials: 6, 7 E/x^3) ----
    # [0, XL) in pieces of width 1/16, degree 7 in u = 2 (16 x - p) - 1: ONE
    # polynomial form for every lane below XL that is not in an all-series
    # warp (no series / middle select), 4 LDS.128 + 7 FMA per value
    U_INV_H, U_DEG = int(os.environ.get("HB_U_INV_H", "16")), int(os.environ.get("HB_U_DEG", "7"))
    U_PIECES = int(XL * U_INV_H)
    out.append("")
    out.append(f"constexpr int kUPieces = {U_PIECES};   // uniform pieces of [0, XL), width 1/{U_INV_H}")
    out.append(f"constexpr int kUDeg = {U_DEG};")
    out.append(f"constexpr double kUInvH = {hexd(mp.mpf(U_INV_H))};")
    for kind, (fname, f) in ((4, ("xH", F_xH)), (5, ("Fx", F_Fx)), (6, ("ex", F_ex)), (7, ("Ex3", F_Ex3))):
        worst, tab = 0, []
        for pc in range(U_PIECES):
            a = mp.mpf(pc) / U_INV_H
            b = a + mp.mpf(1) / U_INV_H
            mono_u = cheb_interp_monomial(f, a, b, U_DEG)
            for j in range(25):
                x = mp.mpf(float(a + (b - a) * (j + mp.mpf(1) / 2) / 25))
                y = mp.mpf(float(x * U_INV_H))
                u = mp.mpf(float(2 * (y - int(mp.floor(y))) - 1))
                worst = max(worst, abs(horner_double(mono_u, u) - f(x)) / abs(f(x)))
            tab.append(mono_u)
        report.append(f"uniform {fname}: {U_PIECES} pieces x degree {U_DEG} on [0, {float(XL)}), "
                      f"max rel err (double Horner) {float(worst):.2e}")
        out.append(f"// {report[-1]}")
        out.append(f"static __device__ __constant__ double kU{kind}[(kUDeg + 1) * kUPieces] = {{")
        for k in range(U_DEG + 1):
            out.append("    " + ", ".join(hexd(tab[pc][k]) for pc in range(U_PIECES)) + ",")
        out.append("};")
    out += ["", "}  // namespace special", "}  // namespace hb", ""]
    path = os.environ.get("HB_SPECIAL_OUT") or os.path.join(
        os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2102_09811_b200", "csrc",
        "hb_special_coeffs.h")
    open(path, "w").write("\n".join(out))
    print("\n".join(report))
    print("wrote", path)


if __name__ == "__main__":
    sys.exit(main())
