// hb_special.cuh -- fused evaluation of the heat-kernel antiderivatives.
//
// With x = rho / (2 sqrt(alpha delta)) every kernel value the assembly needs
// is a rho-dependent factor times ONE function of x (4 pi scaling):
//   V : G^{dtau dt} 4pi = rho/(2 a^2) * H(x),
//       H(x) = erf(x) (1 + 1/(2x^2)) + e^{-x^2} / (sqrt(pi) x)
//   K : a dG^{dtau dt}/dn_y 4pi = -(r.n_y/rho) / (2a) * F(x),
//       F(x) = erf(x) (1 - 1/(2x^2)) + e^{-x^2} / (sqrt(pi) x)
//   D2: a G^{dtau} 4pi = erf(x) / rho
// (obtained from heatbem/_assembly_numba.py:25-76 with delta = rho^2/(4 a x^2)).
// The reference's form of K, (1/(2a) - delta/rho^2) erf + sqrt(delta/(pi a))
// e^{-x^2}/rho, cancels like 1/x^2 for small x; F(x) = x Pf(x^2) does not.
//
//   x <  X0: H = 2/(sqrt(pi) x) + x Ph(t), F = x Pf(t), erf = x Pe(t), t = x^2
//   x >= X0: erf = 1 - E Q(x), E = e^{-x^2}, Q = erfcx (4 polynomial pieces in
//            shared memory), H/F = a + E (1/(sqrt(pi) x) - Q a), a = 1 +- 1/(2x^2)
// Coefficients: csrc/hb_special_coeffs.h (tools/gen_special.py, mpmath).
// Lanes whose x lies on the other side of X0 follow the same instruction
// stream (predicated); a branch is skipped when no active lane needs it.
#pragma once

#include "hb_common.cuh"
#include "hb_special_coeffs.h"

namespace hb {
namespace special {

// shared-memory table: erfcx coefficients, then piece mids and 1/half-widths
constexpr int kTabDoubles = (kQDeg + 1) * kQPieces + 2 * kQPieces;

__device__ __forceinline__ void load_table(double *tab)
{
    for (int i = threadIdx.x; i < (kQDeg + 1) * kQPieces; i += blockDim.x) tab[i] = kQCoef[i];
    for (int i = threadIdx.x; i < kQPieces; i += blockDim.x) {
        tab[(kQDeg + 1) * kQPieces + i] = kQMid[i];
        tab[(kQDeg + 1) * kQPieces + kQPieces + i] = kQInvHalf[i];
    }
}

template <int N>
__device__ __forceinline__ double horner(const double (&c)[N], double t)   // c: __constant__
{
    double p = c[N - 1];
#pragma unroll
    for (int k = N - 2; k >= 0; --k) p = fma(p, t, c[k]);
    return p;
}

// KIND 0: H (single layer), 1: F (double layer), 2: erf (hypersingular D2),
// 3: E(x) = erf(x) - 2x e^{-x^2}/sqrt(pi) (double-layer potential, = x^3 Pg(t)).
// ix = 1/x (formed by the caller from precomputed 1/rho and 1/c); `mask` =
// the lanes executing this call.
template <int KIND>
__device__ __forceinline__ double eval(double x, double ix, const double *__restrict__ tab, unsigned mask)
{
    const double t = __dmul_rn(x, x);
    const bool small = x < kX0;
    double r = 0.0;
    if (__any_sync(mask, small)) {
        if (KIND == 0) r = fma(x, horner(kPh, t), __dmul_rn(kTwoInvSqrtPi, ix));
        else if (KIND == 1) r = __dmul_rn(x, horner(kPf, t));
        else if (KIND == 2) r = __dmul_rn(x, horner(kPe, t));
        else r = __dmul_rn(__dmul_rn(x, t), horner(kPg, t));
    }
    if (__any_sync(mask, !small)) {
        const double E = exp(-t);
        const int pc = (x >= kQBreak1) + (x >= kQBreak2) + (x >= kQBreak3);
        const double xc = fmin(x, kQBreak4);
        const double *mid = tab + (kQDeg + 1) * kQPieces;
        const double u = __dmul_rn(xc - mid[pc], mid[kQPieces + pc]);
        double q = tab[kQDeg * kQPieces + pc];
#pragma unroll
        for (int k = kQDeg - 1; k >= 0; --k) q = fma(q, u, tab[k * kQPieces + pc]);
        double lv;
        if (KIND == 2) {
            lv = fma(-E, q, 1.0);
        } else if (KIND == 3) {
            lv = fma(-E, fma(kTwoInvSqrtPi, x, q), 1.0);
        } else {
            const double hx = __dmul_rn(0.5 * ix, ix);
            const double a = KIND == 0 ? 1.0 + hx : 1.0 - hx;
            lv = fma(E, fma(-q, a, __dmul_rn(kInvSqrtPi, ix)), a);
        }
        if (!small) r = lv;
    }
    return r;
}

// All NJ gap slots of one quadrature point at once: one small-x and one
// large-x region for the whole group, so the NJ independent Horner chains
// interleave (ILP NJ) instead of being serialised by per-slot branches.
template <int KIND, int NJ>
__device__ __forceinline__ void eval_n(const double (&x)[NJ], const double (&ix)[NJ], double (&r)[NJ],
                                       const double *__restrict__ tab, unsigned mask)
{
    double t[NJ];
    bool small[NJ], any_s = false, any_l = false;
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
        t[j] = __dmul_rn(x[j], x[j]);
        small[j] = x[j] < kX0;
        any_s |= small[j];
        any_l |= !small[j];
        r[j] = 0.0;
    }
    if (__any_sync(mask, any_s)) {
#pragma unroll
        for (int j = 0; j < NJ; ++j) {
            if (KIND == 0) r[j] = fma(x[j], horner(kPh, t[j]), __dmul_rn(kTwoInvSqrtPi, ix[j]));
            else if (KIND == 1) r[j] = __dmul_rn(x[j], horner(kPf, t[j]));
            else r[j] = __dmul_rn(x[j], horner(kPe, t[j]));
        }
    }
    if (__any_sync(mask, any_l)) {
        const double *mid = tab + (kQDeg + 1) * kQPieces;
        double E[NJ], u[NJ], q[NJ];
        int pc[NJ];
#pragma unroll
        for (int j = 0; j < NJ; ++j) {
            E[j] = exp(-t[j]);
            pc[j] = (x[j] >= kQBreak1) + (x[j] >= kQBreak2) + (x[j] >= kQBreak3);
            u[j] = __dmul_rn(fmin(x[j], kQBreak4) - mid[pc[j]], mid[kQPieces + pc[j]]);
            q[j] = tab[kQDeg * kQPieces + pc[j]];
        }
#pragma unroll
        for (int k = kQDeg - 1; k >= 0; --k)
#pragma unroll
            for (int j = 0; j < NJ; ++j) q[j] = fma(q[j], u[j], tab[k * kQPieces + pc[j]]);
#pragma unroll
        for (int j = 0; j < NJ; ++j) {
            double lv;
            if (KIND == 2) {
                lv = fma(-E[j], q[j], 1.0);
            } else {
                const double hx = __dmul_rn(0.5 * ix[j], ix[j]);
                const double a = KIND == 0 ? 1.0 + hx : 1.0 - hx;
                lv = fma(E[j], fma(-q[j], a, __dmul_rn(kInvSqrtPi, ix[j])), a);
            }
            if (!small[j]) r[j] = lv;
        }
    }
}

}  // namespace special
}  // namespace hb
