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
//   x <  X0 (= 1):  H = 2/(sqrt(pi) x) + x Ph(t), F = x Pf(t), erf = x Pe(t),
//                   E = x^3 Pg(t), t = x^2 (coefficients uniform across the warp;
//                   degrees 10 / 10 / 11 / 11)
//   X0 <= x < XL:   the function value itself (for the factor-free form x H:
//                   M = (x H - 2/sqrt(pi)) / x^2) as a polynomial in
//                   u = (x - mid_p) / half on 21 uniform pieces of width 1/4
//                   (degree 12 for H, 10 for F and erf, 11 for E: per kind the
//                   lowest degree that keeps the double Horner within 2.3e-16)
//                   (coefficients of the lane's piece from shared memory) --
//                   all four functions are analytic there, no exp is needed
//   x >= XL (6.25): the asymptote, erf = E = 1, H/F = 1 +- 1/(2x^2), which
//                   the exact value rounds to (e^{-x^2}(...) < 2^-53 relative)
// Coefficients: csrc/hb_special_coeffs.h (tools/gen_special.py, mpmath, with
// the max relative error of each piece in double Horner).  A lane's region
// depends on its own x only, so values do not depend on which lanes share a
// warp (slot / window / rank invariance); a region is skipped when no lane of
// the warp needs it.
#pragma once

#include "hb_common.cuh"
#include "hb_special_coeffs.h"

namespace hb {
namespace special {

#ifdef HB_COUNT_BRANCHES
__device__ unsigned long long g_branch_count[4];   // [small?1:0 + large?2:0]
#endif

// shared-memory table of one function: coefficient k of middle-region piece
// p at tab[k * kTabStride + p] (lanes in different pieces read neighbouring
// words), and in column kMidPieces the small-x series coefficient k -- so a
// warp whose lanes straddle x = X0 runs ONE Horner chain, each lane with its
// own variable (t or u) and column.  Rows above a polynomial's degree are
// zero: leading fma(0, v, 0) / fma(0, v, c) steps are exact, so a lane's value
// is bitwise the same as from its own region's chain alone (and so still
// depends on its own x only).
constexpr int kTabStride = kMidPieces + 1;

template <int KIND>
__host__ __device__ constexpr int mid_deg() { return kMidDegK[KIND]; }

// series polynomial of each kind: H and x H use Ph, F and F/x use Pf, erf and
// erf/x use Pe, E uses Pg
template <int KIND>
__host__ __device__ constexpr int series_deg()
{
    return (KIND == 0 || KIND == 4 ? (int)(sizeof(kPh) / sizeof(double))
            : KIND == 1 || KIND == 5 ? (int)(sizeof(kPf) / sizeof(double))
            : KIND == 2 || KIND == 6 ? (int)(sizeof(kPe) / sizeof(double)) : (int)(sizeof(kPg) / sizeof(double))) - 1;
    // (kinds 3 E and 7 E/x^3 share Pg: E = x^3 Pg(t))
}

template <int KIND>
__host__ __device__ constexpr int merged_deg() { return mid_deg<KIND>() > series_deg<KIND>() ? mid_deg<KIND>() : series_deg<KIND>(); }

__host__ __device__ constexpr int cmax(int a, int b) { return a > b ? a : b; }
constexpr int kMergedDegMax = cmax(cmax(cmax(merged_deg<0>(), merged_deg<1>()), cmax(merged_deg<2>(), merged_deg<3>())),
                                   cmax(cmax(merged_deg<4>(), merged_deg<5>()), cmax(merged_deg<6>(), merged_deg<7>())));
constexpr int kTabDoubles = ((kMergedDegMax + 2) & ~1) * kTabStride;   // room for any kind / layout

// the kinds 2-6 (pair kernels, potentials) store coefficients 2m and 2m+1 of a
// column next to each other, at tab[2 (m kTabStride + p) + (k & 1)]: one
// LDS.128 feeds two Horner steps (16-byte slots, distinct pieces in
// consecutive slots)
template <int KIND>
__host__ __device__ constexpr bool packed() { return KIND >= 2; }   // all but the unused H / F forms

template <int KIND>
__device__ __forceinline__ void load_table(double *tab)
{
    const double *mid = KIND == 0 ? kMid0 : KIND == 1 ? kMid1 : KIND == 2 ? kMid2 : KIND == 3 ? kMid3
                      : KIND == 4 ? kMid4 : KIND == 5 ? kMid5 : KIND == 6 ? kMid6 : kMid7;
    const double *ser = (KIND == 0 || KIND == 4) ? kPh : (KIND == 1 || KIND == 5) ? kPf
                      : (KIND == 2 || KIND == 6) ? kPe : kPg;
    constexpr int DM = mid_deg<KIND>(), DS = series_deg<KIND>(), D = merged_deg<KIND>();
    constexpr int ROWS = packed<KIND>() ? ((D + 2) & ~1) : D + 1;
    for (int i = threadIdx.x; i < ROWS * kTabStride; i += blockDim.x) {
        int k, p;
        if (packed<KIND>()) {
            const int slot = i >> 1, m = slot / kTabStride;
            p = slot - m * kTabStride;
            k = 2 * m + (i & 1);
        } else {
            k = i / kTabStride;
            p = i - k * kTabStride;
        }
        double v;
        if (p < kMidPieces) v = k <= DM ? mid[k * kMidPieces + p] : 0.0;
        else v = k <= DS ? ser[k] : 0.0;
        tab[i] = v;
    }
}

// Horner chains q_j = sum_k c_j[k] v_j^k, k = DEG..0, column pointers c_j
// (element offset of the column in tab); fma order identical in both layouts
template <int KIND, int DEG, int NJ>
__device__ __forceinline__ void table_chains(const double *__restrict__ tab, const int (&col)[NJ],
                                             const double (&v)[NJ], double (&q)[NJ])
{
    if constexpr (packed<KIND>()) {
        const double2 *t2 = reinterpret_cast<const double2 *>(tab);
        constexpr int MT = DEG / 2;
        // coefficient pairs prefetched HB_TAB_PREFETCH steps ahead of the chain
        // (the loads do not depend on it): the LDS.128 latency hides behind the
        // previous steps' FMAs instead of stalling every step
#ifndef HB_TAB_PREFETCH
#define HB_TAB_PREFETCH 3
#endif
        constexpr int PF = HB_TAB_PREFETCH < 1 ? 1 : HB_TAB_PREFETCH;
        double2 w[MT + 1][NJ];
#pragma unroll
        for (int m = MT; m >= 0 && m > MT - PF - 1; --m)
#pragma unroll
            for (int j = 0; j < NJ; ++j) w[m][j] = t2[m * kTabStride + col[j]];
#pragma unroll
        for (int j = 0; j < NJ; ++j) q[j] = (DEG & 1) ? fma(w[MT][j].y, v[j], w[MT][j].x) : w[MT][j].x;
#pragma unroll
        for (int m = MT - 1; m >= 0; --m) {
            if (m - PF >= 0) {
#pragma unroll
                for (int j = 0; j < NJ; ++j) w[m - PF][j] = t2[(m - PF) * kTabStride + col[j]];
            }
#pragma unroll
            for (int j = 0; j < NJ; ++j) q[j] = fma(q[j], v[j], w[m][j].y);
#pragma unroll
            for (int j = 0; j < NJ; ++j) q[j] = fma(q[j], v[j], w[m][j].x);
        }
    } else {
#pragma unroll
        for (int j = 0; j < NJ; ++j) q[j] = tab[DEG * kTabStride + col[j]];
#pragma unroll
        for (int k = DEG - 1; k >= 0; --k)
#pragma unroll
            for (int j = 0; j < NJ; ++j) q[j] = fma(q[j], v[j], tab[k * kTabStride + col[j]]);
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

// small-x series (x < X0)
template <int KIND>
__device__ __forceinline__ double series(double x, double t, double ix)
{
    if (KIND == 0) return fma(x, horner(kPh, t), __dmul_rn(kTwoInvSqrtPi, ix));
    if (KIND == 1) return __dmul_rn(x, horner(kPf, t));
    if (KIND == 2) return __dmul_rn(x, horner(kPe, t));
    if (KIND == 3) return __dmul_rn(__dmul_rn(x, t), horner(kPg, t));
    if (KIND == 4) return fma(t, horner(kPh, t), kTwoInvSqrtPi);   // x H = 2/sqrt(pi) + t Ph(t)
    if (KIND == 5) return horner(kPf, t);                          // F / x
    if (KIND == 7) return horner(kPg, t);                          // E / x^3
    return horner(kPe, t);                                         // erf / x
}

// asymptote (x >= XL)
template <int KIND>
__device__ __forceinline__ double asymptote(double x, double ix)
{
    if (KIND == 2 || KIND == 3) return 1.0;
    if (KIND == 6) return ix;                            // erf / x
    if (KIND == 7) return __dmul_rn(__dmul_rn(ix, ix), ix);   // E / x^3
    if (KIND == 4) return fma(0.5, ix, x);               // x H = x + 1/(2x)
    const double hx = __dmul_rn(0.5 * ix, ix);
    if (KIND == 5) return __dmul_rn(ix, 1.0 - hx);       // F / x = (1 - 1/(2x^2)) / x
    return KIND == 0 ? 1.0 + hx : 1.0 - hx;
}

// middle-region piece and local variable: y = (x - X0) / w, piece = floor(y),
// u = 2 (y - piece) - 1 -- every step exact within a piece (w = 1/4), so u
// equals (x - mid) / half exactly
__device__ __forceinline__ int mid_piece(double x, double &u)
{
    const double y = __dmul_rn(x - kX0, kMidInvW);
#ifdef HB_PIECE_FLOOR
    const double pf = fmin(fmax(floor(y), 0.0), (double)(kMidPieces - 1));
    u = fma(2.0, y - pf, -1.0);
    return __double2int_rz(pf);
#else
    // integer floor and clamp (one conversion each way instead of the FP64
    // floor / min / max sequence); identical for middle-region lanes
    // (0 <= y < kMidPieces), other lanes' values are discarded
    const int p = min(max(__double2int_rd(y), 0), kMidPieces - 1);
    u = fma(2.0, y - (double)p, -1.0);
    return p;
#endif
}

// small-x finish of a series polynomial value q = P(t) (as series<KIND>)
template <int KIND>
__device__ __forceinline__ double series_finish(double x, double t, double ix, double q)
{
    if (KIND == 0) return fma(x, q, __dmul_rn(kTwoInvSqrtPi, ix));
    if (KIND == 1 || KIND == 2) return __dmul_rn(x, q);
    if (KIND == 3) return __dmul_rn(__dmul_rn(x, t), q);
    if (KIND == 4) return fma(t, q, kTwoInvSqrtPi);
    return q;
}

// NJ evaluations of one lane at once: one region pass for the whole group,
// so the NJ independent Horner chains interleave (ILP NJ).
// ixf(j) supplies 1/x of evaluation j on demand (the KIND 0 series and the
// asymptotes only), so the common paths do not form it
template <int KIND, int NJ, class IXF>
__device__ __forceinline__ void eval_nf(const double (&x)[NJ], const IXF &ixf, double (&r)[NJ],
                                        const double *__restrict__ tab, unsigned mask)
{
    double t[NJ];
    bool small[NJ], any_ns = false;
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
        t[j] = __dmul_rn(x[j], x[j]);
#if defined(HB_FORCE_SMALL)   // timing experiments only: wrong values
        small[j] = true;
#elif defined(HB_FORCE_MID)
        small[j] = false;
#else
        small[j] = x[j] < kX0;
#endif
        any_ns |= !small[j];
    }
    // common case first: every lane of the warp in the series region -- one
    // compare and one vote, then the constant-bank series
    if (!__any_sync(mask, any_ns)) {
#ifdef HB_COUNT_BRANCHES
        if ((threadIdx.x & 31) == (__ffs(mask) - 1)) atomicAdd(&g_branch_count[1], 1ull);
#endif
#pragma unroll
        for (int j = 0; j < NJ; ++j) r[j] = series<KIND>(x[j], t[j], KIND == 0 ? ixf(j) : 0.0);
        return;
    }
    // region of the other lanes from the integer piece index (one FP64->int
    // conversion; integer compares instead of FP64 ones) and ONE warp
    // reduction of the region bits: 1 small, 2 middle, 4 asymptotic
    bool huge[NJ];
    int pcl[NJ], code = 0;
    double y[NJ];
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
        y[j] = __dmul_rn(x[j] - kX0, kMidInvW);
        const int pi = __double2int_rd(y[j]);   // < 0 for small lanes, >= kMidPieces for asymptotic ones
#if defined(HB_FORCE_MID)
        huge[j] = false;
#else
        huge[j] = !small[j] && pi >= kMidPieces;
#endif
        pcl[j] = min(max(pi, 0), kMidPieces - 1);
        code |= small[j] ? 1 : (huge[j] ? 4 : 2);
    }
    code = __reduce_or_sync(mask, code);
#ifdef HB_COUNT_BRANCHES   // diagnostics: warp-level region mix of the other eval_n calls
    if ((threadIdx.x & 31) == (__ffs(mask) - 1))
        atomicAdd(&g_branch_count[((code & 1) ? 1 : 0) + ((code & 2) ? 2 : 0)], 1ull);
#endif
    // one polynomial pass per warp: ONE table chain in which small lanes use
    // the series column with t and middle lanes their piece with u (merged
    // degree when both occur).  Every chain is computed for all lanes
    // unconditionally (the NJ chains interleave) and lanes keep their own
    // region's value.
    if (code & 2) {
        const bool vote_s = code & 1;
        double v[NJ], q[NJ];
        int col[NJ];
#pragma unroll
        for (int j = 0; j < NJ; ++j) {
            // u = 2 (y - piece) - 1, exact within the piece (as mid_piece)
            const double u = fma(2.0, y[j] - (double)pcl[j], -1.0);
            col[j] = small[j] ? kMidPieces : pcl[j];
            v[j] = small[j] ? t[j] : u;
        }
        if (vote_s) table_chains<KIND, merged_deg<KIND>(), NJ>(tab, col, v, q);
        else table_chains<KIND, mid_deg<KIND>(), NJ>(tab, col, v, q);
#pragma unroll
        for (int j = 0; j < NJ; ++j) {
            asm volatile("" : "+d"(q[j]));
            // huge lanes take this value too and are overwritten by the
            // asymptote below; the factor-free kinds 4-6 finish series and
            // table values alike (x H = 2/sqrt(pi) + t M with M from either,
            // F/x and erf/x are q itself), so they need no select
            const double fs = series_finish<KIND>(x[j], t[j], KIND == 0 ? ixf(j) : 0.0, q[j]);
            r[j] = (KIND >= 4 || small[j]) ? fs : q[j];
        }
    } else {
        // small and huge lanes only: the series for all (huge lanes overwritten)
#pragma unroll
        for (int j = 0; j < NJ; ++j) r[j] = series<KIND>(x[j], t[j], KIND == 0 ? ixf(j) : 0.0);
    }
    if (code & 4) {
#pragma unroll
        for (int j = 0; j < NJ; ++j)
            if (huge[j]) r[j] = asymptote<KIND>(x[j], ixf(j));
    }
}

// ---------------------------------------------------------------------------
// Uniform pieces (the direct pair kernels, kinds 4-6).  A warp whose
// evaluations all lie in the series region (x < X0) takes the constant-bank
// series; any other warp evaluates EVERY lane on the uniform pieces of
// [0, XL) -- piece p = floor(16 x) of width 1/16, degree 7 in
// u = 2 (16 x - p) - 1 (exact) -- with no series / middle select, merged
// chain or region reduction; lanes at or above XL take the asymptote.  A
// lane's form thus depends on the other lanes' x through the all-series vote:
// the direct kernels fix which evaluations share a warp by evaluating whole
// global gap windows (hb_pairs_direct.cu direct_pairs), so blocks stay
// independent of the d-range / row chunk / rank of a call.
// Table: coefficients 2m, 2m+1 of piece p side by side at double2 index
// m kUPieces + p (one LDS.128 per two Horner steps).
// ---------------------------------------------------------------------------
constexpr int kUTabDoubles = (kUDeg + 1) * kUPieces;
static_assert((kUDeg & 1) == 1 && kUTabDoubles % 2 == 0, "uniform pieces: coefficient pairs");

template <int KIND>
__device__ __forceinline__ void load_utable(double *utab)
{
    static_assert(KIND >= 4 && KIND <= 7, "uniform pieces exist for the factor-free kinds 4-7");
    const double *src = KIND == 4 ? kU4 : KIND == 5 ? kU5 : KIND == 6 ? kU6 : kU7;
    for (int i = threadIdx.x; i < kUTabDoubles; i += blockDim.x) {
        const int slot = i >> 1, m = slot / kUPieces, p = slot - m * kUPieces;
        utab[i] = src[(2 * m + (i & 1)) * kUPieces + p];
    }
}

template <int KIND, int NJ, class IXF>
__device__ __forceinline__ void eval_unf(const double (&x)[NJ], const IXF &ixf, double (&r)[NJ],
                                         const double *__restrict__ utab, unsigned mask)
{
    double t[NJ];
    bool any_ns = false;
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
        t[j] = __dmul_rn(x[j], x[j]);
        any_ns |= !(x[j] < kX0);
    }
    if (!__any_sync(mask, any_ns)) {   // every evaluation of the warp in the series region
#pragma unroll
        for (int j = 0; j < NJ; ++j) r[j] = series<KIND>(x[j], t[j], 0.0);
        return;
    }
    const double2 *t2 = reinterpret_cast<const double2 *>(utab);
    constexpr int MT = kUDeg / 2;
    int p[NJ];
    double u[NJ];
    bool huge[NJ], any_h = false;
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
        const double y = __dmul_rn(x[j], kUInvH);   // exact (power of two)
        const int pi = __double2int_rz(y);          // x >= 0: the floor; INT_MAX for inf
        huge[j] = pi >= kUPieces;
        any_h |= huge[j];
        p[j] = min(pi, kUPieces - 1);
        u[j] = fma(2.0, y - (double)p[j], -1.0);    // exact within the piece
    }
    double2 w[MT + 1][NJ];
#pragma unroll
    for (int m = MT; m >= 0; --m)
#pragma unroll
        for (int j = 0; j < NJ; ++j) w[m][j] = t2[m * kUPieces + p[j]];
    double q[NJ];
#pragma unroll
    for (int j = 0; j < NJ; ++j) q[j] = fma(w[MT][j].y, u[j], w[MT][j].x);
#pragma unroll
    for (int m = MT - 1; m >= 0; --m) {
#pragma unroll
        for (int j = 0; j < NJ; ++j) q[j] = fma(q[j], u[j], w[m][j].y);
#pragma unroll
        for (int j = 0; j < NJ; ++j) q[j] = fma(q[j], u[j], w[m][j].x);
    }
#pragma unroll
    for (int j = 0; j < NJ; ++j)   // kinds 4-6 finish like the series (x H = 2/sqrt(pi) + x^2 M)
        r[j] = KIND == 4 ? fma(t[j], q[j], kTwoInvSqrtPi) : q[j];
    if (__any_sync(mask, any_h)) {
#pragma unroll
        for (int j = 0; j < NJ; ++j)
            if (huge[j]) r[j] = asymptote<KIND>(x[j], ixf(j));
    }
}

// Lane-local form of the uniform pieces: every value below XL from its piece,
// whatever the other lanes hold (no votes at all), the asymptote above.  For
// callers whose x is never small -- the per-point gaps of the moment form
// (t = x^2 > kTM) -- where the all-series shortcut of eval_unf cannot fire;
// a value depends on its own x only, so it is independent of the warp's
// composition (d-range, row chunk, rank) by construction.
template <int KIND, int NJ, class IXF>
__device__ __forceinline__ void eval_ulocal(const double (&x)[NJ], const IXF &ixf, double (&r)[NJ],
                                            const double *__restrict__ utab)
{
    const double2 *t2 = reinterpret_cast<const double2 *>(utab);
    constexpr int MT = kUDeg / 2;
    int p[NJ];
    double u[NJ];
    bool huge[NJ];
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
        const double y = __dmul_rn(x[j], kUInvH);   // exact (power of two)
        const int pi = __double2int_rz(y);          // x >= 0: the floor; INT_MAX for inf
        huge[j] = pi >= kUPieces;
        p[j] = min(pi, kUPieces - 1);
        u[j] = fma(2.0, y - (double)p[j], -1.0);    // exact within the piece
    }
    double2 w[MT + 1][NJ];
#pragma unroll
    for (int m = MT; m >= 0; --m)
#pragma unroll
        for (int j = 0; j < NJ; ++j) w[m][j] = t2[m * kUPieces + p[j]];
    double q[NJ];
#pragma unroll
    for (int j = 0; j < NJ; ++j) q[j] = fma(w[MT][j].y, u[j], w[MT][j].x);
#pragma unroll
    for (int m = MT - 1; m >= 0; --m) {
#pragma unroll
        for (int j = 0; j < NJ; ++j) q[j] = fma(q[j], u[j], w[m][j].y);
#pragma unroll
        for (int j = 0; j < NJ; ++j) q[j] = fma(q[j], u[j], w[m][j].x);
    }
    bool any_h = false;
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
        r[j] = KIND == 4 ? fma(__dmul_rn(x[j], x[j]), q[j], kTwoInvSqrtPi) : q[j];
        any_h |= huge[j];
    }
    // (the vote only skips code: the asymptote replaces a lane's own value whoever else is active)
    if (__any_sync(__activemask(), any_h)) {
#pragma unroll
        for (int j = 0; j < NJ; ++j)
            if (huge[j]) r[j] = asymptote<KIND>(x[j], ixf(j));
    }
}

template <int KIND>
__device__ __forceinline__ double eval_u(double x, double ix, const double *__restrict__ utab, unsigned mask)
{
    double r[1];
    const double xs[1] = {x};
    eval_unf<KIND, 1>(xs, [&](int) { return ix; }, r, utab, mask);
    return r[0];
}

template <int KIND, int NJ>
__device__ __forceinline__ void eval_n(const double (&x)[NJ], const double (&ix)[NJ], double (&r)[NJ],
                                       const double *__restrict__ tab, unsigned mask)
{
    eval_nf<KIND, NJ>(x, [&](int j) { return ix[j]; }, r, tab, mask);
}

// KIND 0: H (single layer), 1: F (double layer), 2: erf (hypersingular D2),
// 3: E(x) = erf(x) - 2x e^{-x^2}/sqrt(pi) (double-layer potential); the
// assembly kernels use the factor-free forms 4: x H, 5: F/x, 6: erf/x (the
// per-point factor rho^{+-1} of V / K / D2 becomes a per-gap constant).
// ix = 1/x (formed by the caller from precomputed 1/rho and 1/c; used by the
// KIND 0 series and the asymptotes only); `mask` = the lanes executing this call.
template <int KIND>
__device__ __forceinline__ double eval(double x, double ix, const double *__restrict__ tab, unsigned mask)
{
    double r[1];
    const double xs[1] = {x}, is[1] = {ix};
    eval_n<KIND, 1>(xs, is, r, tab, mask);
    return r[0];
}

}  // namespace special
}  // namespace hb
