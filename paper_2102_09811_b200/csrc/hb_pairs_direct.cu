// hb_pairs_direct.cu -- the direct (all gaps point by point) pair kernel.
//
// Used by hb_assemble (csrc/hb_assembly.cu) for the double-layer and
// hypersingular operators when a call holds few blocks (E_t <= 63): every
// time gap of a 32-gap window is evaluated at every quadrature point, one
// warp per element pair, lanes over gaps -- the single-pass form that beats
// the moment form there because most of its per-point evaluations take the
// cheap series branch.  Larger calls and the single-layer operator use the
// moment form (hb_assembly.cu).  Same staging layout Q[pair][ij][nd] per
// window; the finalize kernels of hb_assembly.cu turn it into blocks.
//
// Replaces heatbem/_assembly_numba.py:111-272 (_toeplitz_pass) for one
// 32-gap window of the _assemble_operator loop (heatbem/assembly.py:215-236),
// with the 3-term AssemblyPlan combination (assembly.py:72-89) fused.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "hb_common.cuh"
#include "hb_special.cuh"

#ifndef HB_PAIR_MINB
#define HB_PAIR_MINB 2
#endif
#ifndef HB_PAIR_WARPS   // warps per CTA of the pair kernels
#define HB_PAIR_WARPS 8
#endif
#ifndef HB_SEP
#define HB_SEP 0     // separable p1 x p1 accumulation (slower at 128 registers; kept for study)
#endif
#ifndef HB_P1P1_GROUPED   // p1 x p1 through the G-point grouped loop (1, default: D2 pair kernel -4 %
#define HB_P1P1_GROUPED 1  // with the per-kind degrees); 0 = one point per iteration
#endif
#ifndef HB_P1P1_MINB
#define HB_P1P1_MINB HB_PAIR_MINB
#endif
#ifndef HB_FUSED
#define HB_FUSED 1   // fused special-function evaluation (hb_special.cuh); 0 = CUDA erf/exp path
#endif

namespace hb {
namespace direct {

struct PairArgs {
    hb_mesh_desc m;
    double step, alpha, d_eps, r_eps;
    double inv2a, inv2a2, inva, kconst;
    int64_t e0, e1;
    int d0, d1, it_lo, it_hi, need_special, nd;
    int halve_diag;
    double *Q;
    unsigned long long *counter;   // work-item counter (zeroed per launch)
    int seg_len;                   // trial elements per separated-pair work item (32, or fewer for few rows)
};

template <int OP, int NIJ>
struct Layout {
    // payload per quadrature point: [rho, s1, s2, W[NIJ]] (OP 0/1) or [rho, s1, W] (OP 2);
    // W = the weight of the factor-free kernel value (hb_special.cuh kinds 4-6):
    // w ht hs for V and D2, w ht hs (-r.n_y)/(2a) for K
    static constexpr int HOFF = (OP == 2) ? 2 : 3;
    static constexpr int PAY_RAW = HOFF + NIJ;
    static constexpr int PAY = (PAY_RAW + 1) & ~1;
};

template <int NIJ, int NJ>
struct LsLayout {
    static constexpr int SLOTS = 16 * NJ;
    static constexpr int SIZE = NIJ * SLOTS + 2 * NIJ;   // + L0 and Lcomb0
};

template <int OP, int NIJ, int NJ>
__host__ __device__ constexpr int smem_doubles_per_warp() { return 32 * Layout<OP, NIJ>::PAY + LsLayout<NIJ, NJ>::SIZE; }

// one point's payload (N doubles, 16-byte aligned) as N/2 LDS.128; loads of
// fields the caller does not use are dead and removed
template <int N>
__device__ __forceinline__ void load_payload(const double *p, double (&v)[N])
{
    static_assert(N % 2 == 0, "payloads are padded to an even number of doubles");
    const double2 *p2 = reinterpret_cast<const double2 *>(p);
#pragma unroll
    for (int i = 0; i < N / 2; ++i) {
        const double2 d = p2[i];
        v[2 * i] = d.x;
        v[2 * i + 1] = d.y;
    }
}

// ---------------------------------------------------------------------------
// per-lane time-gap constants
// ---------------------------------------------------------------------------
template <int OP, int NJ>
struct Slots {
    double dl[NJ], cx[NJ], ic[NJ], kk[NJ], sc[NJ];   // sc: per-gap factor of the factor-free kinds
    __device__ void init(const PairArgs &A, int t)
    {
#pragma unroll
        for (int j = 0; j < NJ; ++j) {
            int it = A.it_lo + t + 16 * j;
            if (it > A.it_hi) it = A.it_hi;   // clamped slots compute finite values, never stored
            const double delta = (double)it * A.step;
            dl[j] = delta;
            ic[j] = 2.0 * sqrt(A.alpha * delta);     // 1 / cx: x = rho cx, 1/x = (1/rho) ic
            cx[j] = 1.0 / ic[j];
            if (OP == 2) kk[j] = 1.0 / sqrt(kPi * A.alpha * delta);
            else kk[j] = sqrt(delta) * A.kconst;
            // V = (x H) ic / (2a^2), K = (F/x) (-rn/(2a)) cx, D2 = (erf/x) cx
            sc[j] = OP == 0 ? ic[j] * A.inv2a2 : cx[j];
        }
    }
};

// ---------------------------------------------------------------------------
// quadrature point generators
// ---------------------------------------------------------------------------
struct RegularGeom {
    static constexpr bool kSeparable = true;   // point q = (p, r): weights and hats factor
    const double *xp, *yp, *w, *hats;
    int nq1;
    __device__ void point(int q, double x[3], double y[3], double &wq, double ht[3], double hs[3]) const
    {
        // p = q / nq1 without the integer division: (q + 1/2) / nq1 is at least
        // 1/(2 nq1) away from an integer, far above the float rounding
        const int p = __float2int_rz(((float)q + 0.5f) * __frcp_rn((float)nq1)), r = q - p * nq1;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            x[c] = __ldg(xp + 3 * p + c);
            y[c] = __ldg(yp + 3 * r + c);
            ht[c] = __ldg(hats + 3 * p + c);
            hs[c] = __ldg(hats + 3 * r + c);
        }
        wq = __ldg(w + p) * __ldg(w + r);
    }
};

struct DuffyGeom {
    static constexpr bool kSeparable = false;
    double a0[3], da1[3], da2[3], b0[3], db1[3], db2[3];
    const double *ts, *ss, *ws;
    int off;
    int invt[3], invs[3];   // original local vertex k sits at permuted position inv[k]
    __device__ static double pick(const double v[3], int i) { return i == 0 ? v[0] : (i == 1 ? v[1] : v[2]); }
    __device__ void point(int q, double x[3], double y[3], double &wq, double ht[3], double hs[3]) const
    {
        const int qd = off + q;
        const double ut = __ldg(ts + 2 * qd), vt = __ldg(ts + 2 * qd + 1);
        const double us = __ldg(ss + 2 * qd), vs = __ldg(ss + 2 * qd + 1);
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            x[c] = a0[c] + ut * da1[c] + vt * da2[c];
            y[c] = b0[c] + us * db1[c] + vs * db2[c];
        }
        wq = __ldg(ws + qd);
        const double tp[3] = {1.0 - ut - vt, ut, vt}, sp[3] = {1.0 - us - vs, us, vs};
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            ht[k] = pick(tp, invt[k]);
            hs[k] = pick(sp, invs[k]);
        }
    }
};

// ---------------------------------------------------------------------------
// kernel value at one (point pair, gap) in the general branch (scaled by 4 pi):
//   op 0: (rho/(2a^2) + delta/(a rho)) erf(x) + sqrt(delta/(pi a^3)) exp(-x^2)
//   op 1: -(rn/rho) [(1/(2a) - delta/rho^2) erf(x) + sqrt(delta/(pi a)) exp(-x^2)/rho]
//         (the -(rn/rho) factor lives in the hat weights)
//   op 2: erf(x) / rho
// Every product/sum is pinned (fma / __dmul_rn): after unrolling the gap
// slots the compiler must not contract the same expression differently per
// slot, or a gap's value would depend on the slot it lands in.
// ---------------------------------------------------------------------------
template <int OP, int NJ>
__device__ __forceinline__ double eval_general(const PairArgs &A, const Slots<OP, NJ> &T, int j, double rho,
                                               double s1, double s2)
{
    const double x = __dmul_rn(rho, T.cx[j]);
    const double e1 = erf(x);
    if (OP == 2) return __dmul_rn(e1, s1);
    const double e2 = exp(-__dmul_rn(x, x));
    if (OP == 0) return fma(fma(T.dl[j], s2, s1), e1, __dmul_rn(T.kk[j], e2));
    return fma(fma(-T.dl[j], s1, A.inv2a), e1, __dmul_rn(__dmul_rn(T.kk[j], s2), e2));
}

// ---------------------------------------------------------------------------
// Warp sums of N per-lane values, value v returned in lane v (v < N): the two
// 16-lane halves folded by one shuffle each, the 16 partials of every value
// summed by one lane through shared memory (`buf`: 16 (N | 1) doubles, odd
// stride: conflict-free) -- N shuffles + 16 loads instead of 5 N shuffles.
// ---------------------------------------------------------------------------
template <int N>
__device__ __forceinline__ double warp_sums_to_lanes(double (&v)[N], double *buf, int lane)
{
    constexpr int S = N | 1;
#pragma unroll
    for (int i = 0; i < N; ++i) v[i] += __shfl_xor_sync(kFull, v[i], 16);
    __syncwarp();
    if (lane < 16) {
#pragma unroll
        for (int i = 0; i < N; ++i) buf[lane * S + i] = v[i];
    }
    __syncwarp();
    double r = 0.0;
    if (lane < N) {
        double p[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) p[k] = buf[k * S + lane];
#pragma unroll
        for (int l = 4; l < 16; l += 4)
#pragma unroll
            for (int k = 0; k < 4; ++k) p[k] += buf[(l + k) * S + lane];
        r = (p[0] + p[1]) + (p[2] + p[3]);
    }
    __syncwarp();
    return r;
}

// ---------------------------------------------------------------------------
// one element pair, all time gaps of the window
// ---------------------------------------------------------------------------
template <int OP, bool TP1, bool SP1, int NJ, class Geom>
__device__ __forceinline__ void eval_pair(const PairArgs &A, const Geom &g, int nq, const double ny[3],
                                          double jac, int64_t slot, const Slots<OP, NJ> &T,
                                          double *geo, double *Ls, int lane, const double *tab)
{
    constexpr int NT = TP1 ? 3 : 1, NS = SP1 ? 3 : 1, NIJ = NT * NS;
    using L = Layout<OP, NIJ>;
    constexpr int PAY = L::PAY, HOFF = L::HOFF;
    constexpr int SLOTS = LsLayout<NIJ, NJ>::SLOTS;
    const int s = lane >> 4, t = lane & 15;

    // p1 x p1 product rules factor: sum_q v w_p w_r ht_i(p) hs_j(r) =
    // sum_p (w_p ht_i(p)) [sum_r v (w_r hs_j(r))] -- 3 FMA per evaluation
    // instead of 9, the row sums flushed when the test point p changes
    constexpr bool SEP = (NIJ == 9) && Geom::kSeparable && HB_FUSED && HB_SEP;
    double acc[NJ][NIJ];
    double inner[NJ][3], arow[3] = {0.0, 0.0, 0.0};
    int prow = -1;
#pragma unroll
    for (int j = 0; j < NJ; ++j)
        for (int c = 0; c < 3; ++c) inner[j][c] = 0.0;
    auto flush = [&]() {
#pragma unroll
        for (int j = 0; j < NJ; ++j) {
#pragma unroll
            for (int i = 0; i < 3; ++i)
#pragma unroll
                for (int c = 0; c < 3; ++c) acc[j][3 * i + c] = fma(arow[i], inner[j][c], acc[j][3 * i + c]);
#pragma unroll
            for (int c = 0; c < 3; ++c) inner[j][c] = 0.0;
        }
    };
    double s0[NIJ], sc[NIJ];
#pragma unroll
    for (int i = 0; i < NIJ; ++i) {
        s0[i] = 0.0;
        sc[i] = 0.0;
#pragma unroll
        for (int j = 0; j < NJ; ++j) acc[j][i] = 0.0;
    }

    for (int base = 0; base < nq; base += 32) {
        const int q = base + lane;
        int small = 0;
        int nzw = OP == 1 ? 0 : 1;   // K: this point's weights are not all zero (r.n_y != 0)
        if (q >= nq) {
            // padding slot of the grouped loop: all zero (x = 0 and 1/x = 0 give
            // finite series values, the zero weights add exact zeros)
            double *p = geo + lane * PAY;
#pragma unroll
            for (int i = 0; i < PAY; ++i) p[i] = 0.0;
        } else {
            double x[3], y[3], wq, ht[3], hs[3];
            g.point(q, x, y, wq, ht, hs);
            const double rx = x[0] - y[0], ry = x[1] - y[1], rz = x[2] - y[2];
            const double rho = sqrt(rx * rx + ry * ry + rz * rz);
            small = rho <= A.r_eps;
            double H[NIJ];
#pragma unroll
            for (int i = 0; i < NT; ++i)
#pragma unroll
                for (int j = 0; j < NS; ++j)
                    H[i * NS + j] = (TP1 || SP1) ? wq * ((TP1 ? ht[i] : 1.0) * (SP1 ? hs[j] : 1.0)) : wq;
            double *p = geo + lane * PAY;
            p[0] = rho;
            if constexpr (SEP) {   // [HOFF..+2] = w_r hs(r), [HOFF+3..+5] = w_p ht(p)
                const int pr = q / g.nq1, rr = q - pr * g.nq1;
                const double wp = __ldg(g.w + pr), wr = __ldg(g.w + rr);
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    p[HOFF + c] = wr * hs[c];
                    p[HOFF + 3 + c] = wp * ht[c];
                }
            }
            if (OP == 0) {
                const double iq = 1.0 / rho;
                const double Aq = rho * A.inv2a2, Bq = A.inva * iq;
                p[1] = Aq;
                p[2] = HB_FUSED ? iq : Bq;
                if constexpr (!SEP) {
#pragma unroll
                    for (int i = 0; i < NIJ; ++i) p[HOFF + i] = H[i];
                }
                if (A.need_special) {
                    const double cq = A.step * Bq + Aq;
#pragma unroll
                    for (int i = 0; i < NIJ; ++i) {
                        s0[i] = fma(H[i], Aq, s0[i]);
                        sc[i] = fma(H[i], cq, sc[i]);
                    }
                }
            } else if (OP == 1) {
                const double rn = rx * ny[0] + ry * ny[1] + rz * ny[2];
                const double iq = 1.0 / rho;
                const double U = small ? 0.0 : -rn * iq, Ur = small ? 0.0 : -rn;
                nzw = Ur != 0.0;
                const double P = 1.0 / __dmul_rn(rho, rho);
                p[1] = HB_FUSED ? iq : P;
                p[2] = iq;
#pragma unroll
                for (int i = 0; i < NIJ; ++i) p[HOFF + i] = HB_FUSED ? (H[i] * Ur) * A.inv2a : H[i] * U;
                if (A.need_special) {
                    const double c0 = A.inv2a, cc = A.inv2a - A.step * P;
#pragma unroll
                    for (int i = 0; i < NIJ; ++i) {
                        s0[i] = fma(H[i] * U, c0, s0[i]);
                        sc[i] = fma(H[i] * U, cc, sc[i]);
                    }
                }
            } else {
                const double iq = 1.0 / rho;
                p[1] = iq;
                if constexpr (!SEP) {
#pragma unroll
                    for (int i = 0; i < NIJ; ++i) p[HOFF + i] = H[i];
                }
                if (A.need_special) {
#pragma unroll
                    for (int i = 0; i < NIJ; ++i) s0[i] = fma(H[i], iq, s0[i]);
                }
            }
        }
        const bool any_small = __any_sync(kFull, small);
        // K: a chunk whose weights are all exactly zero (coplanar triangles:
        // r.n_y == 0 at every point) adds exact zeros -- skip its evaluations
        const bool skip = OP == 1 && !__any_sync(kFull, nzw);
        __syncwarp();
        const int nloc = min(32, nq - base);
        if (skip) {
        } else if (!any_small) {
#if HB_FUSED
            // two quadrature points of the same parity per iteration, evaluated
            // together per gap slot: their x are close, so the small/large-x
            // branch skipping survives, and the two Horner chains interleave
            // uniform trip count for both point-parity halves (tail points of
            // an odd chunk get zero weight), so the branch votes below span the
            // full warp and compile to uniform branches
            const int nloc4 = (nloc + 3) & ~3;
            if constexpr (SEP) {
                for (int k = s; k < nloc4; k += 2) {
                    const bool ok = k < nloc;
                    const double *p = geo + (ok ? k : 0) * PAY;
                    const int pr = (base + k) / g.nq1;
                    if (ok && pr != prow) {
                        if (prow >= 0) flush();
                        prow = pr;
#pragma unroll
                        for (int i = 0; i < 3; ++i) arow[i] = p[HOFF + 3 + i];
                    }
                    const double rho = p[0], s1 = p[1];
                    const double s2 = (OP == 2) ? 0.0 : p[2];
#pragma unroll
                    for (int j = 0; j < NJ; ++j) {
                        const double x = __dmul_rn(rho, T.cx[j]);
                        const double ix = __dmul_rn(OP == 0 ? s2 : s1, T.ic[j]);
                        const double f = special::eval_u<OP + 4>(x, ix, tab, kFull);
                        const double v = ok ? f : 0.0;
#pragma unroll
                        for (int c = 0; c < 3; ++c) inner[j][c] = fma(v, p[HOFF + c], inner[j][c]);
                    }
                }
            } else if constexpr (NIJ == 9 && !HB_P1P1_GROUPED) {
                // p1 x p1: nine hat weights per point -- one point per iteration
                for (int k = s; k < nloc4; k += 2) {
                    const bool ok = k < nloc;
                    const double *p = geo + (ok ? k : 0) * PAY;
                    const double rho = p[0], s1 = p[1];
                    const double s2 = (OP == 2) ? 0.0 : p[2];
#pragma unroll
                    for (int j = 0; j < NJ; ++j) {
                        const double x = __dmul_rn(rho, T.cx[j]);
                        const double ix = __dmul_rn(OP == 0 ? s2 : s1, T.ic[j]);
                        const double f = special::eval_u<OP + 4>(x, ix, tab, kFull);
                        const double v = ok ? f : 0.0;
#pragma unroll
                        for (int i = 0; i < NIJ; ++i) acc[j][i] = fma(v, p[HOFF + i], acc[j][i]);
                    }
                }
            } else {
#ifndef HB_QGROUP
#define HB_QGROUP 2
#endif
                // G points of the same parity per branch region (x close -> the
                // small/large-x skipping survives; G independent Horner chains)
                constexpr int G = HB_QGROUP;
                static_assert(32 % (2 * G) == 0, "padded group loop must stay inside the warp's 32 payload slots");
                const int nlocg = (nloc + 2 * G - 1) / (2 * G) * (2 * G);
                // (slots nloc..nlocg-1 hold the all-zero padding payload)
                // (p1 x p1 keeps the explicit select: measured faster there)
                constexpr bool SEL = NIJ == 9;
                for (int k = s; k < nlocg; k += 2 * G) {
                    double pv[G][PAY];
                    double rho[G], a[G], b[G];
                    bool ok[G];
#pragma unroll
                    for (int g = 0; g < G; ++g) {
                        ok[g] = !SEL || k + 2 * g < nloc;
                        load_payload<PAY>(geo + (ok[g] ? k + 2 * g : 0) * PAY, pv[g]);
                        rho[g] = pv[g][0];
                        a[g] = pv[g][1];
                        b[g] = (OP == 2) ? 0.0 : pv[g][2];
                    }
#pragma unroll
                    for (int j = 0; j < NJ; ++j) {
                        double xs[G], fs[G];
#pragma unroll
                        for (int g = 0; g < G; ++g) xs[g] = __dmul_rn(rho[g], T.cx[j]);
                        const double icj = T.ic[j];
                        special::eval_unf<OP + 4, G>(
                            xs, [&](int g) { return __dmul_rn(OP == 0 ? b[g] : a[g], icj); }, fs, tab, kFull);
#pragma unroll
                        for (int g = 0; g < G; ++g) {
                            const double v = ok[g] ? fs[g] : 0.0;
#pragma unroll
                            for (int i = 0; i < NIJ; ++i) acc[j][i] = fma(v, pv[g][HOFF + i], acc[j][i]);
                        }
                    }
                }
            }
#else
#pragma unroll 1
            for (int k = s; k < nloc; k += 2) {
                const double *p = geo + k * PAY;
                const double rho = p[0], s1 = p[1];
                const double s2 = (OP == 2) ? 0.0 : p[2];
                double val[NJ];
#pragma unroll
                for (int j = 0; j < NJ; ++j) val[j] = eval_general<OP>(A, T, j, rho, s1, s2);
#pragma unroll
                for (int i = 0; i < NIJ; ++i) {
                    const double h = p[HOFF + i];
#pragma unroll
                    for (int j = 0; j < NJ; ++j) acc[j][i] = fma(val[j], h, acc[j][i]);
                }
            }
#endif
        } else {
            if constexpr (SEP) {
                if (prow >= 0) flush();
                prow = -1;
            }
            for (int k = s; k < nloc; k += 2) {
                const double *p = geo + k * PAY;
                const double rho = p[0], s1 = p[1];
                const double s2 = (OP == 2) ? 0.0 : p[2];
                const bool sm = rho <= A.r_eps;
#if HB_FUSED
                const unsigned mask = __activemask();
#endif
#pragma unroll
                for (int j = 0; j < NJ; ++j) {
                    double val;
#if HB_FUSED
                    const double x = __dmul_rn(rho, T.cx[j]);
                    const double ix = __dmul_rn(OP == 0 ? s2 : s1, T.ic[j]);
                    const double f = special::eval_u<OP + 4>(x, ix, tab, mask);
                    // rho <= r_eps limits, divided by the per-gap factor applied at the end
                    if (OP == 0) val = sm ? 2.0 * T.kk[j] / T.sc[j] : f;
                    else if (OP == 1) val = sm ? 0.0 : f;
                    else val = sm ? T.kk[j] / T.sc[j] : f;
#else
                    if (OP == 0) val = sm ? 2.0 * T.kk[j] : eval_general<OP>(A, T, j, rho, s1, s2);
                    else if (OP == 1) val = sm ? 0.0 : eval_general<OP>(A, T, j, rho, s1, s2);
                    else val = sm ? T.kk[j] : eval_general<OP>(A, T, j, rho, s1, s2);
#endif
                    if constexpr (SEP) {
#pragma unroll
                        for (int i = 0; i < 3; ++i)
#pragma unroll
                            for (int c = 0; c < 3; ++c)
                                acc[j][3 * i + c] = fma(val, p[HOFF + 3 + i] * p[HOFF + c], acc[j][3 * i + c]);
                    } else {
#pragma unroll
                        for (int i = 0; i < NIJ; ++i) acc[j][i] = fma(val, p[HOFF + i], acc[j][i]);
                    }
                }
            }
        }
        __syncwarp();
    }
    if constexpr (SEP) {
        if (prow >= 0) flush();
    }

    // fold the two point-parity halves (commutative: both halves get equal bits)
#pragma unroll
    for (int j = 0; j < NJ; ++j)
#pragma unroll
        for (int i = 0; i < NIJ; ++i) acc[j][i] += __shfl_xor_sync(kFull, acc[j][i], 16);
    constexpr int NSP = (OP == 2 ? 1 : 2) * NIJ;   // special sums: s0 (and sc)
    constexpr bool SCATTER = NSP >= 6;
    static_assert(!SCATTER || 16 * (NSP | 1) <= 32 * PAY, "special-sum buffer must fit the payload area");
    double spec = 0.0;   // SCATTER: value `lane` of (s0, sc)
    if (A.need_special) {
        if constexpr (SCATTER) {
            double v[NSP];
#pragma unroll
            for (int i = 0; i < NIJ; ++i) {
                v[i] = s0[i];
                if (OP != 2) v[NIJ + i] = sc[i];
            }
            spec = warp_sums_to_lanes<NSP>(v, geo, lane);
        } else {
#pragma unroll
            for (int o = 16; o >= 1; o >>= 1)
#pragma unroll
                for (int i = 0; i < NIJ; ++i) {
                    s0[i] += __shfl_xor_sync(kFull, s0[i], o);
                    if (OP != 2) sc[i] += __shfl_xor_sync(kFull, sc[i], o);
                }
        }
    }
    const int nslots = A.it_hi - A.it_lo + 1;
    if (s == 0) {
#pragma unroll
        for (int j = 0; j < NJ; ++j) {
            const int sl = t + 16 * j;
            if (sl < nslots) {
#pragma unroll
                for (int i = 0; i < NIJ; ++i) Ls[i * SLOTS + sl] = jac * (HB_FUSED ? acc[j][i] * T.sc[j] : acc[j][i]);
            }
        }
    }
    double *L0 = Ls + NIJ * SLOTS, *Lc = L0 + NIJ;
    if constexpr (SCATTER) {   // L0 = s0, Lc = sc (D2: s0): lane v holds value v
        if (A.need_special && lane < NSP) {
            L0[lane] = jac * spec;
            if (OP == 2) Lc[lane] = jac * spec;
        }
    } else if (lane == 0 && A.need_special) {
#pragma unroll
        for (int i = 0; i < NIJ; ++i) {
            L0[i] = jac * s0[i];
            Lc[i] = jac * (OP == 2 ? s0[i] : sc[i]);
        }
    }
    __syncwarp();
    // 3-term combination (AssemblyPlan.targets) with lanes over blocks d
    double *dst = A.Q + slot * (int64_t)(NIJ * A.nd);
    for (int dd = lane; dd < A.nd; dd += 32) {
        const int d = A.d0 + dd;
#pragma unroll
        for (int i = 0; i < NIJ; ++i) {
            const double *Li = Ls + i * SLOTS;
            double b;
            if (d == 0) {
                const double l1 = Li[1 - A.it_lo];
                b = Lc[i] + (-l1);
            } else {
                const double lm = (d - 1 == 0) ? L0[i] : Li[d - 1 - A.it_lo];
                const double lc = Li[d - A.it_lo];
                const double lp = Li[d + 1 - A.it_lo];
                b = -lm + 2.0 * lc;
                b = b + (-lp);
            }
            dst[i * A.nd + dd] = b;
        }
    }
    __syncwarp();
}

// ---------------------------------------------------------------------------
// K (p0 test x p1 trial) for both orientations of one separated pair.
// The product rule of a separated pair (a, b) uses the same point pairs for
// K(a, b) and K(b, a): rho -- hence x and F(x) at every gap -- is shared, and
// only the per-point weights differ:
//   K(a, b): -(r . n_b)/rho * w hs_j(y_r)      (test a, trial hats on b)
//   K(b, a): +(r . n_a)/rho * w ht_j(x_p)      (test b, trial hats on a)
// with r = x_p - y_r (the reverse orientation's r is -r, exactly).  Each
// point's weight has the bits of the direct computation; one F evaluation
// feeds both sums, halving the special-function work of K.  Every separated
// pair is evaluated as its canonical (min, max) orientation whichever output
// is needed, so the blocks do not depend on the row chunking / rank split.
// ---------------------------------------------------------------------------
constexpr int kDualPay = 8;   // rho, 1/rho, Wf[3], Wr[3]
template <int NJ>
__host__ __device__ constexpr int dual_smem_doubles_per_warp() { return 32 * kDualPay + 2 * LsLayout<3, NJ>::SIZE; }

// 3-term time combination of one staged row of L values (Ls: [NIJ][SLOTS],
// then L0[NIJ], Lcomb0[NIJ]) into Q slot `slot`, lanes over blocks d
template <int NIJ, int NJ>
__device__ __forceinline__ void combine_store(const PairArgs &A, const double *Ls, int64_t slot, int lane)
{
    constexpr int SLOTS = LsLayout<NIJ, NJ>::SLOTS;
    const double *L0 = Ls + NIJ * SLOTS, *Lc = L0 + NIJ;
    double *dst = A.Q + slot * (int64_t)(NIJ * A.nd);
    for (int dd = lane; dd < A.nd; dd += 32) {
        const int d = A.d0 + dd;
#pragma unroll
        for (int i = 0; i < NIJ; ++i) {
            const double *Li = Ls + i * SLOTS;
            double b;
            if (d == 0) {
                const double l1 = Li[1 - A.it_lo];
                b = Lc[i] + (-l1);
            } else {
                const double lm = (d - 1 == 0) ? L0[i] : Li[d - 1 - A.it_lo];
                const double lc = Li[d - A.it_lo];
                const double lp = Li[d + 1 - A.it_lo];
                b = -lm + 2.0 * lc;
                b = b + (-lp);
            }
            dst[i * A.nd + dd] = b;
        }
    }
}

// MODE 0: both outputs; 1: only K(a, b) (forward); 2: only K(b, a) (reverse) --
// the other row lies outside the launch.  Each output's arithmetic is the same
// in every mode (same points, order, fs and weights), so a block entry does not
// depend on which rows share the launch (row chunks, ranks).
template <int NJ, int MODE = 0>
__device__ __forceinline__ void eval_pair_dual(const PairArgs &A, const RegularGeom &g, int nq, const double nb[3],
                                               const double na[3], double jac, int64_t slot_f, int64_t slot_r,
                                               const Slots<1, NJ> &T, double *geo, double *Ls, int lane,
                                               const double *tab)
{
    constexpr bool DF = MODE != 2, DR = MODE != 1;
    constexpr int PAY = kDualPay, SLOTS = LsLayout<3, NJ>::SLOTS, LSZ = LsLayout<3, NJ>::SIZE;
    const int s = lane >> 4, t = lane & 15;
    double af[NJ][3], ar[NJ][3], s0f[3], scf[3], s0r[3], scr[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        s0f[i] = scf[i] = s0r[i] = scr[i] = 0.0;
#pragma unroll
        for (int j = 0; j < NJ; ++j) af[j][i] = ar[j][i] = 0.0;
    }
    for (int base = 0; base < nq; base += 32) {
        const int q = base + lane;
        int small = 0, nzw = 0;
        if (q >= nq) {   // all-zero padding slot (see eval_pair)
            double *p = geo + lane * PAY;
#pragma unroll
            for (int i = 0; i < PAY; ++i) p[i] = 0.0;
        } else {
            double x[3], y[3], wq, ht[3], hs[3];
            g.point(q, x, y, wq, ht, hs);
            const double rx = x[0] - y[0], ry = x[1] - y[1], rz = x[2] - y[2];
            const double rho = sqrt(rx * rx + ry * ry + rz * rz);
            small = rho <= A.r_eps;
            const double rnb = rx * nb[0] + ry * nb[1] + rz * nb[2];
            const double rna = (-rx) * na[0] + (-ry) * na[1] + (-rz) * na[2];   // reverse: r' = -r
            const double iq = 1.0 / rho;
            const double Uf = small ? 0.0 : -rnb * iq, Ur = small ? 0.0 : -rna * iq;
            const double Vf = small ? 0.0 : -rnb, Vr = small ? 0.0 : -rna;   // rho U (factor-free F/x)
            nzw = (DF && Vf != 0.0) || (DR && Vr != 0.0);
            const double P = 1.0 / __dmul_rn(rho, rho);
            double *p = geo + lane * PAY;
            p[0] = rho;
            p[1] = iq;
            double Hf[3], Hr[3];
#pragma unroll
            for (int i = 0; i < 3; ++i) {
                Hf[i] = wq * (1.0 * hs[i]);
                Hr[i] = wq * (1.0 * ht[i]);
                if (DF) p[2 + i] = (Hf[i] * Vf) * A.inv2a;
                if (DR) p[5 + i] = (Hr[i] * Vr) * A.inv2a;
            }
            if (A.need_special) {
                const double c0 = A.inv2a, cc = A.inv2a - A.step * P;
#pragma unroll
                for (int i = 0; i < 3; ++i) {
                    s0f[i] = fma(Hf[i] * Uf, c0, s0f[i]);
                    scf[i] = fma(Hf[i] * Uf, cc, scf[i]);
                    s0r[i] = fma(Hr[i] * Ur, c0, s0r[i]);
                    scr[i] = fma(Hr[i] * Ur, cc, scr[i]);
                }
            }
        }
        const bool any_small = __any_sync(kFull, small);
        const bool skip = !__any_sync(kFull, nzw);   // both orientations' weights all zero (coplanar pair)
        __syncwarp();
        const int nloc = min(32, nq - base);
        if (skip) {
        } else if (!any_small) {
            constexpr int G = HB_QGROUP;
            static_assert(32 % (2 * G) == 0, "padded group loop must stay inside the warp's 32 payload slots");
            const int nlocg = (nloc + 2 * G - 1) / (2 * G) * (2 * G);
            for (int k = s; k < nlocg; k += 2 * G) {   // padding slots are all zero
                double pv[G][PAY];
                double rho[G], a[G];
#pragma unroll
                for (int gg = 0; gg < G; ++gg) {
                    load_payload<PAY>(geo + (k + 2 * gg) * PAY, pv[gg]);
                    rho[gg] = pv[gg][0];
                    a[gg] = pv[gg][1];
                }
#pragma unroll
                for (int j = 0; j < NJ; ++j) {
                    double xs[G], fs[G];
#pragma unroll
                    for (int gg = 0; gg < G; ++gg) xs[gg] = __dmul_rn(rho[gg], T.cx[j]);
                    const double icj = T.ic[j];
                    special::eval_unf<5, G>(xs, [&](int gg) { return __dmul_rn(a[gg], icj); }, fs, tab, kFull);
#pragma unroll
                    for (int gg = 0; gg < G; ++gg) {
#pragma unroll
                        for (int i = 0; i < 3; ++i) {
                            af[j][i] = fma(fs[gg], pv[gg][2 + i], af[j][i]);
                            ar[j][i] = fma(fs[gg], pv[gg][5 + i], ar[j][i]);
                        }
                    }
                }
            }
        } else {
            for (int k = s; k < nloc; k += 2) {
                const double *p = geo + k * PAY;
                const double rho = p[0], s1 = p[1];
                const bool sm = rho <= A.r_eps;
                const unsigned mask = __activemask();
#pragma unroll
                for (int j = 0; j < NJ; ++j) {
                    const double x = __dmul_rn(rho, T.cx[j]);
                    const double ix = __dmul_rn(s1, T.ic[j]);
                    const double f = special::eval_u<5>(x, ix, tab, mask);
                    const double val = sm ? 0.0 : f;
#pragma unroll
                    for (int i = 0; i < 3; ++i) {
                        af[j][i] = fma(val, p[2 + i], af[j][i]);
                        ar[j][i] = fma(val, p[5 + i], ar[j][i]);
                    }
                }
            }
        }
        __syncwarp();
    }
#pragma unroll
    for (int j = 0; j < NJ; ++j)
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            if (DF) af[j][i] += __shfl_xor_sync(kFull, af[j][i], 16);
            if (DR) ar[j][i] += __shfl_xor_sync(kFull, ar[j][i], 16);
        }
    // special sums, value v in lane v: (s0, sc) of the forward output, then of the reverse one
    constexpr int NSP = (DF ? 6 : 0) + (DR ? 6 : 0);
    static_assert(16 * (NSP | 1) <= 32 * PAY, "special-sum buffer must fit the payload area");
    double spec = 0.0;
    if (A.need_special) {
        double v[NSP];
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            if (DF) {
                v[i] = s0f[i];
                v[3 + i] = scf[i];
            }
            if (DR) {
                v[(DF ? 6 : 0) + i] = s0r[i];
                v[(DF ? 9 : 3) + i] = scr[i];
            }
        }
        spec = warp_sums_to_lanes<NSP>(v, geo, lane);
    }
    const int nslots = A.it_hi - A.it_lo + 1;
    double *Lf = Ls, *Lr = Ls + LSZ;
    if (s == 0) {
#pragma unroll
        for (int j = 0; j < NJ; ++j) {
            const int sl = t + 16 * j;
            if (sl < nslots) {
#pragma unroll
                for (int i = 0; i < 3; ++i) {
                    if (DF) Lf[i * SLOTS + sl] = jac * (af[j][i] * T.sc[j]);
                    if (DR) Lr[i * SLOTS + sl] = jac * (ar[j][i] * T.sc[j]);
                }
            }
        }
    }
    if (A.need_special && lane < NSP) {   // [3 SLOTS + 0..2] = s0, [+3..5] = sc
        const bool fwd = DF && lane < 6;
        (fwd ? Lf : Lr)[3 * SLOTS + (fwd ? lane : lane - (DF ? 6 : 0))] = jac * spec;
    }
    __syncwarp();
    if (DF && slot_f >= 0) combine_store<3, NJ>(A, Lf, slot_f, lane);
    if (DR && slot_r >= 0) combine_store<3, NJ>(A, Lr, slot_r, lane);
    __syncwarp();
}

__device__ __forceinline__ double exact_dot3(const double *a, const double *b)
{
    // (a0*b0 + a1*b1) + a2*b2, each step rounded (no FMA contraction)
    return __dadd_rn(__dadd_rn(__dmul_rn(a[0], b[0]), __dmul_rn(a[1], b[1])), __dmul_rn(a[2], b[2]));
}

template <int OP>
__device__ __forceinline__ double pair_jac(const PairArgs &A, int64_t e, int64_t f)
{
    double jac = (__ldg(A.m.areas_dev + e) * __ldg(A.m.areas_dev + f)) * kInvPi;
    if (A.halve_diag && e == f) jac *= 0.5;
    if (OP == 2) {
        double ne[3], nf[3];
        for (int c = 0; c < 3; ++c) {
            ne[c] = __ldg(A.m.normals_dev + 3 * e + c);
            nf[c] = __ldg(A.m.normals_dev + 3 * f + c);
        }
        jac *= exact_dot3(ne, nf);
    }
    return jac;
}

// ---------------------------------------------------------------------------
// pair classification, shared by the pair kernel and hb_pair_classes
// ---------------------------------------------------------------------------
// position of f in e's touching list (binary search, as _assembly_numba.py:139-151), -1 if absent
__device__ __forceinline__ int64_t touching_pos(const hb_mesh_desc &M, int64_t t_lo, int64_t t_hi, int64_t f)
{
    int64_t lo = t_lo, hi = t_hi;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1, v = __ldg(M.tn_idx_dev + mid);
        if (v < f) lo = mid + 1;
        else if (v > f) hi = mid;
        else return mid;
    }
    return -1;
}

// near/far: sqrt((dx*dx + dy*dy) + dz*dz) < 2 max(diam_e, diam_f), every
// operation separately rounded as in _assembly_numba.py:218-223 (no FMA)
__device__ __forceinline__ bool near_test(const hb_mesh_desc &M, const double ce[3], double de, int64_t f)
{
    const double dx = __dsub_rn(ce[0], __ldg(M.centroids_dev + 3 * f));
    const double dy = __dsub_rn(ce[1], __ldg(M.centroids_dev + 3 * f + 1));
    const double dz = __dsub_rn(ce[2], __ldg(M.centroids_dev + 3 * f + 2));
    const double dist = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz)));
    return dist < 2.0 * fmax(de, __ldg(M.diameters_dev + f));
}

// ---------------------------------------------------------------------------
// K1 body: separated pairs of one (test row e, 32-column segment) work item.
// ---------------------------------------------------------------------------
template <int OP, bool TP1, bool SP1, int NJ, bool SYM>
__device__ __forceinline__ void regular_item(const PairArgs &A, int64_t e, int64_t seg, const Slots<OP, NJ> &T,
                                             double *geo, double *Ls, int lane, const double *tab)
{
    const hb_mesh_desc &M = A.m;
    int64_t fb = seg * A.seg_len;
    const int64_t fe = min(fb + A.seg_len, M.E_x);
    if (SYM) fb = max(fb, e);
    if (fb >= fe) return;
    const int64_t t_lo = __ldg(M.tn_indptr_dev + e), t_hi = __ldg(M.tn_indptr_dev + e + 1);
    // classify the segment lane-parallel (lane l: trial fb + l): touching pairs
    // belong to the singular path; near/far by the exact IEEE test
    unsigned todo, nearm;
    {
        const int64_t f = fb + lane;
        bool ok = false, nr = false;
        if (f < fe) {
            double ce[3];
            for (int c = 0; c < 3; ++c) ce[c] = __ldg(M.centroids_dev + 3 * e + c);
            ok = touching_pos(M, t_lo, t_hi, f) < 0;
            nr = ok && near_test(M, ce, __ldg(M.diameters_dev + e), f);
        }
        todo = __ballot_sync(kFull, ok);
        nearm = __ballot_sync(kFull, nr);
    }
    while (todo) {
        const int bit = __ffs(todo) - 1;
        todo &= todo - 1;
        const int64_t f = fb + bit;
        const int64_t slot = (e - A.e0) * M.E_x + f;
        const double jac = pair_jac<OP>(A, e, f);
        if (OP == 2 && jac == 0.0) continue;   // n_x.n_y == 0: no contribution (finalize skips it)
        const bool near = (nearm >> bit) & 1u;
        RegularGeom g;
        const int nq1 = near ? (int)M.n_near : (int)M.n_reg;
        const double *pts = near ? M.near_pts_dev : M.reg_pts_dev;
        g.xp = pts + 3 * e * nq1;
        g.yp = pts + 3 * f * nq1;
        g.w = near ? M.near_w_dev : M.reg_w_dev;
        g.hats = near ? M.near_hats_dev : M.reg_hats_dev;
        g.nq1 = nq1;
        double ny[3];
        for (int c = 0; c < 3; ++c) ny[c] = __ldg(M.normals_dev + 3 * f + c);
        eval_pair<OP, TP1, SP1, NJ>(A, g, nq1 * nq1, ny, jac, slot, T, geo, Ls, lane, tab);
    }
}

// K1 body for K with both orientations: separated pairs (e, f) of one
// (test row e, segment) item, evaluated as the canonical pair (min, max).
// Pairs with both rows in the chunk are produced once (by the smaller row);
// a pair whose other row lies outside the chunk is still evaluated in its
// canonical orientation and only this row's output is stored.
template <int NJ>
__device__ __forceinline__ void regular_item_dual(const PairArgs &A, int64_t e, int64_t seg, const Slots<1, NJ> &T,
                                                  double *geo, double *Ls, int lane, const double *tab)
{
    const hb_mesh_desc &M = A.m;
    const int64_t fb = seg * A.seg_len;
    const int64_t fe = min(fb + A.seg_len, M.E_x);
    if (fb >= fe) return;
    const int64_t t_lo = __ldg(M.tn_indptr_dev + e), t_hi = __ldg(M.tn_indptr_dev + e + 1);
    // classify the segment lane-parallel (lane l: trial fb + l); the near test
    // of the canonical pair (a, b) equals that of (e, f) bitwise (squares of
    // negated differences, symmetric max)
    unsigned todo, nearm;
    {
        const int64_t f = fb + lane;
        bool ok = false, nr = false;
        if (f < fe) {
            const bool f_in = f >= A.e0 && f < A.e1;
            ok = !(f < e && f_in)                              // the canonical pair (f, e) belongs to row f
                 && touching_pos(M, t_lo, t_hi, f) < 0;        // touching pairs: singular path (f == e too)
            if (ok) {
                const int64_t a = f > e ? e : f, b = f > e ? f : e;
                double ca[3];
                for (int c = 0; c < 3; ++c) ca[c] = __ldg(M.centroids_dev + 3 * a + c);
                nr = near_test(M, ca, __ldg(M.diameters_dev + a), b);
            }
        }
        todo = __ballot_sync(kFull, ok);
        nearm = __ballot_sync(kFull, nr);
    }
    while (todo) {
        const int bit = __ffs(todo) - 1;
        todo &= todo - 1;
        const int64_t f = fb + bit;
        const int64_t a = f > e ? e : f, b = f > e ? f : e;
        const int64_t slot_f = (a >= A.e0 && a < A.e1) ? (a - A.e0) * M.E_x + b : -1;   // test a, trial b
        const int64_t slot_r = (b >= A.e0 && b < A.e1) ? (b - A.e0) * M.E_x + a : -1;   // test b, trial a
        const bool near = (nearm >> bit) & 1u;
        RegularGeom g;
        const int nq1 = near ? (int)M.n_near : (int)M.n_reg;
        const double *pts = near ? M.near_pts_dev : M.reg_pts_dev;
        g.xp = pts + 3 * a * nq1;
        g.yp = pts + 3 * b * nq1;
        g.w = near ? M.near_w_dev : M.reg_w_dev;
        g.hats = near ? M.near_hats_dev : M.reg_hats_dev;
        g.nq1 = nq1;
        double nb[3], na[3];
        for (int c = 0; c < 3; ++c) {
            nb[c] = __ldg(M.normals_dev + 3 * b + c);
            na[c] = __ldg(M.normals_dev + 3 * a + c);
        }
        const double jac = pair_jac<1>(A, a, b);
        if (slot_f >= 0 && slot_r >= 0)
            eval_pair_dual<NJ, 0>(A, g, nq1 * nq1, nb, na, jac, slot_f, slot_r, T, geo, Ls, lane, tab);
        else if (slot_f >= 0)
            eval_pair_dual<NJ, 1>(A, g, nq1 * nq1, nb, na, jac, slot_f, slot_r, T, geo, Ls, lane, tab);
        else
            eval_pair_dual<NJ, 2>(A, g, nq1 * nq1, nb, na, jac, slot_f, slot_r, T, geo, Ls, lane, tab);
    }
}

// ---------------------------------------------------------------------------
// K2 body: one touching pair (identical / common edge / common vertex),
// Sauter-Schwab rule on the permuted charts of classify_pair.
// ---------------------------------------------------------------------------
template <int OP, bool TP1, bool SP1, int NJ>
__device__ __forceinline__ void singular_item(const PairArgs &A, int64_t k, const Slots<OP, NJ> &T,
                                              double *geo, double *Ls, int lane, const double *tab)
{
    const hb_mesh_desc &M = A.m;
    const int64_t tpos = __ldg(M.sing_pos_dev + k);
    const int64_t e = __ldg(M.sing_row_dev + tpos);
    const int64_t f = __ldg(M.tn_idx_dev + tpos);
    const int cs = (int)__ldg(M.tn_case_dev + tpos);
    DuffyGeom g;
    int pt[3], ps[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        pt[i] = (int)__ldg(M.tn_permt_dev + 3 * tpos + i);
        ps[i] = (int)__ldg(M.tn_perms_dev + 3 * tpos + i);
    }
#pragma unroll
    for (int q = 0; q < 3; ++q) {   // inverse permutations, register-resident
        g.invt[q] = pt[0] == q ? 0 : (pt[1] == q ? 1 : 2);
        g.invs[q] = ps[0] == q ? 0 : (ps[1] == q ? 1 : 2);
    }
    const double *ve = M.verts_tri_dev + 9 * e, *vf = M.verts_tri_dev + 9 * f;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        const double a0 = __ldg(ve + 3 * pt[0] + c), a1 = __ldg(ve + 3 * pt[1] + c), a2 = __ldg(ve + 3 * pt[2] + c);
        const double b0 = __ldg(vf + 3 * ps[0] + c), b1 = __ldg(vf + 3 * ps[1] + c), b2 = __ldg(vf + 3 * ps[2] + c);
        g.a0[c] = a0; g.da1[c] = a1 - a0; g.da2[c] = a2 - a0;
        g.b0[c] = b0; g.db1[c] = b1 - b0; g.db2[c] = b2 - b0;
    }
    g.ts = M.duf_t_dev;
    g.ss = M.duf_s_dev;
    g.ws = M.duf_w_dev;
    const int off0 = (int)__ldg(M.duf_off_dev + cs), off1 = (int)__ldg(M.duf_off_dev + cs + 1);
    g.off = off0;
    const int64_t slot = (e - A.e0) * M.E_x + f;
    const double jac = pair_jac<OP>(A, e, f);
    if (OP == 2 && jac == 0.0) return;   // n_x.n_y == 0: no contribution (finalize skips it)
    double ny[3];
    for (int c = 0; c < 3; ++c) ny[c] = __ldg(M.normals_dev + 3 * f + c);
    eval_pair<OP, TP1, SP1, NJ>(A, g, off1 - off0, ny, jac, slot, T, geo, Ls, lane, tab);
}

// ---------------------------------------------------------------------------
// Persistent pair kernel: warps pull work items from a global counter.
// Items [0, n_sing) are touching pairs (K2 body, heaviest first in row
// order), items [n_sing, n_sing + rows*nseg) are (row, segment) tiles of
// separated pairs (K1 body).  A warp only ever holds one pair class, so the
// two quadrature families never share a warp; dynamic fetching removes the
// imbalance of upper-triangular / near-diagonal tiles.
// ---------------------------------------------------------------------------
template <int OP, bool TP1, bool SP1, int NJ, bool SYM, bool DUAL = false>
__global__ void __launch_bounds__(HB_PAIR_WARPS * 32, (TP1 && SP1) ? HB_P1P1_MINB : HB_PAIR_MINB) k_pairs(const PairArgs A)
{
    constexpr int NIJ = (TP1 ? 3 : 1) * (SP1 ? 3 : 1);
    extern __shared__ __align__(16) double smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double *tab = smem;
    special::load_utable<OP + 4>(tab);   // factor-free kinds, uniform pieces (hb_special.cuh)
    __syncthreads();
    constexpr int kPerWarp = DUAL ? dual_smem_doubles_per_warp<NJ>() : smem_doubles_per_warp<OP, NIJ, NJ>();
    static_assert(special::kUTabDoubles % 2 == 0 && kPerWarp % 2 == 0 && Layout<OP, NIJ>::PAY % 2 == 0 &&
                      kDualPay % 2 == 0, "payload slots must stay 16-byte aligned (LDS.128)");
    double *geo = smem + special::kUTabDoubles + warp * kPerWarp;
    double *Ls = geo + 32 * Layout<OP, NIJ>::PAY;
    double *Ls_dual = geo + 32 * kDualPay;
    const hb_mesh_desc &M = A.m;
    const int64_t s_lo = __ldg(M.sing_rowptr_dev + A.e0), s_hi = __ldg(M.sing_rowptr_dev + A.e1);
    int64_t n_sing = s_hi - s_lo;
    const int64_t nseg = cdiv(M.E_x, (int64_t)A.seg_len);
    int64_t n_reg = (A.e1 - A.e0) * nseg;
    Slots<OP, NJ> T;
    T.init(A, lane & 15);
    for (;;) {
        unsigned long long it = 0;
        if (lane == 0) it = atomicAdd(A.counter, 1ull);
        it = __shfl_sync(kFull, it, 0);
        const int64_t item = (int64_t)it;
        if (item < n_sing) {
            singular_item<OP, TP1, SP1, NJ>(A, s_lo + item, T, geo, Ls, lane, tab);
        } else if (item - n_sing < n_reg) {
            const int64_t r = item - n_sing;
            if constexpr (DUAL) regular_item_dual<NJ>(A, A.e0 + r / nseg, r % nseg, T, geo, Ls_dual, lane, tab);
            else regular_item<OP, TP1, SP1, NJ, SYM>(A, A.e0 + r / nseg, r % nseg, T, geo, Ls, lane, tab);
        } else {
            break;
        }
    }
}

// ---------------------------------------------------------------------------
struct OpShape {
    int NIJ, NJmax;
};

static OpShape op_shape(const hb_assembly_desc *a)
{
    const int nij = (a->test_p1 ? 3 : 1) * (a->trial_p1 ? 3 : 1);
    return {nij, 2};
}

static int choose_nj(const hb_assembly_desc *a)
{
    const OpShape s = op_shape(a);
    int nj = (int)cdiv(a->E_t, 16);
    return std::max(1, std::min(nj, s.NJmax));
}

template <int OP, bool TP1, bool SP1, int NJ, bool DUAL = false>
static int launch_pairs(const PairArgs &A, cudaStream_t st)
{
    constexpr int NIJ = (TP1 ? 3 : 1) * (SP1 ? 3 : 1);
    constexpr bool SYM = (OP != 1);
    constexpr int per_warp = DUAL ? dual_smem_doubles_per_warp<NJ>() : smem_doubles_per_warp<OP, NIJ, NJ>();
    const size_t sm = ((size_t)HB_PAIR_WARPS * per_warp + special::kUTabDoubles) * sizeof(double);
    auto kp = k_pairs<OP, TP1, SP1, NJ, SYM, DUAL>;
    if (sm > 48 * 1024) cudaFuncSetAttribute(kp, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    int dev = 0, nsm = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kp, HB_PAIR_WARPS * 32, sm);
    const int64_t rows = A.e1 - A.e0;
    // separated-pair items of 32 trial elements, halved while the launch holds
    // fewer than 16 items per resident warp (HB_ITEMS_PER_WARP): the persistent grid's
    // tail is about one item per warp, so few large items leave SMs idle at the
    // end (config 2: 8 items per warp at 32 -> 31 at 8 elements: K 1.36 -> 1.25 ms,
    // D2 1.00 -> 0.89 ms; the values do not depend on the grouping: warp per pair)
    PairArgs B = A;
    const int64_t warps = (int64_t)std::max(1, per_sm) * nsm * HB_PAIR_WARPS;
    static const int seg0 = getenv("HB_SEG_LEN") ? std::max(1, std::min(32, atoi(getenv("HB_SEG_LEN")))) : 32;
    static const int ipw = getenv("HB_ITEMS_PER_WARP") ? std::max(1, atoi(getenv("HB_ITEMS_PER_WARP"))) : 16;
    B.seg_len = seg0;
    static const int min_seg = getenv("HB_MIN_SEG") ? atoi(getenv("HB_MIN_SEG")) : 4;
    const int seg_floor = std::max(1, std::min(32, min_seg));
    while (B.seg_len > seg_floor && rows * cdiv(A.m.E_x, (int64_t)B.seg_len) < ipw * warps) B.seg_len /= 2;
    const int64_t items = rows * cdiv(A.m.E_x, (int64_t)B.seg_len) + rows * A.m.sing_max_per_row;
    const int64_t grid = std::max<int64_t>(1, std::min<int64_t>((int64_t)std::max(1, per_sm) * nsm, cdiv(items, HB_PAIR_WARPS)));
    int rc = cuda_check(cudaMemsetAsync(A.counter, 0, sizeof(unsigned long long), st), "counter reset");
    if (rc) return rc;
    kp<<<(unsigned)grid, HB_PAIR_WARPS * 32, sm, st>>>(B);
    return cuda_check(cudaGetLastError(), "pair kernel");
}

template <int OP, bool TP1, bool SP1>
static int dispatch_nj(int nj, const PairArgs &A, cudaStream_t st)
{
    if constexpr (OP == 1) {
        // K: both orientations of a separated pair per evaluation (HB_K_DUAL=0: off).  A pair
        // whose other row lies outside the launch's rows (row chunks, row-parallel ranks) is
        // evaluated in the same canonical orientation with only the needed output's
        // accumulators, so the blocks stay independent of the row split.
        static const bool dual_on = !getenv("HB_K_DUAL") || atoi(getenv("HB_K_DUAL")) != 0;
        if (dual_on) {
            if (nj == 1) return launch_pairs<OP, TP1, SP1, 1, true>(A, st);
            return launch_pairs<OP, TP1, SP1, 2, true>(A, st);
        }
    }
    if (nj == 1) return launch_pairs<OP, TP1, SP1, 1>(A, st);
    return launch_pairs<OP, TP1, SP1, 2>(A, st);
}

static int run_pairs(const hb_assembly_desc *a, int nj, const PairArgs &A, cudaStream_t st)
{
    if (a->op == 0 && !a->test_p1) return dispatch_nj<0, false, false>(nj, A, st);
    if (a->op == 0 && a->test_p1) return dispatch_nj<0, true, true>(nj, A, st);
    if (a->op == 1) return dispatch_nj<1, false, true>(nj, A, st);
    return dispatch_nj<2, true, true>(nj, A, st);
}

}  // namespace direct

// one 32-gap window [d0, d1) of test rows [e0, e1): pair kernel into the staging Q
// the global direct window [w0, w1) holding block d: [0, 32), then 30 blocks
// each ([32, 62), [62, 92), ...), clipped at E_t -- 32 gaps each
void direct_window(int64_t E_t, int64_t d, int &w0, int &w1)
{
    w0 = d < 32 ? 0 : 32 + 30 * (int)((d - 32) / 30);
    w1 = (int)std::min<int64_t>(E_t, w0 == 0 ? 32 : w0 + 30);
}

int direct_pairs(const hb_mesh_desc *m, const hb_assembly_desc *a, int64_t e0, int64_t e1, int d0, int d1,
                 double *Q, unsigned long long *counter, cudaStream_t st)
{
    using namespace direct;
    PairArgs A{};
    A.m = *m;
    A.step = a->step;
    A.alpha = a->alpha;
    A.d_eps = a->d_eps;
    A.r_eps = a->r_eps;
    A.inv2a = 1.0 / (2.0 * a->alpha);
    A.inv2a2 = 1.0 / (2.0 * a->alpha * a->alpha);
    A.inva = 1.0 / a->alpha;
    A.kconst = (a->op == 0) ? 1.0 / sqrt(kPi * a->alpha * a->alpha * a->alpha) : 1.0 / sqrt(kPi * a->alpha);
    A.halve_diag = (a->test_p1 && a->trial_p1) ? 1 : 0;
    A.Q = Q;
    A.counter = counter;
    A.e0 = e0;
    A.e1 = e1;
    // gaps of the whole global window holding [d0, d1) (direct_window(): [0, 32),
    // [32, 62), [62, 92), ...), whatever part of it the call stores: which
    // evaluations share a warp -- and so every value -- does not depend on the
    // call's d-range (the all-series vote of hb_special.cuh eval_unf)
    int w0, w1;
    direct_window(a->E_t, d0, w0, w1);
    if (d1 > w1) return HB_ERR_INVALID;
    A.d0 = d0;
    A.d1 = d1;
    A.nd = d1 - d0;
    A.it_lo = std::max(1, w0 - 1);
    A.it_hi = w1;
    A.need_special = d0 <= 1;
    const int nj = std::min(choose_nj(a), (int)cdiv(A.it_hi - A.it_lo + 1, 16));
    return run_pairs(a, std::max(1, nj), A, st);
}

}  // namespace hb
