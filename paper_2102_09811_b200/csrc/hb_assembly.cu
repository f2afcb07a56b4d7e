// hb_assembly.cu -- block-Toeplitz assembly of V, V11, K and D2 on sm_100a.
//
// Replaces heatbem/assembly.py:178-242 (_assemble_operator) together with the
// jitted _toeplitz_pass / _scatter_add of heatbem/_assembly_numba.py:111-285.
//
// The reference evaluates every element-pair integral once per time gap
// delta = i_t h (i_t = 0..E_t, "E_t + 1 passes") and combines the passes into
// blocks B^d = -L(d-1) + 2 L(d) - L(d+1), B^0 = Lcomb(0) - L(1)
// (AssemblyPlan.targets, assembly.py:72-89).  Here ONE launch covers all gaps:
//
//   * a warp owns one element pair; its 32 lanes are (s, t) = (lane>>4, lane&15):
//     t selects time gaps i_t = it_lo + t + 16 j (j < NJ, NJ slots per lane),
//     s splits the quadrature points by parity.  The per-pair geometry
//     (rho, 1/rho, hat weights ...) of 32 quadrature points is computed once by
//     the 32 lanes, parked in shared memory and read back as broadcasts, so
//     every lane spends its time in the erf/exp chains of its own gaps --
//     warp-uniform control flow for every pair class, no divergence;
//   * the delta = 0 gap (closed-form limits, no erf) is summed lane-parallel
//     over the points and butterfly-reduced;
//   * the 3-term time combination is applied in shared memory and each block
//     value B^d of the pair is written with lanes over d (coalesced) into a
//     staging row Q[pair][ij][d];
//   * operator-specific finalize kernels turn staging rows into blocks:
//     p0xp0 mirror-transpose (V), node-star gathers for p1 columns (K) and
//     rows+columns (D2, V11, then X + X^T).
//
// Regular (separated) pairs and touching pairs run in separate kernels
// (k_regular / k_singular); the regular kernel classifies near/far on the fly
// with the reference's exact IEEE operation order
// (sqrt((dx*dx + dy*dy) + dz*dz) < 2 max(diam), _assembly_numba.py:218-223)
// using explicitly rounded intrinsics, so the rule choice is bit-identical.
//
// Every per-(pair, gap) sum is taken in an order that depends only on the
// pair and the gap -- never on E_t, the d-window or the row chunk -- so block
// d is bitwise identical however the work is split (1 GPU vs d-sharded ranks,
// E_t = 4 vs E_t = 2 with the same step: the reference's Toeplitz-reuse test).
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

struct PairArgs {
    hb_mesh_desc m;
    double step, alpha, d_eps, r_eps;
    double inv2a, inv2a2, inva, kconst;
    int64_t e0, e1;
    int d0, d1, it_lo, it_hi, need_special, nd;
    int halve_diag;
    double *Q;
    unsigned long long *counter;   // work-item counter (zeroed per launch)
    int debug_class;               // 0 all pairs; 1 / 2 touching / separated only (HB_DEBUG_CLASS)
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
        const int p = q / nq1, r = q - p * nq1;
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
                        const double f = special::eval<OP + 4>(x, ix, tab, kFull);
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
                        const double f = special::eval<OP + 4>(x, ix, tab, kFull);
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
                        special::eval_nf<OP + 4, G>(
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
                    const double f = special::eval<OP + 4>(x, ix, tab, mask);
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
    if (A.need_special) {
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1)
#pragma unroll
            for (int i = 0; i < NIJ; ++i) {
                s0[i] += __shfl_xor_sync(kFull, s0[i], o);
                if (OP != 2) sc[i] += __shfl_xor_sync(kFull, sc[i], o);
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
    if (lane == 0 && A.need_special) {
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
                    special::eval_nf<5, G>(xs, [&](int gg) { return __dmul_rn(a[gg], icj); }, fs, tab, kFull);
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
                    const double f = special::eval<5>(x, ix, tab, mask);
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
    if (A.need_special) {
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1)
#pragma unroll
            for (int i = 0; i < 3; ++i) {
                if (DF) {
                    s0f[i] += __shfl_xor_sync(kFull, s0f[i], o);
                    scf[i] += __shfl_xor_sync(kFull, scf[i], o);
                }
                if (DR) {
                    s0r[i] += __shfl_xor_sync(kFull, s0r[i], o);
                    scr[i] += __shfl_xor_sync(kFull, scr[i], o);
                }
            }
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
    if (lane == 0 && A.need_special) {
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            if (DF) {
                Lf[3 * SLOTS + i] = jac * s0f[i];
                Lf[3 * SLOTS + 3 + i] = jac * scf[i];
            }
            if (DR) {
                Lr[3 * SLOTS + i] = jac * s0r[i];
                Lr[3 * SLOTS + 3 + i] = jac * scr[i];
            }
        }
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

// class codes: 0 far, 1 near, 2 identical, 3 common edge, 4 common vertex
__global__ void k_pair_classes(const hb_mesh_desc M, int64_t e0, int64_t e1, int8_t *out)
{
    const int64_t n = (e1 - e0) * M.E_x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t e = e0 + i / M.E_x, f = i % M.E_x;
        const int64_t tp = touching_pos(M, __ldg(M.tn_indptr_dev + e), __ldg(M.tn_indptr_dev + e + 1), f);
        if (tp >= 0) {
            out[i] = (int8_t)(2 + __ldg(M.tn_case_dev + tp));
        } else {
            double ce[3];
            for (int c = 0; c < 3; ++c) ce[c] = __ldg(M.centroids_dev + 3 * e + c);
            out[i] = near_test(M, ce, __ldg(M.diameters_dev + e), f) ? 1 : 0;
        }
    }
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
    double ce[3];
    for (int c = 0; c < 3; ++c) ce[c] = __ldg(M.centroids_dev + 3 * e + c);
    const double de = __ldg(M.diameters_dev + e);

    for (int64_t f = fb; f < fe; ++f) {
        // touching pairs belong to the singular path
        if (touching_pos(M, t_lo, t_hi, f) >= 0) continue;
        const int64_t slot = (e - A.e0) * M.E_x + f;
        const double jac = pair_jac<OP>(A, e, f);
        if (OP == 2 && jac == 0.0) continue;   // n_x.n_y == 0: no contribution (finalize skips it)
        const bool near = near_test(M, ce, de, f);
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
    for (int64_t f = fb; f < fe; ++f) {
        const bool f_in = f >= A.e0 && f < A.e1;
        if (f < e && f_in) continue;                           // the canonical pair (f, e) belongs to row f
        if (touching_pos(M, t_lo, t_hi, f) >= 0) continue;     // touching pairs: singular path (f == e too)
        const int64_t a = f > e ? e : f, b = f > e ? f : e;
        const int64_t slot_f = (a >= A.e0 && a < A.e1) ? (a - A.e0) * M.E_x + b : -1;   // test a, trial b
        const int64_t slot_r = (b >= A.e0 && b < A.e1) ? (b - A.e0) * M.E_x + a : -1;   // test b, trial a
        double ca[3];
        for (int c = 0; c < 3; ++c) ca[c] = __ldg(M.centroids_dev + 3 * a + c);
        const bool near = near_test(M, ca, __ldg(M.diameters_dev + a), b);
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
    special::load_table<OP + 4>(tab);   // factor-free kinds (hb_special.cuh)
    __syncthreads();
    constexpr int kPerWarp = DUAL ? dual_smem_doubles_per_warp<NJ>() : smem_doubles_per_warp<OP, NIJ, NJ>();
    static_assert(special::kTabDoubles % 2 == 0 && kPerWarp % 2 == 0 && Layout<OP, NIJ>::PAY % 2 == 0 &&
                      kDualPay % 2 == 0, "payload slots must stay 16-byte aligned (LDS.128)");
    double *geo = smem + special::kTabDoubles + warp * kPerWarp;
    double *Ls = geo + 32 * Layout<OP, NIJ>::PAY;
    double *Ls_dual = geo + 32 * kDualPay;
    const hb_mesh_desc &M = A.m;
    const int64_t s_lo = __ldg(M.sing_rowptr_dev + A.e0), s_hi = __ldg(M.sing_rowptr_dev + A.e1);
    int64_t n_sing = s_hi - s_lo;
    const int64_t nseg = cdiv(M.E_x, (int64_t)A.seg_len);
    int64_t n_reg = (A.e1 - A.e0) * nseg;
    if (A.debug_class == 1) n_reg = 0;      // study hook: touching pairs only
    if (A.debug_class == 2) n_sing = 0;     // study hook: separated pairs only
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
// finalize kernels
// ---------------------------------------------------------------------------
struct FinArgs {
    const double *Q;
    double *out;          // blocks_dev, block (d - d_begin) at out + (d - d_begin) R C
    double *const *bptr;  // optional per-block destinations (row-parallel: the d-owner's memory)
    int64_t E_x, N_x, R, C, e0, e1;
    int d0, nd, d_begin;
    const int64_t *star_indptr, *star_elem, *star_local, *tri_nodes;
    const double *normals;
    int skip_zero_dot;    // D2: pairs with n_e . n_f == 0 were not staged
    int star_max;
    const int64_t *tile_eptr, *tile_elem;   // curl tile plan (32-node tiles)
    const int32_t *star_pos;
};

// destination of block d - d_begin = b: the caller's per-block pointer (another
// GPU's memory over NVLink in a row-parallel run) or the contiguous blocks
__device__ __forceinline__ double *fin_block(const FinArgs &F, int64_t b)
{
    return F.bptr ? F.bptr[b] : F.out + b * F.R * F.C;
}

// V (p0 x p0, symmetric): tile of 4 rows x 32 columns x 32 blocks through smem;
// direct rows coalesced over f, mirror rows in 32-byte runs over e.
__global__ void __launch_bounds__(256) k_fin_p0p0(const FinArgs F)
{
    __shared__ double tile[4][32][33];
    const int64_t f0 = (int64_t)blockIdx.x * 32, eb = F.e0 + (int64_t)blockIdx.y * 4;
    if (f0 + 31 < eb) return;   // tile entirely below the diagonal: nothing staged
    const int tid = threadIdx.x;
    for (int dc = 0; dc < F.nd; dc += 32) {
        const int ndc = min(32, F.nd - dc);
        for (int idx = tid; idx < 4 * 32 * 32; idx += 256) {
            const int el = idx >> 10, fl = (idx >> 5) & 31, dl = idx & 31;
            const int64_t e = eb + el, f = f0 + fl;
            if (e < F.e1 && f < F.E_x && f >= e && dl < ndc)
                tile[el][fl][dl] = F.Q[((e - F.e0) * F.E_x + f) * F.nd + dc + dl];
        }
        __syncthreads();
        for (int idx = tid; idx < 4 * 32 * 32; idx += 256) {
            const int el = idx >> 10, dl = (idx >> 5) & 31, fl = idx & 31;
            const int64_t e = eb + el, f = f0 + fl;
            if (e < F.e1 && f < F.E_x && f >= e && dl < ndc) {
                const int64_t b = F.d0 + dc + dl - F.d_begin;
                fin_block(F, b)[e * F.C + f] = tile[el][fl][dl];
            }
        }
        for (int idx = tid; idx < 4 * 32 * 32; idx += 256) {
            const int fl = idx >> 7, dl = (idx >> 2) & 31, el = idx & 3;
            const int64_t e = eb + el, f = f0 + fl;
            if (e < F.e1 && f < F.E_x && f > e && dl < ndc) {
                const int64_t b = F.d0 + dc + dl - F.d_begin;
                fin_block(F, b)[f * F.C + e] = tile[el][fl][dl];
            }
        }
        __syncthreads();
    }
}

// K (p0 test x p1 trial): out[d][e][n] = sum_{(f,j) in star(n), f ascending} Q[e,f][j][d]
__global__ void __launch_bounds__(256) k_fin_p0p1(const FinArgs F)
{
    __shared__ double tile[32][33];
    const int64_t n0 = (int64_t)blockIdx.y * 32, e = F.e0 + blockIdx.x;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const double *Qe = F.Q + (e - F.e0) * F.E_x * 3 * F.nd;
    for (int dc = 0; dc < F.nd; dc += 32) {
        const int ndc = min(32, F.nd - dc);
        for (int nl = warp; nl < 32; nl += kWarps) {
            const int64_t n = n0 + nl;
            double acc = 0.0;
            if (n < F.N_x && lane < ndc) {
                const int64_t s0 = __ldg(F.star_indptr + n), s1 = __ldg(F.star_indptr + n + 1);
                for (int64_t s = s0; s < s1; ++s) {
                    const int64_t f = __ldg(F.star_elem + s), j = __ldg(F.star_local + s);
                    acc += Qe[(f * 3 + j) * F.nd + dc + lane];
                }
            }
            tile[nl][lane] = acc;
        }
        __syncthreads();
        for (int dl = warp; dl < ndc; dl += kWarps) {
            const int64_t n = n0 + lane;
            if (n < F.N_x) {
                const int64_t b = F.d0 + dc + dl - F.d_begin;
                fin_block(F, b)[e * F.C + n] = tile[lane][dl];
            }
        }
        __syncthreads();
    }
}

// D2 / V11 (p1 x p1): X[d][m][n] += sum_{(e,i) in star(m), e in chunk}
//                                   sum_{(f,j) in star(n), f >= e} Q[e,f][3i+j][d]
// CTA = (owner of node m, 32-node column tile), warp per column node n, lane
// per block d.  Which (e,f) were staged (f >= e, and n_e . n_f != 0 for D2)
// is decided once per CTA as a bitmask over the column tile's element list
// (the mesh's curl tile plan); the star product loop is then a bit test and
// a predicated load -- unstaged pairs add +0.0, which leaves the sum as is.
constexpr int kFinMaxW = 8;   // bitmask words per star entry (tile lists <= 256 elements)

__global__ void __launch_bounds__(256) k_fin_p1p1_accum(const FinArgs F)
{
    __shared__ double tile[32][33];
    extern __shared__ __align__(16) double fsm[];
    // CTA x = (element of the chunk, local node): node m is handled by the
    // CTA of the first chunk element in its (element-sorted) star only
    const int64_t n0 = (int64_t)blockIdx.y * 32, eo = F.e0 + blockIdx.x / 3;
    const int64_t m = __ldg(F.tri_nodes + 3 * eo + blockIdx.x % 3);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t sm0 = __ldg(F.star_indptr + m), sm1 = __ldg(F.star_indptr + m + 1);
    int64_t first = -1;
    for (int64_t a = sm0; a < sm1 && first < 0; ++a) {
        const int64_t e = __ldg(F.star_elem + a);
        if (e >= F.e0) first = e;
    }
    if (first != eo) return;
    const int smax = F.star_max;
    int64_t *sQ = (int64_t *)fsm;                          // [star_max] Q offset of (e - e0, 3i)
    int64_t *sE = sQ + smax;                               // [star_max] e
    int64_t *wFJ = sE + smax;                              // [kWarps][star_max] (9f + j) nd of node n's star
    unsigned *okm = (unsigned *)(wFJ + kWarps * smax);     // [star_max][kFinMaxW]
    int *wP = (int *)(okm + smax * kFinMaxW);              // [kWarps][star_max] tile position of f
    __shared__ int na_s;
    if (threadIdx.x == 0) {
        int na = 0;
        for (int64_t a = sm0; a < sm1; ++a) {
            const int64_t e = __ldg(F.star_elem + a);
            if (e < F.e0 || e >= F.e1) continue;
            sE[na] = e;
            sQ[na] = (e - F.e0) * F.E_x * 9 * (int64_t)F.nd + 3 * __ldg(F.star_local + a) * F.nd;
            ++na;
        }
        na_s = na;
    }
    __syncthreads();
    const int na = na_s;
    const int64_t tB0 = F.tile_eptr[blockIdx.y], tB = F.tile_eptr[blockIdx.y + 1] - tB0;
    {   // staged-pair bitmask: warp w owns word w (tile positions 32w..32w+31)
        const int p = 32 * warp + lane;
        int64_t f = -1;
        double nf[3] = {0.0, 0.0, 0.0};
        if (p < tB) {
            f = F.tile_elem[tB0 + p];
            for (int c = 0; c < 3; ++c) nf[c] = __ldg(F.normals + 3 * f + c);
        }
        for (int a = 0; a < na; ++a) {
            const int64_t e = sE[a];
            bool ok = p < tB && f >= e;
            if (F.skip_zero_dot) {
                const double ne[3] = {__ldg(F.normals + 3 * e), __ldg(F.normals + 3 * e + 1),
                                      __ldg(F.normals + 3 * e + 2)};
                ok = ok && exact_dot3(ne, nf) != 0.0;
            }
            const unsigned word = __ballot_sync(kFull, ok);
            if (lane == 0) okm[a * kFinMaxW + warp] = word;
        }
    }
    __syncthreads();
    const bool dok = lane < F.nd;
    int64_t *myFJ = wFJ + warp * smax;
    int *myP = wP + warp * smax;
    for (int dc = 0; dc < F.nd; dc += 32) {
        const int ndc = min(32, F.nd - dc);
        // stage X[d][m][n0..n0+31] (coalesced over n), add this chunk's
        // elements one at a time in ascending e, write back: the sequence of
        // additions is X = ((0 + s_e1) + s_e2) + ... whatever the row chunking
        for (int dl = warp; dl < ndc; dl += kWarps) {
            const int64_t n = n0 + lane;
            const int64_t b = F.d0 + dc + dl - F.d_begin;
            tile[lane][dl] = n < F.N_x ? F.out[(b * F.R + m) * F.C + n] : 0.0;
        }
        __syncthreads();
        const bool lok = dok && lane < ndc;
        for (int nl = warp; nl < 32; nl += kWarps) {
            const int64_t n = n0 + nl;
            if (n >= F.N_x) break;
            const int sn0 = (int)__ldg(F.star_indptr + n), nb = (int)__ldg(F.star_indptr + n + 1) - sn0;
            for (int b = lane; b < nb; b += 32) {
                myFJ[b] = (9 * __ldg(F.star_elem + sn0 + b) + __ldg(F.star_local + sn0 + b)) * F.nd;
                myP[b] = F.star_pos[sn0 + b];
            }
            __syncwarp();
            double x = tile[nl][lane];
            // stars of <= 32 entries: lanes test the staged bit of entry b (lane b), a ballot
            // gives the staged entries and only those are loaded (ascending b, as before;
            // the skipped +0.0 additions were exact identities).  Longer stars: the full loop.
            const int pb = lane < nb ? myP[lane] : 0;
            for (int a = 0; a < na; ++a) {
                const double *Qe = F.Q + sQ[a] + dc + lane;
                const unsigned *om = okm + a * kFinMaxW;
                double se = 0.0;
                if (nb <= 32) {
                    unsigned mask = __ballot_sync(kFull, lane < nb && ((om[pb >> 5] >> (pb & 31)) & 1u));
                    while (mask) {   // four staged entries per round: their loads are in flight together
                        int b[4];
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            b[u] = mask ? __ffs(mask) - 1 : -1;
                            mask &= mask - 1;
                        }
                        double qv[4];
#pragma unroll
                        for (int u = 0; u < 4; ++u) qv[u] = (lok && b[u] >= 0) ? Qe[myFJ[b[u] < 0 ? 0 : b[u]]] : 0.0;
#pragma unroll
                        for (int u = 0; u < 4; ++u)
                            if (b[u] >= 0) se += qv[u];
                    }
                } else {
#pragma unroll 4
                    for (int b = 0; b < nb; ++b) {
                        const int p = myP[b];
                        const bool ok = lok && ((om[p >> 5] >> (p & 31)) & 1u);
                        const double q = ok ? Qe[myFJ[b]] : 0.0;
                        se += q;
                    }
                }
                x += se;
            }
            tile[nl][lane] = x;
            __syncwarp();
        }
        __syncthreads();
        for (int dl = warp; dl < ndc; dl += kWarps) {
            const int64_t n = n0 + lane;
            if (n < F.N_x) {
                const int64_t b = F.d0 + dc + dl - F.d_begin;
                F.out[(b * F.R + m) * F.C + n] = tile[lane][dl];
            }
        }
        __syncthreads();
    }
}

// in-place X <- X + X^T on square blocks, 32x32 tile pairs (upper tile grid)
__global__ void __launch_bounds__(256) k_symmetrize(double *out, int64_t N, int64_t b_lo)
{
    __shared__ double A[32][33], B[32][33];
    const int64_t ntile = cdiv(N, 32);
    const int64_t tb = blockIdx.x;   // linear index into upper-triangular tile pairs
    // decode (ti <= tj) from tb
    int64_t ti = 0, rem = tb;
    while (rem >= ntile - ti) { rem -= ntile - ti; ++ti; }
    const int64_t tj = ti + rem;
    double *X = out + (b_lo + blockIdx.y) * N * N;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    for (int r = ty; r < 32; r += 8) {
        const int64_t i = ti * 32 + r, j = tj * 32 + tx;
        A[r][tx] = (i < N && j < N) ? X[i * N + j] : 0.0;
        const int64_t i2 = tj * 32 + r, j2 = ti * 32 + tx;
        B[r][tx] = (i2 < N && j2 < N) ? X[i2 * N + j2] : 0.0;
    }
    __syncthreads();
    for (int r = ty; r < 32; r += 8) {
        const int64_t i = ti * 32 + r, j = tj * 32 + tx;
        if (i < N && j < N) X[i * N + j] = A[r][tx] + B[tx][r];
        const int64_t i2 = tj * 32 + r, j2 = ti * 32 + tx;
        if (ti != tj && i2 < N && j2 < N) X[i2 * N + j2] = B[r][tx] + A[tx][r];
    }
}

// ---------------------------------------------------------------------------
// host orchestration
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

static bool combo_ok(const hb_assembly_desc *a)
{
    if (a->op == HB_OP_SINGLE_LAYER)
        return a->symmetric && a->test_p1 == a->trial_p1;
    if (a->op == HB_OP_DOUBLE_LAYER) return !a->symmetric && !a->test_p1 && a->trial_p1;
    if (a->op == HB_OP_HYPERSINGULAR2) return a->symmetric && a->test_p1 && a->trial_p1;
    return false;
}

constexpr size_t kCounterBytes = 256;

static size_t row_bytes(const hb_mesh_desc *m, const hb_assembly_desc *a)
{
    const int nj = choose_nj(a);
    const int64_t W = std::min<int64_t>(16 * nj, a->d_end - a->d_begin);
    return (size_t)m->E_x * op_shape(a).NIJ * W * sizeof(double);
}

template <int OP, bool TP1, bool SP1, int NJ, bool DUAL = false>
static int launch_pairs(const PairArgs &A, cudaStream_t st)
{
    constexpr int NIJ = (TP1 ? 3 : 1) * (SP1 ? 3 : 1);
    constexpr bool SYM = (OP != 1);
    constexpr int per_warp = DUAL ? dual_smem_doubles_per_warp<NJ>() : smem_doubles_per_warp<OP, NIJ, NJ>();
    const size_t sm = ((size_t)HB_PAIR_WARPS * per_warp + special::kTabDoubles) * sizeof(double);
    auto kp = k_pairs<OP, TP1, SP1, NJ, SYM, DUAL>;
    if (sm > 48 * 1024) cudaFuncSetAttribute(kp, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    int dev = 0, nsm = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kp, HB_PAIR_WARPS * 32, sm);
    const int64_t rows = A.e1 - A.e0;
    // separated-pair items of 32 trial elements, or shorter when few test rows
    // (a row-parallel rank) would leave fewer than 4 items per resident warp
    PairArgs B = A;
    const int64_t warps = (int64_t)std::max(1, per_sm) * nsm * HB_PAIR_WARPS;
    B.seg_len = 32;
    while (B.seg_len > 4 && rows * cdiv(A.m.E_x, (int64_t)B.seg_len) < 4 * warps) B.seg_len /= 2;
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

}  // namespace hb

using namespace hb;

extern "C" size_t hb_assemble_min_workspace(const hb_mesh_desc *m, const hb_assembly_desc *a)
{
    if (!m || !a) return 0;
    return row_bytes(m, a) + kCounterBytes;
}

extern "C" size_t hb_assemble_full_workspace(const hb_mesh_desc *m, const hb_assembly_desc *a)
{
    if (!m || !a) return 0;
    return row_bytes(m, a) * (size_t)m->E_x + kCounterBytes;
}

namespace hb {
// brackets launches with events when stats are requested
struct LaunchTimer {
    hb_assembly_stats *st;
    cudaStream_t s;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> pair_ev, fin_ev;
    int64_t launches = 0, pair_launches = 0;
    cudaEvent_t begin(cudaStream_t s_)
    {
        if (!st) return nullptr;
        cudaEvent_t e;
        cudaEventCreate(&e);
        cudaEventRecord(e, s_);
        return e;
    }
    void end(cudaEvent_t b, bool is_pair, cudaStream_t s_)
    {
        if (!st) return;
        cudaEvent_t e;
        cudaEventCreate(&e);
        cudaEventRecord(e, s_);
        (is_pair ? pair_ev : fin_ev).emplace_back(b, e);
    }
    int finish()
    {
        if (!st) return HB_OK;
        int rc = cuda_check(cudaStreamSynchronize(s), "stats sync");
        for (auto &pr : pair_ev) { float ms = 0; cudaEventElapsedTime(&ms, pr.first, pr.second); st->pair_ms += ms; }
        for (auto &pr : fin_ev) { float ms = 0; cudaEventElapsedTime(&ms, pr.first, pr.second); st->finalize_ms += ms; }
        for (auto *v : {&pair_ev, &fin_ev})
            for (auto &pr : *v) { cudaEventDestroy(pr.first); cudaEventDestroy(pr.second); }
        st->launches += launches;
        st->pair_launches += pair_launches;
        return rc;
    }
};
}  // namespace hb

extern "C" int hb_assemble(const hb_mesh_desc *m, const hb_assembly_desc *a, void *stream)
{
    if (!m || !a) { set_error("hb_assemble: null descriptor"); return HB_ERR_INVALID; }
    if (!combo_ok(a)) {
        set_error("hb_assemble: unsupported op/space combination (op=%d test_p1=%d trial_p1=%d sym=%d)",
                  a->op, a->test_p1, a->trial_p1, a->symmetric);
        return HB_ERR_UNSUPPORTED;
    }
    if (a->E_t < 1 || a->d_begin < 0 || a->d_end > a->E_t || a->d_begin >= a->d_end || m->E_x < 1 ||
        m->N_x < 3 || !(a->step > 0) || !(a->alpha > 0)) {
        set_error("hb_assemble: invalid sizes or parameters (E_t=%lld d=[%lld,%lld) E_x=%lld)",
                  (long long)a->E_t, (long long)a->d_begin, (long long)a->d_end, (long long)m->E_x);
        return HB_ERR_INVALID;
    }
    const int64_t r0 = a->row_end > a->row_begin ? a->row_begin : 0;
    const int64_t r1 = a->row_end > a->row_begin ? a->row_end : m->E_x;
    if (r0 < 0 || r1 > m->E_x || r0 >= r1 || (a->test_p1 && a->trial_p1 && a->block_ptrs_dev)) {
        set_error("hb_assemble: bad test-row range [%lld, %lld) (p1 x p1 operators accumulate over rows: "
                  "contiguous blocks only; a row range gives those rows' partial sum)", (long long)r0,
                  (long long)r1);
        return HB_ERR_INVALID;
    }
    if (!a->blocks_dev && !a->block_ptrs_dev) {
        set_error("hb_assemble: no output (blocks_dev and block_ptrs_dev are NULL)");
        return HB_ERR_INVALID;
    }
    if (a->test_p1 && a->trial_p1 &&
        (!m->curl_tile_eptr_dev || !m->curl_tile_elem_dev || !m->curl_star_pos_dev ||
         m->curl_tile_emax > 32 * kFinMaxW)) {
        set_error("hb_assemble: p1 x p1 needs the mesh tile plan with <= %d elements per 32-node tile", 32 * kFinMaxW);
        return HB_ERR_UNSUPPORTED;
    }
    cudaStream_t st = (cudaStream_t)stream;
    const int nj = choose_nj(a);
    const int W = 16 * nj;
    const size_t rb = row_bytes(m, a);
    if (!a->workspace_dev || a->workspace_bytes < rb + kCounterBytes) {
        set_error("hb_assemble: workspace %zu bytes < one row chunk (%zu bytes)", a->workspace_bytes, rb);
        return HB_ERR_WORKSPACE;
    }
    const size_t q_bytes = (a->workspace_bytes - kCounterBytes) & ~(size_t)255;
    const int64_t rows_per_chunk = std::max<int64_t>(1, std::min<int64_t>(m->E_x, (int64_t)(q_bytes / rb)));
    const int64_t R = a->test_p1 ? m->N_x : m->E_x, C = a->trial_p1 ? m->N_x : m->E_x;
    const int64_t nb = a->d_end - a->d_begin;
    const bool p1p1 = a->test_p1 && a->trial_p1;
    if (p1p1) {
        int rc = cuda_check(cudaMemsetAsync(a->blocks_dev, 0, (size_t)nb * R * C * sizeof(double), st), "memset");
        if (rc) return rc;
    }

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
    A.halve_diag = p1p1 ? 1 : 0;
#ifdef HB_DIAGNOSTICS   // timing study only: restrict the pair classes (results incomplete)
    if (const char *dc = getenv("HB_DEBUG_CLASS")) A.debug_class = atoi(dc);
#endif
    A.Q = (double *)a->workspace_dev;
    A.counter = (unsigned long long *)((char *)a->workspace_dev + q_bytes);

    LaunchTimer LT{a->stats, st};
    if (p1p1) LT.launches += 0;   // memset is not a kernel
    int64_t d0 = a->d_begin;
    while (d0 < a->d_end) {
        // slots i_t in [max(1, d0-1), d1] must fit the W lanes-x-slots of a warp
        const int64_t d1 = std::min<int64_t>(a->d_end, (d0 <= 1) ? (int64_t)W : d0 + W - 2);
        A.d0 = (int)d0;
        A.d1 = (int)d1;
        A.nd = (int)(d1 - d0);
        A.it_lo = (int)std::max<int64_t>(1, d0 - 1);
        A.it_hi = (int)d1;
        A.need_special = d0 <= 1;
        // a short (tail) window needs only the lanes-x-slots its gaps occupy
        const int nj_w = std::min(nj, (int)cdiv(A.it_hi - A.it_lo + 1, 16));
        for (int64_t e0 = r0; e0 < r1; e0 += rows_per_chunk) {
            const int64_t e1 = std::min(r1, e0 + rows_per_chunk);
            A.e0 = e0;
            A.e1 = e1;
            cudaEvent_t ev = LT.begin(st);
            int rc = run_pairs(a, nj_w, A, st);
            if (rc) return rc;
            LT.end(ev, true, st);
            LT.launches += 1;
            LT.pair_launches += 1;
            ev = LT.begin(st);
            FinArgs F{};
            F.Q = A.Q;
            F.out = a->blocks_dev;
            F.bptr = a->block_ptrs_dev;
            F.E_x = m->E_x; F.N_x = m->N_x; F.R = R; F.C = C; F.e0 = e0; F.e1 = e1;
            F.d0 = (int)d0; F.nd = A.nd; F.d_begin = (int)a->d_begin;
            F.star_indptr = m->star_indptr_dev; F.star_elem = m->star_elem_dev;
            F.star_local = m->star_local_dev; F.tri_nodes = m->tri_nodes_dev;
            F.normals = m->normals_dev; F.skip_zero_dot = a->op == HB_OP_HYPERSINGULAR2;
            F.star_max = (int)m->star_max;
            F.tile_eptr = m->curl_tile_eptr_dev; F.tile_elem = m->curl_tile_elem_dev; F.star_pos = m->curl_star_pos_dev;
            if (!a->test_p1 && !a->trial_p1) {
                dim3 g((unsigned)cdiv(m->E_x, 32), (unsigned)cdiv(e1 - e0, 4));
                k_fin_p0p0<<<g, 256, 0, st>>>(F);
            } else if (!a->test_p1) {
                dim3 g((unsigned)(e1 - e0), (unsigned)cdiv(m->N_x, 32));
                k_fin_p0p1<<<g, 256, 0, st>>>(F);
            } else {
                dim3 g((unsigned)(3 * (e1 - e0)), (unsigned)cdiv(m->N_x, 32));
                const size_t fsm = (size_t)m->star_max * ((2 + kWarps) * sizeof(int64_t) + kFinMaxW * sizeof(unsigned) +
                                                          kWarps * sizeof(int));
                k_fin_p1p1_accum<<<g, 256, fsm, st>>>(F);
            }
            rc = cuda_check(cudaGetLastError(), "finalize");
            if (rc) return rc;
            LT.end(ev, false, st);
            LT.launches += 1;
        }
        if (p1p1) {
            const int64_t nt = cdiv(R, 32);
            dim3 g((unsigned)(nt * (nt + 1) / 2), (unsigned)(d1 - d0));
            cudaEvent_t ev = LT.begin(st);
            k_symmetrize<<<g, 256, 0, st>>>(a->blocks_dev, R, d0 - a->d_begin);
            int rc = cuda_check(cudaGetLastError(), "symmetrize");
            if (rc) return rc;
            LT.end(ev, false, st);
            LT.launches += 1;
        }
        d0 = d1;
    }
    return LT.finish();
}

extern "C" int hb_pair_classes(const hb_mesh_desc *m, int64_t e0, int64_t e1, int8_t *out_dev, void *stream)
{
    if (!m || e0 < 0 || e1 > m->E_x || e0 >= e1 || !out_dev) {
        set_error("hb_pair_classes: bad arguments");
        return HB_ERR_INVALID;
    }
    const int64_t n = (e1 - e0) * m->E_x;
    k_pair_classes<<<(unsigned)std::min<int64_t>(cdiv(n, 256), 148 * 32), 256, 0, (cudaStream_t)stream>>>(*m, e0, e1,
                                                                                                        out_dev);
    return cuda_check(cudaGetLastError(), "hb_pair_classes");
}

#ifdef HB_COUNT_BRANCHES
// diagnostics build only: warp-level branch mix of the pair kernels' eval_n calls
extern "C" int hb_debug_branch_counts(unsigned long long *out4, int reset)
{
    cudaMemcpyFromSymbol(out4, hb::special::g_branch_count, 4 * sizeof(unsigned long long));
    if (reset) {
        unsigned long long z[4] = {0, 0, 0, 0};
        cudaMemcpyToSymbol(hb::special::g_branch_count, z, sizeof(z));
    }
    return cuda_check(cudaGetLastError(), "hb_debug_branch_counts");
}
#endif
