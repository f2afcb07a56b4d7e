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
#include "hb_moment_coeffs.h"
#include "hb_special.cuh"

#ifndef HB_PAIR_MINB
#define HB_PAIR_MINB 2
#endif
#ifndef HB_PAIR_WARPS   // warps per CTA of the pair kernels
#define HB_PAIR_WARPS 8
#endif
#ifndef HB_P1P1_MINB
#define HB_P1P1_MINB HB_PAIR_MINB
#endif
#ifndef HB_FUSE1
#define HB_FUSE1 1   // p0 x p0 touching / near pairs: moments and per-point gaps in one payload pass
#endif
#ifndef HB_QGROUP
#define HB_QGROUP 2   // quadrature points of the same parity per evaluation group (independent chains)
#endif

namespace hb {

// one factor-free kernel value on the lane-local uniform pieces (hb_special.cuh eval_ulocal)
template <int KIND>
__device__ __forceinline__ double eval_one(double x, double ix, const double *__restrict__ utab)
{
    double r[1];
    const double xs[1] = {x};
    special::eval_ulocal<KIND, 1>(xs, [&](int) { return ix; }, r, utab);
    return r[0];
}


struct PairArgs {
    hb_mesh_desc m;
    double step, alpha, d_eps, r_eps;
    double inv2a, inv2a2, inva, kconst;
    double inv_u2;                 // 1 / u^2 = 1 / (4 alpha h): rho~^2 = rho^2 / u^2
    double mom_S, mom_q0;          // moment form: L(i) = jac S sum_k a_k M_k i^(q0 - k)
    int64_t e0, e1;
    int d0, d1, need_special, nd;   // blocks [d0, d1) of this launch, nd = d1 - d0
    int moments;                    // 1: moment form for the blocks d >= dmom of a pair; 0: all gaps per point
    const double *Tm;              // moment table [kNK][nd] + term thresholds (k_moment_table)
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

constexpr int kPwDoubles = 32 * 17;   // per-warp moment scratch: DMMA fragments (12 rows of stride 36), then the moments Ms

template <int OP, int NIJ, int NJ>
__host__ __device__ constexpr int smem_doubles_per_warp_base()
{
    return 32 * Layout<OP, NIJ>::PAY + LsLayout<NIJ, NJ>::SIZE + kPwDoubles;
}

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
// per-point gap window of a pair: gaps it_lo..it_hi feed the blocks
// [w0, w1) (it_lo = max(1, w0 - 1), it_hi = w1, <= 32 gap slots)
// ---------------------------------------------------------------------------
struct Win {
    int w0, w1, it_lo, it_hi;
};

// a lane's NJ gap slots sl = t + 16 j of window W: cx = 1/(2 sqrt(a delta))
// (x = rho cx), ic = 1/cx, kk (rho <= r_eps limits), sc (per-gap factor of
// the factor-free kinds: V = (x H) ic / (2a^2), K = (F/x) (-rn/(2a)) cx,
// D2 = (erf/x) cx).  Slots past it_hi are clamped (finite values, never stored).
template <int OP, int NJ>
struct Slots {
    double cx[NJ], ic[NJ], kk[NJ], sc[NJ];
    __device__ __forceinline__ void init(const PairArgs &A, const Win &W, int t)
    {
#pragma unroll
        for (int j = 0; j < NJ; ++j) {
            int it = W.it_lo + t + 16 * j;
            if (it > W.it_hi) it = W.it_hi;
            const double delta = (double)it * A.step;
            ic[j] = 2.0 * sqrt(A.alpha * delta);
            cx[j] = 1.0 / ic[j];
            kk[j] = (OP == 2) ? 1.0 / sqrt(kPi * A.alpha * delta) : sqrt(delta) * A.kconst;
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
// Moment form.  At gaps where every quadrature point of a pair has
// t = x^2 <= kTM, the factor-free kernel value is a power series in
// t = rho~^2 / i (rho~ = rho / u, u = 2 sqrt(alpha h), gap i = delta / h):
//   L(i) = jac S sum_k a_k M_k i^(q0 - k),   M_k = sum_p W_p rho~_p^(2k)
//   B^d  = jac sum_k M_k Tm_k(d),            Tm_k(d) = S a_k D2[i^(q0 - k)](d)
// with the pair's gap-independent moments M_k and the time second
// difference D2[g](d) = -g(d-1) + 2 g(d) - g(d+1) of the powers taken in
// closed form.  The reference's B^d = -L(d-1) + 2 L(d) - L(d+1) cancels like
// 1/(4 d^2) and amplifies the rounding of every L; here the rounding errors of
// the moments do not depend on d and are not amplified.
// V: S = u / (2 a^2), q0 = 1/2 (x H); K: S = 1/u, q0 = -1/2 (F/x);
// D2: S = 1/u, q0 = -1/2 (erf/x).  Coefficients: hb_moment_coeffs.h.
// A pair's moment gap istar = ceil(max_p rho~_p^2 / kTM) follows from its own
// points; blocks d >= max(2, istar + 1) come from the moments, blocks below
// from L(i) evaluated point by point (gaps <= istar + 1).  The split and
// the per-point lane layout depend on the pair only -- never on the launch's
// d range, the row chunk or the rank -- so every block entry is bitwise
// independent of how the work is cut.  Terms beyond the t-dependent count of
// kMom*Thr are below 2^-56 of the leading one.
// ---------------------------------------------------------------------------
constexpr int kNK = moments::kNK;    // 32: lane k of a warp owns moment k
static_assert(kPwDoubles >= 9 * kNK, "moment scratch holds the moments of nine weights");
static_assert(kNK == 32, "one moment per lane");

template <int OP>
__device__ __forceinline__ double mom_coef(int k)
{
    return OP == 0 ? moments::kMomV[k] : OP == 1 ? moments::kMomK[k] : moments::kMomE[k];
}

template <int OP>
__device__ __forceinline__ double mom_thr(int k)
{
    return OP == 0 ? moments::kMomVThr[k] : OP == 1 ? moments::kMomKThr[k] : moments::kMomEThr[k];
}

// D2[i^q](d) = -(d-1)^q + 2 d^q - (d+1)^q = -2 d^q (expm1(m) cosh(dl) + 2 sinh^2(dl/2)),
// m = (q/2) log1p(-1/d^2), dl = q atanh(1/d): no cancellation beyond a factor ~2
__device__ __forceinline__ double second_diff_pow(double d, double q)
{
    const double r = 1.0 / d;
    const double m = 0.5 * q * log1p(-r * r);
    const double dl = q * atanh(r);
    const double sh = sinh(0.5 * dl);
    return -2.0 * pow(d, q) * (expm1(m) * cosh(dl) + 2.0 * sh * sh);
}

// moment table of a launch: Tm[k][dd] = S a_k D2[i^(q0-k)](d0 + dd) for d >= 2
// (0 below), then the kNK + 1 term-count thresholds
template <int OP>
__global__ void k_moment_table(double *Tm, int d0, int nd, double S, double q0)
{
    const int n = kNK * nd;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n + kNK + 1; i += gridDim.x * blockDim.x) {
        if (i < n) {
            const int k = i / nd, dd = i - k * nd, d = d0 + dd;
            Tm[i] = d >= 2 ? (S * mom_coef<OP>(k)) * second_diff_pow((double)d, q0 - k) : 0.0;
        } else {
            Tm[i] = mom_thr<OP>(i - n);
        }
    }
}

__device__ __forceinline__ void dmma884(double &d0, double &d1, double a, double b);

// One weight per point (p0 x p0): the 32 moments of a chunk as ONE rank-32
// product on the FP64 tensor cores.  With k = 8 n + g,
//   M_k = sum_p r_p^g (W_p r_p^(8 n))  =  (A B)[g][n],
// A[g][p] = r_p^g (g < 8), B[p][n] = W_p r_p^(8 n) (n < 4; columns 4-7 zero):
// lane p forms its point's 8 + 4 values with 11 multiplications (instead of 32
// powers and 32 stores), eight m8n8k4 DMMAs (4 points each) accumulate into the
// C fragment cf (lane (g, t): columns 2t, 2t + 1) across the pair's chunks.
// Scratch Pw: A rows at stride 36 (conflict-free stores, 2-wavefront fragment
// loads), then the four B rows.  Padding points (all-zero payload, r = 0)
// contribute exact zeros.
constexpr int kMmStride = 36;
static_assert(12 * kMmStride <= kPwDoubles, "DMMA moment scratch must fit the per-warp moment scratch");

template <int PAY, int WOFF>
__device__ __forceinline__ void chunk_moments_mma(const double *geo, double *Pw, double r, double (&cf)[2], int lane)
{
    const double W = geo[lane * PAY + WOFF];
    const double r2 = __dmul_rn(r, r), r3 = __dmul_rn(r2, r), r4 = __dmul_rn(r2, r2);
    const double r5 = __dmul_rn(r4, r), r6 = __dmul_rn(r4, r2), r7 = __dmul_rn(r4, r3), r8 = __dmul_rn(r4, r4);
    const double w8 = __dmul_rn(W, r8), r16 = __dmul_rn(r8, r8), w16 = __dmul_rn(W, r16), w24 = __dmul_rn(w16, r8);
    double *Ar = Pw + lane, *Br = Pw + 8 * kMmStride + lane;
    Ar[0] = 1.0;
    Ar[kMmStride] = r;
    Ar[2 * kMmStride] = r2;
    Ar[3 * kMmStride] = r3;
    Ar[4 * kMmStride] = r4;
    Ar[5 * kMmStride] = r5;
    Ar[6 * kMmStride] = r6;
    Ar[7 * kMmStride] = r7;
    Br[0] = W;
    Br[kMmStride] = w8;
    Br[2 * kMmStride] = w16;
    Br[3 * kMmStride] = w24;
    __syncwarp();
    const int g = lane >> 2, t = lane & 3;
    const double *af = Pw + g * kMmStride + t, *bf = Pw + (8 + (g & 3)) * kMmStride + t;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        const double a = af[4 * q];
        const double b = g < 4 ? bf[4 * q] : 0.0;
        dmma884(cf[0], cf[1], a, b);
    }
    __syncwarp();
}

// park the DMMA moments in Pw as Ms[k], k = 8 n + g (lane (g, t): n = 2t, 2t + 1 < 4)
__device__ __forceinline__ void store_moments_mma(const double (&cf)[2], double *Pw, int lane)
{
    const int g = lane >> 2, t = lane & 3;
    __syncwarp();
    if (t < 2) {
        Pw[8 * (2 * t) + g] = cf[0];
        Pw[8 * (2 * t + 1) + g] = cf[1];
    }
    __syncwarp();
}

// NW weights per point (p0 x p1, p1 x p1, K's two orientations): the same
// product with B[p][(i, n)] = W_i(p) r_p^(8 n), column c = 4 i + n, in
// ceil(4 NW / 8) column tiles; the B element is formed in registers from the
// payload weight and the staged power r_p^(8 n) (rows 8..11 of the scratch).
template <int NW>
__host__ __device__ constexpr int mom_tiles() { return (4 * NW + 7) / 8; }

template <int PAY, int WOFF, int NW>
__device__ __forceinline__ void chunk_moments_mma_n(const double *geo, double *Pw, double r,
                                                    double (&cf)[mom_tiles<NW>()][2], int lane)
{
    constexpr int NT = mom_tiles<NW>();
    const double r2 = __dmul_rn(r, r), r3 = __dmul_rn(r2, r), r4 = __dmul_rn(r2, r2);
    const double r5 = __dmul_rn(r4, r), r6 = __dmul_rn(r4, r2), r7 = __dmul_rn(r4, r3), r8 = __dmul_rn(r4, r4);
    const double r16 = __dmul_rn(r8, r8), r24 = __dmul_rn(r16, r8);
    double *Ar = Pw + lane;
    Ar[0] = 1.0;
    Ar[kMmStride] = r;
    Ar[2 * kMmStride] = r2;
    Ar[3 * kMmStride] = r3;
    Ar[4 * kMmStride] = r4;
    Ar[5 * kMmStride] = r5;
    Ar[6 * kMmStride] = r6;
    Ar[7 * kMmStride] = r7;
    Ar[8 * kMmStride] = 1.0;
    Ar[9 * kMmStride] = r8;
    Ar[10 * kMmStride] = r16;
    Ar[11 * kMmStride] = r24;
    __syncwarp();
    const int g = lane >> 2, t = lane & 3;
    const double *af = Pw + g * kMmStride + t, *rf = Pw + (8 + (g & 3)) * kMmStride + t;
    const double *wf = geo + t * PAY + WOFF + (g >> 2);
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        const double a = af[4 * q], rb = rf[4 * q];
#pragma unroll
        for (int tau = 0; tau < NT; ++tau) {
            // column c = 8 tau + g = 4 i + n: weight i = 2 tau + (g >> 2), power n = g & 3
            const bool live = 2 * tau + (g >> 2) < NW;
            const double b = live ? __dmul_rn(wf[4 * q * PAY + 2 * tau], rb) : 0.0;
            dmma884(cf[tau][0], cf[tau][1], a, b);
        }
    }
    __syncwarp();
}

// park them in Pw as Ms[i][k], k = 8 n + g (lane (g, t): columns 8 tau + 2t, + 1)
template <int NW>
__device__ __forceinline__ void store_moments_mma_n(const double (&cf)[mom_tiles<NW>()][2], double *Pw, int lane)
{
    const int g = lane >> 2, t = lane & 3;
    __syncwarp();
#pragma unroll
    for (int tau = 0; tau < mom_tiles<NW>(); ++tau)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int c = 8 * tau + 2 * t + h, i = c >> 2, n = c & 3;
            if (i < NW) Pw[i * kNK + 8 * n + g] = cf[tau][h];
        }
    __syncwarp();
}

// blocks [dmom, d1) of the launch from the moments Ms, lanes over d; the
// series is cut at the lane's own term count (t = rmax / (d - 1))
template <int NIJ>
__device__ __forceinline__ void combine_moments(const PairArgs &A, int64_t slot, int lane, const double *Ms,
                                                double jac, int dmom, double rmax)
{
    double *dst = A.Q + slot * (int64_t)(NIJ * A.nd);
    const double *thr = A.Tm + kNK * A.nd;
    for (int dd0 = max(dmom, A.d0) - A.d0; dd0 < A.nd; dd0 += 32) {
        const int dd = dd0 + lane;
        const bool an = dd < A.nd;
        int nk = 0;
        if (an) {   // smallest term count whose threshold covers t (thresholds ascending, thr[kNK] = kTM)
            const double t = rmax / (double)(A.d0 + dd - 1);
            int lo = 1, hi = kNK;
            while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                if (t <= __ldg(thr + mid)) hi = mid;
                else lo = mid + 1;
            }
            nk = lo;
        }
        const int nkw = __reduce_max_sync(kFull, nk);
        double b[NIJ];
#pragma unroll
        for (int i = 0; i < NIJ; ++i) b[i] = 0.0;
        const double *tm = A.Tm + (an ? dd : 0);
        for (int k = 0; k < nkw; ++k) {
            const double tk = __ldg(tm + k * A.nd);
            if (k < nk) {
#pragma unroll
                for (int i = 0; i < NIJ; ++i) b[i] = fma(Ms[i * kNK + k], tk, b[i]);
            }
        }
        if (an) {
#pragma unroll
            for (int i = 0; i < NIJ; ++i) dst[i * A.nd + dd] = jac * b[i];
        }
    }
}

// blocks [W.w0, W.w1) by the 3-term combination of the staged L row of the
// window (Ls: [NIJ][SLOTS], then L0[NIJ], Lcomb0[NIJ]), lanes over d
template <int NIJ, int SLOTS>
__device__ __forceinline__ void combine_window(const PairArgs &A, const Win &W, const double *Ls, int64_t slot,
                                               int lane)
{
    const double *L0 = Ls + NIJ * SLOTS, *Lc = L0 + NIJ;
    double *dst = A.Q + slot * (int64_t)(NIJ * A.nd);
    for (int d = W.w0 + lane; d < W.w1; d += 32) {
        const int dd = d - A.d0;
#pragma unroll
        for (int i = 0; i < NIJ; ++i) {
            const double *Li = Ls + i * SLOTS;
            double b;
            if (d == 0) {
                const double l1 = Li[1 - W.it_lo];
                b = Lc[i] + (-l1);
            } else {
                const double lm = (d - 1 == 0) ? L0[i] : Li[d - 1 - W.it_lo];
                const double lc = Li[d - W.it_lo];
                const double lp = Li[d + 1 - W.it_lo];
                b = -lm + 2.0 * lc;
                b = b + (-lp);
            }
            dst[i * A.nd + dd] = b;
        }
    }
}

// pair's moment gap from its largest rho~^2 (warp-uniform)
__device__ __forceinline__ int moment_istar(double rmax)
{
    const double is = ceil(rmax / moments::kTM);
    return is < 1.0 ? 1 : (is > 1e9 ? 1000000000 : (int)is);
}

// lanes per point group of the per-point evaluation: the pair's per-point
// gaps are 1..istar+1, so GW = 4 / 8 lanes cover them with 8 / 4 point
// groups; larger istar use 16 lanes x NJ slots (2 point groups)
__device__ __forceinline__ int pair_gw(int istar) { return istar + 1 <= 4 ? 4 : (istar + 1 <= 8 ? 8 : 16); }

// ---------------------------------------------------------------------------
// per-point evaluation of one chunk of nloc points for the lane's nje gap
// slots; gw lanes per point group, npg = 32 / gw point groups (lane's group
// pg = lane / gw takes points pg, pg + npg, ...; with G points per step).
// gw and nje are warp-uniform runtime values (one code copy for all layouts).
// ---------------------------------------------------------------------------
template <int OP, int NIJ, int PAY, int HOFF, int NJ>
__device__ __forceinline__ void eval_points(const PairArgs &A, const Slots<OP, NJ> &T, const double *geo, int nloc,
                                            bool any_small, int pg, int npg, int nje, double (&acc)[NJ][NIJ],
                                            const double *tab)
{
    const int NPG = npg;
    if (!any_small) {
        // G points of one group per step (x close -> the small/large-x
        // skipping survives; G independent Horner chains); uniform trip count
        // for all groups (padding slots hold the all-zero payload), so the
        // branch votes span the full warp
        constexpr int G = HB_QGROUP;
        const int STEP = NPG * G;   // divides 32: the padded loop stays inside the warp's 32 payload slots
        const int nlocg = (nloc + STEP - 1) / STEP * STEP;
        constexpr bool SEL = NIJ == 9;   // p1 x p1 keeps the explicit select: measured faster there
        for (int k = pg; k < nlocg; k += STEP) {
            double pv[G][PAY];
            double rho[G], a[G], b[G];
            bool ok[G];
#pragma unroll
            for (int g = 0; g < G; ++g) {
                ok[g] = !SEL || k + NPG * g < nloc;
                load_payload<PAY>(geo + (ok[g] ? k + NPG * g : 0) * PAY, pv[g]);
                rho[g] = pv[g][0];
                a[g] = pv[g][1];
                b[g] = (OP == 2) ? 0.0 : pv[g][2];
            }
#pragma unroll
            for (int j = 0; j < NJ; ++j) {
                if (j >= nje) break;
                double xs[G], fs[G];
#pragma unroll
                for (int g = 0; g < G; ++g) xs[g] = __dmul_rn(rho[g], T.cx[j]);
                const double icj = T.ic[j];
                special::eval_ulocal<OP + 4, G>(
                    xs, [&](int g) { return __dmul_rn(OP == 0 ? b[g] : a[g], icj); }, fs, tab);
#pragma unroll
                for (int g = 0; g < G; ++g) {
                    const double v = ok[g] ? fs[g] : 0.0;
#pragma unroll
                    for (int i = 0; i < NIJ; ++i) acc[j][i] = fma(v, pv[g][HOFF + i], acc[j][i]);
                }
            }
        }
    } else {
        for (int k = pg; k < nloc; k += NPG) {
            const double *p = geo + k * PAY;
            const double rho = p[0], s1 = p[1];
            const double s2 = (OP == 2) ? 0.0 : p[2];
            const bool sm = rho <= A.r_eps;
#pragma unroll
            for (int j = 0; j < NJ; ++j) {
                if (j >= nje) break;
                const double x = __dmul_rn(rho, T.cx[j]);
                const double ix = __dmul_rn(OP == 0 ? s2 : s1, T.ic[j]);
                const double f = eval_one<OP + 4>(x, ix, tab);
                // rho <= r_eps limits, divided by the per-gap factor applied at the end
                double val;
                if (OP == 0) val = sm ? 2.0 * T.kk[j] / T.sc[j] : f;
                else if (OP == 1) val = sm ? 0.0 : f;
                else val = sm ? T.kk[j] / T.sc[j] : f;
#pragma unroll
                for (int i = 0; i < NIJ; ++i) acc[j][i] = fma(val, p[HOFF + i], acc[j][i]);
            }
        }
    }
}

// sum the point groups (butterfly over the lane bits >= log2(gw); every lane
// ends with the same bits) and stage L for the window slots of gaps < gend
template <int OP, int NIJ, int NJ, int SLOTS>
__device__ __forceinline__ void stage_L(const Win &W, const Slots<OP, NJ> &T, double (&acc)[NJ][NIJ], double jac,
                                        int gend, int gw, int nje, double *Ls, int lane)
{
    for (int o = 16; o >= gw; o >>= 1)
#pragma unroll
        for (int j = 0; j < NJ; ++j) {
            if (j >= nje) break;
#pragma unroll
            for (int i = 0; i < NIJ; ++i) acc[j][i] += __shfl_xor_sync(kFull, acc[j][i], o);
        }
    const int t = lane & (gw - 1), nslots = W.it_hi - W.it_lo + 1;
    if (lane < gw) {
#pragma unroll
        for (int j = 0; j < NJ; ++j) {
            const int sl = t + 16 * j;
            if (j < nje && sl < nslots && W.it_lo + sl < gend) {
#pragma unroll
                for (int i = 0; i < NIJ; ++i) Ls[i * SLOTS + sl] = jac * (acc[j][i] * T.sc[j]);
            }
        }
    }
}

// ---------------------------------------------------------------------------
// payload of quadrature point q (lane's slot): rho, per-op scalars, weights;
// returns rho~^2 and the small / nonzero-weight flags; SPECIAL adds the
// delta = 0 sums (closed-form limits) of the point
// ---------------------------------------------------------------------------
template <int OP, bool TP1, bool SP1, class Geom>
__device__ __forceinline__ void point_payload(const PairArgs &A, const Geom &g, int q, int nq, const double ny[3],
                                              bool SPECIAL, double *p, double &rt2, int &small, int &nzw,
                                              double (&s0)[(TP1 ? 3 : 1) * (SP1 ? 3 : 1)],
                                              double (&sc)[(TP1 ? 3 : 1) * (SP1 ? 3 : 1)])
{
    constexpr int NT = TP1 ? 3 : 1, NS = SP1 ? 3 : 1, NIJ = NT * NS;
    using L = Layout<OP, NIJ>;
    constexpr int PAY = L::PAY, HOFF = L::HOFF;
    small = 0;
    nzw = OP == 1 ? 0 : 1;   // K: this point's weights are not all zero (r.n_y != 0)
    rt2 = 0.0;
    if (q >= nq) {
        // padding slot of the grouped loop: all zero (x = 0 and 1/x = 0 give
        // finite series values, the zero weights add exact zeros)
#pragma unroll
        for (int i = 0; i < PAY; ++i) p[i] = 0.0;
        return;
    }
    double x[3], y[3], wq, ht[3], hs[3];
    g.point(q, x, y, wq, ht, hs);
    const double rx = x[0] - y[0], ry = x[1] - y[1], rz = x[2] - y[2];
    const double r2 = rx * rx + ry * ry + rz * rz;
    const double rho = sqrt(r2);
    rt2 = r2 * A.inv_u2;
    small = rho <= A.r_eps;
    double H[NIJ];
#pragma unroll
    for (int i = 0; i < NT; ++i)
#pragma unroll
        for (int j = 0; j < NS; ++j)
            H[i * NS + j] = (TP1 || SP1) ? wq * ((TP1 ? ht[i] : 1.0) * (SP1 ? hs[j] : 1.0)) : wq;
    p[0] = rho;
    if (OP == 0) {
        const double iq = 1.0 / rho;
        const double Aq = rho * A.inv2a2, Bq = A.inva * iq;
        p[1] = Aq;
        p[2] = iq;
#pragma unroll
        for (int i = 0; i < NIJ; ++i) p[HOFF + i] = H[i];
        if (SPECIAL) {
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
        p[1] = iq;
        p[2] = iq;
#pragma unroll
        for (int i = 0; i < NIJ; ++i) p[HOFF + i] = (H[i] * Ur) * A.inv2a;
        if (SPECIAL) {
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
#pragma unroll
        for (int i = 0; i < NIJ; ++i) p[HOFF + i] = H[i];
        if (SPECIAL) {
#pragma unroll
            for (int i = 0; i < NIJ; ++i) s0[i] = fma(H[i], iq, s0[i]);
        }
    }
}

// per-point L of one window for one lane layout: gap slots [it_lo, gend)
// over all point chunks, staged into Ls
template <int OP, bool TP1, bool SP1, int NJ, class Geom>
__device__ __noinline__ void pair_points(const PairArgs &A, const Win &W, const Geom &g, int nq, const double ny[3],
                                         double jac, int gend, int gw, int nje, double *geo, double *Ls, int lane,
                                         const double *tab)
{
    constexpr int NIJ = (TP1 ? 3 : 1) * (SP1 ? 3 : 1);
    using L = Layout<OP, NIJ>;
    constexpr int PAY = L::PAY, HOFF = L::HOFF;
    constexpr int SLOTS = LsLayout<NIJ, NJ>::SLOTS;
    Slots<OP, NJ> T;
    T.init(A, W, lane & (gw - 1));
    const int pg = lane / gw, npg = 32 / gw;
    double acc[NJ][NIJ];
#pragma unroll
    for (int j = 0; j < NJ; ++j)
#pragma unroll
        for (int i = 0; i < NIJ; ++i) acc[j][i] = 0.0;
    double dummy[NIJ];
    for (int base = 0; base < nq; base += 32) {
        double rt2;
        int small, nzw;
        point_payload<OP, TP1, SP1>(A, g, base + lane, nq, ny, false, geo + lane * PAY, rt2, small, nzw, dummy, dummy);
        const bool any_small = __any_sync(kFull, small);
        const bool skip = OP == 1 && !__any_sync(kFull, nzw);   // all-zero K chunk: exact zeros
        __syncwarp();
        if (!skip) eval_points<OP, NIJ, PAY, HOFF, NJ>(A, T, geo, min(32, nq - base), any_small, pg, npg, nje, acc, tab);
        __syncwarp();
    }
    stage_L<OP, NIJ, NJ, SLOTS>(W, T, acc, jac, gend, gw, nje, Ls, lane);
}

// the per-point windows of a pair: blocks [d0, dend) in windows of <= 32 gap
// slots (the first from block 0 or 1 holds 32 blocks, later ones 30); per
// window the gaps up to istar + 1, then the 3-term combination
template <int NIJ, int SLOTS, class PointsFn>
__device__ __forceinline__ void per_point_windows(const PairArgs &A, int dend, int istar, double *Ls, int64_t slot,
                                                  int lane, const PointsFn &points)
{
    int w0 = A.d0;
    while (w0 < dend) {
        Win W;
        W.w0 = w0;
        W.w1 = min(dend, w0 <= 1 ? 32 : w0 + 30);
        W.it_lo = max(1, w0 - 1);
        W.it_hi = W.w1;
        const int npp = min(W.it_hi, istar + 1) - W.it_lo + 1;
        if (npp > 0) points(W, npp);
        __syncwarp();
        combine_window<NIJ, SLOTS>(A, W, Ls, slot, lane);
        __syncwarp();
        w0 = W.w1;
    }
}

// ---------------------------------------------------------------------------
// one element pair, all blocks [d0, d1) of the launch.  Phase 1: payload over
// all point chunks -> the pair's largest rho~^2 (hence istar), the delta = 0
// sums and (when the launch may hold moment blocks) the moments.  Phase 2:
// point-by-point L for the gaps below istar + 2, window by window (payload
// recomputed: same bits; the phases never hold their registers at the same
// time), 3-term blocks below dmom = max(2, istar + 1), moment blocks above.
// rt2_lo: a lower bound of the pair's rho~^2 (squared centroid distance).
// ---------------------------------------------------------------------------
template <int OP, bool TP1, bool SP1, int NJ, class Geom>
__device__ __noinline__ void eval_pair(const PairArgs &A, const Geom &g, int nq, const double ny[3],
                                          double jac, double rt2_lo, double rt2_hi, int64_t slot, double *geo,
                                          double *Ls, double *Pw, int lane, const double *tab)
{
    constexpr int NT = TP1 ? 3 : 1, NS = SP1 ? 3 : 1, NIJ = NT * NS;
    using L = Layout<OP, NIJ>;
    constexpr int PAY = L::PAY, HOFF = L::HOFF;
    constexpr int SLOTS = LsLayout<NIJ, NJ>::SLOTS;
    double *p_lane = geo + lane * PAY;
    double *L0 = Ls + NIJ * SLOTS, *Lc = L0 + NIJ;
    const bool try_mom = A.moments && A.d1 - 1 >= max(2, moment_istar(rt2_lo) + 1);

    // Single pass (p0 x p0, HB_FUSE1): with the moment split taken from the
    // vertex bound rt2_hi the per-point gaps are known before the payload pass,
    // so each point chunk feeds the moments AND the per-point gaps at once
    // (no second payload pass); taken when those gaps fit the first window.
    if constexpr (NIJ == 1 && HB_FUSE1) {
        const int istar_f = moment_istar(rt2_hi), dmom_f = max(2, istar_f + 1);
        if (try_mom && rt2_hi > 0.0 && A.d0 <= 1 && A.d1 > dmom_f && dmom_f <= 32) {
            Win W;
            W.w0 = A.d0;
            W.w1 = dmom_f;
            W.it_lo = max(1, A.d0 - 1);
            W.it_hi = W.w1;
            const int gw = pair_gw(istar_f);
            const int npp = min(W.it_hi, istar_f + 1) - W.it_lo + 1;
            const int nje = (gw == 16 && npp > 16) ? NJ : 1;
            Slots<OP, NJ> T;
            T.init(A, W, lane & (gw - 1));
            const int pg = lane / gw, npg = 32 / gw;
            double acc[NJ][NIJ], mom[1][2] = {{0.0, 0.0}}, s0[NIJ], sc[NIJ];   // mom: the DMMA C fragment
#pragma unroll
            for (int i = 0; i < NIJ; ++i) {
                s0[i] = sc[i] = 0.0;
#pragma unroll
                for (int j = 0; j < NJ; ++j) acc[j][i] = 0.0;
            }
            for (int base = 0; base < nq; base += 32) {
                double rt2;
                int small, nzw;
                point_payload<OP, TP1, SP1>(A, g, base + lane, nq, ny, A.need_special, p_lane, rt2, small, nzw, s0,
                                            sc);
                const bool any_small = __any_sync(kFull, small);
                __syncwarp();
                const int nloc = min(32, nq - base);
                chunk_moments_mma<PAY, HOFF>(geo, Pw, rt2, mom[0], lane);   // (NIJ == 1: mom[0] = the C fragment)
                __syncwarp();
                eval_points<OP, NIJ, PAY, HOFF, NJ>(A, T, geo, nloc, any_small, pg, npg, nje, acc, tab);
                __syncwarp();
            }
            if (A.need_special) {
#pragma unroll
                for (int o = 16; o >= 1; o >>= 1)
#pragma unroll
                    for (int i = 0; i < NIJ; ++i) {
                        s0[i] += __shfl_xor_sync(kFull, s0[i], o);
                        sc[i] += __shfl_xor_sync(kFull, sc[i], o);
                    }
                if (lane == 0) {
#pragma unroll
                    for (int i = 0; i < NIJ; ++i) {
                        L0[i] = jac * s0[i];
                        Lc[i] = jac * sc[i];
                    }
                }
            }
            store_moments_mma(mom[0], Pw, lane);
            stage_L<OP, NIJ, NJ, SLOTS>(W, T, acc, jac, istar_f + 2, gw, nje, Ls, lane);
            __syncwarp();
            combine_window<NIJ, SLOTS>(A, W, Ls, slot, lane);
            __syncwarp();
            // the bound: every term count the series cut needs is covered
            combine_moments<NIJ>(A, slot, lane, Pw, jac, dmom_f, rt2_hi);
            __syncwarp();
            return;
        }
    }

    // ---- phase 1 ----
    double rmax = 0.0;
    {
        double s0[NIJ], sc[NIJ], cf[2] = {0.0, 0.0}, cfn[mom_tiles<NIJ>()][2];   // DMMA C fragments of the moments
#pragma unroll
        for (int i = 0; i < NIJ; ++i) s0[i] = sc[i] = 0.0;
#pragma unroll
        for (int tau = 0; tau < mom_tiles<NIJ>(); ++tau) cfn[tau][0] = cfn[tau][1] = 0.0;
        for (int base = 0; base < nq; base += 32) {
            double rt2;
            int small, nzw;
            point_payload<OP, TP1, SP1>(A, g, base + lane, nq, ny, A.need_special, p_lane, rt2, small, nzw, s0, sc);
            rmax = fmax(rmax, rt2);
            const bool skip = OP == 1 && !__any_sync(kFull, nzw);   // all-zero K chunk: exact zeros
            __syncwarp();
            if (try_mom && !skip) {
                // p0 x p0: the same tensor-core moments as the single-pass path (same bits)
                if constexpr (NIJ == 1) chunk_moments_mma<PAY, HOFF>(geo, Pw, rt2, cf, lane);
                else chunk_moments_mma_n<PAY, HOFF, NIJ>(geo, Pw, rt2, cfn, lane);
            }
            __syncwarp();
        }
        if (A.need_special) {
#pragma unroll
            for (int o = 16; o >= 1; o >>= 1)
#pragma unroll
                for (int i = 0; i < NIJ; ++i) {
                    s0[i] += __shfl_xor_sync(kFull, s0[i], o);
                    if (OP != 2) sc[i] += __shfl_xor_sync(kFull, sc[i], o);
                }
            if (lane == 0) {
#pragma unroll
                for (int i = 0; i < NIJ; ++i) {
                    L0[i] = jac * s0[i];
                    Lc[i] = jac * (OP == 2 ? s0[i] : sc[i]);
                }
            }
        }
        if (try_mom) {
            if constexpr (NIJ == 1) store_moments_mma(cf, Pw, lane);
            else store_moments_mma_n<NIJ>(cfn, Pw, lane);
        }
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) rmax = fmax(rmax, __shfl_xor_sync(kFull, rmax, o));
    // p0 x p0 with the single-pass path: the split always comes from the vertex
    // bound, so the blocks do not depend on which path a launch takes
    if (NIJ == 1 && HB_FUSE1 && rt2_hi > 0.0) rmax = rt2_hi;
    // without the moment form every gap is evaluated point by point
    const int istar = A.moments ? moment_istar(rmax) : (1 << 29);
    const int dmom = max(2, istar + 1);
    const bool use_mom = try_mom && A.d1 > dmom;

    // ---- phase 2: per-point windows below dmom, moment blocks from dmom ----
    const int gend = istar + 2;
    const int gw = pair_gw(istar);
    per_point_windows<NIJ, SLOTS>(A, use_mom ? min(A.d1, dmom) : A.d1, istar, Ls, slot, lane,
                                  [&](const Win &W, int npp) {
        pair_points<OP, TP1, SP1, NJ>(A, W, g, nq, ny, jac, gend, gw, (gw == 16 && npp > 16) ? NJ : 1, geo, Ls, lane,
                                      tab);
    });
    if (use_mom) combine_moments<NIJ>(A, slot, lane, Pw, jac, dmom, rmax);
    __syncwarp();
}

// ---------------------------------------------------------------------------
// K (p0 test x p1 trial) for both orientations of one separated pair.
// The product rule of a separated pair (a, b) uses the same point pairs for
// K(a, b) and K(b, a): rho -- hence x and F(x) at every gap, and the powers
// of the moment form -- is shared, and only the per-point weights differ:
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
__host__ __device__ constexpr int dual_smem_doubles_per_warp_base() { return 32 * kDualPay + 2 * LsLayout<3, NJ>::SIZE + kPwDoubles; }

// payload of one point of the dual K pair (both orientations' weights);
// `special` adds the delta = 0 sums of both orientations
__device__ __forceinline__ void dual_payload(const PairArgs &A, const RegularGeom &g, int q, int nq, const double nb[3],
                                             const double na[3], bool special, double *p, double &rt2, int &small,
                                             int &nzw, double (&s0f)[3], double (&scf)[3], double (&s0r)[3],
                                             double (&scr)[3])
{
    small = 0;
    nzw = 0;
    rt2 = 0.0;
    if (q >= nq) {   // all-zero padding slot (see point_payload)
#pragma unroll
        for (int i = 0; i < kDualPay; ++i) p[i] = 0.0;
        return;
    }
    double x[3], y[3], wq, ht[3], hs[3];
    g.point(q, x, y, wq, ht, hs);
    const double rx = x[0] - y[0], ry = x[1] - y[1], rz = x[2] - y[2];
    const double r2 = rx * rx + ry * ry + rz * rz;
    const double rho = sqrt(r2);
    rt2 = r2 * A.inv_u2;
    small = rho <= A.r_eps;
    const double rnb = rx * nb[0] + ry * nb[1] + rz * nb[2];
    const double rna = (-rx) * na[0] + (-ry) * na[1] + (-rz) * na[2];   // reverse: r' = -r
    const double iq = 1.0 / rho;
    const double Vf = small ? 0.0 : -rnb, Vr = small ? 0.0 : -rna;   // rho U (factor-free F/x)
    nzw = Vf != 0.0 || Vr != 0.0;
    p[0] = rho;
    p[1] = iq;
    double Hf[3], Hr[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        Hf[i] = wq * (1.0 * hs[i]);
        Hr[i] = wq * (1.0 * ht[i]);
        p[2 + i] = (Hf[i] * Vf) * A.inv2a;
        p[5 + i] = (Hr[i] * Vr) * A.inv2a;
    }
    if (special) {
        const double Uf = small ? 0.0 : -rnb * iq, Ur = small ? 0.0 : -rna * iq;
        const double P = 1.0 / __dmul_rn(rho, rho);
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

// per-point L of one window of the dual pair (both orientations; stage_f /
// stage_r: which staged rows are needed), runtime lane layout gw / nje
template <int NJ>
__device__ __noinline__ void dual_points(const PairArgs &A, const Win &W, const RegularGeom &g, int nq,
                                         const double nb[3], const double na[3], double jac, int gend, int gw,
                                         int nje, bool stage_f, bool stage_r, double *geo, double *Lf, double *Lr,
                                         int lane, const double *tab)
{
    constexpr int PAY = kDualPay, SLOTS = LsLayout<3, NJ>::SLOTS;
    Slots<1, NJ> T;
    T.init(A, W, lane & (gw - 1));
    const int pg = lane / gw, NPG = 32 / gw;
    double af[NJ][3], ar[NJ][3];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < NJ; ++j) af[j][i] = ar[j][i] = 0.0;
    double d3[3];
    for (int base = 0; base < nq; base += 32) {
        double rt2;
        int small, nzw;
        dual_payload(A, g, base + lane, nq, nb, na, false, geo + lane * PAY, rt2, small, nzw, d3, d3, d3, d3);
        const bool any_small = __any_sync(kFull, small);
        const bool skip = !__any_sync(kFull, nzw);   // both orientations' weights all zero (coplanar pair)
        __syncwarp();
        const int nloc = min(32, nq - base);
        if (skip) {
        } else if (!any_small) {
            constexpr int G = HB_QGROUP;
            const int STEP = NPG * G;   // divides 32
            const int nlocg = (nloc + STEP - 1) / STEP * STEP;
            for (int k = pg; k < nlocg; k += STEP) {   // padding slots are all zero
                double pv[G][PAY];
                double rho[G], a[G];
#pragma unroll
                for (int gg = 0; gg < G; ++gg) {
                    load_payload<PAY>(geo + (k + NPG * gg) * PAY, pv[gg]);
                    rho[gg] = pv[gg][0];
                    a[gg] = pv[gg][1];
                }
#pragma unroll
                for (int j = 0; j < NJ; ++j) {
                    if (j >= nje) break;
                    double xs[G], fs[G];
#pragma unroll
                    for (int gg = 0; gg < G; ++gg) xs[gg] = __dmul_rn(rho[gg], T.cx[j]);
                    const double icj = T.ic[j];
                    special::eval_ulocal<5, G>(xs, [&](int gg) { return __dmul_rn(a[gg], icj); }, fs, tab);
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
            for (int k = pg; k < nloc; k += NPG) {
                const double *p = geo + k * PAY;
                const double rho = p[0], s1 = p[1];
                const bool sm = rho <= A.r_eps;
#pragma unroll
                for (int j = 0; j < NJ; ++j) {
                    if (j >= nje) break;
                    const double x = __dmul_rn(rho, T.cx[j]);
                    const double ix = __dmul_rn(s1, T.ic[j]);
                    const double f = eval_one<5>(x, ix, tab);
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
    if (stage_f) stage_L<1, 3, NJ, SLOTS>(W, T, af, jac, gend, gw, nje, Lf, lane);
    if (stage_r) stage_L<1, 3, NJ, SLOTS>(W, T, ar, jac, gend, gw, nje, Lr, lane);
}

// delta = 0 sums of the dual pair (L0 / Lc of both staged rows)
template <int NJ>
__device__ __forceinline__ void dual_specials_reduce(double (&s0f)[3], double (&scf)[3], double (&s0r)[3],
                                                     double (&scr)[3], double jac, double *Lf, double *Lr, int lane)
{
    constexpr int SLOTS = LsLayout<3, NJ>::SLOTS;
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1)
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            s0f[i] += __shfl_xor_sync(kFull, s0f[i], o);
            scf[i] += __shfl_xor_sync(kFull, scf[i], o);
            s0r[i] += __shfl_xor_sync(kFull, s0r[i], o);
            scr[i] += __shfl_xor_sync(kFull, scr[i], o);
        }
    if (lane == 0) {
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            Lf[3 * SLOTS + i] = jac * s0f[i];
            Lf[3 * SLOTS + 3 + i] = jac * scf[i];
            Lr[3 * SLOTS + i] = jac * s0r[i];
            Lr[3 * SLOTS + 3 + i] = jac * scr[i];
        }
    }
}

// blocks [d0, dend) of the dual pair from per-point L, window by window
template <int NJ>
__device__ __forceinline__ void dual_point_blocks(const PairArgs &A, const RegularGeom &g, int nq, const double nb[3],
                                                  const double na[3], double jac, int istar, int dend, int64_t slot_f,
                                                  int64_t slot_r, double *geo, double *Ls, int lane, const double *tab)
{
    constexpr int SLOTS = LsLayout<3, NJ>::SLOTS, LSZ = LsLayout<3, NJ>::SIZE;
    double *Lf = Ls, *Lr = Ls + LSZ;
    const int gend = istar + 2;
    const int gw = pair_gw(istar);
    int w0 = A.d0;
    while (w0 < dend) {
        Win W;
        W.w0 = w0;
        W.w1 = min(dend, w0 <= 1 ? 32 : w0 + 30);
        W.it_lo = max(1, w0 - 1);
        W.it_hi = W.w1;
        const int npp = min(W.it_hi, istar + 1) - W.it_lo + 1;
        if (npp > 0)
            dual_points<NJ>(A, W, g, nq, nb, na, jac, gend, gw, (gw == 16 && npp > 16) ? NJ : 1, slot_f >= 0,
                            slot_r >= 0, geo, Lf, Lr, lane, tab);
        __syncwarp();
        if (slot_f >= 0) combine_window<3, SLOTS>(A, W, Lf, slot_f, lane);
        if (slot_r >= 0) combine_window<3, SLOTS>(A, W, Lr, slot_r, lane);
        __syncwarp();
        w0 = W.w1;
    }
}

// One dual pair, warp per pair (near pairs): phase 1 (rmax, delta = 0 sums,
// moments rows 0..2 forward, 3..5 reverse), per-point blocks below dmom,
// moment blocks from dmom.  Both orientations are always evaluated (each
// output's arithmetic is the same whichever rows the launch holds); only the
// outputs with a slot (>= 0) are stored.
template <int NJ>
__device__ __noinline__ void eval_pair_dual(const PairArgs &A, const RegularGeom &g, int nq, const double nb[3],
                                            const double na[3], double jac, double rt2_lo, int64_t slot_f,
                                            int64_t slot_r, double *geo, double *Ls, double *Pw, int lane,
                                            const double *tab)
{
    constexpr int PAY = kDualPay, LSZ = LsLayout<3, NJ>::SIZE;
    double *p_lane = geo + lane * PAY;
    double *Lf = Ls, *Lr = Ls + LSZ;
    const bool try_mom = A.moments && A.d1 - 1 >= max(2, moment_istar(rt2_lo) + 1);
    double rmax = 0.0;
    {
        double cfn[mom_tiles<6>()][2], s0f[3], scf[3], s0r[3], scr[3];   // cfn: DMMA C fragments of the moments
#pragma unroll
        for (int i = 0; i < 3; ++i) s0f[i] = scf[i] = s0r[i] = scr[i] = 0.0;
#pragma unroll
        for (int tau = 0; tau < mom_tiles<6>(); ++tau) cfn[tau][0] = cfn[tau][1] = 0.0;
        for (int base = 0; base < nq; base += 32) {
            double rt2;
            int small, nzw;
            dual_payload(A, g, base + lane, nq, nb, na, A.need_special, p_lane, rt2, small, nzw, s0f, scf, s0r, scr);
            rmax = fmax(rmax, rt2);
            const bool skip = !__any_sync(kFull, nzw);
            __syncwarp();
            if (try_mom && !skip) chunk_moments_mma_n<PAY, 2, 6>(geo, Pw, rt2, cfn, lane);
            __syncwarp();
        }
        if (A.need_special) dual_specials_reduce<NJ>(s0f, scf, s0r, scr, jac, Lf, Lr, lane);
        if (try_mom) store_moments_mma_n<6>(cfn, Pw, lane);
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) rmax = fmax(rmax, __shfl_xor_sync(kFull, rmax, o));
    // without the moment form every gap is evaluated point by point
    const int istar = A.moments ? moment_istar(rmax) : (1 << 29);
    const int dmom = max(2, istar + 1);
    const bool use_mom = try_mom && A.d1 > dmom;
    dual_point_blocks<NJ>(A, g, nq, nb, na, jac, istar, use_mom ? min(A.d1, dmom) : A.d1, slot_f, slot_r, geo, Ls,
                          lane, tab);
    if (use_mom) {
        if (slot_f >= 0) combine_moments<3>(A, slot_f, lane, Pw, jac, dmom, rmax);
        if (slot_r >= 0) combine_moments<3>(A, slot_r, lane, Pw + 3 * kNK, jac, dmom, rmax);
    }
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

// lower bound of a separated pair's largest rho~^2: the symmetric triangle
// rules have the centroid as weighted mean, so by convexity the largest point
// distance is at least the centroid distance (1 - 1e-12 covers rounding)
// an upper bound of a pair's rho~^2 from its vertices (every quadrature point
// lies in its triangle): max over the 9 vertex pairs, rounded up by 1e-12 --
// a function of the pair alone, so a moment split taken from it is the same
// whatever the launch
__device__ __forceinline__ double rt2_upper(const PairArgs &A, int64_t e, int64_t f)
{
    const double *ve = A.m.verts_tri_dev + 9 * e, *vf = A.m.verts_tri_dev + 9 * f;
    double q = 0.0;
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) {
            double s = 0.0;
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                const double d = __ldg(ve + 3 * i + c) - __ldg(vf + 3 * j + c);
                s = fma(d, d, s);
            }
            q = fmax(q, s);
        }
    return q * A.inv_u2 * (1.0 + 1e-12);
}

__device__ __forceinline__ double rt2_lower(const PairArgs &A, int64_t e, int64_t f)
{
    double q = 0.0;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        const double d = __ldg(A.m.centroids_dev + 3 * e + c) - __ldg(A.m.centroids_dev + 3 * f + c);
        q = fma(d, d, q);
    }
    return q * A.inv_u2 * (1.0 - 1e-12);
}

// per-warp shared-memory areas of the pair kernels
struct WarpMem {
    double *geo, *Ls, *Pw;
    const double *rw, *rh;   // regular rule weights / hats (CTA copy, far batches)
};

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
// Far-pair batches (separated pairs on the regular product rule).  The
// moments of a batch are computed lane-parallel with FMA-dense register loops
// -- lane (pair ps, k-group g) runs over the pair's point pairs and owns the
// moments k in [KPL g, KPL g + KPL) -- instead of the warp-per-pair transposes
// through shared memory, and the moment blocks of the whole batch come from
// ONE small GEMM on the FP64 tensor cores,
//   B[d][n] = sum_k Tm[k][d] M[k][n],   n = output i * PB + pair ps,
// with mma.sync m8n8k4 f64 (8 k-steps of the 32 terms per 8 x 8 tile).  The
// blocks below a pair's dmom keep the warp-per-pair per-point path.  The
// moments of a far pair are always formed this way, so a block entry still
// depends on the pair only.
//   V (NW 1): KPL 16, PB 16      K dual (NW 6): KPL 4, PB 4
//   p1 x p1 (NW 9, separable hat weights): KPL 4, PB 4
// ---------------------------------------------------------------------------
template <int NW>
struct FarCfg;
template <>
struct FarCfg<1> {
    static constexpr int KPL = 16, PB = 16;
};
template <>
struct FarCfg<6> {
    static constexpr int KPL = 4, PB = 4;
};
template <>
struct FarCfg<9> {
    static constexpr int KPL = 4, PB = 4;
};
template <int NW>
__host__ __device__ constexpr int far_ntile() { return (NW * FarCfg<NW>::PB + 7) / 8; }
// row stride of Ms[k][n]: 8 ntile + 4 (= 4 or 12 mod 16: conflict-free B fragments)
template <int NW>
__host__ __device__ constexpr int far_nstr() { return 8 * far_ntile<NW>() + 4; }
template <int NW>
__host__ __device__ constexpr int far_smem_doubles() { return kNK * far_nstr<NW>() + 5 * FarCfg<NW>::PB; }

// per-pair data of a batch (shared memory, after Ms)
template <int NW>
struct FarPairs {
    double *jac, *rmax;
    int64_t *slot_f, *slot_r;
    int *dmom, *lane;   // first moment block; lane (segment position) of the pair
    __device__ FarPairs(double *base)
        : jac(base + kNK * far_nstr<NW>()), rmax(jac + FarCfg<NW>::PB),
          slot_f(reinterpret_cast<int64_t *>(rmax + FarCfg<NW>::PB)), slot_r(slot_f + FarCfg<NW>::PB),
          dmom(reinterpret_cast<int *>(slot_r + FarCfg<NW>::PB)), lane(dmom + FarCfg<NW>::PB) {}
};

// a far pair's points staged in shared memory (x: test element a, y: trial
// element b, 3 coordinates each) and the regular rule's weights and hats
// (CTA copy): plain shared-memory loads in the lane loops
struct FarGeom {
    const double *xp, *yp, *w, *hats;
    int nq1;
};
constexpr int kFarMaxRule = 7;    // far batches when the regular rule has <= 7 points
constexpr int kRuleDoubles = 4 * 16;

// copy the batch's point coordinates: lane (ps, g) copies entries g, g + LPP, ...
// of its pair into Xs[ps][0..6 nq1) (stride 6 nq1 + 1)
template <int LPP>
__device__ __forceinline__ void stage_far_points(const hb_mesh_desc &M, int64_t a, int64_t b, double *Xs, int g)
{
    const int n3 = 3 * (int)M.n_reg;
    const double *pa = M.reg_pts_dev + a * n3, *pb = M.reg_pts_dev + b * n3;
    for (int c = g; c < 2 * n3; c += LPP) Xs[c] = c < n3 ? __ldg(pa + c) : __ldg(pb + c - n3);
}

// t^(KPL g): the first power of the lane's k-group (KPL a power of two)
template <int KPL>
__device__ __forceinline__ double group_start_pow(double t, int g)
{
    double s = t;
#pragma unroll
    for (int q = 1; q < KPL; q <<= 1) s = __dmul_rn(s, s);   // t^KPL
    double p = 1.0;
#pragma unroll
    for (int b = 1; b < 32 / KPL; b <<= 1) {
        if (g & b) p = __dmul_rn(p, s);
        s = __dmul_rn(s, s);
    }
    return p;
}

__device__ __forceinline__ void dmma884(double &d0, double &d1, double a, double b)
{
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

// DMMA combine of a batch: blocks d in [dlo, d1) of all its pairs; entries
// below a pair's dmom are left to the per-point path
template <int NW, int NIJ>
__device__ __forceinline__ void far_combine(const PairArgs &A, const double *Ms, const FarPairs<NW> &P, int npairs,
                                            int dlo, int lane)
{
    constexpr int PB = FarCfg<NW>::PB, NT = far_ntile<NW>(), NSTR = far_nstr<NW>();
    const int gq = lane >> 2, tq = lane & 3;
    // per output column (2 per lane per tile): pair, output, dmom
    for (int dt = dlo; dt < A.d1; dt += 8) {
        const int d = dt + gq;
        double acc[NT][2];
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) acc[nt][0] = acc[nt][1] = 0.0;
        const bool drow = d < A.d1;
#pragma unroll
        for (int ks = 0; ks < kNK / 4; ++ks) {
            const double a = drow ? __ldg(A.Tm + (4 * ks + tq) * A.nd + (d - A.d0)) : 0.0;
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) dmma884(acc[nt][0], acc[nt][1], a, Ms[(4 * ks + tq) * NSTR + 8 * nt + gq]);
        }
        if (!drow) continue;
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int n = 8 * nt + 2 * tq + h;
                const int i = n / PB, ps = n - i * PB;
                if (i >= NW || ps >= npairs) continue;
                if (d < P.dmom[ps]) continue;
                int64_t slot;
                int io;
                if (NW == 6) {   // K dual: outputs 0..2 forward (slot_f), 3..5 reverse (slot_r)
                    slot = i < 3 ? P.slot_f[ps] : P.slot_r[ps];
                    io = i < 3 ? i : i - 3;
                } else {
                    slot = P.slot_f[ps];
                    io = i;
                }
                if (slot < 0) continue;
                A.Q[slot * (int64_t)(NIJ * A.nd) + io * A.nd + (d - A.d0)] = P.jac[ps] * acc[nt][h];
            }
    }
}

// moments of a V pair (p0 x p0) on the regular rule: lane (ps, g) = (lane >> 1, lane & 1)
__device__ __forceinline__ void far_moments_v(const PairArgs &A, const FarGeom &G, double (&mom)[16], double &rmax,
                                              int g)
{
    const double *xp = G.xp, *yp = G.yp, *w = G.w;
    const int nq1 = G.nq1;
    rmax = 0.0;
#pragma unroll
    for (int k = 0; k < 16; ++k) mom[k] = 0.0;
    for (int p = 0; p < nq1; ++p) {
        const double x0 = (xp + 3 * p)[0], x1 = (xp + 3 * p + 1)[0], x2 = (xp + 3 * p + 2)[0];
        const double wp = (w + p)[0];
#pragma unroll 2
        for (int r = 0; r < nq1; ++r) {
            const double rx = x0 - (yp + 3 * r)[0], ry = x1 - (yp + 3 * r + 1)[0], rz = x2 - (yp + 3 * r + 2)[0];
            const double t = (rx * rx + ry * ry + rz * rz) * A.inv_u2;
            rmax = fmax(rmax, t);
            const double W = wp * (w + r)[0];
            double pw = group_start_pow<16>(t, g);
#pragma unroll
            for (int k = 0; k < 16; ++k) {
                mom[k] = fma(W, pw, mom[k]);
                pw = __dmul_rn(pw, t);
            }
        }
    }
}

// moments of a K pair, both orientations (canonical a < b): lane (ps, g) = (lane >> 2, lane & 3)
__device__ __forceinline__ void far_moments_k(const PairArgs &A, const FarGeom &G, const double nb[3],
                                              const double na[3], double (&mom)[6][FarCfg<6>::KPL], int g)
{
    constexpr int KPL = FarCfg<6>::KPL;
#pragma unroll
    for (int i = 0; i < 6; ++i)
#pragma unroll
        for (int k = 0; k < KPL; ++k) mom[i][k] = 0.0;
    const int nq1 = G.nq1;
    for (int p = 0; p < nq1; ++p) {
        const double x0 = G.xp[3 * p], x1 = G.xp[3 * p + 1], x2 = G.xp[3 * p + 2];
        const double wp = G.w[p];
        double ht[3];
#pragma unroll
        for (int c = 0; c < 3; ++c) ht[c] = G.hats[3 * p + c];
        for (int r = 0; r < nq1; ++r) {
            const double rx = x0 - G.yp[3 * r], ry = x1 - G.yp[3 * r + 1], rz = x2 - G.yp[3 * r + 2];
            const double t = (rx * rx + ry * ry + rz * rz) * A.inv_u2;
            const double rnb = rx * nb[0] + ry * nb[1] + rz * nb[2];
            const double rna = (-rx) * na[0] + (-ry) * na[1] + (-rz) * na[2];
            const double wq = wp * G.w[r];
            double Wt[6];
#pragma unroll
            for (int i = 0; i < 3; ++i) {
                Wt[i] = ((wq * (1.0 * G.hats[3 * r + i])) * (-rnb)) * A.inv2a;
                Wt[3 + i] = ((wq * (1.0 * ht[i])) * (-rna)) * A.inv2a;
            }
            double pw = group_start_pow<KPL>(t, g);
#pragma unroll
            for (int k = 0; k < KPL; ++k) {
#pragma unroll
                for (int i = 0; i < 6; ++i) mom[i][k] = fma(Wt[i], pw, mom[i][k]);
                pw = __dmul_rn(pw, t);
            }
        }
    }
}

// moments of a p1 x p1 pair (separable hat weights (w_p ht_i(p)) (w_r hs_j(r))):
// lane (ps, g) = (lane >> 3, lane & 7)
__device__ __forceinline__ void far_moments_p1p1(const PairArgs &A, const FarGeom &G, double (&mom)[9][4],
                                                 double &rmax, int g)
{
    rmax = 0.0;
#pragma unroll
    for (int i = 0; i < 9; ++i)
#pragma unroll
        for (int k = 0; k < 4; ++k) mom[i][k] = 0.0;
    const int nq1 = G.nq1;
    for (int p = 0; p < nq1; ++p) {
        const double x0 = (G.xp + 3 * p)[0], x1 = (G.xp + 3 * p + 1)[0], x2 = (G.xp + 3 * p + 2)[0];
        const double wp = (G.w + p)[0];
        double N[3][4];
#pragma unroll
        for (int j = 0; j < 3; ++j)
#pragma unroll
            for (int k = 0; k < 4; ++k) N[j][k] = 0.0;
        for (int r = 0; r < nq1; ++r) {
            const double rx = x0 - (G.yp + 3 * r)[0], ry = x1 - (G.yp + 3 * r + 1)[0],
                         rz = x2 - (G.yp + 3 * r + 2)[0];
            const double t = (rx * rx + ry * ry + rz * rz) * A.inv_u2;
            rmax = fmax(rmax, t);
            const double wr = (G.w + r)[0];
            double b[3];
#pragma unroll
            for (int j = 0; j < 3; ++j) b[j] = wr * (G.hats + 3 * r + j)[0];
            double pw = group_start_pow<4>(t, g);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
#pragma unroll
                for (int j = 0; j < 3; ++j) N[j][k] = fma(b[j], pw, N[j][k]);
                pw = __dmul_rn(pw, t);
            }
        }
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            const double a = wp * (G.hats + 3 * p + i)[0];
#pragma unroll
            for (int j = 0; j < 3; ++j)
#pragma unroll
                for (int k = 0; k < 4; ++k) mom[3 * i + j][k] = fma(a, N[j][k], mom[3 * i + j][k]);
        }
    }
}

// ---------------------------------------------------------------------------
// Fused lane-level K far path.  For far pairs whose per-point gaps
// 1..istar+1 number at most 8 (the common case at moderate E_t), lane
// (ps, g) of the batch forms from the pair's point pairs the moments k in
// [4g, 4g + 4) of both orientations and the kernel value F/x at its gap
// g + 1 -- no per-pair warp-serial phase.  The blocks d < dmom follow from the 3-term combination of those L
// values, the blocks d >= dmom from the moments (DMMA combine).
// ---------------------------------------------------------------------------
constexpr int kFusedMaxGap = 8;   // per-point gaps 1..8: one per lane of a pair

// largest rho~^2 of a far pair: lane g of the pair takes the point pairs q = g mod LPP
template <int LPP>
__device__ __forceinline__ double far_rmax(const PairArgs &A, const FarGeom &G, int g)
{
    const int nq1 = G.nq1, nq = nq1 * nq1;
    double rmax = 0.0;
    for (int q = g; q < nq; q += LPP) {
        const int p = q / nq1, r = q - p * nq1;
        const double rx = G.xp[3 * p] - G.yp[3 * r], ry = G.xp[3 * p + 1] - G.yp[3 * r + 1],
                     rz = G.xp[3 * p + 2] - G.yp[3 * r + 2];
        rmax = fmax(rmax, (rx * rx + ry * ry + rz * rz) * A.inv_u2);
    }
#pragma unroll
    for (int o = 1; o < LPP; o <<= 1) rmax = fmax(rmax, __shfl_xor_sync(kFull, rmax, o));
    return rmax;
}

// gap constants of gap i (as Slots::init): cx = 1/(2 sqrt(a delta)), ic = 1/cx, sc = cx (K)
__device__ __forceinline__ void gap_consts(const PairArgs &A, int i, double &cx, double &ic)
{
    const double delta = (double)max(i, 1) * A.step;
    ic = 2.0 * sqrt(A.alpha * delta);
    cx = 1.0 / ic;
}

// lane (ps, g) of a K dual batch (4 pairs x 8 lanes), second walk over the
// pair's point pairs (the moments are formed by far_moments_k first): when
// `pp`, the per-point sum of gap g + 1 (acc[o], o: 3 forward, 3 reverse
// outputs); `spec`: the delta = 0 sums of the point pairs q = g mod 8.  Called
// warp-uniformly (every lane takes part in the region votes).
__device__ __forceinline__ void far_pp_k(const PairArgs &A, const FarGeom &G, const double nb[3], const double na[3],
                                         int g, bool pp, bool spec, double (&acc)[6], double (&s0f)[3],
                                         double (&scf)[3], double (&s0r)[3], double (&scr)[3], const double *tab)
{
    constexpr int LPP = 32 / FarCfg<6>::PB;
#pragma unroll
    for (int i = 0; i < 6; ++i) acc[i] = 0.0;
#pragma unroll
    for (int i = 0; i < 3; ++i) s0f[i] = scf[i] = s0r[i] = scr[i] = 0.0;
    double cx, ic;
    gap_consts(A, g + 1, cx, ic);
    const int nq1 = G.nq1;
    int q = 0;
    for (int p = 0; p < nq1; ++p) {
        const double x0 = G.xp[3 * p], x1 = G.xp[3 * p + 1], x2 = G.xp[3 * p + 2];
        const double wp = G.w[p];
        for (int r = 0; r < nq1; ++r, ++q) {
            const double rx = x0 - G.yp[3 * r], ry = x1 - G.yp[3 * r + 1], rz = x2 - G.yp[3 * r + 2];
            const double r2 = rx * rx + ry * ry + rz * rz;
            const double rnb = rx * nb[0] + ry * nb[1] + rz * nb[2];
            const double rna = (-rx) * na[0] + (-ry) * na[1] + (-rz) * na[2];
            const double wq = wp * G.w[r];
            const double rho = sqrt(r2);
            double xs[1] = {__dmul_rn(rho, cx)}, fs[1];
            special::eval_ulocal<5, 1>(xs, [&](int) { return __dmul_rn(1.0 / rho, ic); }, fs, tab);
            if (pp) {
#pragma unroll
                for (int i = 0; i < 3; ++i) {
                    const double wf = ((wq * (1.0 * G.hats[3 * r + i])) * (-rnb)) * A.inv2a;
                    const double wr = ((wq * (1.0 * G.hats[3 * p + i])) * (-rna)) * A.inv2a;
                    acc[i] = fma(fs[0], wf, acc[i]);
                    acc[3 + i] = fma(fs[0], wr, acc[3 + i]);
                }
            }
            if (spec && (q % LPP) == g) {
                const double iq = 1.0 / rho;
                const double Uf = -rnb * iq, Ur = -rna * iq;
                const double P = 1.0 / __dmul_rn(rho, rho);
                const double c0 = A.inv2a, cc = A.inv2a - A.step * P;
#pragma unroll
                for (int i = 0; i < 3; ++i) {
                    const double hf = wq * (1.0 * G.hats[3 * r + i]), hr = wq * (1.0 * G.hats[3 * p + i]);
                    s0f[i] = fma(hf * Uf, c0, s0f[i]);
                    scf[i] = fma(hf * Uf, cc, scf[i]);
                    s0r[i] = fma(hr * Ur, c0, s0r[i]);
                    scr[i] = fma(hr * Ur, cc, scr[i]);
                }
            }
        }
    }
}

// blocks d in [d0, min(d1, dmom)) of a fused K pair from its staged L row
// Lrow[o][0..9] (o: 6 outputs; index 0 = L0, 1..8 = gaps, 9 = Lcomb0),
// lane (ps, g): block g
__device__ __forceinline__ void fused_blocks_k(const PairArgs &A, const double *Lrow, int dmom, int64_t slot_f,
                                               int64_t slot_r, int g)
{
    {
        const int d = g;
        if (d < A.d0 || d >= A.d1 || d >= dmom) return;
#pragma unroll
        for (int o = 0; o < 6; ++o) {
            const int64_t slot = o < 3 ? slot_f : slot_r;
            if (slot < 0) continue;
            const double *Li = Lrow + o * 10;
            double b;
            if (d == 0) {
                b = Li[9] + (-Li[1]);
            } else {
                b = -Li[d - 1] + 2.0 * Li[d];
                b = b + (-Li[d + 1]);
            }
            A.Q[slot * (int64_t)(3 * A.nd) + (o % 3) * A.nd + (d - A.d0)] = b;
        }
    }
}

// ---------------------------------------------------------------------------
// K far batches from a per-point payload (HB_KFAR_PAYLOAD): the geometry of a
// pair's point pairs -- t = rho~^2, rho, 1/rho and both orientations' six
// weights -- is formed ONCE per point pair by the pair's 8 lanes into shared
// memory, and the moment loop (lane: 4 moments x 6 outputs) and the per-point
// gap loop (lane: one gap) read it back, instead of every lane recomputing
// sqrt, 1/rho, the normal products and the weights per point pair.
// Payload of point pair q of pair ps: Pk[(ps nq + q) kKPay + .] =
//   [t, rho, 1/rho, -, Wf0, Wf1, Wf2, Wr0, Wr1, Wr2]   (LDS.128-aligned pairs)
// ---------------------------------------------------------------------------
#ifndef HB_KFAR_PAYLOAD
#define HB_KFAR_PAYLOAD 1
#endif
constexpr int kKPay = 10;
constexpr int kKFarPts = 36;   // payload room: regular rules of <= 6 points (the default order 4)

// lane (ps, g) of the batch forms the payload of point pairs q = g, g + 8, ...;
// returns the pair's largest t (reduced over its 8 lanes)
__device__ __forceinline__ double far_payload_k(const PairArgs &A, const FarGeom &G, const double nb[3],
                                                const double na[3], double *Pk, int g)
{
    constexpr int LPP = 32 / FarCfg<6>::PB;
    const int nq1 = G.nq1, nq = nq1 * nq1;
    double tmax = 0.0;
    for (int q = g; q < nq; q += LPP) {
        const int p = q / nq1, r = q - p * nq1;
        const double rx = G.xp[3 * p] - G.yp[3 * r], ry = G.xp[3 * p + 1] - G.yp[3 * r + 1],
                     rz = G.xp[3 * p + 2] - G.yp[3 * r + 2];
        const double r2 = rx * rx + ry * ry + rz * rz;
        const double t = r2 * A.inv_u2;
        tmax = fmax(tmax, t);
        const double rho = sqrt(r2);
        const double rnb = rx * nb[0] + ry * nb[1] + rz * nb[2];
        const double rna = (-rx) * na[0] + (-ry) * na[1] + (-rz) * na[2];
        const double wq = G.w[p] * G.w[r];
        double *o = Pk + q * kKPay;
        o[0] = t;
        o[1] = rho;
        o[2] = 1.0 / rho;
        o[3] = 0.0;
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            o[4 + i] = ((wq * (1.0 * G.hats[3 * r + i])) * (-rnb)) * A.inv2a;
            o[7 + i] = ((wq * (1.0 * G.hats[3 * p + i])) * (-rna)) * A.inv2a;
        }
    }
#pragma unroll
    for (int o = 1; o < LPP; o <<= 1) tmax = fmax(tmax, __shfl_xor_sync(kFull, tmax, o));
    return tmax;
}

// moments k in [KPL g, KPL g + KPL) of both orientations from the payload
__device__ __forceinline__ void far_moments_k2(const double *Pk, int nq, double (&mom)[6][FarCfg<6>::KPL], int g)
{
    constexpr int KPL = FarCfg<6>::KPL;
#pragma unroll
    for (int i = 0; i < 6; ++i)
#pragma unroll
        for (int k = 0; k < KPL; ++k) mom[i][k] = 0.0;
#pragma unroll 2
    for (int q = 0; q < nq; ++q) {
        const double2 *o = reinterpret_cast<const double2 *>(Pk + q * kKPay);
        const double t = o[0].x;
        const double2 w01 = o[2], w23 = o[3], w45 = o[4];
        const double Wt[6] = {w01.x, w01.y, w23.x, w23.y, w45.x, w45.y};
        double pw = group_start_pow<KPL>(t, g);
#pragma unroll
        for (int k = 0; k < KPL; ++k) {
#pragma unroll
            for (int i = 0; i < 6; ++i) mom[i][k] = fma(Wt[i], pw, mom[i][k]);
            pw = __dmul_rn(pw, t);
        }
    }
}

// lane (ps, g): when `pp`, the per-point sum of gap g + 1 (acc[o]); `spec`: the
// delta = 0 sums of the point pairs q = g mod 8 -- from the payload.  Called
// warp-uniformly (every lane takes part in the region votes).
__device__ __forceinline__ void far_pp_k2(const PairArgs &A, const double *Pk, int nq, int g, bool pp, bool spec,
                                          double (&acc)[6], double (&s0f)[3], double (&scf)[3], double (&s0r)[3],
                                          double (&scr)[3], const double *tab)
{
    constexpr int LPP = 32 / FarCfg<6>::PB;
#pragma unroll
    for (int i = 0; i < 6; ++i) acc[i] = 0.0;
#pragma unroll
    for (int i = 0; i < 3; ++i) s0f[i] = scf[i] = s0r[i] = scr[i] = 0.0;
    double cx, ic;
    gap_consts(A, g + 1, cx, ic);
    const double k2 = 2.0 * A.alpha * A.step;   // cc / c0 = 1 - step P / inv2a
    for (int q = 0; q < nq; ++q) {
        const double2 *o = reinterpret_cast<const double2 *>(Pk + q * kKPay);
        const double2 tr = o[0], ii = o[1], w01 = o[2], w23 = o[3], w45 = o[4];
        const double rho = tr.y, iq = ii.x;
        const double W[6] = {w01.x, w01.y, w23.x, w23.y, w45.x, w45.y};
        double xs[1] = {__dmul_rn(rho, cx)}, fs[1];
        special::eval_ulocal<5, 1>(xs, [&](int) { return __dmul_rn(iq, ic); }, fs, tab);
        if (pp) {
#pragma unroll
            for (int i = 0; i < 6; ++i) acc[i] = fma(fs[0], W[i], acc[i]);
        }
        if (spec && (q % LPP) == g) {
            // (w hs (-r.n) / rho) c0 = W iq, (...) cc = W iq (1 - 2 a h / rho^2)
            const double f = 1.0 - k2 * __dmul_rn(iq, iq);
#pragma unroll
            for (int i = 0; i < 3; ++i) {
                const double af = W[i] * iq, ar = W[3 + i] * iq;
                s0f[i] += af;
                scf[i] = fma(af, f, scf[i]);
                s0r[i] += ar;
                scr[i] = fma(ar, f, scr[i]);
            }
        }
    }
}

// Fused lane-level V far path (2 lanes per pair): lane (ps, g) evaluates
// x H at the pair's gaps g + 1, g + 3, g + 5, g + 7 (four interleaved Horner
// chains) over its point pairs and, when `spec`, the delta = 0 sums of the
// point pairs q = g mod 2.  Called warp-uniformly.
__device__ __forceinline__ void far_pp_v(const PairArgs &A, const FarGeom &G, int g, bool pp, bool spec,
                                         double (&acc)[4], double &s0, double &sc, const double *tab)
{
    double cmp[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[j] = cmp[j] = 0.0;
    s0 = sc = 0.0;
    double cx[4], ic[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) gap_consts(A, g + 1 + 2 * j, cx[j], ic[j]);
    const int nq1 = G.nq1;
    int q = 0;
    for (int p = 0; p < nq1; ++p) {
        const double x0 = G.xp[3 * p], x1 = G.xp[3 * p + 1], x2 = G.xp[3 * p + 2];
        const double wp = G.w[p];
        for (int r = 0; r < nq1; ++r, ++q) {
            const double rx = x0 - G.yp[3 * r], ry = x1 - G.yp[3 * r + 1], rz = x2 - G.yp[3 * r + 2];
            const double rho = sqrt(rx * rx + ry * ry + rz * rz);
            const double wq = wp * G.w[r];
            double xs[4], fs[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) xs[j] = __dmul_rn(rho, cx[j]);
            // (1 / rho only where a lane takes the asymptote: the division stays off the common path)
            special::eval_ulocal<4, 4>(xs, [&](int j) { return __dmul_rn(1.0 / rho, ic[j]); }, fs, tab);
            if (pp) {
                // compensated sum (TwoProd by fma + TwoSum): the point sum of a gap
                // carries no rounding of its own, so the time second difference
                // below dmom amplifies only the per-point evaluation errors
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const double pr = __dmul_rn(fs[j], wq);
                    const double pe = fma(fs[j], wq, -pr);
                    const double sm = __dadd_rn(acc[j], pr);
                    const double bp = __dsub_rn(sm, acc[j]);
                    const double er = __dadd_rn(__dsub_rn(acc[j], __dsub_rn(sm, bp)), __dsub_rn(pr, bp));
                    cmp[j] = __dadd_rn(cmp[j], __dadd_rn(er, pe));
                    acc[j] = sm;
                }
            }
            if (spec && (q & 1) == g) {
                const double iq = 1.0 / rho;
                const double Aq = rho * A.inv2a2, Bq = A.inva * iq;
                const double cq = A.step * Bq + Aq;
                s0 = fma(wq, Aq, s0);
                sc = fma(wq, cq, sc);
            }
        }
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[j] = __dadd_rn(acc[j], cmp[j]);
}

// blocks d in [d0, min(d1, dmom)) of a fused V pair from its staged L row
// Lrow[0] = L0, [1..8] = gaps, [9] = Lcomb0; lane (ps, g): blocks g, g + 2, g + 4, g + 6
__device__ __forceinline__ void fused_blocks_v(const PairArgs &A, const double *Lrow, int dmom, int64_t slot, int g)
{
#pragma unroll
    for (int h = 0; h < 4; ++h) {
        const int d = g + 2 * h;
        if (d < A.d0 || d >= A.d1 || d >= dmom) continue;
        double b;
        if (d == 0) {
            b = Lrow[9] + (-Lrow[1]);
        } else {
            b = -Lrow[d - 1] + 2.0 * Lrow[d];
            b = b + (-Lrow[d + 1]);
        }
        A.Q[slot * (int64_t)A.nd + (d - A.d0)] = b;
    }
}

// delta = 0 sums of a pair without moments (far-batch pairs): L0 / Lc of the staged row
template <int OP, bool TP1, bool SP1, int NJ, class Geom>
__device__ __forceinline__ void pair_specials(const PairArgs &A, const Geom &g, int nq, const double ny[3],
                                              double jac, double *geo, double *Ls, int lane)
{
    constexpr int NIJ = (TP1 ? 3 : 1) * (SP1 ? 3 : 1);
    constexpr int PAY = Layout<OP, NIJ>::PAY, SLOTS = LsLayout<NIJ, NJ>::SLOTS;
    double s0[NIJ], sc[NIJ];
#pragma unroll
    for (int i = 0; i < NIJ; ++i) s0[i] = sc[i] = 0.0;
    for (int base = 0; base < nq; base += 32) {
        double rt2;
        int small, nzw;
        point_payload<OP, TP1, SP1>(A, g, base + lane, nq, ny, true, geo + lane * PAY, rt2, small, nzw, s0, sc);
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1)
#pragma unroll
        for (int i = 0; i < NIJ; ++i) {
            s0[i] += __shfl_xor_sync(kFull, s0[i], o);
            if (OP != 2) sc[i] += __shfl_xor_sync(kFull, sc[i], o);
        }
    if (lane == 0) {
        double *L0 = Ls + NIJ * SLOTS, *Lc = L0 + NIJ;
#pragma unroll
        for (int i = 0; i < NIJ; ++i) {
            L0[i] = jac * s0[i];
            Lc[i] = jac * (OP == 2 ? s0[i] : sc[i]);
        }
    }
    __syncwarp();
}


// blocks [d0, dend) of a pair from per-point L (windows), given its istar
template <int OP, bool TP1, bool SP1, int NJ, class Geom>
__device__ __forceinline__ void pair_point_blocks(const PairArgs &A, const Geom &g, int nq, const double ny[3],
                                                  double jac, int istar, int dend, int64_t slot, double *geo,
                                                  double *Ls, int lane, const double *tab)
{
    constexpr int NIJ = (TP1 ? 3 : 1) * (SP1 ? 3 : 1);
    constexpr int SLOTS = LsLayout<NIJ, NJ>::SLOTS;
    const int gend = istar + 2;
    const int gw = pair_gw(istar);
    per_point_windows<NIJ, SLOTS>(A, dend, istar, Ls, slot, lane, [&](const Win &W, int npp) {
        pair_points<OP, TP1, SP1, NJ>(A, W, g, nq, ny, jac, gend, gw, (gw == 16 && npp > 16) ? NJ : 1, geo, Ls, lane,
                                      tab);
    });
}


__device__ __forceinline__ RegularGeom regular_geom(const hb_mesh_desc &M, int64_t a, int64_t b, bool near)
{
    RegularGeom g;
    const int nq1 = near ? (int)M.n_near : (int)M.n_reg;
    const double *pts = near ? M.near_pts_dev : M.reg_pts_dev;
    g.xp = pts + 3 * a * nq1;
    g.yp = pts + 3 * b * nq1;
    g.w = near ? M.near_w_dev : M.reg_w_dev;
    g.hats = near ? M.near_hats_dev : M.reg_hats_dev;
    g.nq1 = nq1;
    return g;
}

// lane of the n-th set bit of m (n < popc(m)), warp-uniform inputs
__device__ __forceinline__ int nth_bit(unsigned m, int n)
{
    for (int k = 0; k < n; ++k) m &= m - 1;
    return __ffs(m) - 1;
}

// smallest first moment block over the batch's pairs (lanes of pair ps: ps < npairs)
__device__ __forceinline__ int batch_dlo(const PairArgs &A, double rmax, bool valid)
{
    const int dm = valid ? max(2, moment_istar(rmax) + 1) : 0x7fffffff;
    return max(A.d0, __reduce_min_sync(kFull, dm));
}

// ---------------------------------------------------------------------------
// K1 body: separated pairs of one (test row e, 32-column segment) work item.
// The segment is classified lane-parallel; near pairs run warp per pair,
// far pairs in batches (V, V11, D2: moments in registers, DMMA combine).
// ---------------------------------------------------------------------------
template <int OP, bool TP1, bool SP1, int NJ, bool SYM, int CLS>
__device__ __forceinline__ void regular_item(const PairArgs &A, int64_t e, int64_t seg, const WarpMem &W, int lane,
                                             const double *tab)
{
    constexpr int NIJ = (TP1 ? 3 : 1) * (SP1 ? 3 : 1);
    const hb_mesh_desc &M = A.m;
    int64_t fb = seg * A.seg_len;
    const int64_t fe = min(fb + A.seg_len, M.E_x);
    if (SYM) fb = max(fb, e);
    if (fb >= fe) return;
    const int64_t t_lo = __ldg(M.tn_indptr_dev + e), t_hi = __ldg(M.tn_indptr_dev + e + 1);
    double ce[3];
    for (int c = 0; c < 3; ++c) ce[c] = __ldg(M.centroids_dev + 3 * e + c);
    const double de = __ldg(M.diameters_dev + e);

    // lane l classifies f = fb + l (touching pairs belong to the singular path;
    // D2 pairs with n_x.n_y == 0 contribute nothing and are not staged)
    const int64_t f = fb + lane;
    bool ok = f < fe && touching_pos(M, t_lo, t_hi, f) < 0;
    double jac = 0.0;
    if (ok) {
        jac = pair_jac<OP>(A, e, f);
        if (OP == 2 && jac == 0.0) ok = false;
    }
    const bool near = ok && near_test(M, ce, de, f);
    constexpr bool FARC = NIJ == 1 || NIJ == 9;
    const bool FAR = FARC && A.moments && M.n_reg <= kFarMaxRule;
    // CLS 2: far pairs only (batches), 3: the rest (near pairs, warp per pair)
    const unsigned nearm = CLS == 2 ? 0u : __ballot_sync(kFull, ok && (near || !FAR));
    const unsigned farm = CLS == 3 ? 0u : __ballot_sync(kFull, ok && !near && FAR);

    for (unsigned m = nearm; m; m &= m - 1) {
        const int l = __ffs(m) - 1;
        const int64_t ff = fb + l;
        const double jf = __shfl_sync(kFull, jac, l);
        const bool nf = (__shfl_sync(kFull, (int)near, l)) != 0;
        const RegularGeom g = regular_geom(M, e, ff, nf);
        double ny[3];
        for (int c = 0; c < 3; ++c) ny[c] = __ldg(M.normals_dev + 3 * ff + c);
        eval_pair<OP, TP1, SP1, NJ>(A, g, g.nq1 * g.nq1, ny, jf, rt2_lower(A, e, ff), rt2_upper(A, e, ff),
                                    (e - A.e0) * M.E_x + ff, W.geo,
                                    W.Ls, W.Pw, lane, tab);
    }
    if constexpr (FARC) {
        constexpr int PB = FarCfg<NIJ>::PB, KPL = FarCfg<NIJ>::KPL, LPP = 32 / PB, NSTR = far_nstr<NIJ>();
        double *Ms = W.geo;
        FarPairs<NIJ> P(W.geo);
        unsigned m = farm;
        while (m) {
            const int npairs = min(PB, __popc(m));
            const int ps = lane / LPP, gk = lane % LPP;
            const bool pv = ps < npairs;
            const int l = pv ? nth_bit(m, ps) : 0;
            const int64_t ff = fb + l;
            double rmax;
            __syncwarp();
            const int n3 = 3 * (int)M.n_reg;
            double *Xs = W.geo + ps * (2 * n3 + 1);
            stage_far_points<LPP>(M, e, ff, Xs, gk);
            __syncwarp();
            const FarGeom fg{Xs, Xs + n3, W.rw, W.rh, (int)M.n_reg};
            bool fused = false;
            if constexpr (NIJ == 1) {
                // the pair's largest rho~^2 first: it decides istar, dmom and whether
                // its per-point gaps fit the fused lane path (<= 8 gaps, 4 per lane)
                rmax = far_rmax<LPP>(A, fg, gk);
                const int istar = moment_istar(rmax), dmom = max(2, istar + 1);
                fused = pv && istar + 1 <= kFusedMaxGap;
                const bool pp = fused && A.d0 < dmom;
                const bool pp_any = __any_sync(kFull, pp);
                double mom[16], rdummy;
                far_moments_v(A, fg, mom, rdummy, gk);
                double acc[4], s0, sc;
                if (pp_any) far_pp_v(A, fg, gk, pp, pp && A.need_special, acc, s0, sc, tab);
                __syncwarp();   // the staged points are overwritten from here on
                if (pp_any) {
                    const double jq = __shfl_sync(kFull, jac, l);
                    double *Lrow = W.geo + ps * 10;
                    if (A.need_special) {
                        s0 += __shfl_xor_sync(kFull, s0, 1);
                        sc += __shfl_xor_sync(kFull, sc, 1);
                    }
                    if (pp) {
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            const int i = gk + 1 + 2 * j;
                            double cxj, icj;
                            gap_consts(A, i, cxj, icj);
                            Lrow[i] = jq * (acc[j] * (icj * A.inv2a2));
                        }
                        if (A.need_special && gk == 0) {
                            Lrow[0] = jq * s0;
                            Lrow[9] = jq * sc;
                        }
                    }
                    __syncwarp();
                    if (pp) fused_blocks_v(A, Lrow, dmom, (e - A.e0) * M.E_x + ff, gk);
                    __syncwarp();
                }
#pragma unroll
                for (int k = 0; k < KPL; ++k) Ms[(KPL * gk + k) * NSTR + ps] = pv ? mom[k] : 0.0;
            } else {
                double mom[9][4];
                far_moments_p1p1(A, fg, mom, rmax, gk);
                __syncwarp();
#pragma unroll
                for (int k = 0; k < KPL; ++k)
#pragma unroll
                    for (int i = 0; i < 9; ++i) Ms[(KPL * gk + k) * NSTR + i * PB + ps] = pv ? mom[i][k] : 0.0;
            }
            const double jf = __shfl_sync(kFull, jac, l);
            if (gk == 0 && pv) {
                P.jac[ps] = jf;
                P.rmax[ps] = fused ? -1.0 : rmax;   // < 0: no warp-path per-point work left
                P.dmom[ps] = max(2, moment_istar(rmax) + 1);
                P.lane[ps] = l;
                P.slot_f[ps] = (e - A.e0) * M.E_x + ff;
                P.slot_r[ps] = -1;
            }
            const int dlo = batch_dlo(A, rmax, pv);
            __syncwarp();
            far_combine<NIJ, NIJ>(A, Ms, P, npairs, dlo, lane);
            __syncwarp();
            // blocks below each pair's dmom: per-point L, warp per pair
            for (int q = 0; q < npairs; ++q) {
                const int dmom = P.dmom[q];
                if (A.d0 >= dmom || P.rmax[q] < 0.0) continue;
                const int istar = moment_istar(P.rmax[q]);
                const int lq = P.lane[q];
                const int64_t fq = fb + lq;
                const double jq = P.jac[q];
                const RegularGeom gq = regular_geom(M, e, fq, false);
                double ny[3];
                for (int c = 0; c < 3; ++c) ny[c] = __ldg(M.normals_dev + 3 * fq + c);
                const int64_t slot = (e - A.e0) * M.E_x + fq;
                if (A.need_special) pair_specials<OP, TP1, SP1, NJ>(A, gq, gq.nq1 * gq.nq1, ny, jq, W.geo, W.Ls, lane);
                pair_point_blocks<OP, TP1, SP1, NJ>(A, gq, gq.nq1 * gq.nq1, ny, jq, istar, min(A.d1, dmom), slot, W.geo,
                                                    W.Ls, lane, tab);
                __syncwarp();
            }
            for (int q = 0; q < npairs; ++q) m &= m - 1;
        }
    }
}

// K1 body for K with both orientations: separated pairs (e, f) of one
// (test row e, segment) item, evaluated as the canonical pair (min, max).
// Pairs with both rows in the chunk are produced once (by the smaller row);
// a pair whose other row lies outside the chunk is still evaluated in its
// canonical orientation and only this row's output is stored.  Near pairs
// run warp per pair, far pairs in batches (moments of both orientations in
// registers, DMMA combine).
template <int NJ, int CLS>
__device__ __forceinline__ void regular_item_dual(const PairArgs &A, int64_t e, int64_t seg, const WarpMem &W,
                                                  int lane, const double *tab)
{
    const hb_mesh_desc &M = A.m;
    const int64_t fb = seg * A.seg_len;
    const int64_t fe = min(fb + A.seg_len, M.E_x);
    if (fb >= fe) return;
    const int64_t t_lo = __ldg(M.tn_indptr_dev + e), t_hi = __ldg(M.tn_indptr_dev + e + 1);
    const int64_t f = fb + lane;
    const bool f_in = f >= A.e0 && f < A.e1;
    // the canonical pair (f, e) of f < e in the chunk belongs to row f; touching pairs (f == e
    // too) belong to the singular path
    const bool ok = f < fe && !(f < e && f_in) && touching_pos(M, t_lo, t_hi, f) < 0;
    const int64_t a = f > e ? e : f, b = f > e ? f : e;
    bool near = false;
    if (ok) {
        double ca[3];
        for (int c = 0; c < 3; ++c) ca[c] = __ldg(M.centroids_dev + 3 * a + c);
        near = near_test(M, ca, __ldg(M.diameters_dev + a), b);
    }
    // CLS 2: far pairs only (batches), 3: the rest (near pairs, warp per pair)
    const bool FAR = A.moments && M.n_reg <= kFarMaxRule;
    const unsigned nearm = CLS == 2 ? 0u : __ballot_sync(kFull, ok && (near || !FAR));
    const unsigned farm = CLS == 3 ? 0u : __ballot_sync(kFull, ok && !near && FAR);
    auto slots = [&](int64_t aa, int64_t bb, int64_t &sf, int64_t &sr) {
        sf = (aa >= A.e0 && aa < A.e1) ? (aa - A.e0) * M.E_x + bb : -1;   // test a, trial b
        sr = (bb >= A.e0 && bb < A.e1) ? (bb - A.e0) * M.E_x + aa : -1;   // test b, trial a
    };
    for (unsigned m = nearm; m; m &= m - 1) {
        const int l = __ffs(m) - 1;
        const int64_t ff = fb + l;
        const int64_t aa = ff > e ? e : ff, bb = ff > e ? ff : e;
        int64_t slot_f, slot_r;
        slots(aa, bb, slot_f, slot_r);
        const RegularGeom g = regular_geom(M, aa, bb, __shfl_sync(kFull, (int)near, l) != 0);
        double nb[3], na[3];
        for (int c = 0; c < 3; ++c) {
            nb[c] = __ldg(M.normals_dev + 3 * bb + c);
            na[c] = __ldg(M.normals_dev + 3 * aa + c);
        }
        const double jac = pair_jac<1>(A, aa, bb);
        const double rlo = rt2_lower(A, aa, bb);
        const int nq = g.nq1 * g.nq1;
        eval_pair_dual<NJ>(A, g, nq, nb, na, jac, rlo, slot_f, slot_r, W.geo, W.Ls, W.Pw, lane, tab);
    }
    constexpr int PB = FarCfg<6>::PB, KPL = FarCfg<6>::KPL, LPP = 32 / PB, NSTR = far_nstr<6>();
    double *Ms = W.geo;
    FarPairs<6> P(W.geo);
    unsigned m = farm;
    while (m) {
        const int npairs = min(PB, __popc(m));
        const int ps = lane / LPP, gk = lane % LPP;
        const bool pv = ps < npairs;
        const int l = pv ? nth_bit(m, ps) : 0;
        const int64_t ff = fb + l;
        const int64_t aa = ff > e ? e : ff, bb = ff > e ? ff : e;
        double nb[3], na[3];
        for (int c = 0; c < 3; ++c) {
            nb[c] = __ldg(M.normals_dev + 3 * bb + c);
            na[c] = __ldg(M.normals_dev + 3 * aa + c);
        }
        double mom[6][KPL], acc[6], s0f[3], scf[3], s0r[3], scr[3];
        __syncwarp();
        const int n3 = 3 * (int)M.n_reg;
        double *Xs = W.geo + ps * (2 * n3 + 1);
        stage_far_points<LPP>(M, aa, bb, Xs, gk);
        __syncwarp();
        const FarGeom g{Xs, Xs + n3, W.rw, W.rh, (int)M.n_reg};
        const int nqf = (int)(M.n_reg * M.n_reg);
#if HB_KFAR_PAYLOAD
        const bool kpay = nqf <= kKFarPts;   // warp-uniform
        double *Pk = W.geo + ((PB * (2 * n3 + 1) + 1) & ~1) + ps * nqf * kKPay;
        // the payload, with the pair's largest rho~^2: it decides istar, dmom and
        // whether the per-point gaps fit the fused lane path
        const double rmax = kpay ? far_payload_k(A, g, nb, na, Pk, gk) : far_rmax<LPP>(A, g, gk);
        __syncwarp();
#else
        const double rmax = far_rmax<LPP>(A, g, gk);
#endif
        const int istar = moment_istar(rmax), dmom = max(2, istar + 1);
        const bool fused = pv && istar + 1 <= kFusedMaxGap;
        const bool pp = fused && A.d0 < dmom;
        const bool pp_any = __any_sync(kFull, pp);
        int64_t sf = -1, sr = -1;
        slots(aa, bb, sf, sr);
        const double jac = pair_jac<1>(A, aa, bb);
#if HB_KFAR_PAYLOAD
        if (kpay) {
            far_moments_k2(Pk, nqf, mom, gk);
            if (pp_any) far_pp_k2(A, Pk, nqf, gk, pp, pp && A.need_special, acc, s0f, scf, s0r, scr, tab);
        } else {
            far_moments_k(A, g, nb, na, mom, gk);
            if (pp_any) far_pp_k(A, g, nb, na, gk, pp, pp && A.need_special, acc, s0f, scf, s0r, scr, tab);
        }
#else
        far_moments_k(A, g, nb, na, mom, gk);
        if (pp_any) far_pp_k(A, g, nb, na, gk, pp, pp && A.need_special, acc, s0f, scf, s0r, scr, tab);
#endif
        __syncwarp();   // the staged points are overwritten from here on
        if (pp_any) {
            // staged L row per pair: [o][0] = L0, [o][1..8] = gaps, [o][9] = Lcomb0
            double *Lrow = W.geo + ps * 60;
            if (A.need_special) {
#pragma unroll
                for (int o = 1; o < LPP; o <<= 1)
#pragma unroll
                    for (int i = 0; i < 3; ++i) {
                        s0f[i] += __shfl_xor_sync(kFull, s0f[i], o);
                        scf[i] += __shfl_xor_sync(kFull, scf[i], o);
                        s0r[i] += __shfl_xor_sync(kFull, s0r[i], o);
                        scr[i] += __shfl_xor_sync(kFull, scr[i], o);
                    }
            }
            if (pp) {
                double cxh, ich;
                gap_consts(A, gk + 1, cxh, ich);
#pragma unroll
                for (int o = 0; o < 6; ++o) Lrow[o * 10 + gk + 1] = jac * (acc[o] * cxh);
                if (A.need_special && gk == 0) {
#pragma unroll
                    for (int i = 0; i < 3; ++i) {
                        Lrow[i * 10] = jac * s0f[i];
                        Lrow[i * 10 + 9] = jac * scf[i];
                        Lrow[(3 + i) * 10] = jac * s0r[i];
                        Lrow[(3 + i) * 10 + 9] = jac * scr[i];
                    }
                }
            }
            __syncwarp();
            if (pp) fused_blocks_k(A, Lrow, dmom, sf, sr, gk);
            __syncwarp();
        }
#pragma unroll
        for (int k = 0; k < KPL; ++k)
#pragma unroll
            for (int i = 0; i < 6; ++i) Ms[(KPL * gk + k) * NSTR + i * PB + ps] = pv ? mom[i][k] : 0.0;
        if (gk == 0 && pv) {
            P.jac[ps] = jac;
            P.rmax[ps] = fused ? -1.0 : rmax;   // < 0: no warp-path per-point work left
            P.dmom[ps] = dmom;
            P.lane[ps] = l;
            P.slot_f[ps] = sf;
            P.slot_r[ps] = sr;
        }
        const int dlo = max(A.d0, __reduce_min_sync(kFull, pv ? dmom : 0x7fffffff));
        __syncwarp();
        far_combine<6, 3>(A, Ms, P, npairs, dlo, lane);
        __syncwarp();
        // pairs outside the fused path: per-point blocks warp per pair
        for (int q = 0; q < npairs; ++q) {
            const int dmom = P.dmom[q];
            if (A.d0 >= dmom || P.rmax[q] < 0.0) continue;
            const int istar = moment_istar(P.rmax[q]);
            const int lq = P.lane[q];
            const int64_t fq = fb + lq;
            const int64_t aq = fq > e ? e : fq, bq = fq > e ? fq : e;
            const double jq = P.jac[q];
            const int64_t sf = P.slot_f[q], sr = P.slot_r[q];
            const RegularGeom gq = regular_geom(M, aq, bq, false);
            double nbq[3], naq[3];
            for (int c = 0; c < 3; ++c) {
                nbq[c] = __ldg(M.normals_dev + 3 * bq + c);
                naq[c] = __ldg(M.normals_dev + 3 * aq + c);
            }
            const int nq = gq.nq1 * gq.nq1, dend = min(A.d1, dmom);
            if (A.need_special) {
                double s0f[3] = {0, 0, 0}, scf[3] = {0, 0, 0}, s0r[3] = {0, 0, 0}, scr[3] = {0, 0, 0};
                for (int base = 0; base < nq; base += 32) {
                    double rt2;
                    int small, nzw;
                    dual_payload(A, gq, base + lane, nq, nbq, naq, true, W.geo + lane * kDualPay, rt2, small, nzw,
                                 s0f, scf, s0r, scr);
                }
                dual_specials_reduce<NJ>(s0f, scf, s0r, scr, jq, W.Ls, W.Ls + LsLayout<3, NJ>::SIZE, lane);
                __syncwarp();
            }
            dual_point_blocks<NJ>(A, gq, nq, nbq, naq, jq, istar, dend, sf, sr, W.geo, W.Ls, lane, tab);
            __syncwarp();
        }
        for (int q = 0; q < npairs; ++q) m &= m - 1;
    }
}

// per-warp shared memory: the warp-per-pair layout (payload, staged L row,
// moment scratch), or the far batch's Ms + pair data where larger (they are
// never live at the same time)
template <int OP, int NIJ, int NJ>
__host__ __device__ constexpr int smem_doubles_per_warp()
{
    if constexpr (NIJ == 1 || NIJ == 9) {
        return smem_doubles_per_warp_base<OP, NIJ, NJ>() > far_smem_doubles<NIJ>()
                   ? smem_doubles_per_warp_base<OP, NIJ, NJ>() : far_smem_doubles<NIJ>();
    } else {
        return smem_doubles_per_warp_base<OP, NIJ, NJ>();
    }
}
// K far batches from a payload: the staged points of the batch + PB x 36 x kKPay
// payload doubles (the regular rule of <= kFarMaxRule points: 49 point pairs)
__host__ __device__ constexpr int kfar_payload_doubles()
{
    return HB_KFAR_PAYLOAD ? ((FarCfg<6>::PB * (6 * kFarMaxRule + 1) + 1) & ~1) + FarCfg<6>::PB * kKFarPts * kKPay
                           : 0;
}

template <int NJ>
__host__ __device__ constexpr int dual_smem_doubles_per_warp()
{
    constexpr int a = dual_smem_doubles_per_warp_base<NJ>() > far_smem_doubles<6>()
                          ? dual_smem_doubles_per_warp_base<NJ>() : far_smem_doubles<6>();
    return a > kfar_payload_doubles() ? a : kfar_payload_doubles();
}

// ---------------------------------------------------------------------------
// K2 body: one touching pair (identical / common edge / common vertex),
// Sauter-Schwab rule on the permuted charts of classify_pair.
// ---------------------------------------------------------------------------
template <int OP, bool TP1, bool SP1, int NJ>
__device__ __forceinline__ void singular_item(const PairArgs &A, int64_t k, const WarpMem &W, int lane,
                                              const double *tab)
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
    // touching pairs: no lower bound of rho~^2 (0)
    eval_pair<OP, TP1, SP1, NJ>(A, g, off1 - off0, ny, jac, 0.0, rt2_upper(A, e, f), slot, W.geo, W.Ls, W.Pw, lane,
                                tab);
}

// ---------------------------------------------------------------------------
// Persistent pair kernel: warps pull work items from a global counter.
// Items [0, n_sing) are touching pairs (K2 body, heaviest first in row
// order), items [n_sing, n_sing + rows*nseg) are (row, segment) tiles of
// separated pairs (K1 body).  A warp only ever holds one pair class, so the
// two quadrature families never share a warp; dynamic fetching removes the
// imbalance of upper-triangular / near-diagonal tiles.
// ---------------------------------------------------------------------------
template <int OP, bool TP1, bool SP1, int NJ, bool SYM, bool DUAL, int CLS>
__global__ void __launch_bounds__(HB_PAIR_WARPS * 32, (TP1 && SP1) ? HB_P1P1_MINB : HB_PAIR_MINB) k_pairs(const PairArgs A)
{
    constexpr int NIJ = (TP1 ? 3 : 1) * (SP1 ? 3 : 1);
    extern __shared__ __align__(16) double smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double *tab = smem;
    special::load_utable<OP + 4>(tab);   // factor-free kinds, uniform pieces (hb_special.cuh)
    double *rule = smem + special::kUTabDoubles;
    if (A.m.n_reg <= kFarMaxRule) {
        for (int i = threadIdx.x; i < 4 * (int)A.m.n_reg; i += blockDim.x)
            rule[i] = i < A.m.n_reg ? __ldg(A.m.reg_w_dev + i) : __ldg(A.m.reg_hats_dev + i - A.m.n_reg);
    }
    __syncthreads();
    constexpr int kPerWarp = DUAL ? dual_smem_doubles_per_warp<NJ>() : smem_doubles_per_warp<OP, NIJ, NJ>();
    static_assert(special::kUTabDoubles % 2 == 0 && kPerWarp % 2 == 0 && Layout<OP, NIJ>::PAY % 2 == 0 &&
                      kDualPay % 2 == 0, "payload slots must stay 16-byte aligned (LDS.128)");
    double *geo = smem + special::kUTabDoubles + kRuleDoubles + warp * kPerWarp;
    WarpMem W;
    W.geo = geo;
    W.Ls = geo + 32 * (DUAL ? kDualPay : Layout<OP, NIJ>::PAY);
    W.Pw = W.Ls + (DUAL ? 2 * LsLayout<3, NJ>::SIZE : LsLayout<NIJ, NJ>::SIZE);
    W.rw = rule;
    W.rh = rule + A.m.n_reg;
    const hb_mesh_desc &M = A.m;
    const int64_t s_lo = __ldg(M.sing_rowptr_dev + A.e0), s_hi = __ldg(M.sing_rowptr_dev + A.e1);
    int64_t n_sing = s_hi - s_lo;
    const int64_t nseg = cdiv(M.E_x, (int64_t)A.seg_len);
    int64_t n_reg = (A.e1 - A.e0) * nseg;
    if (CLS == 1) n_reg = 0;                 // touching pairs only
    if (CLS == 2 || CLS == 3) n_sing = 0;    // separated pairs: far (2) / near (3); 4: touching, then near
    constexpr int RCLS = CLS == 4 ? 3 : CLS;
    for (;;) {
        unsigned long long it = 0;
        if (lane == 0) it = atomicAdd(A.counter, 1ull);
        it = __shfl_sync(kFull, it, 0);
        const int64_t item = (int64_t)it;
        if (item < n_sing) {
            singular_item<OP, TP1, SP1, NJ>(A, s_lo + item, W, lane, tab);
        } else if (item - n_sing < n_reg) {
            const int64_t r = item - n_sing;
            if constexpr (DUAL) regular_item_dual<NJ, RCLS>(A, A.e0 + r / nseg, r % nseg, W, lane, tab);
            else regular_item<OP, TP1, SP1, NJ, SYM, RCLS>(A, A.e0 + r / nseg, r % nseg, W, lane, tab);
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
    int node_grid;        // p1 x p1 finalize: grid x = node (rows cover most of the mesh) instead of (chunk element, local node)
    const int64_t *tile_eptr, *tile_elem;   // curl tile plan (32-node tiles)
    const int32_t *star_pos;
    int nrs;                                // row-sharded destination: shards, bounds, base pointers
    const int64_t *rs_bounds;
    double *const *rs_ptrs;
    // fused curl transform (k_fin_p1p1_accum<true>): the single layer's staging
    // Qv[(e - e0) E_x + f][ndv] of the same row chunk, the window's offset in
    // it, alpha^2 and the surface curls (E_x, 3, 3)
    const double *Qv;
    int ndv, dv_off;
    double a2;
    const double *curls;
};

// address of entry (row, col) of block d - d_begin = b: the caller's per-block
// pointer (another GPU's memory over NVLink in a d-sharded row-parallel run),
// the owner of the row in a row-sharded run, or the contiguous blocks
__device__ __forceinline__ double *fin_addr(const FinArgs &F, int64_t b, int64_t row, int64_t col)
{
    if (F.nrs > 0) {
        int k = 0;   // owner of the row: <= 8-ish shards, linear scan of cached bounds
        while (k + 1 < F.nrs && row >= __ldg(F.rs_bounds + k + 1)) ++k;
        const int64_t lo = __ldg(F.rs_bounds + k), rows = __ldg(F.rs_bounds + k + 1) - lo;
        return F.rs_ptrs[k] + (b * rows + (row - lo)) * F.C + col;
    }
    return (F.bptr ? F.bptr[b] : F.out + b * F.R * F.C) + row * F.C + col;
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
                *fin_addr(F, b, e, f) = tile[el][fl][dl];
            }
        }
        for (int idx = tid; idx < 4 * 32 * 32; idx += 256) {
            const int fl = idx >> 7, dl = (idx >> 2) & 31, el = idx & 3;
            const int64_t e = eb + el, f = f0 + fl;
            if (e < F.e1 && f < F.E_x && f > e && dl < ndc) {
                const int64_t b = F.d0 + dc + dl - F.d_begin;
                *fin_addr(F, b, f, e) = tile[el][fl][dl];
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
                *fin_addr(F, b, e, n) = tile[lane][dl];
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
constexpr int kFlatMax = 96;  // flat (a, b) lists of the p1 x p1 finalize: star sizes up to ~9 x 9

// FUSE: D = D2 + alpha^2 curl^T V curl in the same pass (hb_assemble_vd).  Every
// pair (e, f >= e) of the chunk adds alpha^2 (c_ei . c_fj) V_ef to X[m][n]
// beside its staged D2 value (c: surface curl of hat i on e; V_ef from the
// single layer's staging of the same rows, halved for e == f like D2's
// diagonal), so X + X^T is D: sum over (e, i) in star(m), (f, j) in star(n) of
// D2 + alpha^2 (c_ei . c_fj) V_ef -- the curl transform of
// hypersingular_from_single_layer (heatbem/assembly.py:314-334) without a
// pass of its own over V.
template <bool FUSE>
__global__ void __launch_bounds__(256) k_fin_p1p1_accum(const FinArgs F)
{
    __shared__ double tile[32][33];
    extern __shared__ __align__(16) double fsm[];
    // CTA x = (element of the chunk, local node): node m is handled by the
    // CTA of the first chunk element in its (element-sorted) star only
    const int64_t n0 = (int64_t)blockIdx.y * 32;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    int64_t m;
    if (F.node_grid) {
        // one CTA column per node (row ranges covering most of the mesh: fewer CTAs
        // than three candidates per chunk element, none of them empty-handed)
        m = blockIdx.x;
    } else {
        const int64_t eo = F.e0 + blockIdx.x / 3;
        m = __ldg(F.tri_nodes + 3 * eo + blockIdx.x % 3);
        const int64_t a0 = __ldg(F.star_indptr + m), a1 = __ldg(F.star_indptr + m + 1);
        int64_t first = -1;
        for (int64_t a = a0; a < a1 && first < 0; ++a) {
            const int64_t e = __ldg(F.star_elem + a);
            if (e >= F.e0) first = e;
        }
        if (first != eo) return;
    }
    const int64_t sm0 = __ldg(F.star_indptr + m), sm1 = __ldg(F.star_indptr + m + 1);
    const int smax = F.star_max;
    int64_t *sQ = (int64_t *)fsm;                          // [star_max] Q offset of (e - e0, 3i)
    int64_t *sE = sQ + smax;                               // [star_max] e
    int64_t *wFJ = sE + smax;                              // [kWarps][star_max] (9f + j) nd of node n's star
    unsigned *okm = (unsigned *)(wFJ + kWarps * smax);     // [star_max][kFinMaxW]
    int *wP = (int *)(okm + smax * kFinMaxW);              // [kWarps][star_max] tile position of f
    // FUSE only: [star_max][4] curl of (e, i) | [kWarps][star_max][4] alpha^2 curl of (f, j), f
    double *sC = (double *)(wP + kWarps * smax + (smax * kWarps & 1));
    double *wC = sC + 4 * smax;
    __shared__ int na_s;
    __shared__ int64_t fOff[FUSE ? 1 : kWarps][FUSE ? 1 : kFlatMax];   // flat (a, b) list per warp
    __shared__ int fA[FUSE ? 1 : kWarps][FUSE ? 1 : kFlatMax];
    if (threadIdx.x == 0) {
        int na = 0;
        for (int64_t a = sm0; a < sm1; ++a) {
            const int64_t e = __ldg(F.star_elem + a);
            if (e < F.e0 || e >= F.e1) continue;
            sE[na] = e;
            sQ[na] = (e - F.e0) * F.E_x * 9 * (int64_t)F.nd + 3 * __ldg(F.star_local + a) * F.nd;
            if (FUSE) {
                const double *c = F.curls + 9 * e + 3 * __ldg(F.star_local + a);
                sC[4 * na] = __ldg(c);
                sC[4 * na + 1] = __ldg(c + 1);
                sC[4 * na + 2] = __ldg(c + 2);
            }
            ++na;
        }
        na_s = na;
    }
    __syncthreads();
    const int na = na_s;
    if (na == 0) return;   // (node grid: no element of the node's star in this row range)
    const int64_t tB0 = F.tile_eptr[blockIdx.y], tB = F.tile_eptr[blockIdx.y + 1] - tB0;
    // staged-pair bitmasks: warp w owns word w (tile positions 32w..32w+31);
    // okm: D2 staged (f >= e, n_e . n_f != 0); FUSE: okv, every f >= e (V staged)
    unsigned *okv = okm;
    __shared__ unsigned okv_s[FUSE ? 64 * kFinMaxW : 1];
    if (FUSE) okv = okv_s;
    {
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
            if (FUSE) {
                const unsigned wv = __ballot_sync(kFull, ok);
                if (lane == 0) okv[a * kFinMaxW + warp] = wv;
            }
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
            double *myC = wC + warp * 4 * smax;
            for (int b = lane; b < nb; b += 32) {
                const int64_t fb = __ldg(F.star_elem + sn0 + b), jb = __ldg(F.star_local + sn0 + b);
                myFJ[b] = (9 * fb + jb) * F.nd;
                myP[b] = F.star_pos[sn0 + b];
                if (FUSE) {
                    const double *c = F.curls + 9 * fb + 3 * jb;
                    myC[4 * b] = F.a2 * __ldg(c);
                    myC[4 * b + 1] = F.a2 * __ldg(c + 1);
                    myC[4 * b + 2] = F.a2 * __ldg(c + 2);
                    myC[4 * b + 3] = __longlong_as_double(fb);
                }
            }
            __syncwarp();
            double x = tile[nl][lane];
            // stars of <= 32 entries: lanes test the staged bit of entry b (lane b), a ballot
            // gives the staged entries and only those are loaded (ascending b, as before;
            // the skipped +0.0 additions were exact identities).  Longer stars: the full loop.
            const int pb = lane < nb ? myP[lane] : 0;
            // flat list of the staged (a, b) entries in (a, b) order, loaded eight at a
            // time: the same additions in the same order as the per-a loop (se over b,
            // then x += se for every a, empty ones included), with more loads in flight
            const bool flat_ok = !FUSE && nb <= 32 && na * nb <= kFlatMax;
            if (flat_ok) {
                int cnt = 0;
                for (int a = 0; a < na; ++a) {
                    const unsigned *om = okm + a * kFinMaxW;
                    const bool st = lane < nb && ((om[pb >> 5] >> (pb & 31)) & 1u);
                    const unsigned mask = __ballot_sync(kFull, st);
                    if (st) {
                        const int slot = cnt + __popc(mask & ((1u << lane) - 1u));
                        fOff[warp][slot] = sQ[a] + myFJ[lane];
                        fA[warp][slot] = a;
                    }
                    cnt += __popc(mask);
                }
                __syncwarp();
                double se = 0.0;
                int cur = 0;
                for (int i = 0; i < cnt; i += 8) {
                    double qv[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u) qv[u] = (lok && i + u < cnt) ? F.Q[fOff[warp][i + u] + dc + lane] : 0.0;
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        if (i + u >= cnt) break;
                        const int a = fA[warp][i + u];
                        for (; cur < a; ++cur) {
                            x += se;
                            se = 0.0;
                        }
                        se += qv[u];
                    }
                }
                for (; cur < na; ++cur) {
                    x += se;
                    se = 0.0;
                }
                __syncwarp();
            }
            for (int a = 0; a < (flat_ok ? 0 : na); ++a) {
                const double *Qe = F.Q + sQ[a] + dc + lane;
                const unsigned *om = okm + a * kFinMaxW;
                double se = 0.0;
                if (FUSE && nb <= 32) {
                    // every (f, j) of star(n) with f >= e: staged D2 value (0 where D2
                    // skipped the pair) + (alpha^2 c_ei . c_fj) V_ef, in star order.
                    // Lane b holds entry b's coefficient; four entries per round
                    // with their eight loads in flight together
                    const int64_t e = sE[a];
                    const double *Qve = F.Qv + (e - F.e0) * F.E_x * (int64_t)F.ndv + F.dv_off + dc + lane;
                    const unsigned *ov = okv + a * kFinMaxW;
                    bool vb = false, db = false;
                    double sb = 0.0;
                    int64_t fbl = 0;
                    if (lane < nb) {
                        vb = (ov[pb >> 5] >> (pb & 31)) & 1u;
                        db = (om[pb >> 5] >> (pb & 31)) & 1u;
                        fbl = __double_as_longlong(myC[4 * lane + 3]);
                        sb = fma(sC[4 * a + 2], myC[4 * lane + 2], fma(sC[4 * a + 1], myC[4 * lane + 1],
                                                                       sC[4 * a] * myC[4 * lane]));
                        if (fbl == e) sb *= 0.5;
                    }
                    unsigned mask = __ballot_sync(kFull, vb);
                    const unsigned dmask = __ballot_sync(kFull, db);
                    while (mask) {
                        int b[4];
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            b[u] = mask ? __ffs(mask) - 1 : -1;
                            mask &= mask - 1;
                        }
                        double su[4], qd[4], qv[4];
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            const int bu = b[u] < 0 ? 0 : b[u];
                            su[u] = __shfl_sync(kFull, sb, bu);
                            const int64_t fu = __shfl_sync(kFull, fbl, bu);
                            qd[u] = (lok && b[u] >= 0 && ((dmask >> bu) & 1u)) ? Qe[myFJ[bu]] : 0.0;
                            qv[u] = (lok && b[u] >= 0) ? Qve[fu * F.ndv] : 0.0;
                        }
#pragma unroll
                        for (int u = 0; u < 4; ++u)
                            if (b[u] >= 0) se += fma(su[u], qv[u], qd[u]);
                    }
                } else if (FUSE) {
                    const int64_t e = sE[a];
                    const double ce0 = sC[4 * a], ce1 = sC[4 * a + 1], ce2 = sC[4 * a + 2];
                    const double *Qve = F.Qv + (e - F.e0) * F.E_x * (int64_t)F.ndv + F.dv_off + dc + lane;
                    const unsigned *ov = okv + a * kFinMaxW;
                    for (int b = 0; b < nb; ++b) {
                        const int p = myP[b];
                        if (!((ov[p >> 5] >> (p & 31)) & 1u)) continue;   // f < e: the mirrored half
                        const int64_t fb = __double_as_longlong(myC[4 * b + 3]);
                        double s = fma(ce2, myC[4 * b + 2], fma(ce1, myC[4 * b + 1], ce0 * myC[4 * b]));
                        if (fb == e) s *= 0.5;
                        const bool d2 = (om[p >> 5] >> (p & 31)) & 1u;
                        const double qd = (lok && d2) ? Qe[myFJ[b]] : 0.0;
                        const double qv = lok ? Qve[fb * F.ndv] : 0.0;
                        se += fma(s, qv, qd);
                    }
                } else if (nb <= 32) {
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
// gap slots per per-point window: 16 lanes x NJ = 2
constexpr int kNJ = 2;

static int op_nij(const hb_assembly_desc *a) { return (a->test_p1 ? 3 : 1) * (a->trial_p1 ? 3 : 1); }

static bool combo_ok(const hb_assembly_desc *a)
{
    if (a->op == HB_OP_SINGLE_LAYER)
        return a->symmetric && a->test_p1 == a->trial_p1;
    if (a->op == HB_OP_DOUBLE_LAYER) return !a->symmetric && !a->test_p1 && a->trial_p1;
    if (a->op == HB_OP_HYPERSINGULAR2) return a->symmetric && a->test_p1 && a->trial_p1;
    return false;
}

constexpr size_t kCounterBytes = 256;

// Which blocks the moment form computes: blocks d >= moment_from(op, E_t).
// * E_t < 64 (config 2 size): V throughout (its moments beat the per-point
//   gaps there: 1.03 vs 1.23 ms), K and D2 never (direct kernel: K's
//   dual-orientation body feeds both orientations from one F evaluation).
// * E_t >= 64: V and D2 direct below block 32 and moments from block 32; K
//   (E_t >= 128) from block 62 (a direct-window edge).
//   At small gaps each pair's moment block lies high (many per-point gaps below
//   it) and the direct kernel is faster; above, the moments win (B200, config
//   5, pair ms per block range direct / moments: V [0,32) 282 / 383,
//   [32,62) 212 / 88, [62,92) 175 / 41; D2 174 / 318, 134 / 115, 121 / 83;
//   K 393 / 923, 296 / 267, 244 / 176).
// A function of (op, E_t) only, so a block is computed the same way whatever
// d-range a call (chunk, rank) covers: d-sharded calls agree bitwise.
// HB_MOMENTS=0/1 overrides (never / always), HB_MOMENT_FROM the switch block.
static int64_t moment_from(const hb_assembly_desc *a)
{
    static const int env = getenv("HB_MOMENTS") ? (atoi(getenv("HB_MOMENTS")) != 0) : -1;
    static const int64_t sw = getenv("HB_MOMENT_FROM") ? atoll(getenv("HB_MOMENT_FROM")) : 32;
    static const int64_t ksw = getenv("HB_K_MOMENT_FROM") ? atoll(getenv("HB_K_MOMENT_FROM")) : 62;
    const int64_t never = INT64_MAX / 4;
    if (env == 1) return 0;
    if (env == 0) return never;
    if (a->op == HB_OP_DOUBLE_LAYER)   // K: the moment form pays only far out (config 3, E_t 64: it does not)
        return a->E_t >= 128 ? std::max<int64_t>(sw, ksw) : never;
    if (a->E_t >= 64) return sw;
    return a->op == HB_OP_SINGLE_LAYER ? 0 : never;
}

// the moment form for a call (a part of one) that starts at d_begin
static int use_moments(const hb_assembly_desc *a) { return a->d_begin >= moment_from(a) ? 1 : 0; }

// the direct and moment parts of a call's blocks [d_begin, d_end)
struct CallPart {
    int64_t lo, hi;
    bool mom;
};
static int call_parts(const hb_assembly_desc *a, CallPart (&p)[2])
{
    const int64_t sw = std::max(a->d_begin, std::min(a->d_end, moment_from(a)));
    int n = 0;
    if (a->d_begin < sw) p[n++] = {a->d_begin, sw, false};
    if (sw < a->d_end) p[n++] = {sw, a->d_end, true};
    return n;
}

// staging of one test row: every trial element x NIJ x the blocks of one
// launch (all blocks of the moment part, a 32-gap window of the direct part)
static size_t row_bytes(const hb_mesh_desc *m, const hb_assembly_desc *a)
{
    CallPart p[2];
    const int n = call_parts(a, p);
    int64_t nd = 1;
    for (int i = 0; i < n; ++i) nd = std::max(nd, p[i].mom ? p[i].hi - p[i].lo : std::min<int64_t>(p[i].hi - p[i].lo, 32));
    return (size_t)m->E_x * op_nij(a) * (size_t)nd * sizeof(double);
}

// moment table of the moment part (k_moment_table), 256-byte rounded
static size_t tm_bytes(const hb_assembly_desc *a)
{
    CallPart p[2];
    const int n = call_parts(a, p);
    for (int i = 0; i < n; ++i)
        if (p[i].mom) {
            const size_t k = (size_t)kNK * (size_t)(p[i].hi - p[i].lo) + kNK + 1;
            return (k * sizeof(double) + 255) & ~(size_t)255;
        }
    return 0;
}

// one class of pair items: CLS 1 touching pairs (Sauter-Schwab), 3 separated
// near pairs (warp per pair), 2 separated far pairs (batches).  The classes
// run as separate launches so that each kernel's working set of instructions
// is one path.
template <int OP, bool TP1, bool SP1, int NJ, bool DUAL, int CLS>
static int launch_class(const PairArgs &A, cudaStream_t st)
{
    constexpr int NIJ = (TP1 ? 3 : 1) * (SP1 ? 3 : 1);
    constexpr bool SYM = (OP != 1);
    constexpr int per_warp = DUAL ? dual_smem_doubles_per_warp<NJ>() : smem_doubles_per_warp<OP, NIJ, NJ>();
    const size_t sm = ((size_t)HB_PAIR_WARPS * per_warp + special::kUTabDoubles + kRuleDoubles) * sizeof(double);
    auto kp = k_pairs<OP, TP1, SP1, NJ, SYM, DUAL, CLS>;
    if (sm > 48 * 1024) cudaFuncSetAttribute(kp, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    int dev = 0, nsm = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kp, HB_PAIR_WARPS * 32, sm);
    const int64_t rows = A.e1 - A.e0;
    // separated-pair items of 32 trial elements, halved while the launch holds
    // fewer than 16 items per resident warp (the persistent grid's tail is about
    // one item per warp: config 2 V pair kernels 1.02 -> 0.975 ms; a row-parallel
    // rank's few rows likewise)
    PairArgs B = A;
    const int64_t warps = (int64_t)std::max(1, per_sm) * nsm * HB_PAIR_WARPS;
    B.seg_len = 32;
    // far batches (CLS 2) keep 32 trial elements per item: a batch combines up to
    // 16 pairs of one item on the tensor cores (floor 4 for a rank of 8 at config 2:
    // V 0.49 ms, floor 32: 0.37 ms)
    static const int min_seg = getenv("HB_MIN_SEG") ? atoi(getenv("HB_MIN_SEG")) : 4;
    static const int min_far = getenv("HB_MIN_SEG_FAR") ? atoi(getenv("HB_MIN_SEG_FAR")) : 32;
    const int seg_floor = std::max(1, std::min(32, CLS == 2 ? min_far : min_seg));
    static const int ipw = getenv("HB_ITEMS_PER_WARP_M") ? std::max(1, atoi(getenv("HB_ITEMS_PER_WARP_M"))) : 16;
    while (B.seg_len > seg_floor && rows * cdiv(A.m.E_x, (int64_t)B.seg_len) < ipw * warps) B.seg_len /= 2;
    const int64_t items = (CLS == 1 || CLS == 4 ? rows * A.m.sing_max_per_row : 0) +
                          (CLS == 1 ? 0 : rows * cdiv(A.m.E_x, (int64_t)B.seg_len));
    // (near-pair items: most segments hold none and exit after the classification)
    if (items == 0) return HB_OK;
    const int64_t grid = std::max<int64_t>(1, std::min<int64_t>((int64_t)std::max(1, per_sm) * nsm, cdiv(items, HB_PAIR_WARPS)));
    int rc = cuda_check(cudaMemsetAsync(A.counter, 0, sizeof(unsigned long long), st), "counter reset");
    if (rc) return rc;
    kp<<<(unsigned)grid, HB_PAIR_WARPS * 32, sm, st>>>(B);
    return cuda_check(cudaGetLastError(), "pair kernel");
}

static bool merge_tn()
{
    static const bool merge = !getenv("HB_MERGE_TN") || atoi(getenv("HB_MERGE_TN")) != 0;
    return merge;
}

template <int OP, bool TP1, bool SP1, int NJ, bool DUAL = false>
static int launch_pairs(const PairArgs &A, cudaStream_t st)
{
    // touching and near pairs (warp per pair) in one launch: the cheap segment
    // items fill in behind the heavy touching ones (one kernel tail instead of
    // two); HB_MERGE_TN=0: separate launches
    // (all three classes in one launch: measured slower -- V 1.38 vs 1.10 ms at
    // config 2 -- the far batches' register-heavy path and the warp-per-pair
    // path then share SMs)
    int rc;
    if (merge_tn()) {
        rc = launch_class<OP, TP1, SP1, NJ, DUAL, 4>(A, st);
    } else {
        rc = launch_class<OP, TP1, SP1, NJ, DUAL, 1>(A, st);
        if (!rc) rc = launch_class<OP, TP1, SP1, NJ, DUAL, 3>(A, st);
    }
    if (!rc && A.moments) rc = launch_class<OP, TP1, SP1, NJ, DUAL, 2>(A, st);   // far batches
    return rc;
}

static int run_pairs(const hb_assembly_desc *a, const PairArgs &A, cudaStream_t st)
{
    if (a->op == 0 && !a->test_p1) return launch_pairs<0, false, false, kNJ>(A, st);
    if (a->op == 0 && a->test_p1) return launch_pairs<0, true, true, kNJ>(A, st);
    if (a->op == 1) {
        // K: both orientations of a separated pair per evaluation (HB_K_DUAL=0: off).  A pair
        // whose other row lies outside the launch's rows (row chunks, row-parallel ranks) is
        // evaluated in the same canonical orientation with only the needed output's
        // accumulators, so the blocks stay independent of the row split.
        static const bool dual_on = !getenv("HB_K_DUAL") || atoi(getenv("HB_K_DUAL")) != 0;
        if (dual_on) return launch_pairs<1, false, true, kNJ, true>(A, st);
        return launch_pairs<1, false, true, kNJ>(A, st);
    }
    return launch_pairs<2, true, true, kNJ>(A, st);
}

// the direct pair kernel (csrc/hb_pairs_direct.cu): one 32-gap window
int direct_pairs(const hb_mesh_desc *m, const hb_assembly_desc *a, int64_t e0, int64_t e1, int d0, int d1,
                 double *Q, unsigned long long *counter, cudaStream_t st);
void direct_window(int64_t E_t, int64_t d, int &w0, int &w1);   // hb_pairs_direct.cu

static int moment_table(const hb_assembly_desc *a, const PairArgs &A, double *Tm, cudaStream_t st)
{
    const int nd = (int)(a->d_end - a->d_begin);
    const int n = kNK * nd + kNK + 1;
    const unsigned grid = (unsigned)std::max(1, std::min(148, (n + 255) / 256));
    if (a->op == HB_OP_SINGLE_LAYER) k_moment_table<0><<<grid, 256, 0, st>>>(Tm, (int)a->d_begin, nd, A.mom_S, A.mom_q0);
    else if (a->op == HB_OP_DOUBLE_LAYER) k_moment_table<1><<<grid, 256, 0, st>>>(Tm, (int)a->d_begin, nd, A.mom_S, A.mom_q0);
    else k_moment_table<2><<<grid, 256, 0, st>>>(Tm, (int)a->d_begin, nd, A.mom_S, A.mom_q0);
    return cuda_check(cudaGetLastError(), "moment table");
}

}  // namespace hb

using namespace hb;

extern "C" size_t hb_assemble_min_workspace(const hb_mesh_desc *m, const hb_assembly_desc *a)
{
    if (!m || !a) return 0;
    return row_bytes(m, a) + tm_bytes(a) + kCounterBytes;
}

extern "C" size_t hb_assemble_full_workspace(const hb_mesh_desc *m, const hb_assembly_desc *a)
{
    if (!m || !a) return 0;
    return row_bytes(m, a) * (size_t)m->E_x + tm_bytes(a) + kCounterBytes;
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

namespace hb {
// pair-kernel arguments of one operator call (everything but the staging
// pointers and the row range)
static PairArgs make_pair_args(const hb_mesh_desc *m, const hb_assembly_desc *a)
{
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
    {   // moment form: u = 2 sqrt(alpha h); V: S = u / (2 a^2), q0 = 1/2; K, D2: S = 1/u, q0 = -1/2
        const double u = 2.0 * sqrt(a->alpha * a->step);
        A.inv_u2 = 1.0 / (u * u);
        A.mom_S = (a->op == HB_OP_SINGLE_LAYER) ? u * A.inv2a2 : 1.0 / u;
        A.mom_q0 = (a->op == HB_OP_SINGLE_LAYER) ? 0.5 : -0.5;
    }
    A.halve_diag = (a->test_p1 && a->trial_p1) ? 1 : 0;
    // one launch per test-row chunk covers all blocks [d_begin, d_end) in the
    // moment form: each pair computes its moments once and its per-point gap
    // windows inside the kernel
    A.d0 = (int)a->d_begin;
    A.d1 = (int)a->d_end;
    A.nd = (int)(a->d_end - a->d_begin);
    A.need_special = a->d_begin <= 1;
    A.moments = use_moments(a);
    return A;
}

// gap windows of a call: the moment form covers all blocks in one; the direct
// form windows of <= 32 gap slots (the first from block 0 or 1 holds 32 blocks,
// later ones 30)
// direct windows are the global ones of direct_window ([0, 32), [32, 62), ...)
// clipped to the call's range: a call's blocks are computed in the same warps
// whatever its d-range (d-sharded ranks, chunks reproduce the 1-GPU blocks)
static int64_t window_end(const hb_assembly_desc *a, bool moments, int64_t d0)
{
    if (moments) return a->d_end;
    int w0, w1;
    direct_window(a->E_t, d0, w0, w1);
    return std::min<int64_t>(a->d_end, w1);
}

// the pair kernels of rows [e0, e1) and blocks [d0, d1) into staging A.Q
static int pairs_window(const hb_mesh_desc *m, const hb_assembly_desc *a, PairArgs &A, int64_t e0, int64_t e1,
                        int64_t d0, int64_t d1, LaunchTimer &LT, cudaStream_t st)
{
    A.e0 = e0;
    A.e1 = e1;
    cudaEvent_t ev = LT.begin(st);
    int rc;
    if (A.moments) {
        rc = run_pairs(a, A, st);   // touching + near pairs, far batches (or three launches)
        LT.launches += merge_tn() ? 2 : 3;
        LT.pair_launches += merge_tn() ? 2 : 3;
    } else {
        rc = direct_pairs(m, a, e0, e1, (int)d0, (int)d1, A.Q, A.counter, st);
        LT.launches += 1;
        LT.pair_launches += 1;
    }
    if (rc) return rc;
    LT.end(ev, true, st);
    return HB_OK;
}

static FinArgs fin_args(const hb_mesh_desc *m, const hb_assembly_desc *a, const double *Q, int64_t e0, int64_t e1,
                        int64_t d0, int nd_w)
{
    FinArgs F{};
    F.Q = Q;
    F.out = a->blocks_dev;
    F.bptr = a->block_ptrs_dev;
    F.nrs = (int)a->n_row_shards;
    F.rs_bounds = a->row_shard_bounds_dev;
    F.rs_ptrs = a->row_shard_ptrs_dev;
    F.E_x = m->E_x; F.N_x = m->N_x;
    F.R = a->test_p1 ? m->N_x : m->E_x;
    F.C = a->trial_p1 ? m->N_x : m->E_x;
    F.e0 = e0; F.e1 = e1;
    F.d0 = (int)d0; F.nd = nd_w; F.d_begin = (int)a->d_begin;
    F.star_indptr = m->star_indptr_dev; F.star_elem = m->star_elem_dev;
    F.star_local = m->star_local_dev; F.tri_nodes = m->tri_nodes_dev;
    F.normals = m->normals_dev; F.skip_zero_dot = a->op == HB_OP_HYPERSINGULAR2;
    F.star_max = (int)m->star_max;
    F.tile_eptr = m->curl_tile_eptr_dev; F.tile_elem = m->curl_tile_elem_dev; F.star_pos = m->curl_star_pos_dev;
    return F;
}

static size_t fin_p1p1_smem(const hb_mesh_desc *m, bool fuse)
{
    const size_t sm = (size_t)m->star_max;
    size_t b = sm * ((2 + kWarps) * sizeof(int64_t) + kFinMaxW * sizeof(unsigned) + kWarps * sizeof(int));
    if (fuse) b += sizeof(double) * 4 * sm * (1 + kWarps);
    return b;
}

// staging -> blocks for one window of one row chunk
static int finalize_window(const hb_mesh_desc *m, const hb_assembly_desc *a, const FinArgs &F, LaunchTimer &LT,
                           cudaStream_t st)
{
    cudaEvent_t ev = LT.begin(st);
    const int64_t rows = F.e1 - F.e0;
    if (!a->test_p1 && !a->trial_p1) {
        dim3 g((unsigned)cdiv(m->E_x, 32), (unsigned)cdiv(rows, 4));
        k_fin_p0p0<<<g, 256, 0, st>>>(F);
    } else if (!a->test_p1) {
        dim3 g((unsigned)rows, (unsigned)cdiv(m->N_x, 32));
        k_fin_p0p1<<<g, 256, 0, st>>>(F);
    } else {
        FinArgs G = F;
        static const int ng_env = getenv("HB_FIN_NODE_GRID") ? atoi(getenv("HB_FIN_NODE_GRID")) : -1;
        G.node_grid = ng_env >= 0 ? ng_env : (3 * rows >= m->N_x ? 1 : 0);
        dim3 g((unsigned)(G.node_grid ? m->N_x : 3 * rows), (unsigned)cdiv(m->N_x, 32));
        if (G.Qv) k_fin_p1p1_accum<true><<<g, 256, fin_p1p1_smem(m, true), st>>>(G);
        else k_fin_p1p1_accum<false><<<g, 256, fin_p1p1_smem(m, false), st>>>(G);
    }
    int rc = cuda_check(cudaGetLastError(), "finalize");
    if (rc) return rc;
    LT.end(ev, false, st);
    LT.launches += 1;
    return HB_OK;
}

// X <- X + X^T on every block of a p1 x p1 call
static int symmetrize_blocks(double *blocks, int64_t R, int64_t nb, LaunchTimer &LT, cudaStream_t st)
{
    const int64_t nt = cdiv(R, 32);
    for (int64_t b0 = 0; b0 < nb; b0 += 65535) {
        dim3 g((unsigned)(nt * (nt + 1) / 2), (unsigned)std::min<int64_t>(65535, nb - b0));
        cudaEvent_t ev = LT.begin(st);
        k_symmetrize<<<g, 256, 0, st>>>(blocks, R, b0);
        int rc = cuda_check(cudaGetLastError(), "symmetrize");
        if (rc) return rc;
        LT.end(ev, false, st);
        LT.launches += 1;
    }
    return HB_OK;
}

static int check_desc(const hb_mesh_desc *m, const hb_assembly_desc *a, const char *who)
{
    if (!combo_ok(a)) {
        set_error("%s: unsupported op/space combination (op=%d test_p1=%d trial_p1=%d sym=%d)", who, a->op,
                  a->test_p1, a->trial_p1, a->symmetric);
        return HB_ERR_UNSUPPORTED;
    }
    if (a->E_t < 1 || a->d_begin < 0 || a->d_end > a->E_t || a->d_begin >= a->d_end || m->E_x < 1 ||
        m->N_x < 3 || !(a->step > 0) || !(a->alpha > 0)) {
        set_error("%s: invalid sizes or parameters (E_t=%lld d=[%lld,%lld) E_x=%lld)", who, (long long)a->E_t,
                  (long long)a->d_begin, (long long)a->d_end, (long long)m->E_x);
        return HB_ERR_INVALID;
    }
    if (a->test_p1 && a->trial_p1 &&
        (!m->curl_tile_eptr_dev || !m->curl_tile_elem_dev || !m->curl_star_pos_dev ||
         m->curl_tile_emax > 32 * kFinMaxW)) {
        set_error("%s: p1 x p1 needs the mesh tile plan with <= %d elements per 32-node tile", who, 32 * kFinMaxW);
        return HB_ERR_UNSUPPORTED;
    }
    return HB_OK;
}

// the single layer's descriptor of a fused V + D call
static hb_assembly_desc vd_single_layer(const hb_assembly_desc *d2, double *V_blocks_dev)
{
    hb_assembly_desc v = *d2;
    v.op = HB_OP_SINGLE_LAYER;
    v.test_p1 = v.trial_p1 = 0;
    v.symmetric = 1;
    v.blocks_dev = V_blocks_dev;
    v.stats = nullptr;
    return v;
}
}  // namespace hb

extern "C" int hb_assemble(const hb_mesh_desc *m, const hb_assembly_desc *a, void *stream)
{
    if (!m || !a) { set_error("hb_assemble: null descriptor"); return HB_ERR_INVALID; }
    int rc = check_desc(m, a, "hb_assemble");
    if (rc) return rc;
    const int64_t r0 = a->row_end > a->row_begin ? a->row_begin : 0;
    const int64_t r1 = a->row_end > a->row_begin ? a->row_end : m->E_x;
    if (r0 < 0 || r1 > m->E_x || r0 >= r1 || (a->test_p1 && a->trial_p1 && a->block_ptrs_dev)) {
        set_error("hb_assemble: bad test-row range [%lld, %lld) (p1 x p1 operators accumulate over rows: "
                  "contiguous blocks only; a row range gives those rows' partial sum)", (long long)r0,
                  (long long)r1);
        return HB_ERR_INVALID;
    }
    if (a->n_row_shards < 0 ||
        (a->n_row_shards > 0 && (a->test_p1 || a->block_ptrs_dev || !a->row_shard_bounds_dev ||
                                 !a->row_shard_ptrs_dev))) {
        set_error("hb_assemble: row-sharded output needs p0 test functions, bounds and pointers, and no "
                  "block_ptrs_dev");
        return HB_ERR_INVALID;
    }
    if (!a->blocks_dev && !a->block_ptrs_dev && a->n_row_shards == 0) {
        set_error("hb_assemble: no output (blocks_dev, block_ptrs_dev and row shards all absent)");
        return HB_ERR_INVALID;
    }
    cudaStream_t st = (cudaStream_t)stream;
    const size_t rb = row_bytes(m, a), tb = tm_bytes(a);
    if (!a->workspace_dev || a->workspace_bytes < rb + tb + kCounterBytes) {
        set_error("hb_assemble: workspace %zu bytes < one row chunk (%zu bytes)", a->workspace_bytes,
                  rb + tb + kCounterBytes);
        return HB_ERR_WORKSPACE;
    }
    // workspace: [staging Q: row chunks][moment table][counter]
    const size_t q_bytes = (a->workspace_bytes - kCounterBytes - tb) & ~(size_t)255;
    const int64_t rows_per_chunk = std::max<int64_t>(1, std::min<int64_t>(m->E_x, (int64_t)(q_bytes / rb)));
    const int64_t R = a->test_p1 ? m->N_x : m->E_x;
    const int64_t nb = a->d_end - a->d_begin;
    const bool p1p1 = a->test_p1 && a->trial_p1;
    if (p1p1) {
        rc = cuda_check(cudaMemsetAsync(a->blocks_dev, 0, (size_t)nb * R * R * sizeof(double), st), "memset");
        if (rc) return rc;
    }
    double *Tm = (double *)((char *)a->workspace_dev + q_bytes);
    LaunchTimer LT{a->stats, st};
    CallPart parts[2];
    const int nparts = call_parts(a, parts);
    for (int ip = 0; ip < nparts; ++ip) {
        // the part's blocks: its own pair arguments and windows; the finalize
        // stores through the call's descriptor (block offsets from d_begin)
        hb_assembly_desc ap = *a;
        ap.d_begin = parts[ip].lo;
        ap.d_end = parts[ip].hi;
        PairArgs A = make_pair_args(m, &ap);
        A.Q = (double *)a->workspace_dev;
        A.Tm = Tm;
        A.counter = (unsigned long long *)((char *)a->workspace_dev + q_bytes + tb);
        if (A.moments) {
            cudaEvent_t ev = LT.begin(st);
            rc = moment_table(&ap, A, Tm, st);
            if (rc) return rc;
            LT.end(ev, false, st);
            LT.launches += 1;
        }
        for (int64_t d0 = ap.d_begin; d0 < ap.d_end;) {
            const int64_t d1 = window_end(&ap, A.moments, d0);
            for (int64_t e0 = r0; e0 < r1; e0 += rows_per_chunk) {
                const int64_t e1 = std::min(r1, e0 + rows_per_chunk);
                rc = pairs_window(m, &ap, A, e0, e1, d0, d1, LT, st);
                if (rc) return rc;
                rc = finalize_window(m, a, fin_args(m, a, A.Q, e0, e1, d0, (int)(d1 - d0)), LT, st);
                if (rc) return rc;
            }
            d0 = d1;
        }
    }
    if (p1p1) {
        rc = symmetrize_blocks(a->blocks_dev, R, nb, LT, st);
        if (rc) return rc;
    }
    return LT.finish();
}

// fused V + D (hb_assemble_vd): staging of one test row for both operators
static size_t vd_row_bytes(const hb_mesh_desc *m, const hb_assembly_desc *d2)
{
    const hb_assembly_desc v = vd_single_layer(d2, nullptr);
    return row_bytes(m, &v) + row_bytes(m, d2);
}

static size_t vd_fixed_bytes(const hb_assembly_desc *d2)
{
    const hb_assembly_desc v = vd_single_layer(d2, nullptr);
    return tm_bytes(&v) + tm_bytes(d2) + kCounterBytes;
}

extern "C" size_t hb_assemble_vd_min_workspace(const hb_mesh_desc *m, const hb_assembly_desc *d2)
{
    if (!m || !d2) return 0;
    return vd_row_bytes(m, d2) + vd_fixed_bytes(d2) + 512;
}

extern "C" size_t hb_assemble_vd_full_workspace(const hb_mesh_desc *m, const hb_assembly_desc *d2)
{
    if (!m || !d2) return 0;
    return vd_row_bytes(m, d2) * (size_t)m->E_x + vd_fixed_bytes(d2) + 512;
}

extern "C" int hb_assemble_vd(const hb_mesh_desc *m, const hb_assembly_desc *d2, double *V_blocks_dev,
                              const double *curls_dev, void *stream)
{
    if (!m || !d2 || !curls_dev || !d2->blocks_dev) {
        set_error("hb_assemble_vd: null descriptor, curls or D blocks");
        return HB_ERR_INVALID;
    }
    if (d2->op != HB_OP_HYPERSINGULAR2 || d2->row_end > d2->row_begin || d2->block_ptrs_dev || d2->n_row_shards) {
        set_error("hb_assemble_vd: needs the hypersingular (D2) descriptor over all rows, contiguous blocks");
        return HB_ERR_INVALID;
    }
    int rc = check_desc(m, d2, "hb_assemble_vd");
    if (rc) return rc;
    if (m->star_max > 64) {
        set_error("hb_assemble_vd: node stars of more than 64 elements");
        return HB_ERR_UNSUPPORTED;
    }
    const hb_assembly_desc v = vd_single_layer(d2, V_blocks_dev);
    {
        CallPart pv[2], pd[2];
        if (call_parts(&v, pv) != 1 || call_parts(d2, pd) != 1) {
            set_error("hb_assemble_vd: calls whose blocks straddle the direct / moment switch (E_t >= 64) are not "
                      "fused; use hb_assemble + hb_curl_combine");
            return HB_ERR_UNSUPPORTED;
        }
    }
    cudaStream_t st = (cudaStream_t)stream;
    const size_t rbv = row_bytes(m, &v), rbd = row_bytes(m, d2), tbv = tm_bytes(&v), tbd = tm_bytes(d2);
    if (!d2->workspace_dev || d2->workspace_bytes < hb_assemble_vd_min_workspace(m, d2)) {
        set_error("hb_assemble_vd: workspace %zu bytes < one row chunk (%zu bytes)", d2->workspace_bytes,
                  hb_assemble_vd_min_workspace(m, d2));
        return HB_ERR_WORKSPACE;
    }
    // workspace: [Q_V: row chunk][Q_D2: row chunk][Tm_V][Tm_D2][counter]
    const size_t avail = d2->workspace_bytes - tbv - tbd - kCounterBytes - 512;
    const int64_t rows_per_chunk = std::max<int64_t>(1, std::min<int64_t>(m->E_x, (int64_t)(avail / (rbv + rbd))));
    char *ws = (char *)d2->workspace_dev;
    const size_t qv_bytes = ((size_t)rows_per_chunk * rbv + 255) & ~(size_t)255;
    const size_t qd_bytes = ((size_t)rows_per_chunk * rbd + 255) & ~(size_t)255;
    PairArgs AV = make_pair_args(m, &v), AD = make_pair_args(m, d2);
    if (!AV.moments && AD.moments) {
        set_error("hb_assemble_vd: direct single layer with a moment-form D2 (HB_MOMENTS override) is not fused");
        return HB_ERR_UNSUPPORTED;
    }
    AV.Q = (double *)ws;
    AD.Q = (double *)(ws + qv_bytes);
    AV.Tm = (double *)(ws + qv_bytes + qd_bytes);
    AD.Tm = (double *)(ws + qv_bytes + qd_bytes + tbv);
    AV.counter = AD.counter = (unsigned long long *)(ws + qv_bytes + qd_bytes + tbv + tbd);
    const int64_t N = m->N_x, nb = d2->d_end - d2->d_begin;
    rc = cuda_check(cudaMemsetAsync(d2->blocks_dev, 0, (size_t)nb * N * N * sizeof(double), st), "memset");
    if (rc) return rc;
    LaunchTimer LT{d2->stats, st};
    if (AV.moments) { rc = moment_table(&v, AV, const_cast<double *>(AV.Tm), st); if (rc) return rc; LT.launches += 1; }
    if (AD.moments) { rc = moment_table(d2, AD, const_cast<double *>(AD.Tm), st); if (rc) return rc; LT.launches += 1; }
    for (int64_t e0 = 0; e0 < m->E_x; e0 += rows_per_chunk) {
        const int64_t e1 = std::min(m->E_x, e0 + rows_per_chunk);
        if (AV.moments) {   // V staging of all blocks of the call
            rc = pairs_window(m, &v, AV, e0, e1, v.d_begin, v.d_end, LT, st);
            if (!rc && V_blocks_dev) rc = finalize_window(m, &v, fin_args(m, &v, AV.Q, e0, e1, v.d_begin, (int)nb), LT, st);
            if (rc) return rc;
        }
        for (int64_t d0 = d2->d_begin; d0 < d2->d_end;) {
            const int64_t d1 = window_end(d2, AD.moments, d0);
            if (!AV.moments) {   // direct V: the same windows as the direct D2
                rc = pairs_window(m, &v, AV, e0, e1, d0, d1, LT, st);
                if (!rc && V_blocks_dev)
                    rc = finalize_window(m, &v, fin_args(m, &v, AV.Q, e0, e1, d0, (int)(d1 - d0)), LT, st);
                if (rc) return rc;
            }
            rc = pairs_window(m, d2, AD, e0, e1, d0, d1, LT, st);
            if (rc) return rc;
            FinArgs F = fin_args(m, d2, AD.Q, e0, e1, d0, (int)(d1 - d0));
            F.Qv = AV.Q;
            F.ndv = AV.moments ? (int)nb : (int)(d1 - d0);
            F.dv_off = AV.moments ? (int)(d0 - d2->d_begin) : 0;
            F.a2 = d2->alpha * d2->alpha;
            F.curls = curls_dev;
            rc = finalize_window(m, d2, F, LT, st);
            if (rc) return rc;
            d0 = d1;
        }
    }
    rc = symmetrize_blocks(d2->blocks_dev, N, nb, LT, st);
    if (rc) return rc;
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
