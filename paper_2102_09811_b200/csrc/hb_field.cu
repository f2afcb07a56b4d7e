// hb_field.cu -- interior potentials (representation formula), sm_100a.
//
// Replaces heatbem/_field_numba.py:15-79 (_eval_potential).  For an
// evaluation point (x, t = k h + eps) the reference sums, per element e and
// quadrature node q,
//     s = sum_{m=0..k} c_m G(rho, m h + eps)      (+ dens[k] G(rho, 0) if cur)
//     c_m = dens[k-1-m] - dens[k-m] * [k-m < k or cur]
// and recomputes every G for every output time.  The G values depend on
// (x, eps, m) only, so outputs that share (x, eps) -- one spatial point at
// all time-step ends -- share them: one CTA owns such a group; its warps split
// the elements, the lanes of a warp first evaluate G(m), m = 0..kmax, once
// per (e, q) into shared memory, then each lane contracts them with the
// density differences of its two output times (one merged loop, so lanes
// with short and long histories stay in step).  Per-warp partial sums are
// added in fixed warp order: results are deterministic.
//
// Kernels (x = rho / (2 sqrt(a gap)), gap = m h + eps):
//   single layer: G^{dtau}         = erf(x) / (4 pi a rho)
//   double layer: a dG^{dtau}/dn_y = rn / (4 pi rho^3) * E(x),
//                 E(x) = erf(x) - 2x e^{-x^2}/sqrt(pi)
// erf and E come from the fused evaluator (hb_special.cuh); E is evaluated
// without the small-x cancellation of the reference's
// erf(x)/rho - e^{-x^2}/sqrt(pi a gap) form.  The reference's branches are
// kept: gap <= d_eps (first for the single layer), rho <= r_eps.
// The sums keep the reference's order (m, then q, then e within a warp).
#include <algorithm>
#include <cmath>
#include <cstdlib>

#include <cooperative_groups.h>

#include "hb_common.cuh"
#include "hb_special.cuh"

namespace cg = cooperative_groups;

namespace hb {

struct PotArgs {
    int kind;
    int64_t n_groups, E_t, E_x, nq;
    const double *gx;          // (n_groups, 3)
    const double *geps;        // (n_groups,)
    const int64_t *gptr;       // (n_groups+1,) outputs of each group
    const int64_t *k;          // (n_out,) completed intervals per output (ascending in a group)
    const uint8_t *cur;        // (n_out,)
    const int64_t *out_idx;    // (n_out,) position in the caller's point list
    const double *dens_t;      // (E_x, nq, E_t) density, time fastest
    const double *qpts, *qw, *areas, *normals;
    double step, alpha, d_eps, r_eps;
    double *out;
    int kcap;                  // per-warp smem capacity of the G / A / B / C arrays
    int skip_eps0;             // k_potential_tiles: leave eps = 0 groups to k_potential_reg
};

constexpr int kPotWarps = 8;
constexpr int kOut = 64;       // outputs per pass (2 per lane)

template <int KIND>
__global__ void __launch_bounds__(kPotWarps * 32) k_potential(const PotArgs P)
{
    extern __shared__ __align__(16) double psm[];
    double *tab = psm;
    special::load_table<KIND == 0 ? 2 : 3>(tab);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double *red = psm + special::kTabDoubles;                  // [kPotWarps][kOut]
    double *G = red + kPotWarps * kOut + warp * 4 * P.kcap;    // G(m)
    double *A = G + P.kcap;                                    // dens[j], 0 outside [0, E_t)
    double *B = A + P.kcap;                                    // A[j-1] - A[j]
    double *C = B + P.kcap;                                    // 1 / (2 sqrt(a gap_m))
    __syncthreads();
    const double inv4pi = 0.25 * kInvPi;
    for (int64_t grp = blockIdx.x; grp < P.n_groups; grp += gridDim.x) {
        const double px = P.gx[3 * grp], py = P.gx[3 * grp + 1], pz = P.gx[3 * grp + 2];
        const double eps = P.geps[grp];
        const int64_t o0 = P.gptr[grp], o1 = P.gptr[grp + 1];
        for (int64_t ob = o0; ob < o1; ob += kOut) {
            const int64_t oi1 = ob + lane, oi2 = ob + kOut - 1 - lane;
            const bool ok1 = oi1 < o1, ok2 = oi2 < o1;
            const int k1 = ok1 ? (int)P.k[oi1] : 0, k2 = ok2 ? (int)P.k[oi2] : 0;
            const bool cu1 = ok1 && P.cur[oi1] != 0, cu2 = ok2 && P.cur[oi2] != 0;
            int kmax = max(k1, k2);
            for (int o = 16; o >= 1; o >>= 1) kmax = max(kmax, __shfl_xor_sync(kFull, kmax, o));
            const int rounds = kmax / 32 + 1;
            for (int m = lane; m <= kmax; m += 32) C[m] = 1.0 / (2.0 * sqrt(P.alpha * ((double)m * P.step + eps)));
            __syncwarp();
            double acc1 = 0.0, acc2 = 0.0;
            for (int64_t e = warp; e < P.E_x; e += kPotWarps) {
                const double nyx = __ldg(P.normals + 3 * e), nyy = __ldg(P.normals + 3 * e + 1),
                             nyz = __ldg(P.normals + 3 * e + 2);
                double el1 = 0.0, el2 = 0.0;
                for (int64_t q = 0; q < P.nq; ++q) {
                    const double *y = P.qpts + 3 * (e * P.nq + q);
                    const double rx = px - __ldg(y), ry = py - __ldg(y + 1), rz = pz - __ldg(y + 2);
                    const double rho = sqrt(rx * rx + ry * ry + rz * rz);
                    const double rn = rx * nyx + ry * nyy + rz * nyz;
                    const bool rsmall = rho <= P.r_eps;
                    const double lim0 = KIND == 0 ? 1.0 / (4.0 * kPi * P.alpha * rho) : (rsmall ? 0.0 : inv4pi * rn / (rho * rho * rho));
                    const double *dq = P.dens_t + (e * P.nq + q) * P.E_t;
                    for (int r = 0; r < rounds; ++r) {
                        const int m = lane + 32 * r;
                        const int mc = m <= kmax ? m : kmax;
                        const double gap = (double)mc * P.step + eps;
                        const double x = __dmul_rn(rho, C[mc]);
                        const double f = special::eval<KIND == 0 ? 2 : 3>(x, 0.0, tab, kFull);
                        double g;
                        if (gap <= P.d_eps) g = lim0;
                        else if (rsmall) g = KIND == 0 ? 1.0 / (4.0 * sqrt((kPi * kPi * kPi) * (P.alpha * P.alpha * P.alpha) * gap)) : 0.0;
                        else g = __dmul_rn(lim0, f);
                        const double a = m < P.E_t ? __ldg(dq + m) : 0.0;
                        const double am = (m >= 1 && m - 1 < P.E_t) ? __ldg(dq + m - 1) : 0.0;
                        if (m <= kmax) {
                            G[m] = g;
                            A[m] = a;
                            B[m] = am - a;
                        }
                    }
                    __syncwarp();
                    // m = 0: c = dens[k-1] - dens[k] [cur];  m >= 1: c = B[k - m]
                    const double c1 = (k1 >= 1 ? A[k1 - 1] : 0.0) - (cu1 ? A[k1] : 0.0);
                    const double c2 = (k2 >= 1 ? A[k2 - 1] : 0.0) - (cu2 ? A[k2] : 0.0);
                    // two independent accumulation chains per output (even / odd m)
                    const int n1 = ok1 ? k1 : 0, n2 = ok2 ? k2 : 0;
                    double s1 = fma(c1, G[0], 0.0), s2 = fma(c2, G[0], 0.0), s1b = 0.0, s2b = 0.0;
                    {
                        const double *b = B + k1;
                        int m = 1;
                        for (; m + 1 <= n1; m += 2) {
                            s1b = fma(b[-m], G[m], s1b);
                            s1 = fma(b[-m - 1], G[m + 1], s1);
                        }
                        if (m <= n1) s1b = fma(b[-m], G[m], s1b);
                    }
                    {
                        const double *b = B + k2;
                        int m = 1;
                        for (; m + 1 <= n2; m += 2) {
                            s2b = fma(b[-m], G[m], s2b);
                            s2 = fma(b[-m - 1], G[m + 1], s2);
                        }
                        if (m <= n2) s2b = fma(b[-m], G[m], s2b);
                    }
                    s1 += s1b;
                    s2 += s2b;
                    if (cu1 && k1 < P.E_t) s1 = fma(A[k1], lim0, s1);
                    if (cu2 && k2 < P.E_t) s2 = fma(A[k2], lim0, s2);
                    const double w = __ldg(P.qw + q);
                    el1 = fma(w, s1, el1);
                    el2 = fma(w, s2, el2);
                    __syncwarp();
                }
                const double a2 = 2.0 * __ldg(P.areas + e);
                acc1 = fma(a2, el1, acc1);
                acc2 = fma(a2, el2, acc2);
            }
            red[warp * kOut + lane] = acc1;
            red[warp * kOut + kOut - 1 - lane] = acc2;
            __syncthreads();
            if (warp == 0) {
                for (int h = 0; h < 2; ++h) {
                    const int o = h == 0 ? lane : kOut - 1 - lane;
                    const int64_t oi = ob + o;
                    if (oi < o1) {
                        double v = 0.0;
                        for (int w = 0; w < kPotWarps; ++w) v += red[w * kOut + o];
                        P.out[P.out_idx[oi]] = v;
                    }
                }
            }
            __syncthreads();
        }
    }
}

// ---------------------------------------------------------------------------
// Tiled form for histories kmax <= 64 (config 4: every output time of 1e5
// points).  With W = 2 area_e w_q, A_eq[k] = W dens[k] (0 for k >= E_t) and
// B_eq[j] = W (dens[j-1] - dens[j]), the reference's sum is
//     u(k) = sum_{m=0..k} S[k-m][m] + (cur ? U[k] : U0[k]),
//     S[j][m] = sum_eq B_eq[j] G_eq[m],  U[k] = sum_eq A_eq[k] lim0_eq,
//     U0[k] = sum_eq A_eq[k] G_eq[0]
// (the m = 0 coefficient dens[k-1] - cur dens[k] is B[k] + (1 - cur) dens[k],
// and the current-interval term adds cur dens[k] lim0).  S is a small GEMM
// over the 36 864 (element, node) pairs: one CTA owns kTP points, stages the
// density rows of kTC pairs once for all of them, evaluates their G values
// into shared memory, and accumulates 4 x 4 register tiles of S (only the 153
// tiles with j + m <= 64; (point, tile) items spread <= 2 per thread).  The
// anti-diagonal sums are reduced in a fixed order: deterministic.
constexpr int kTP = 3;                  // points per CTA
#ifndef HB_POT_TC
#define HB_POT_TC 16
#endif
#ifndef HB_POT_UNROLL
#define HB_POT_UNROLL 4
#endif
constexpr int kTC = HB_POT_TC;          // (element, node) pairs per chunk
constexpr int kTUnroll = HB_POT_UNROLL;
constexpr int kTK = 68;                 // j, m in [0, 68): 17 tiles of 4
constexpr int kTW = 85;                 // padded row: element m at m + m / 4 (chunks of 4 at a
                                        // 40-byte stride -> tiles of a warp hit distinct banks)
__device__ __forceinline__ int tpad(int m) { return m + (m >> 2); }
constexpr int kNTile = 153;             // tiles (jt, mt), jt + mt <= 16
constexpr int kTItems = kTP * kNTile;   // 459
constexpr int kTThreads = 256;
constexpr int kTMaxK = 64;

// tiles enumerated jt-major (lanes of a warp mostly share the j-tile: the B
// loads broadcast): id = off(jt) + mt, off(jt) = 17 jt - jt (jt - 1) / 2
__device__ __forceinline__ int tile_off(int jt) { return 17 * jt - jt * (jt - 1) / 2; }
__device__ __forceinline__ void tile_of(int t, int &jt, int &mt)
{
    jt = 0;
    while (tile_off(jt + 1) <= t) ++jt;
    mt = t - tile_off(jt);
}

template <int KIND>
__global__ void __launch_bounds__(kTThreads, 2) k_potential_tiles(const PotArgs P)
{
    extern __shared__ __align__(16) double tsm[];
    double *tab = tsm;
    double *As = tab + special::kTabDoubles;          // [kTC][kTW]
    double *Bs = As + kTC * kTW;                      // [kTC][kTW]
    double *Gs = Bs + kTC * kTW;                      // [kTP][kTC][kTW]; later T [kTItems][7]
    double *Ls = Gs + kTP * kTC * kTW;                // [kTP][kTC]
    double *Cm = Ls + kTP * kTC;                      // [kTP][kTK]: 1 / (2 sqrt(a (m h + eps)))
    double *Gq = Cm + kTP * kTK;                      // [kTP][kTC][2]: rho
    double *Rs = Gq + kTP * kTC * 2;                  // [3][kTP][65]: R, U, U0
    special::load_table<KIND == 0 ? 2 : 3>(tab);
    const int tid = threadIdx.x, lane = tid & 31;
    const int64_t g0 = (int64_t)blockIdx.x * kTP;
    const int64_t EQ = P.E_x * P.nq;
    double px[kTP], py[kTP], pz[kTP];
    if (P.skip_eps0) {   // every group of this CTA at a time-step end: k_potential_reg owns them
        bool any = false;
        for (int p = 0; p < kTP; ++p) any |= g0 + p < P.n_groups && P.geps[g0 + p] != 0.0;
        if (!any) return;
    }
    int kmax = 0;
#pragma unroll
    for (int p = 0; p < kTP; ++p) {
        const int64_t g = min(g0 + p, P.n_groups - 1);
        px[p] = P.gx[3 * g]; py[p] = P.gx[3 * g + 1]; pz[p] = P.gx[3 * g + 2];
        if (g0 + p < P.n_groups) kmax = max(kmax, (int)P.k[P.gptr[g + 1] - 1]);
    }
    for (int i = tid; i < kTP * kTK; i += kTThreads) {
        const int p = i / kTK, m = i % kTK;
        const int64_t g = min(g0 + p, P.n_groups - 1);
        Cm[i] = 1.0 / (2.0 * sqrt(P.alpha * ((double)m * P.step + P.geps[g])));
    }
    // this thread's (point, tile) items
    int it_p[2], it_j[2], it_m[2];
    bool it_ok[2];
#pragma unroll
    for (int r = 0; r < 2; ++r) {
        const int item = tid + r * kTThreads;
        it_ok[r] = item < kTItems;
        const int ii = it_ok[r] ? item : 0;
        int jt, mt;
        tile_of(ii % kNTile, jt, mt);
        it_p[r] = ii / kNTile;
        it_j[r] = 4 * jt;
        it_m[r] = 4 * mt;
    }
    double acc[2][16];
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
        for (int c = 0; c < 16; ++c) acc[r][c] = 0.0;
    const bool xt = tid < kTP * 65;       // X-term cell (p, k)
    const int xp = xt ? tid / 65 : 0, xk = xt ? tid % 65 : 0;
    double U = 0.0, U0 = 0.0;
    const double inv4pi = 0.25 * kInvPi;
    constexpr int kEvalIters = (kTP * kTC * kTK + kTThreads - 1) / kTThreads;
    for (int64_t eq0 = 0; eq0 < EQ; eq0 += kTC) {
        __syncthreads();   // previous chunk fully consumed
        for (int i = tid; i < kTC * kTK; i += kTThreads) {
            const int el = i / kTK, kk = i % kTK;
            const int64_t eq = eq0 + el;
            double a = 0.0, am = 0.0, W = 0.0;
            if (eq < EQ) {
                const double *dq = P.dens_t + eq * P.E_t;
                W = 2.0 * __ldg(P.areas + eq / P.nq) * __ldg(P.qw + eq % P.nq);
                if (kk < P.E_t) a = __ldg(dq + kk);
                if (kk >= 1 && kk - 1 < P.E_t) am = __ldg(dq + kk - 1);
            }
            As[el * kTW + tpad(kk)] = W * a;
            Bs[el * kTW + tpad(kk)] = W * (am - a);
        }
        if (tid < kTP * kTC) {   // per (point, pair): rho and the gap-independent factor lim0
            const int p = tid / kTC, el = tid % kTC;
            const int64_t eq = eq0 + el;
            const int64_t e = eq < EQ ? eq / P.nq : 0, eqc = eq < EQ ? eq : 0;
            const double rx = (p == 0 ? px[0] : p == 1 ? px[1] : px[2]) - P.qpts[3 * eqc];
            const double ry = (p == 0 ? py[0] : p == 1 ? py[1] : py[2]) - P.qpts[3 * eqc + 1];
            const double rz = (p == 0 ? pz[0] : p == 1 ? pz[1] : pz[2]) - P.qpts[3 * eqc + 2];
            const double rho = sqrt(rx * rx + ry * ry + rz * rz);
            const double rn = rx * P.normals[3 * e] + ry * P.normals[3 * e + 1] + rz * P.normals[3 * e + 2];
            const bool rsmall = rho <= P.r_eps;
            const double lim0 = KIND == 0 ? 1.0 / (4.0 * kPi * P.alpha * rho)
                                          : (rsmall ? 0.0 : inv4pi * rn / (rho * rho * rho));
            Gq[tid * 2] = rho;
            Ls[tid] = eq < EQ ? lim0 : 0.0;
        }
        __syncthreads();
        // kernel values G(rho, m h + eps) for kTP points x kTC pairs x m < kTK
        // (uniform trip count: every lane takes part in the warp votes)
#pragma unroll 1
        for (int r = 0; r < kEvalIters; ++r) {
            const int i = tid + r * kTThreads;
            const bool ok = i < kTP * kTC * kTK;
            const int ic = ok ? i : 0;
            const int p = ic / (kTC * kTK), el = (ic / kTK) % kTC, m = ic % kTK;
            const double rho = Gq[(p * kTC + el) * 2];
            const bool rsmall = rho <= P.r_eps;
            const double lim0 = Ls[p * kTC + el];
            const int64_t g = min(g0 + p, P.n_groups - 1);
            const double gap = (double)m * P.step + P.geps[g];
            const double x = __dmul_rn(rho, Cm[p * kTK + m]);
            const double f = special::eval<KIND == 0 ? 2 : 3>(x, 0.0, tab, kFull);
            double gv;
            if (gap <= P.d_eps) gv = lim0;
            else if (rsmall) gv = KIND == 0 ? 1.0 / (4.0 * sqrt((kPi * kPi * kPi) * (P.alpha * P.alpha * P.alpha) * gap)) : 0.0;
            else gv = __dmul_rn(lim0, f);
            if (ok) Gs[(p * kTC + el) * kTW + tpad(m)] = (m <= kmax && eq0 + el < EQ) ? gv : 0.0;
        }
        __syncthreads();
#pragma unroll kTUnroll
        for (int el = 0; el < kTC; ++el) {
#pragma unroll
            for (int r = 0; r < 2; ++r) {
                if (!it_ok[r]) continue;
                const double *b = Bs + el * kTW + tpad(it_j[r]);
                const double *gg = Gs + (it_p[r] * kTC + el) * kTW + tpad(it_m[r]);
                const double b0 = b[0], b1 = b[1], b2 = b[2], b3 = b[3];
                const double gv[4] = {gg[0], gg[1], gg[2], gg[3]};
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    acc[r][0 * 4 + c] = fma(b0, gv[c], acc[r][0 * 4 + c]);
                    acc[r][1 * 4 + c] = fma(b1, gv[c], acc[r][1 * 4 + c]);
                    acc[r][2 * 4 + c] = fma(b2, gv[c], acc[r][2 * 4 + c]);
                    acc[r][3 * 4 + c] = fma(b3, gv[c], acc[r][3 * 4 + c]);
                }
            }
            if (xt) {
                const double a = As[el * kTW + tpad(xk)];
                U = fma(a, Ls[xp * kTC + el], U);
                U0 = fma(a, Gs[(xp * kTC + el) * kTW], U0);
            }
        }
    }
    __syncthreads();
    // anti-diagonal partial sums of each item: T[item][d], d = a + b (a ascending)
    double *T = Gs;
#pragma unroll
    for (int r = 0; r < 2; ++r) {
        if (!it_ok[r]) continue;
        const int item = tid + r * kTThreads;
#pragma unroll
        for (int d = 0; d < 7; ++d) {
            double sdg = 0.0;
#pragma unroll
            for (int a = 0; a < 4; ++a) {
                const int bcol = d - a;
                if (bcol >= 0 && bcol < 4) sdg += acc[r][a * 4 + bcol];
            }
            T[item * 7 + d] = sdg;
        }
    }
    __syncthreads();
    if (xt) {   // R[p][k]: tiles of anti-diagonal band s = jt + mt with 4s <= k <= 4s + 6
        double R = 0.0;
        for (int sd = max(0, (xk - 6 + 3) / 4); sd <= min(16, xk / 4); ++sd)
            for (int jt = 0; jt <= sd; ++jt) R += T[(xp * kNTile + tile_off(jt) + (sd - jt)) * 7 + (xk - 4 * sd)];
        Rs[xp * 65 + xk] = R;
        Rs[kTP * 65 + xp * 65 + xk] = U;
        Rs[2 * kTP * 65 + xp * 65 + xk] = U0;
    }
    __syncthreads();
    for (int p = 0; p < kTP; ++p) {
        const int64_t g = g0 + p;
        if (g >= P.n_groups) break;
        for (int64_t o = P.gptr[g] + tid; o < P.gptr[g + 1]; o += kTThreads) {
            const int k = (int)P.k[o];
            const bool cu = P.cur[o] != 0;
            P.out[P.out_idx[o]] = Rs[p * 65 + k] + Rs[(cu ? 1 : 2) * kTP * 65 + p * 65 + k];
        }
    }
    (void)lane;
}

// ---------------------------------------------------------------------------
// Register-blocked form for points at time-step ends (eps = 0, histories
// kmax <= KM; config 4 and represent_grid).  With W = 2 area_e w_q,
// B[j] = W (dens[j-1] - dens[j]) and A1[k] = W dens[k-1] (dens = 0 outside
// [0, E_t)), the reference's sum with cur = false is
//     u(k) = sum_eq  A1[k] G(0) + sum_{m=1..k} B[k-m] G(m)
// (its m = 0 coefficient dens[k-1] multiplies G(0) = lim0: gap 0 <= d_eps),
// and u(0) = 0.  The outputs k = 1..KM are cut into four blocks of R = KM/4;
// thread (point p, half h) owns blocks h and 3 - h, so both halves do the same
// number of FMAs.  For a block [k0, k0 + R) the thread walks m = 0..k0+R-1,
// loading G(m) of its point (shared memory, own column) and keeping the
// window B[k0 + i - m], i < R, in registers: one new broadcast load per m
// feeds R FMAs (the tile form above needs two shared loads per FMA).  Terms
// with k - m < 0 are skipped at compile time (template recursion over m).
// The G values of the CTA's 64 points are evaluated cooperatively with the
// lanes of a warp over m (neighbouring gaps: mostly one special-function
// region per warp).  Per eq: A (geometry, B / A1 rows) | sync | B (kernel
// values) | sync | C (contraction).  A cluster of S CTAs splits the eq range
// of the same points; the partial sums are added across the cluster through
// distributed shared memory in rank order (deterministic).  Groups with
// eps != 0 are left to k_potential_tiles (P.skip_eps0).
constexpr int kRP = 64;                  // points per CTA
constexpr int kRT = 2 * kRP;             // threads: (half, point)
constexpr int kRS = kRP + 1;             // G row stride (doubles): conflict-free rows and columns

template <int KM, int STRIDE = kRS>
struct RegBlock {
    static constexpr int R = KM / 4;
    // stage M of block K0: acc[i] += w[i] G(M) for the live i, then shift the
    // window by one (w[i] <- w[i-1], w[0] <- B[K0 - M - 1])
    template <int K0, int M>
    static __device__ __forceinline__ void step(double (&acc)[R], double (&w)[R], const double *Gc,
                                                const double *b)
    {
        if constexpr (M < K0 + R) {
            const double g = Gc[M * STRIDE];
#pragma unroll
            for (int i = 0; i < R; ++i)
                if (K0 + i - M >= 0) acc[i] = fma(w[i], g, acc[i]);
#pragma unroll
            for (int i = R - 1; i >= 1; --i) w[i] = w[i - 1];
            if constexpr (K0 - M - 1 >= 0) w[0] = b[K0 - M - 1];
            step<K0, M + 1>(acc, w, Gc, b);
        }
    }
    template <int K0>
    static __device__ __forceinline__ void run(double (&acc)[R], const double *Gc, const double *b,
                                               const double *a1)
    {
        const double g0 = Gc[0];
        double w[R];
#pragma unroll
        for (int i = 0; i < R; ++i) {
            acc[i] = fma(a1[K0 + i], g0, acc[i]);
            w[i] = b[K0 + i - 1];   // window for m = 1
        }
        step<K0, 1>(acc, w, Gc, b);
    }
};

template <int KIND, int KM>
#ifndef HB_POT_MINB
#define HB_POT_MINB 4
#endif
#ifndef HB_POT_ONEPASS
#define HB_POT_ONEPASS 0
#endif
__global__ void __launch_bounds__(kRT, HB_POT_MINB) k_potential_reg(const PotArgs P, int n_split)
{
    constexpr int R = KM / 4;
    extern __shared__ __align__(16) double rsm[];
    double *tab = rsm;
    double *Gs = tab + special::kTabDoubles;   // [KM + 1][kRS]: G(m) of point p at m * kRS + p
    double *Bs = Gs + (KM + 1) * kRS;          // [2][2][KM + 2]: B, A1 (double-buffered by eq parity)
    double *Rs = Bs + 4 * (KM + 2);            // [kRP] rho
    special::load_table<KIND == 0 ? 2 : 3>(tab);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int half = tid / kRP, pt = tid % kRP;   // warp-uniform half
    const int split = blockIdx.x % n_split;
    const int64_t pblock = blockIdx.x / n_split;
    const int64_t g = pblock * kRP + pt;
    const int64_t gc = g < P.n_groups ? g : P.n_groups - 1;
    const double px = P.gx[3 * gc], py = P.gx[3 * gc + 1], pz = P.gx[3 * gc + 2];
    const int64_t EQ = P.E_x * P.nq;
    const int64_t eq_lo = EQ * split / n_split, eq_hi = EQ * (split + 1) / n_split;
    // lane constants of the kernel-value phase: gaps m = lane + 1 + 32 s
    constexpr int kS = KM >= 64 ? 2 : 1;
    double cm[kS], gsmall[kS];
    bool gzero[kS];
#pragma unroll
    for (int s = 0; s < kS; ++s) {
        const double gap = (double)(lane + 1 + 32 * s) * P.step;
        cm[s] = 1.0 / (2.0 * sqrt(P.alpha * gap));
        gsmall[s] = KIND == 0 ? 1.0 / (4.0 * sqrt((kPi * kPi * kPi) * (P.alpha * P.alpha * P.alpha) * gap)) : 0.0;
        gzero[s] = gap <= P.d_eps;
    }
    const double inv4pi = 0.25 * kInvPi;
    double accA[R], accB[R];   // blocks half and 3 - half
#pragma unroll
    for (int i = 0; i < R; ++i) { accA[i] = 0.0; accB[i] = 0.0; }
    int64_t e = eq_lo / P.nq, q = eq_lo % P.nq;
    for (int64_t eq = eq_lo; eq < eq_hi; ++eq) {
        const int buf = (int)(eq & 1);
        // ---- A: point vs node eq (half 0 threads); the eq's B / A1 rows ----
        if (half == 0) {
            const double *y = P.qpts + 3 * eq;
            const double rx = px - __ldg(y), ry = py - __ldg(y + 1), rz = pz - __ldg(y + 2);
            const double rho = sqrt(rx * rx + ry * ry + rz * rz);
            double lim0;
            if (KIND == 0) {
                lim0 = 1.0 / (4.0 * kPi * P.alpha * rho);
            } else {
                const double rn = rx * __ldg(P.normals + 3 * e) + ry * __ldg(P.normals + 3 * e + 1) +
                                  rz * __ldg(P.normals + 3 * e + 2);
                lim0 = rho <= P.r_eps ? 0.0 : inv4pi * rn / (rho * rho * rho);
            }
            Rs[pt] = rho;
            Gs[pt] = lim0;   // G(0)
        } else {
            const double W = 2.0 * __ldg(P.areas + e) * __ldg(P.qw + q);
            const double *dq = P.dens_t + eq * P.E_t;
            for (int j = pt; j <= KM; j += kRP) {
                const double d = j < P.E_t ? __ldg(dq + j) : 0.0;
                const double dm = (j >= 1 && j - 1 < P.E_t) ? __ldg(dq + j - 1) : 0.0;
                Bs[(2 * buf) * (KM + 2) + j] = W * (dm - d);
                Bs[(2 * buf + 1) * (KM + 2) + j] = W * dm;
            }
        }
        if (++q == P.nq) { q = 0; ++e; }
        __syncthreads();
        // ---- B: kernel values G(rho_p, m h), m = 1..KM, lanes over m ----
#pragma unroll 1
        for (int p = warp; p < kRP; p += kRT / 32) {
            const double rho = Rs[p], lim0 = Gs[p];
            const bool rsmall = rho <= P.r_eps;
            double x[kS], ix[kS], r[kS];
#pragma unroll
            for (int s = 0; s < kS; ++s) { x[s] = __dmul_rn(rho, cm[s]); ix[s] = 0.0; }
#if HB_POT_ONEPASS
            special::eval_n<KIND == 0 ? 2 : 3, kS>(x, ix, r, tab, kFull);
#else
            // one pass per 32 gaps: the far gaps (m > 32) are mostly all in
            // the series region, so that pass runs one chain, not two
#pragma unroll
            for (int s = 0; s < kS; ++s) {
                double xs[1] = {x[s]}, is[1] = {0.0}, rs[1];
                special::eval_n<KIND == 0 ? 2 : 3, 1>(xs, is, rs, tab, kFull);
                r[s] = rs[0];
            }
#endif
#pragma unroll
            for (int s = 0; s < kS; ++s) {
                const int m = lane + 1 + 32 * s;
                const double gv = gzero[s] ? lim0 : rsmall ? gsmall[s] : __dmul_rn(lim0, r[s]);
                if (m <= KM) Gs[m * kRS + p] = gv;
            }
        }
        __syncthreads();
        // ---- C: contraction, blocks (half, 3 - half) of this thread's point ----
        {
            const double *b = Bs + (2 * buf) * (KM + 2), *a1 = Bs + (2 * buf + 1) * (KM + 2);
            const double *Gc = Gs + pt;
            if (half == 0) {
                RegBlock<KM>::template run<1>(accA, Gc, b, a1);
                RegBlock<KM>::template run<1 + 3 * R>(accB, Gc, b, a1);
            } else {
                RegBlock<KM>::template run<1 + R>(accA, Gc, b, a1);
                RegBlock<KM>::template run<1 + 2 * R>(accB, Gc, b, a1);
            }
        }
    }
    // ---- partial sums of the cluster's eq slices, added in rank order ----
    __syncthreads();
    double *Os = Gs;   // [kRP][KM + 2]: u(k) of point p at p * (KM + 2) + k
    {
        const int ka = 1 + (half == 0 ? 0 : R), kb = 1 + (half == 0 ? 3 * R : 2 * R);
#pragma unroll
        for (int i = 0; i < R; ++i) {
            Os[pt * (KM + 2) + ka + i] = accA[i];
            Os[pt * (KM + 2) + kb + i] = accB[i];
        }
        if (half == 0) Os[pt * (KM + 2)] = 0.0;   // u(0) = 0 at eps = 0
    }
    cg::cluster_group cl = cg::this_cluster();
    cl.sync();
    for (int p = split + n_split * (tid / 32); p < kRP; p += n_split * (kRT / 32)) {   // warp per point
        const int64_t gg = pblock * kRP + p;
        if (gg >= P.n_groups || P.geps[gg] != 0.0) continue;
        for (int64_t o = P.gptr[gg] + lane; o < P.gptr[gg + 1]; o += 32) {
            const int k = (int)P.k[o];
            double v = 0.0;
            for (int s = 0; s < n_split; ++s) v += cl.map_shared_rank(Os, s)[p * (KM + 2) + k];
            P.out[P.out_idx[o]] = v;
        }
    }
    cl.sync();
}

template <int KIND, int KM>
int launch_potential_reg(const PotArgs &P, cudaStream_t stream)
{
    auto kern = k_potential_reg<KIND, KM>;
    const size_t sm = sizeof(double) * (special::kTabDoubles +
                                        std::max<size_t>((KM + 1) * kRS + 4 * (KM + 2) + kRP, kRP * (KM + 2)));
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    int dev = 0, nsm = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kRT, sm);
    const int64_t slots = (int64_t)std::max(1, per_sm) * nsm;
    const int64_t nb = cdiv(P.n_groups, kRP);
    // eq split (cluster size) with the fullest last wave; ties -> fewer splits
    int best = 1;
    double best_eff = 0.0;
    for (int s = 1; s <= 8; ++s) {
        if ((int64_t)s * 64 > P.E_x * P.nq) break;
        const double waves = (double)(nb * s) / (double)slots;
        const double eff = waves / std::ceil(waves);
        if (eff > best_eff + 1e-3) { best_eff = eff; best = s; }
    }
    if (const char *f = getenv("HB_POT_SPLIT")) best = std::max(1, std::min(8, atoi(f)));
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)(nb * best));
    cfg.blockDim = dim3(kRT);
    cfg.dynamicSmemBytes = sm;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = best;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cuda_check(cudaLaunchKernelEx(&cfg, kern, P, best), "hb_potential (register-blocked)");
}

// ---------------------------------------------------------------------------
// Fused representation formula on a grid (represent_grid: M points x output
// times k <= 64, eps = 0): u = V~q - W g in ONE pass.  The single- and
// double-layer kernel values share x = rho / (2 sqrt(a m h)), the region
// votes and the middle-region piece, so one evaluation yields erf(x) and
// E(x) as two independent Horner chains.  The contraction is k_potential_reg's
// (RegBlock): thread types 0/1 of a point own the single-layer blocks
// (h, 3 - h), types 2/3 the double-layer ones (B / A1 rows stored negated),
// and the two partial results are added per output at the end.  Otherwise as
// k_potential_reg (cooperative kernel values, eq split over a cluster).
constexpr int kFP = 32;                  // points per CTA
constexpr int kFT = 4 * kFP;             // threads: (quarter, point)
constexpr int kFS = kFP + 1;             // G row stride (doubles)

// erf(x) and E(x) of one lane at once (hb_special.cuh regions): one compare
// and one vote for the common all-small warp, else ONE table chain per
// function in which small lanes use the series column (values bitwise their
// own region's, as in special::eval_nf)
__device__ __forceinline__ void eval_erf_E(double x, const double *__restrict__ tabS, const double *__restrict__ tabD,
                                           double &rs, double &rd)
{
    const double t = __dmul_rn(x, x);
    const bool small = x < special::kX0;
    if (!__any_sync(kFull, !small)) {
        rs = special::series<2>(x, t, 0.0);
        rd = special::series<3>(x, t, 0.0);
        return;
    }
    const bool midr = !small && x < special::kXL, huge = !small && !midr;
    if (__any_sync(kFull, midr)) {
        double u;
        const int pc = special::mid_piece(x, u);
        const int col[1] = {small ? special::kMidPieces : pc};
        const double v[1] = {small ? t : u};
        double qs[1], qd[1];
        if (__any_sync(kFull, small)) {
            special::table_chains<2, special::merged_deg<2>(), 1>(tabS, col, v, qs);
            special::table_chains<3, special::merged_deg<3>(), 1>(tabD, col, v, qd);
        } else {
            special::table_chains<2, special::mid_deg<2>(), 1>(tabS, col, v, qs);
            special::table_chains<3, special::mid_deg<3>(), 1>(tabD, col, v, qd);
        }
        asm volatile("" : "+d"(qs[0]), "+d"(qd[0]));
        rs = small ? special::series_finish<2>(x, t, 0.0, qs[0]) : qs[0];
        rd = small ? special::series_finish<3>(x, t, 0.0, qd[0]) : qd[0];
    } else {
        rs = special::series<2>(x, t, 0.0);
        rd = special::series<3>(x, t, 0.0);
    }
    if (__any_sync(kFull, huge)) {
        if (huge) { rs = 1.0; rd = 1.0; }
    }
}

// factor-free forms for k_represent_elem (HB_REP_FF): erf(x)/x and E(x)/x^3
// (kinds 6, 7) -- the per-point factors 1/rho and rn/rho^3 of the two
// potentials turn into per-gap constants cm/(4 pi alpha) and cm^3 applied
// once to the node sums; no finishing multiplies or region selects per value
__device__ __forceinline__ void eval_ex_Ex3(double x, double ix, const double *__restrict__ tabS,
                                            const double *__restrict__ tabD, double &rs, double &rd)
{
    const double t = __dmul_rn(x, x);
    const bool small = x < special::kX0;
    if (!__any_sync(kFull, !small)) {
        rs = special::series<6>(x, t, 0.0);
        rd = special::series<7>(x, t, 0.0);
        return;
    }
    const bool midr = !small && x < special::kXL, huge = !small && !midr;
    if (__any_sync(kFull, midr)) {
        double u;
        const int pc = special::mid_piece(x, u);
        const int col[1] = {small ? special::kMidPieces : pc};
        const double v[1] = {small ? t : u};
        double qs[1], qd[1];
        if (__any_sync(kFull, small)) {
            special::table_chains<6, special::merged_deg<6>(), 1>(tabS, col, v, qs);
            special::table_chains<7, special::merged_deg<7>(), 1>(tabD, col, v, qd);
        } else {
            special::table_chains<6, special::mid_deg<6>(), 1>(tabS, col, v, qs);
            special::table_chains<7, special::mid_deg<7>(), 1>(tabD, col, v, qd);
        }
        rs = qs[0];
        rd = qd[0];
    } else {
        rs = special::series<6>(x, t, 0.0);
        rd = special::series<7>(x, t, 0.0);
    }
    if (__any_sync(kFull, huge)) {
        if (huge) {
            rs = ix;
            rd = __dmul_rn(__dmul_rn(ix, ix), ix);
        }
    }
}

// The same two values from the uniform pieces of [0, XL) (kinds 6 and 7: width
// 1/16, degree 7, one shared piece index; hb_special.cuh): a warp whose lanes
// -- the gaps m of one (point, node) -- all lie in the series region takes the
// constant-bank series, any other warp evaluates every lane on its piece with
// no series / middle select or merged chain (two chains of 7 steps instead of
// two merged ones of 11).  Which lanes share a warp is fixed by (point, node,
// lane pass), so a value does not depend on the launch split.
__device__ __forceinline__ void eval_ex_Ex3_u(double x, double ix, const double *__restrict__ utabS,
                                              const double *__restrict__ utabD, double &rs, double &rd)
{
    const double t = __dmul_rn(x, x);
    if (!__any_sync(kFull, !(x < special::kX0))) {
        rs = special::series<6>(x, t, 0.0);
        rd = special::series<7>(x, t, 0.0);
        return;
    }
    const double2 *s2 = reinterpret_cast<const double2 *>(utabS), *d2 = reinterpret_cast<const double2 *>(utabD);
    constexpr int MT = special::kUDeg / 2, NP = special::kUPieces;
    const double y = __dmul_rn(x, special::kUInvH);   // exact (power of two)
    const int pi = __double2int_rz(y);
    const bool huge = pi >= NP;
    const int p = min(pi, NP - 1);
    const double u = fma(2.0, y - (double)p, -1.0);   // exact within the piece
    double2 ws[MT + 1], wd[MT + 1];
#pragma unroll
    for (int m = MT; m >= 0; --m) {
        ws[m] = s2[m * NP + p];
        wd[m] = d2[m * NP + p];
    }
    double qs = fma(ws[MT].y, u, ws[MT].x), qd = fma(wd[MT].y, u, wd[MT].x);
#pragma unroll
    for (int m = MT - 1; m >= 0; --m) {
        qs = fma(qs, u, ws[m].y);
        qd = fma(qd, u, wd[m].y);
        qs = fma(qs, u, ws[m].x);
        qd = fma(qd, u, wd[m].x);
    }
    rs = huge ? ix : qs;
    rd = huge ? __dmul_rn(__dmul_rn(ix, ix), ix) : qd;
}

#ifndef HB_REP_FF
#define HB_REP_FF 1
#endif

struct RepArgs {
    int64_t n_points, n_times, E_t, E_x, nq;
    const double *x;        // (n_points, 3)
    const int64_t *k;       // (n_times,) ascending, <= KM
    const double *dens_s, *dens_d;   // (E_x, nq, E_t) time fastest
    const double *qpts, *qw, *areas, *normals;
    double step, alpha, d_eps, r_eps;
    double *out;            // (n_points, n_times)
};

#ifndef HB_REP_MINB
#define HB_REP_MINB 3
#endif
template <int KM>
__global__ void __launch_bounds__(kFT, HB_REP_MINB) k_represent_reg(const RepArgs P, int n_split)
{
    constexpr int R = KM / 4;
    constexpr int BT = 4 * (KM + 2);
    extern __shared__ __align__(16) double fsm[];
    double *tabS = fsm, *tabD = tabS + special::kTabDoubles;
    double *Gs = tabD + special::kTabDoubles;   // [KM + 1][kFS]
    double *Gd = Gs + (KM + 1) * kFS;           // [KM + 1][kFS]
    double *Bt = Gd + (KM + 1) * kFS;           // [2][BT]
    double *Rs = Bt + 2 * BT;                   // [kFP]
    special::load_table<2>(tabS);
    special::load_table<3>(tabD);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int quarter = tid / kFP, pt = tid % kFP;   // warp-uniform quarter
    const int split = blockIdx.x % n_split;
    const int64_t pblock = blockIdx.x / n_split;
    const int64_t g = pblock * kFP + pt;
    const int64_t gc = g < P.n_points ? g : P.n_points - 1;
    const double px = P.x[3 * gc], py = P.x[3 * gc + 1], pz = P.x[3 * gc + 2];
    const int64_t EQ = P.E_x * P.nq;
    const int64_t eq_lo = EQ * split / n_split, eq_hi = EQ * (split + 1) / n_split;
    constexpr int kS = KM >= 64 ? 2 : 1;
    double cm[kS], gsmall[kS];
    bool gzero[kS];
#pragma unroll
    for (int s = 0; s < kS; ++s) {
        const double gap = (double)(lane + 1 + 32 * s) * P.step;
        cm[s] = 1.0 / (2.0 * sqrt(P.alpha * gap));
        gsmall[s] = 1.0 / (4.0 * sqrt((kPi * kPi * kPi) * (P.alpha * P.alpha * P.alpha) * gap));
        gzero[s] = gap <= P.d_eps;
    }
    const double inv4pi = 0.25 * kInvPi;
    double accA[R], accB[R];
#pragma unroll
    for (int i = 0; i < R; ++i) { accA[i] = 0.0; accB[i] = 0.0; }
    int64_t e = eq_lo / P.nq, q = eq_lo % P.nq;
    for (int64_t eq = eq_lo; eq < eq_hi; ++eq) {
        double *bt = Bt + (int)(eq & 1) * BT;
        // ---- A: point geometry (quarter 0); the eq's B / A1 rows (quarters 1-3) ----
        if (quarter == 0) {
            const double *y = P.qpts + 3 * eq;
            const double rx = px - __ldg(y), ry = py - __ldg(y + 1), rz = pz - __ldg(y + 2);
            const double rho = sqrt(rx * rx + ry * ry + rz * rz);
            const double rn = rx * __ldg(P.normals + 3 * e) + ry * __ldg(P.normals + 3 * e + 1) +
                              rz * __ldg(P.normals + 3 * e + 2);
            Rs[pt] = rho;
            Gs[pt] = 1.0 / (4.0 * kPi * P.alpha * rho);
            Gd[pt] = rho <= P.r_eps ? 0.0 : inv4pi * rn / (rho * rho * rho);
        } else {
            const double W = 2.0 * __ldg(P.areas + e) * __ldg(P.qw + q);
            const double *ds = P.dens_s + eq * P.E_t, *dd = P.dens_d + eq * P.E_t;
            for (int j = tid - kFP; j <= KM; j += kFT - kFP) {
                const double s0 = j < P.E_t ? __ldg(ds + j) : 0.0;
                const double s1 = (j >= 1 && j - 1 < P.E_t) ? __ldg(ds + j - 1) : 0.0;
                const double d0 = j < P.E_t ? __ldg(dd + j) : 0.0;
                const double d1 = (j >= 1 && j - 1 < P.E_t) ? __ldg(dd + j - 1) : 0.0;
                bt[j] = W * (s1 - s0);
                bt[(KM + 2) + j] = W * s1;
                bt[2 * (KM + 2) + j] = -(W * (d1 - d0));
                bt[3 * (KM + 2) + j] = -(W * d1);
            }
        }
        if (++q == P.nq) { q = 0; ++e; }
        __syncthreads();
        // ---- B: kernel values of both potentials, lanes over m ----
#pragma unroll 1
        for (int p = warp; p < kFP; p += kFT / 32) {
            const double rho = Rs[p], l0s = Gs[p], l0d = Gd[p];
            const bool rsmall = rho <= P.r_eps;
#pragma unroll
            for (int s = 0; s < kS; ++s) {
                double fs, fd;
                eval_erf_E(__dmul_rn(rho, cm[s]), tabS, tabD, fs, fd);
                const int m = lane + 1 + 32 * s;
                const double vs = gzero[s] ? l0s : rsmall ? gsmall[s] : __dmul_rn(l0s, fs);
                const double vd = gzero[s] ? l0d : rsmall ? 0.0 : __dmul_rn(l0d, fd);
                if (m <= KM) {
                    Gs[m * kFS + p] = vs;
                    Gd[m * kFS + p] = vd;
                }
            }
        }
        __syncthreads();
        // ---- C: contraction; quarters 0/1: single layer, blocks (h, 3 - h);
        //      quarters 2/3: double layer (B / A1 rows negated) ----
        {
            const int pot = quarter >> 1, h = quarter & 1;
            const double *Gc = (pot ? Gd : Gs) + pt;
            const double *b = bt + 2 * pot * (KM + 2), *a1 = b + (KM + 2);
            if (h == 0) {
                RegBlock<KM, kFS>::template run<1>(accA, Gc, b, a1);
                RegBlock<KM, kFS>::template run<1 + 3 * R>(accB, Gc, b, a1);
            } else {
                RegBlock<KM, kFS>::template run<1 + R>(accA, Gc, b, a1);
                RegBlock<KM, kFS>::template run<1 + 2 * R>(accB, Gc, b, a1);
            }
        }
    }
    __syncthreads();
    double *Os = Gs;   // [2][kFP][KM + 2]: single, negated double (spans Gs and Gd)
    {
        const int pot = quarter >> 1, h = quarter & 1;
        const int ka = 1 + (h == 0 ? 0 : R), kb = 1 + (h == 0 ? 3 * R : 2 * R);
        double *o = Os + (pot * kFP + pt) * (KM + 2);
#pragma unroll
        for (int i = 0; i < R; ++i) {
            o[ka + i] = accA[i];
            o[kb + i] = accB[i];
        }
        if (h == 0) o[0] = 0.0;   // u(0) = 0 at eps = 0
    }
    cg::cluster_group cl = cg::this_cluster();
    cl.sync();
    for (int p = split + n_split * warp; p < kFP; p += n_split * (kFT / 32)) {   // warp per point
        const int64_t gg = pblock * kFP + p;
        if (gg >= P.n_points) continue;
        for (int64_t o = lane; o < P.n_times; o += 32) {
            const int k = (int)P.k[o];
            double v = 0.0;
            for (int s = 0; s < n_split; ++s) {
                const double *os = cl.map_shared_rank(Os, s);
                v += os[p * (KM + 2) + k] + os[(kFP + p) * (KM + 2) + k];
            }
            P.out[gg * P.n_times + o] = v;
        }
    }
    cl.sync();
}

// ---------------------------------------------------------------------------
// k_represent_mma: k_represent_reg with the time contraction on the FP64
// tensor cores (mma.sync m8n8k4 f64, DMMA).  Per element quadrature node eq
// and potential, the contraction is a small GEMM over the m (time-gap) axis:
//   Out[p][k] += sum_m G[p][m] T[m][k],  T[0][k] = A1[k], T[m][k] = B[k - m]
//   (1 <= m <= k), 0 for m > k
// with points p as the M dimension (8-point tiles), output steps k = 1..KM as
// N (8-step tiles) and m = 0..KM (+ zero padding) as K (4-gap steps); tiles
// that lie entirely above the diagonal (m > k) are skipped at compile time.
// Warp w owns potential w >> 1 and points 16 (w & 1) .. +15 (two M tiles x
// KM/8 N tiles of accumulators).  G is stored per point (row stride KM + 4,
// == 4 mod 16 doubles: conflict-free fragment loads and phase-B stores), B
// with KM + 4 leading zeros (no index test for k < m).  One DMMA replaces 8
// DFMA issue slots; the sums run in a fixed order (deterministic).
// ---------------------------------------------------------------------------
__device__ __forceinline__ void dmma884(double &d0, double &d1, double a, double b)
{
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

template <int KM>
struct RepMmaLayout {
    static constexpr int KS = (KM + 4) / 4;   // 4-gap K steps covering m = 0..KM
    static constexpr int GS = 4 * KS;         // G row stride (== 4 mod 16 for KM in {16, 32, 64})
    static constexpr int NT = KM / 8;         // 8-step N tiles
    static constexpr int ZP = GS;             // zeros before each B row
    static constexpr int BR = ZP + KM + 1;    // B row length
    static_assert(GS % 16 == 4, "conflict-free G fragment loads need a row stride of 4 mod 16");
    static constexpr size_t doubles()
    {
        return 2 * (size_t)special::kTabDoubles + 2 * kFP * GS + 2 * 2 * BR + 2 * 2 * (KM + 1) + 3 * kFP;
    }
};

template <int KM>
__global__ void __launch_bounds__(kFT, 4) k_represent_mma(const RepArgs P, int n_split)
{
    using L = RepMmaLayout<KM>;
    constexpr int KS = L::KS, GS = L::GS, NT = L::NT, ZP = L::ZP, BR = L::BR;
    extern __shared__ __align__(16) double fsm[];
    double *tabS = fsm, *tabD = tabS + special::kTabDoubles;
    double *Gt = tabD + special::kTabDoubles;   // [2 pot][kFP][GS]
    double *Bz = Gt + 2 * kFP * GS;             // [2 buf][2 pot][BR]
    double *A1 = Bz + 2 * 2 * BR;               // [2 buf][2 pot][KM + 1]
    double *Rs = A1 + 2 * 2 * (KM + 1);         // [kFP]
    double *L0s = Rs + kFP, *L0d = L0s + kFP;   // [kFP] G at m = 0
    special::load_table<2>(tabS);
    special::load_table<3>(tabD);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int i = tid; i < 2 * kFP * GS; i += kFT) Gt[i] = 0.0;   // padding rows m > KM stay zero
    for (int i = tid; i < 2 * 2 * BR; i += kFT) Bz[i] = 0.0;     // leading zeros stay zero
    const int split = blockIdx.x % n_split;
    const int64_t pblock = blockIdx.x / n_split;
    const int pt = tid % kFP;
    const int64_t g = pblock * kFP + pt;
    const int64_t gc = g < P.n_points ? g : P.n_points - 1;
    const double px = P.x[3 * gc], py = P.x[3 * gc + 1], pz = P.x[3 * gc + 2];
    const int64_t EQ = P.E_x * P.nq;
    const int64_t eq_lo = EQ * split / n_split, eq_hi = EQ * (split + 1) / n_split;
    constexpr int kS = KM >= 64 ? 2 : 1;
    double cm[kS], gsmall[kS];
    bool gzero[kS];
#pragma unroll
    for (int s = 0; s < kS; ++s) {
        const double gap = (double)(lane + 1 + 32 * s) * P.step;
        cm[s] = 1.0 / (2.0 * sqrt(P.alpha * gap));
        gsmall[s] = 1.0 / (4.0 * sqrt((kPi * kPi * kPi) * (P.alpha * P.alpha * P.alpha) * gap));
        gzero[s] = gap <= P.d_eps;
    }
    const double inv4pi = 0.25 * kInvPi;
    const int pot = warp >> 1, mt0 = 2 * (warp & 1);
    const int gq = lane >> 2, tq = lane & 3;   // fragment row group / thread in group
    double acc[2][NT][2];
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int n = 0; n < NT; ++n) acc[a][n][0] = acc[a][n][1] = 0.0;
    __syncthreads();
    int64_t e = eq_lo / P.nq, q = eq_lo % P.nq;
    for (int64_t eq = eq_lo; eq < eq_hi; ++eq) {
        const int buf = (int)(eq & 1);
        // ---- A: point geometry (warp 0); the eq's B / A1 rows (warps 1-3) ----
        if (warp == 0) {
            const double *y = P.qpts + 3 * eq;
            const double rx = px - __ldg(y), ry = py - __ldg(y + 1), rz = pz - __ldg(y + 2);
            const double rho = sqrt(rx * rx + ry * ry + rz * rz);
            const double rn = rx * __ldg(P.normals + 3 * e) + ry * __ldg(P.normals + 3 * e + 1) +
                              rz * __ldg(P.normals + 3 * e + 2);
            Rs[pt] = rho;
            L0s[pt] = 1.0 / (4.0 * kPi * P.alpha * rho);
            L0d[pt] = rho <= P.r_eps ? 0.0 : inv4pi * rn / (rho * rho * rho);
        } else {
            const double W = 2.0 * __ldg(P.areas + e) * __ldg(P.qw + q);
            const double *ds = P.dens_s + eq * P.E_t, *dd = P.dens_d + eq * P.E_t;
            double *bs = Bz + (2 * buf) * BR + ZP, *bd = bs + BR;
            double *as = A1 + (2 * buf) * (KM + 1), *ad = as + (KM + 1);
            for (int j = tid - kFP; j <= KM; j += kFT - kFP) {
                const double s0 = j < P.E_t ? __ldg(ds + j) : 0.0;
                const double s1 = (j >= 1 && j - 1 < P.E_t) ? __ldg(ds + j - 1) : 0.0;
                const double d0 = j < P.E_t ? __ldg(dd + j) : 0.0;
                const double d1 = (j >= 1 && j - 1 < P.E_t) ? __ldg(dd + j - 1) : 0.0;
                bs[j] = W * (s1 - s0);
                as[j] = W * s1;
                bd[j] = -(W * (d1 - d0));
                ad[j] = -(W * d1);
            }
        }
        if (++q == P.nq) { q = 0; ++e; }
        __syncthreads();
        // ---- B: kernel values of both potentials, lanes over m (G rows per point) ----
#pragma unroll 1
        for (int p = warp; p < kFP; p += kFT / 32) {
            const double rho = Rs[p], l0s = L0s[p], l0d = L0d[p];
            const bool rsmall = rho <= P.r_eps;
            double *gs = Gt + p * GS, *gd = Gt + (kFP + p) * GS;
            if (lane == 0) {
                gs[0] = l0s;
                gd[0] = l0d;
            }
#pragma unroll
            for (int s = 0; s < kS; ++s) {
                double fs, fd;
                eval_erf_E(__dmul_rn(rho, cm[s]), tabS, tabD, fs, fd);
                const int m = lane + 1 + 32 * s;
                const double vs = gzero[s] ? l0s : rsmall ? gsmall[s] : __dmul_rn(l0s, fs);
                const double vd = gzero[s] ? l0d : rsmall ? 0.0 : __dmul_rn(l0d, fd);
                if (m <= KM) {
                    gs[m] = vs;
                    gd[m] = vd;
                }
            }
        }
        __syncthreads();
        // ---- C: DMMA contraction (warp: potential `pot`, M tiles mt0, mt0 + 1) ----
        {
            const double *gp = Gt + (pot * kFP + 8 * mt0 + gq) * GS + tq;
            const double *bz = Bz + (2 * buf + pot) * BR + ZP, *a1 = A1 + (2 * buf + pot) * (KM + 1);
#pragma unroll
            for (int ks = 0; ks < KS; ++ks) {
                const double a0 = gp[4 * ks], a1f = gp[8 * GS + 4 * ks];
                const int m = 4 * ks + tq;
#pragma unroll
                for (int n = 0; n < NT; ++n) {
                    if (8 * n + 8 < 4 * ks) continue;   // whole tile above the diagonal (m > k)
                    const int k = 1 + 8 * n + gq;
                    const double b = (ks == 0 && tq == 0) ? a1[k] : bz[k - m];
                    dmma884(acc[0][n][0], acc[0][n][1], a0, b);
                    dmma884(acc[1][n][0], acc[1][n][1], a1f, b);
                }
            }
        }
    }
    __syncthreads();
    double *Os = Gt;   // [2][kFP][KM + 2]: single, negated double (fits in Gt)
#pragma unroll
    for (int a = 0; a < 2; ++a) {
        double *o = Os + (pot * kFP + 8 * (mt0 + a) + gq) * (KM + 2);
#pragma unroll
        for (int n = 0; n < NT; ++n) {
            o[1 + 8 * n + 2 * tq] = acc[a][n][0];
            o[1 + 8 * n + 2 * tq + 1] = acc[a][n][1];
        }
        if (tq == 0) o[0] = 0.0;   // u(0) = 0 at eps = 0
    }
    cg::cluster_group cl = cg::this_cluster();
    cl.sync();
    for (int p = split + n_split * warp; p < kFP; p += n_split * (kFT / 32)) {   // warp per point
        const int64_t gg = pblock * kFP + p;
        if (gg >= P.n_points) continue;
        for (int64_t o = lane; o < P.n_times; o += 32) {
            const int k = (int)P.k[o];
            double v = 0.0;
            for (int s = 0; s < n_split; ++s) {
                const double *os = cl.map_shared_rank(Os, s);
                v += os[p * (KM + 2) + k] + os[(kFP + p) * (KM + 2) + k];
            }
            P.out[gg * P.n_times + o] = v;
        }
    }
    cl.sync();
}

template <int KM>
int launch_represent_mma(const RepArgs &P, cudaStream_t stream)
{
    auto kern = k_represent_mma<KM>;
    const size_t sm = sizeof(double) * RepMmaLayout<KM>::doubles();
    static_assert(2 * kFP * (KM + 2) <= 2 * kFP * RepMmaLayout<KM>::GS, "output staging must fit in G");
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    int dev = 0, nsm = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kFT, sm);
    const int64_t slots = (int64_t)std::max(1, per_sm) * nsm;
    const int64_t nb = cdiv(P.n_points, kFP);
    int best = 1;
    double best_eff = 0.0;
    for (int s = 1; s <= 8; ++s) {
        if ((int64_t)s * 64 > P.E_x * P.nq) break;
        const double waves = (double)(nb * s) / (double)slots;
        const double eff = waves / std::ceil(waves);
        if (eff > best_eff + 1e-3) { best_eff = eff; best = s; }
    }
    if (const char *f = getenv("HB_POT_SPLIT")) best = std::max(1, std::min(8, atoi(f)));
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)(nb * best));
    cfg.blockDim = dim3(kFT);
    cfg.dynamicSmemBytes = sm;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = best;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cuda_check(cudaLaunchKernelEx(&cfg, kern, P, best), "hb_represent_grid");
}

// ---------------------------------------------------------------------------
// k_represent_elem: the representation formula with the time contraction
// done ONCE PER ELEMENT instead of once per element quadrature node.  The
// density differences of a node are element data: the p0 density is constant
// on the element and the p1 density at node q is sum_i hat_i(q) g_{v_i}, so
//   sum_q G_q[p][m] W_q B_q[k - m]
//     = sum_m (sum_q W_q G_q[p][m]) Bq[k - m]                       (single)
//     + sum_i sum_m (sum_q W_q hat_i(q) G_q[p][m]) Bg_i[k - m]      (double)
// with W_q = 2 area_e qw_q: the kernel values of the nq nodes are first
// summed into four per-element arrays H (single; double x 3 vertices) and the
// element then needs 4 Toeplitz products instead of 2 nq (12 at config 4) --
// on the FP64 tensor cores as in k_represent_mma (warp w: points 8w..8w+7,
// all four products).  Inputs: the p0 density per element (E_x, E_t) and the
// p1 density at each element's vertices (E_x, 3, E_t), time fastest.
// ---------------------------------------------------------------------------
struct RepElemArgs {
    int64_t n_points, n_times, E_t, E_x, nq;
    const double *x;          // (n_points, 3)
    const int64_t *k;         // (n_times,) ascending, <= KM
    const double *dens_e;     // (E_x, E_t)
    const double *dens_v;     // (E_x, 3, E_t)
    const double *hats;       // (nq, 3)
    const double *qpts, *qw, *areas, *normals;
    double step, alpha, d_eps, r_eps;
    double eps;               // evaluation times k h + eps (0: time-step ends)
    double *out;              // (n_points, n_times)
    int kblock;               // LONG kernels: this launch forms the outputs k in (KM kblock, KM kblock + KM]
};

constexpr int kFTE = 256;   // k_represent_elem threads (8 warps, 32 points)
// shared-memory doubles per special-function table of k_represent_elem (uniform pieces with HB_REP_FF)
constexpr int kRepTab = special::kUTabDoubles > special::kTabDoubles ? special::kUTabDoubles : special::kTabDoubles;

template <int KM>
struct RepElemLayout {
    static constexpr int KS = (KM + 4) / 4, GS = 4 * KS, NT = KM / 8, ZP = GS, BR = ZP + KM + 1;
    static_assert(GS % 16 == 4, "conflict-free H fragment loads need a row stride of 4 mod 16");
    // kt: time steps held per density vector (KM, or KM (kblock + 1) for the LONG kernels)
    static size_t doubles(int64_t nq, int64_t kt = KM)
    {
        return 2 * (size_t)kRepTab + 4 * kFP * GS + (HB_REP_FF ? 5 : 3) * (size_t)nq * kFP +
               2 * 4 * (size_t)(ZP + kt + 1) + 2 * 2 * 4 * (size_t)(kt + 1);
    }
};

// EPS (eps > 0, the reference's current-interval case, _field_numba.py:53-76):
// out[k] = sum_{m=0..k} G(m h + eps) B[k - m] + G(0) W dens[k] -- the m = 0 row
// is a regular kernel value and the G(0) term rides in the spare K row XR = KM + 1
// against the element's density vector.
//
// LONG (histories longer than KM steps, eps = 0): the launch forms the output
// block J = kblock, k = KM J + k', k' in 1..KM, from the gap windows
// w = 0..J (gaps m = KM w + m', m' in 1..KM; G(0) in window 0):
//   out[k] = sum_w sum_m' H_w[m'] T[KM (J - w) + k' - m']
// -- window J is the triangular product of the short kernel, the windows below
// are full tiles.  Each window's kernel values are evaluated into the same H
// rows and contracted on the tensor cores before the next one; one launch per
// output block (hb_represent_grid_elem loops J), so gap window w is evaluated
// by the launches J >= w.
template <int KM, bool EPS, bool LONG = false>
__global__ void __launch_bounds__(kFTE, 2) k_represent_elem(const RepElemArgs P, int n_split)
{
    using L = RepElemLayout<KM>;
    constexpr int KS = L::KS, GS = L::GS, NT = L::NT, ZP = L::ZP;
    constexpr int MOFS = EPS ? 0 : 1, XR = KM + 1;
    static_assert(XR < GS, "the G(0) row must fit in the K padding");
    static_assert(!(EPS && LONG), "long histories: time-step ends only");
    const int J = LONG ? P.kblock : 0;
    const int KT = KM * (J + 1);            // time steps held per density vector
    const int BR = ZP + KT + 1, AS = KT + 1;
    extern __shared__ __align__(16) double fsm[];
    const int nq = (int)P.nq;
    double *tabS = fsm, *tabD = tabS + kRepTab;
    double *H = tabD + kRepTab;                 // [4][kFP][GS]: W G (single), W hat_i G (double, i = 0..2)
    double *Rn = H + 4 * kFP * GS;              // [nq][kFP] rho
    double *L0s = Rn + nq * kFP, *L0d = L0s + nq * kFP;   // [nq][kFP] G at m = 0
    double *Tv = L0d + nq * kFP;                // [2 buf][4][BR]: density differences, zeros before
    double *Av = Tv + 2 * 4 * BR;               // [2 buf][4][AS]: m = 0 row
    double *Dv = Av + 2 * 4 * AS;               // [2 buf][4][AS]: density (EPS: the G(0) term)
    double *Ri = Dv + 2 * 4 * AS;               // HB_REP_FF: [nq][kFP] 1/rho
    double *Rq = Ri + nq * kFP;                 // HB_REP_FF: [nq][kFP] rn / (4 pi) (0 for rho <= r_eps)
#if HB_REP_FF
    special::load_utable<6>(tabS);
    special::load_utable<7>(tabD);
#else
    special::load_table<2>(tabS);
    special::load_table<3>(tabD);
#endif
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int i = tid; i < 4 * kFP * GS; i += kFTE) H[i] = 0.0;   // padding rows m > KM stay zero
    for (int i = tid; i < 2 * 4 * BR; i += kFTE) Tv[i] = 0.0;    // leading zeros stay zero
    const int split = blockIdx.x % n_split;
    const int64_t pblock = blockIdx.x / n_split;
    const int64_t e_lo = P.E_x * split / n_split, e_hi = P.E_x * (split + 1) / n_split;
    constexpr int kS = (KM + 1 - MOFS + 31) / 32;   // lane passes over m = MOFS..KM
    double cm[kS], gsmall[kS], icm[kS];
    bool gzero[kS];
    auto gap_constants = [&](int w) {   // gaps KM w + m', m' = lane + MOFS + 32 s
#pragma unroll
        for (int s = 0; s < kS; ++s) {
            const double gap = (double)(KM * w + lane + MOFS + 32 * s) * P.step + (EPS ? P.eps : 0.0);
            icm[s] = 2.0 * sqrt(P.alpha * gap);
            cm[s] = 1.0 / icm[s];
            gsmall[s] = 1.0 / (4.0 * sqrt((kPi * kPi * kPi) * (P.alpha * P.alpha * P.alpha) * gap));
            gzero[s] = gap <= P.d_eps;
        }
    };
    if (!LONG) gap_constants(0);
    const double inv4pi = 0.25 * kInvPi;
    const int gq = lane >> 2, tq = lane & 3;
    // phase C: warp w owns M tile (points 8 (w & 3) ..) and the N tiles n = 2 j + (w >> 2)
    // (odd / even interleave balances the skipped upper-triangle tiles)
    constexpr int NH = (NT + 1) / 2;
    const int mt = warp & 3, nh = warp >> 2;
    double accS[NH][2], accD[NH][2];
#pragma unroll
    for (int n = 0; n < NH; ++n) accS[n][0] = accS[n][1] = accD[n][0] = accD[n][1] = 0.0;
    __syncthreads();
    for (int64_t e = e_lo; e < e_hi; ++e) {
        const int buf = (int)(e & 1);
        // ---- A: geometry of every (node, point); the element's density vectors ----
        const double nx = __ldg(P.normals + 3 * e), ny = __ldg(P.normals + 3 * e + 1), nz = __ldg(P.normals + 3 * e + 2);
        for (int it = tid; it < nq * kFP; it += kFTE) {
            const int node = it / kFP, p = it - node * kFP;
            const int64_t gp = min(pblock * kFP + p, P.n_points - 1);
            const double *y = P.qpts + 3 * (e * P.nq + node);
            const double rx = __ldg(P.x + 3 * gp) - __ldg(y), ry = __ldg(P.x + 3 * gp + 1) - __ldg(y + 1),
                         rz = __ldg(P.x + 3 * gp + 2) - __ldg(y + 2);
            const double rho = sqrt(rx * rx + ry * ry + rz * rz);
            const double rn = rx * nx + ry * ny + rz * nz;
            Rn[it] = rho;
            L0s[it] = 1.0 / (4.0 * kPi * P.alpha * rho);
            L0d[it] = rho <= P.r_eps ? 0.0 : inv4pi * rn / (rho * rho * rho);
            if (HB_REP_FF) {
                Ri[it] = 1.0 / rho;
                Rq[it] = rho <= P.r_eps ? 0.0 : inv4pi * rn;
            }
        }
        {
            double *tv = Tv + buf * 4 * BR + ZP, *av = Av + buf * 4 * AS, *dd = Dv + buf * 4 * AS;
            const double *de = P.dens_e + e * P.E_t, *dv = P.dens_v + e * 3 * P.E_t;
            for (int it = tid; it < 4 * AS; it += kFTE) {
                const int v = it / AS, j = it - v * AS;
                const double *d = v == 0 ? de : dv + (v - 1) * P.E_t;
                const double cur = j < P.E_t ? __ldg(d + j) : 0.0;
                const double prev = (j >= 1 && j - 1 < P.E_t) ? __ldg(d + j - 1) : 0.0;
                // single layer: B = s1 - s0, A1 = s1; double layer negated (u = V~q - W g)
                tv[v * BR + j] = v == 0 ? prev - cur : -(prev - cur);
                av[v * AS + j] = v == 0 ? prev : -prev;
                if (EPS) dd[v * AS + j] = v == 0 ? cur : -cur;
            }
        }
        __syncthreads();
        const double a2 = 2.0 * __ldg(P.areas + e);
#pragma unroll 1
        for (int w = 0; w <= J; ++w) {   // gap windows (one, w = 0, unless LONG)
        if (LONG) {
            if (w > 0) __syncthreads();   // the previous window's products have read H
            gap_constants(w);
        }
        // ---- B: kernel values of every node, summed over the nodes in registers
        //      (lanes over m, node ascending) and stored once into H ----
#pragma unroll 1
        for (int p = warp; p < kFP; p += kFTE / 32) {
            double hsum[4][kS], hz[4];
#pragma unroll
            for (int v = 0; v < 4; ++v) {
                hz[v] = 0.0;
#pragma unroll
                for (int s = 0; s < kS; ++s) hsum[v][s] = 0.0;
            }
#pragma unroll 1
            for (int node = 0; node < nq; ++node) {
                const double W = a2 * __ldg(P.qw + node);
                const double wh0 = W * __ldg(P.hats + 3 * node), wh1 = W * __ldg(P.hats + 3 * node + 1),
                             wh2 = W * __ldg(P.hats + 3 * node + 2);
                const double rho = Rn[node * kFP + p], l0s = L0s[node * kFP + p], l0d = L0d[node * kFP + p];
                const bool rsmall = rho <= P.r_eps;
                hz[0] = fma(W, l0s, hz[0]);
                hz[1] = fma(wh0, l0d, hz[1]);
                hz[2] = fma(wh1, l0d, hz[2]);
                hz[3] = fma(wh2, l0d, hz[3]);
#if HB_REP_FF
                const double ri = Ri[node * kFP + p], rq = Rq[node * kFP + p];
                (void)rsmall;
#pragma unroll
                for (int s = 0; s < kS; ++s) {
                    double fs, fd;
                    eval_ex_Ex3_u(__dmul_rn(rho, cm[s]), __dmul_rn(ri, icm[s]), tabS, tabD, fs, fd);
                    // (scaled by cm / (4 pi a) and cm^3 after the node sum; rho <= r_eps:
                    // erf(x)/x -> 2/sqrt(pi), the reference's limit, and rq = 0)
                    const double vs = gzero[s] ? l0s : fs;
                    const double vd = gzero[s] ? l0d : __dmul_rn(rq, fd);
                    hsum[0][s] = fma(W, vs, hsum[0][s]);
                    hsum[1][s] = fma(wh0, vd, hsum[1][s]);
                    hsum[2][s] = fma(wh1, vd, hsum[2][s]);
                    hsum[3][s] = fma(wh2, vd, hsum[3][s]);
                }
#else
#pragma unroll
                for (int s = 0; s < kS; ++s) {
                    double fs, fd;
                    eval_erf_E(__dmul_rn(rho, cm[s]), tabS, tabD, fs, fd);
                    const double vs = gzero[s] ? l0s : rsmall ? gsmall[s] : __dmul_rn(l0s, fs);
                    const double vd = gzero[s] ? l0d : rsmall ? 0.0 : __dmul_rn(l0d, fd);
                    hsum[0][s] = fma(W, vs, hsum[0][s]);
                    hsum[1][s] = fma(wh0, vd, hsum[1][s]);
                    hsum[2][s] = fma(wh1, vd, hsum[2][s]);
                    hsum[3][s] = fma(wh2, vd, hsum[3][s]);
                }
#endif
            }
#if HB_REP_FF
#pragma unroll
            for (int s = 0; s < kS; ++s) {
                if (!gzero[s]) {
                    const double cs = cm[s] * (0.25 * kInvPi / P.alpha), cd = cm[s] * cm[s] * cm[s];
                    hsum[0][s] *= cs;
#pragma unroll
                    for (int v = 1; v < 4; ++v) hsum[v][s] *= cd;
                }
            }
#endif
#pragma unroll
            for (int v = 0; v < 4; ++v) {
                double *h = H + (v * kFP + p) * GS;
                // G(0) sums: the m = 0 row (of window 0), or row XR
                if (lane == 0) h[EPS ? XR : 0] = (LONG && w > 0) ? 0.0 : hz[v];
#pragma unroll
                for (int s = 0; s < kS; ++s) {
                    const int m = lane + MOFS + 32 * s;
                    if (m <= KM) h[m] = hsum[v][s];
                }
            }
        }
        __syncthreads();
        // ---- C: four Toeplitz products per element on the tensor cores ----
        {
            const double *hp = H + (8 * mt + gq) * GS + tq;
            // window w against the densities KM (J - w) steps back; the m = 0 row of
            // window 0 against the previous step's density of the output k = KM J + k'
            const double *tv = Tv + buf * 4 * BR + ZP + KM * (J - w), *av = Av + buf * 4 * AS + KM * J,
                         *dd = Dv + buf * 4 * AS;
            const bool diag = !LONG || w == J;   // the triangular window: tiles above the diagonal are empty
#pragma unroll
            for (int ks = 0; ks < KS; ++ks) {
                double a[4];
#pragma unroll
                for (int v = 0; v < 4; ++v) a[v] = hp[v * kFP * GS + 4 * ks];
                const int m = 4 * ks + tq;
#pragma unroll
                for (int j = 0; j < NH; ++j) {
                    const int n = 2 * j + nh;
                    // whole tile above the diagonal (m > k) -- except the G(0) row XR (EPS)
                    if (n >= NT || (diag && 8 * n + 8 < 4 * ks && !(EPS && ks == XR / 4))) continue;
                    const int k = 1 + 8 * n + gq;
                    double b[4];
#pragma unroll
                    for (int v = 0; v < 4; ++v)
                        b[v] = (EPS && m == XR) ? dd[v * AS + k]
                             : (!EPS && ks == 0 && tq == 0 && (!LONG || w == 0)) ? av[v * AS + k] : tv[v * BR + k - m];
                    dmma884(accS[j][0], accS[j][1], a[0], b[0]);
                    dmma884(accD[j][0], accD[j][1], a[1], b[1]);
                    dmma884(accD[j][0], accD[j][1], a[2], b[2]);
                    dmma884(accD[j][0], accD[j][1], a[3], b[3]);
                }
            }
        }
        }   // gap windows
    }
    __syncthreads();
    double *Os = H;   // [2][kFP][KM + 2]: single, negated double
    {
        double *os = Os + (8 * mt + gq) * (KM + 2), *od = Os + (kFP + 8 * mt + gq) * (KM + 2);
#pragma unroll
        for (int j = 0; j < NH; ++j) {
            const int n = 2 * j + nh;
            if (n >= NT) continue;
            os[1 + 8 * n + 2 * tq] = accS[j][0];
            os[1 + 8 * n + 2 * tq + 1] = accS[j][1];
            od[1 + 8 * n + 2 * tq] = accD[j][0];
            od[1 + 8 * n + 2 * tq + 1] = accD[j][1];
        }
        if (tq == 0 && nh == 0) { os[0] = 0.0; od[0] = 0.0; }   // u(0) = 0 at eps = 0
    }
    cg::cluster_group cl = cg::this_cluster();
    cl.sync();
    for (int p = split + n_split * warp; p < kFP; p += n_split * (kFTE / 32)) {   // warp per point
        const int64_t gg = pblock * kFP + p;
        if (gg >= P.n_points) continue;
        for (int64_t o = lane; o < P.n_times; o += 32) {
            int k = (int)P.k[o];
            if (LONG) {   // this launch's output block only (k = 0 belongs to block 0)
                k -= KM * J;
                if (k > KM || k < (J == 0 ? 0 : 1)) continue;
            }
            double v = 0.0;
            for (int s = 0; s < n_split; ++s) {
                const double *os = cl.map_shared_rank(Os, s);
                v += os[p * (KM + 2) + k] + os[(kFP + p) * (KM + 2) + k];
            }
            // k = 0 inside the first step (eps > 0) is not this kernel's case
            // (header: k >= 1 when eps > 0): NaN, never a silent 0
            if (EPS && k == 0) v = __longlong_as_double(0x7ff8000000000000ll);
            P.out[gg * P.n_times + o] = v;
        }
    }
    cl.sync();
}

template <int KM, bool EPS, bool LONG = false>
int launch_represent_elem(const RepElemArgs &P, cudaStream_t stream)
{
    auto kern = k_represent_elem<KM, EPS, LONG>;
    const size_t sm = sizeof(double) * RepElemLayout<KM>::doubles(P.nq, LONG ? (int64_t)KM * (P.kblock + 1) : KM);
    if (sm > 227 * 1024) {
        set_error("hb_represent_grid_elem: %d output blocks of %d steps do not fit shared memory", P.kblock + 1, KM);
        return HB_ERR_UNSUPPORTED;
    }
    constexpr int kFT = kFTE;
    static_assert(2 * kFP * (KM + 2) <= 4 * kFP * RepElemLayout<KM>::GS, "output staging must fit in H");
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    int dev = 0, nsm = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kFT, sm);
    const int64_t slots = (int64_t)std::max(1, per_sm) * nsm;
    const int64_t nb = cdiv(P.n_points, kFP);
    // element split over a cluster only when the point blocks alone fill the GPU
    // poorly: the split adds a cluster barrier and the DSMEM reduction
    int best = 1;
    double best_eff = 0.0;
    for (int s = 1; s <= 8; ++s) {
        if ((int64_t)s * 8 > P.E_x) break;
        const double waves = (double)(nb * s) / (double)slots;
        const double eff = waves / std::ceil(waves);
        if (eff >= 0.9) { best = s; break; }
        if (eff > best_eff + 1e-3) { best_eff = eff; best = s; }
    }
    if (const char *f = getenv("HB_POT_SPLIT")) best = std::max(1, std::min(8, atoi(f)));
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)(nb * best));
    cfg.blockDim = dim3(kFT);
    cfg.dynamicSmemBytes = sm;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = best;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cuda_check(cudaLaunchKernelEx(&cfg, kern, P, best), "hb_represent_grid_elem");
}

template <int KM>
int launch_represent_reg(const RepArgs &P, cudaStream_t stream)
{
    auto kern = k_represent_reg<KM>;
    const size_t sm = sizeof(double) * (2 * special::kTabDoubles +
                                        std::max<size_t>(2 * (KM + 1) * kFS + 8 * (KM + 2) + kFP,
                                                         2 * kFP * (KM + 2)));
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    int dev = 0, nsm = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kFT, sm);
    const int64_t slots = (int64_t)std::max(1, per_sm) * nsm;
    const int64_t nb = cdiv(P.n_points, kFP);
    int best = 1;
    double best_eff = 0.0;
    for (int s = 1; s <= 8; ++s) {
        if ((int64_t)s * 64 > P.E_x * P.nq) break;
        const double waves = (double)(nb * s) / (double)slots;
        const double eff = waves / std::ceil(waves);
        if (eff > best_eff + 1e-3) { best_eff = eff; best = s; }
    }
    if (const char *f = getenv("HB_POT_SPLIT")) best = std::max(1, std::min(8, atoi(f)));
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)(nb * best));
    cfg.blockDim = dim3(kFT);
    cfg.dynamicSmemBytes = sm;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = best;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cuda_check(cudaLaunchKernelEx(&cfg, kern, P, best), "hb_represent_grid");
}

}  // namespace hb

using namespace hb;

// Outputs sharing (x, eps) form one group (gptr); k ascending within a group.
extern "C" int hb_potential(int kind, int64_t n_groups, int64_t E_t, int64_t E_x, int64_t nq,
                            const double *gx_dev, const double *geps_dev, const int64_t *gptr_dev,
                            const int64_t *k_dev, const uint8_t *cur_dev, const int64_t *out_idx_dev,
                            int64_t kmax, const double *dens_t_dev, const double *qpts_dev,
                            const double *qw_dev, const double *areas_dev, const double *normals_dev,
                            double step, double alpha, double d_eps, double r_eps, double *out_dev,
                            void *stream)
{
    if (kind < 0 || kind > 1 || n_groups < 0 || E_t < 1 || E_x < 1 || nq < 1 || kmax < 0 || !out_dev) {
        set_error("hb_potential: bad arguments");
        return HB_ERR_INVALID;
    }
    if (n_groups == 0) return HB_OK;
    PotArgs P{};
    P.kind = kind; P.n_groups = n_groups; P.E_t = E_t; P.E_x = E_x; P.nq = nq;
    P.gx = gx_dev; P.geps = geps_dev; P.gptr = gptr_dev; P.k = k_dev; P.cur = cur_dev; P.out_idx = out_idx_dev;
    P.dens_t = dens_t_dev; P.qpts = qpts_dev; P.qw = qw_dev; P.areas = areas_dev; P.normals = normals_dev;
    P.step = step; P.alpha = alpha; P.d_eps = d_eps; P.r_eps = r_eps; P.out = out_dev;
    if (kmax <= kTMaxK && !getenv("HB_POT_GENERAL") && !getenv("HB_POT_TILES")) {
        // eps = 0 groups: register-blocked form; the rest: tiled form (below)
        int rc;
        if (kmax <= 16) rc = kind == 0 ? launch_potential_reg<0, 16>(P, (cudaStream_t)stream)
                                       : launch_potential_reg<1, 16>(P, (cudaStream_t)stream);
        else if (kmax <= 32) rc = kind == 0 ? launch_potential_reg<0, 32>(P, (cudaStream_t)stream)
                                            : launch_potential_reg<1, 32>(P, (cudaStream_t)stream);
        else rc = kind == 0 ? launch_potential_reg<0, 64>(P, (cudaStream_t)stream)
                            : launch_potential_reg<1, 64>(P, (cudaStream_t)stream);
        if (rc != HB_OK) return rc;
        P.skip_eps0 = 1;
    }
    if (kmax <= kTMaxK && !getenv("HB_POT_GENERAL")) {   // tiled form (config 4 and shorter histories)
        const size_t sm = sizeof(double) * (special::kTabDoubles + 2 * kTC * kTW + kTP * kTC * kTW + kTP * kTC +
                                            kTP * kTK + kTP * kTC * 2 + 3 * kTP * 65);
        auto kern = kind == 0 ? k_potential_tiles<0> : k_potential_tiles<1>;
        if (sm > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        kern<<<(unsigned)cdiv(n_groups, kTP), kTThreads, sm, (cudaStream_t)stream>>>(P);
        return cuda_check(cudaGetLastError(), "hb_potential");
    }
    P.kcap = (int)((kmax / 32 + 1) * 32);
    const size_t sm = (special::kTabDoubles + (size_t)kPotWarps * kOut + (size_t)kPotWarps * 4 * P.kcap) * sizeof(double);
    if (sm > 220 * 1024) { set_error("hb_potential: time history too long (%lld)", (long long)kmax); return HB_ERR_INVALID; }
    auto kern = kind == 0 ? k_potential<0> : k_potential<1>;
    if (sm > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    int dev = 0, nsm = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kPotWarps * 32, sm);
    const int64_t grid = std::min<int64_t>(n_groups, (int64_t)std::max(1, per_sm) * nsm * 4);
    kern<<<(unsigned)grid, kPotWarps * 32, sm, (cudaStream_t)stream>>>(P);
    return cuda_check(cudaGetLastError(), "hb_potential");
}

// u = V~q - W g at every point x_i and every output time k_j (k ascending,
// eps = 0): represent_grid (heatbem/field.py:184-190 on a space-time grid).
extern "C" int hb_represent_grid(int64_t n_points, int64_t n_times, int64_t E_t, int64_t E_x, int64_t nq,
                                 const double *x_dev, const int64_t *k_dev, int64_t kmax,
                                 const double *dens_single_dev, const double *dens_double_dev,
                                 const double *qpts_dev, const double *qw_dev, const double *areas_dev,
                                 const double *normals_dev, double step, double alpha, double d_eps, double r_eps,
                                 double *out_dev, void *stream)
{
    if (n_points < 0 || n_times < 0 || E_t < 1 || E_x < 1 || nq < 1 || kmax < 0 || kmax > 64 ||
        (n_points > 0 && n_times > 0 && (!x_dev || !k_dev || !dens_single_dev || !dens_double_dev || !out_dev))) {
        set_error("hb_represent_grid: bad arguments (kmax %lld: at most 64 output steps)", (long long)kmax);
        return HB_ERR_INVALID;
    }
    if (n_points == 0 || n_times == 0) return HB_OK;
    RepArgs P{};
    P.n_points = n_points; P.n_times = n_times; P.E_t = E_t; P.E_x = E_x; P.nq = nq;
    P.x = x_dev; P.k = k_dev; P.dens_s = dens_single_dev; P.dens_d = dens_double_dev;
    P.qpts = qpts_dev; P.qw = qw_dev; P.areas = areas_dev; P.normals = normals_dev;
    P.step = step; P.alpha = alpha; P.d_eps = d_eps; P.r_eps = r_eps; P.out = out_dev;
    cudaStream_t st = (cudaStream_t)stream;
    // time contraction on the FP64 tensor cores (HB_REP_MMA=0: the DFMA register-blocked form)
    static const bool mma = !getenv("HB_REP_MMA") || atoi(getenv("HB_REP_MMA")) != 0;
    if (mma) {
        if (kmax <= 16) return launch_represent_mma<16>(P, st);
        if (kmax <= 32) return launch_represent_mma<32>(P, st);
        return launch_represent_mma<64>(P, st);
    }
    if (kmax <= 16) return launch_represent_reg<16>(P, st);
    if (kmax <= 32) return launch_represent_reg<32>(P, st);
    return launch_represent_reg<64>(P, st);
}

constexpr int kRepMaxBlocks = 8;   // histories up to 512 steps on the per-element kernel

extern "C" int hb_represent_grid_elem(int64_t n_points, int64_t n_times, int64_t E_t, int64_t E_x, int64_t nq,
                                      const double *x_dev, const int64_t *k_dev, int64_t kmax,
                                      const double *dens_elem_dev, const double *dens_vert_dev,
                                      const double *hats_dev, const double *qpts_dev, const double *qw_dev,
                                      const double *areas_dev, const double *normals_dev, double step, double alpha,
                                      double d_eps, double r_eps, double eps, double *out_dev, void *stream)
{
    if (n_points < 0 || n_times < 0 || E_t < 1 || E_x < 1 || nq < 1 || nq > 64 || kmax < 0 ||
        (kmax > 64 && (eps > 0.0 || kmax > 64 * kRepMaxBlocks)) || !(eps >= 0.0 && eps < step) ||
        (n_points > 0 && n_times > 0 &&
         (!x_dev || !k_dev || !dens_elem_dev || !dens_vert_dev || !hats_dev || !out_dev))) {
        set_error("hb_represent_grid_elem: bad arguments (kmax %lld: at most 64 output steps inside a step, "
                  "%d at time-step ends)", (long long)kmax, 64 * kRepMaxBlocks);
        return HB_ERR_INVALID;
    }
    if (n_points == 0 || n_times == 0) return HB_OK;
    RepElemArgs P{};
    P.n_points = n_points; P.n_times = n_times; P.E_t = E_t; P.E_x = E_x; P.nq = nq;
    P.x = x_dev; P.k = k_dev; P.dens_e = dens_elem_dev; P.dens_v = dens_vert_dev; P.hats = hats_dev;
    P.qpts = qpts_dev; P.qw = qw_dev; P.areas = areas_dev; P.normals = normals_dev;
    P.step = step; P.alpha = alpha; P.d_eps = d_eps; P.r_eps = r_eps; P.eps = eps; P.out = out_dev;
    cudaStream_t st = (cudaStream_t)stream;
    if (eps > 0.0) {
        if (kmax <= 16) return launch_represent_elem<16, true>(P, st);
        if (kmax <= 32) return launch_represent_elem<32, true>(P, st);
        return launch_represent_elem<64, true>(P, st);
    }
    if (kmax <= 16) return launch_represent_elem<16, false>(P, st);
    if (kmax <= 32) return launch_represent_elem<32, false>(P, st);
    if (kmax <= 64) return launch_represent_elem<64, false>(P, st);
    // longer histories: one launch per block of 64 output steps, each over the gap windows below it
    for (int J = 0; 64 * J < kmax; ++J) {
        P.kblock = J;
        const int rc = launch_represent_elem<64, false, true>(P, st);
        if (rc) return rc;
    }
    return HB_OK;
}
