// hb_solver.cu -- block lower-triangular Toeplitz products for the solve.
//
// Replaces the numpy loops of heatbem/solver.py:47-73 (apply_toeplitz) and
// :178-182 (history sums of forward_block_solve).  One CTA owns a tile of 16
// output rows x 16 time steps and walks the (d, column) space in 32-wide
// chunks staged through shared memory; every output is a fixed-order sum
// (d ascending, column ascending), so results are bitwise deterministic.
#include <algorithm>
#include <cstdlib>

#include "hb_common.cuh"

namespace hb {

constexpr int kTR = 16, kTK = 16, kTC = 32;

// y[k][r] (+)= sign * sum_{d = d_lo(k)}^{k} sum_c A^d(r, c) x[k - d][c]
// A^d(r, c) = blocks[d][r][c] (or blocks[d][c][r] when transposed);
// diagonal_only: only d == 0 with x[k] for every k.
__global__ void __launch_bounds__(256) k_toeplitz(const double *__restrict__ blocks, int64_t R, int64_t C,
                                                  int transpose, int diagonal_only, int64_t n_steps,
                                                  int64_t k_lo, int64_t d_min, int64_t d_off, int64_t n_blocks,
                                                  const double *__restrict__ x, double *__restrict__ y,
                                                  int accumulate_neg)
{
    __shared__ double As[kTR][kTC + 1];
    __shared__ double Xs[kTK][kTC + 1];
    const int64_t n_out = transpose ? C : R, n_in = transpose ? R : C;
    const int tr = threadIdx.x & 15, tk = threadIdx.x >> 4;
    const int64_t r0 = (int64_t)blockIdx.x * kTR, k0 = k_lo + (int64_t)blockIdx.y * kTK;
    const int64_t r = r0 + tr, k = k0 + tk;
    double acc = 0.0;
    const int64_t kmax_tile = min(k0 + kTK - 1, n_steps - 1);
    const int64_t dmax = diagonal_only ? 0 : min(kmax_tile, d_off + n_blocks - 1);
    for (int64_t d = max(d_min, d_off); d <= dmax; ++d) {
        const double *Ad = blocks + (d - d_off) * R * C;
        for (int64_t c0 = 0; c0 < n_in; c0 += kTC) {
            // stage A^d(r0.., c0..) and x[k - d][c0..] for the tile's k
            for (int i = threadIdx.x; i < kTR * kTC; i += 256) {
                const int rr = i / kTC, cc = i % kTC;
                const int64_t gr = r0 + rr, gc = c0 + cc;
                double v = 0.0;
                if (gr < n_out && gc < n_in) v = transpose ? Ad[gc * C + gr] : Ad[gr * C + gc];
                As[rr][cc] = v;
            }
            for (int i = threadIdx.x; i < kTK * kTC; i += 256) {
                const int kk = i / kTC, cc = i % kTC;
                const int64_t gk = k0 + kk, gc = c0 + cc;
                const int64_t src = diagonal_only ? gk : gk - d;
                double v = 0.0;
                if (gk < n_steps && src >= 0 && gc < n_in) v = x[src * n_in + gc];
                Xs[kk][cc] = v;
            }
            __syncthreads();
            if (k < n_steps && (diagonal_only || d <= k)) {
#pragma unroll 8
                for (int cc = 0; cc < kTC; ++cc) acc = fma(As[tr][cc], Xs[tk][cc], acc);
            }
            __syncthreads();
        }
    }
    if (r < n_out && k < n_steps) {
        double *dst = y + k * n_out + r;
        if (accumulate_neg) *dst = *dst - acc;
        else *dst = acc;
    }
}

// ---------------------------------------------------------------------------
// Forward substitution (solver.py:165-184) as one call: per time step k the
// history h = sum_{d=1..k} A^d x[k-d] (warp per output row: lanes stream a
// block row, fixed-order butterfly), then x[k] = (A^0)^{-1} (rhs[k] - h) with
// the inverse cached by the caller (warp per row).  2 E_t launches, no host
// round trips.
// ---------------------------------------------------------------------------
__device__ __forceinline__ double warp_sum(double v)
{
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
    return v;
}

// A^d(r, c) = blocks[d][r][c]; 4 warps per output row r (the c range split
// in 4 interleaved quarters), partials added in warp order
constexpr int kHW = 4;
// (R output rows -- all of a square operator, or one rank's row shard -- by
// C columns; blocks d = 1..min(k, n_blocks - 1))
__global__ void __launch_bounds__(256) k_hist_rows(const double *__restrict__ blocks, int64_t R, int64_t C,
                                                   int64_t n_blocks, int64_t k, const double *__restrict__ x,
                                                   double *__restrict__ h)
{
    __shared__ double part[8];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, sub = warp % kHW;
    const int64_t r = (int64_t)blockIdx.x * (8 / kHW) + warp / kHW;
    double acc = 0.0;
    if (r < R) {
        const int64_t dmax = min(k, n_blocks - 1);
        for (int64_t d = 1; d <= dmax; ++d) {
            const double *a = blocks + (d * R + r) * C;
            const double *xv = x + (k - d) * C;
#pragma unroll 4
            for (int64_t c = lane + 32 * sub; c < C; c += 32 * kHW) acc = fma(__ldg(a + c), __ldg(xv + c), acc);
        }
    }
    acc = warp_sum(acc);
    if (lane == 0) part[warp] = acc;
    __syncthreads();
    if (sub == 0 && lane == 0 && r < R) {
        double v = 0.0;
        for (int w = 0; w < kHW; ++w) v += part[warp + w];
        h[r] = v;
    }
}

// Toeplitz product, non-transposed: y[k][r] = sum_{d<=k} A^d(r, :) x[k-d] for a
// tile of up to kMK output times; one warp per (row, time tile): every element
// of A^d(r, :) is loaded once and updates the tile's times k >= d (x from L1)
constexpr int kMK = 8;
// the warp-per-row form re-reads a block row once per time tile: short
// histories only (config 2: 0.46 vs 1.47 ms); long ones (config 5, 256 steps)
// keep the shared-memory tiles of k_toeplitz, which reuse each staged tile
constexpr int64_t kRowsMaxSteps = 64;
__global__ void __launch_bounds__(256) k_toep_rows(const double *__restrict__ blocks, int64_t n_out, int64_t n_in,
                                                   int64_t n_steps, const double *__restrict__ x,
                                                   double *__restrict__ y, int64_t d_off, int64_t n_blocks)
{
    const int lane = threadIdx.x & 31;
    const int64_t wid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t r = wid % n_out, k0 = (wid / n_out) * kMK;
    if (k0 >= n_steps) return;
    const int nk = (int)(n_steps - k0 < kMK ? n_steps - k0 : (int64_t)kMK);
    double acc[kMK];
#pragma unroll
    for (int i = 0; i < kMK; ++i) acc[i] = 0.0;
    // blocks hold A^d for d in [d_off, d_off + n_blocks) (the full operator: d_off = 0)
    const int64_t dmax = min(k0 + nk - 1, d_off + n_blocks - 1);
    for (int64_t d = d_off; d <= dmax; ++d) {
        const double *a = blocks + ((d - d_off) * n_out + r) * n_in;
        const int ilo = (int)(d > k0 ? d - k0 : 0);       // tile times k = k0 + i with k >= d
        for (int64_t c = lane; c < n_in; c += 32) {
            const double av = __ldg(a + c);
            const double *xc = x + (k0 - d) * n_in + c;
#pragma unroll
            for (int i = 0; i < kMK; ++i)
                if (i >= ilo && i < nk) acc[i] = fma(av, __ldg(xc + i * n_in), acc[i]);
        }
    }
#pragma unroll
    for (int i = 0; i < kMK; ++i) {
        const double v = warp_sum(acc[i]);
        if (lane == 0 && i < nk) y[(k0 + i) * n_out + r] = v;
    }
}

// transposed, A^d(r, c) = blocks[d][c][r]: lanes = 32 consecutive outputs r,
// the 8 warps split the input index c, partials added in warp order
__global__ void __launch_bounds__(256) k_hist_cols(const double *__restrict__ blocks, int64_t n, int64_t k,
                                                   const double *__restrict__ x, double *__restrict__ h)
{
    __shared__ double part[8][33];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t r = (int64_t)blockIdx.x * 32 + lane;
    double acc = 0.0;
    if (r < n) {
        for (int64_t d = 1; d <= k; ++d) {
            const double *a = blocks + d * n * n + r;
            const double *xv = x + (k - d) * n;
            for (int64_t c = warp; c < n; c += 8) acc = fma(__ldg(a + c * n), __ldg(xv + c), acc);
        }
    }
    part[warp][lane] = acc;
    __syncthreads();
    if (warp == 0 && r < n) {
        double v = 0.0;
        for (int w = 0; w < 8; ++w) v += part[w][lane];
        h[r] = v;
    }
}

// x_k[i] = sum_j inv[i][j] (rhs_k[j] - h[j]); kHW warps per row i (the j range
// split in interleaved quarters, partials added in warp order)
__global__ void __launch_bounds__(256) k_inv_apply(const double *__restrict__ inv, int64_t n,
                                                   const double *__restrict__ rhs_k, const double *__restrict__ h,
                                                   int has_h, double *__restrict__ x_k)
{
    __shared__ double part[8];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, sub = warp % kHW;
    const int64_t i = (int64_t)blockIdx.x * (8 / kHW) + warp / kHW;
    double acc = 0.0;
    if (i < n) {
        const double *a = inv + i * n;
#pragma unroll 4
        for (int64_t j = lane + 32 * sub; j < n; j += 32 * kHW) {
            const double v = has_h ? __ldg(rhs_k + j) - __ldg(h + j) : __ldg(rhs_k + j);
            acc = fma(__ldg(a + j), v, acc);
        }
    }
    acc = warp_sum(acc);
    if (lane == 0) part[warp] = acc;
    __syncthreads();
    if (sub == 0 && lane == 0 && i < n) {
        double v = 0.0;
        for (int w = 0; w < kHW; ++w) v += part[warp + w];
        x_k[i] = v;
    }
}

// ---------------------------------------------------------------------------
// Blocked forward substitution: the steps in tiles of kFT.  Per tile [k0,
// k0 + nk) the history from earlier tiles (the "far" terms, k - d < k0) of
// all nk steps in one pass that reads each block once (k_hist_far); inside
// the tile, per step, only the near terms d <= k - k0 (blocks 1..kFT-1,
// L2-resident) and the inverse apply.  Block reads per solve: about
// E_t^2 / (2 kFT) instead of E_t^2 / 2.
// ---------------------------------------------------------------------------
constexpr int kFT = 8;

// H[i][r] = sum_{d >= 1} A^d(r, :) x[k0 + i - d] over the terms with
// 0 <= k0 + i - d < k0, i < nk; 4 warps per row split the columns, each lane
// keeps x[k0 + i - d][c] (i < kFT) of the current d in registers -- one new x
// load per element of A as d grows; sums in fixed order (column, d, lanes, warps)
// (R output rows -- all of a square operator or one rank's row shard -- by C columns)
__global__ void __launch_bounds__(256, 3) k_hist_far(const double *__restrict__ blocks, int64_t R, int64_t C,
                                                  int64_t n_blocks, int64_t k0, int nk, const double *__restrict__ x,
                                                  double *__restrict__ H)
{
    __shared__ double part[8][kFT];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, sub = warp % kHW;
    const int64_t r = (int64_t)blockIdx.x * (8 / kHW) + warp / kHW;
    double acc[kFT];
#pragma unroll
    for (int i = 0; i < kFT; ++i) acc[i] = 0.0;
    if (r < R) {
        const int64_t dmax = min(k0 + nk - 1, n_blocks - 1);
        for (int64_t c = lane + 32 * sub; c < C; c += 32 * kHW) {
            double xw[kFT];   // xw[i] = x[k0 + i - d][c], 0 unless 0 <= k0 + i - d < k0
#pragma unroll
            for (int i = 0; i < kFT; ++i) xw[i] = 0.0;
            const double *a = blocks + r * C + c;
            for (int64_t db = 1; db <= dmax; db += kFT) {
                // the loads of kFT blocks d first (independent: in flight together), then the FMAs
                double av[kFT], xn[kFT];
#pragma unroll
                for (int u = 0; u < kFT; ++u) {
                    const int64_t d = db + u;
                    av[u] = d <= dmax ? __ldg(a + d * R * C) : 0.0;
                    xn[u] = (d <= dmax && k0 - d >= 0) ? __ldg(x + (k0 - d) * C + c) : 0.0;
                }
#pragma unroll
                for (int u = 0; u < kFT; ++u) {
#pragma unroll
                    for (int i = kFT - 1; i > 0; --i) xw[i] = xw[i - 1];
                    xw[0] = xn[u];
#pragma unroll
                    for (int i = 0; i < kFT; ++i) acc[i] = fma(av[u], xw[i], acc[i]);
                }
            }
        }
    }
#pragma unroll
    for (int i = 0; i < kFT; ++i) acc[i] = warp_sum(acc[i]);
    if (lane == 0) {
#pragma unroll
        for (int i = 0; i < kFT; ++i) part[warp][i] = acc[i];
    }
    __syncthreads();
    if (sub == 0 && lane < nk && r < R) {
        double v = 0.0;
        for (int w = 0; w < kHW; ++w) v += part[warp + w][lane];
        H[lane * R + r] = v;
    }
}

// h[r] = Hk[r] (far terms, if any) + sum_{d=1..dn} A^d(r, :) x[k - d] (near
// terms, dn < kFT; the blocks are L2-resident across the tile's steps)
__global__ void __launch_bounds__(256) k_hist_near(const double *__restrict__ blocks, int64_t R, int64_t C,
                                                   int64_t k, int64_t dn, const double *__restrict__ x,
                                                   const double *__restrict__ Hk, double *__restrict__ h)
{
    __shared__ double part[8];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, sub = warp % kHW;
    const int64_t r = (int64_t)blockIdx.x * (8 / kHW) + warp / kHW;
    double acc = 0.0;
    if (r < R) {
        // column-outer, d-inner: the dn loads of a column are in flight together
        for (int64_t c = lane + 32 * sub; c < C; c += 32 * kHW) {
            double av[kFT - 1], xv[kFT - 1];
#pragma unroll
            for (int d = 1; d < kFT; ++d) {
                av[d - 1] = d <= dn ? __ldg(blocks + (d * R + r) * C + c) : 0.0;
                xv[d - 1] = d <= dn ? __ldg(x + (k - d) * C + c) : 0.0;
            }
#pragma unroll
            for (int d = 1; d < kFT; ++d)
                if (d <= dn) acc = fma(av[d - 1], xv[d - 1], acc);
        }
    }
    acc = warp_sum(acc);
    if (lane == 0) part[warp] = acc;
    __syncthreads();
    if (sub == 0 && lane == 0 && r < R) {
        double v = Hk ? Hk[r] : 0.0;
        for (int w = 0; w < kHW; ++w) v += part[warp + w];
        h[r] = v;
    }
}

constexpr int kNW = 8;
// x_k[i] = sum_j inv[i][j] (rhs_k[j] - h[j]) for the blocked substitution: one
// row per CTA, 8 warps over interleaved 32-column slices, partials in warp order
__global__ void __launch_bounds__(256) k_inv_apply_row(const double *__restrict__ inv, int64_t n,
                                                       const double *__restrict__ rhs_k,
                                                       const double *__restrict__ h, int has_h,
                                                       double *__restrict__ x_k)
{
    __shared__ double part[kNW];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t i = blockIdx.x;
    const double *a = inv + i * n;
    double acc = 0.0;
#pragma unroll 4
    for (int64_t j = lane + 32 * warp; j < n; j += 32 * kNW) {
        const double v = has_h ? __ldg(rhs_k + j) - __ldg(h + j) : __ldg(rhs_k + j);
        acc = fma(__ldg(a + j), v, acc);
    }
    acc = warp_sum(acc);
    if (lane == 0) part[warp] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double v = 0.0;
        for (int w = 0; w < kNW; ++w) v += part[w];
        x_k[i] = v;
    }
}

}  // namespace hb

using namespace hb;

// ---------------------------------------------------------------------------
// Large operators (>= kMmaMinRows output rows; plain or transposed): the block-Toeplitz
// product as one tensor-core GEMM per block d,
//   Y[k][r] += sum_c X[k - d][c] A^d[r][c]   (k >= d),
// with mma.sync m8n8k4 f64 (DMMA): M = steps (a CTA owns a 64-step tile,
// 8-step fragments), N = 32 output rows per CTA (4 warps; warp w: rows
// 8w..8w+7), K = the input index in 32-wide chunks staged in shared memory
// (row stride 36: conflict-free fragment loads) -- per (chunk, d) the A^d tile
// and the 96-row x window of the step tile.  TR (K', D^T): the A^d tile is
// staged as [in 32][out 32] and read as the B fragment B[k = in][n = out].  Every element of A is read from HBM once per
// 64-step tile (the warp-per-row kernel re-reads it once per 8-step tile);
// sums run in a fixed order (chunk, d, K step).
// ---------------------------------------------------------------------------
constexpr int kMmaMinRows = 1024;
constexpr int kMR = 32, kMC = 32, kMS = kMC + 4, kMT = 4 * kMR;   // kMT threads: warp w owns rows 8w..8w+7

__device__ __forceinline__ void dmma884s(double &d0, double &d1, double a, double b)
{
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

// the DMMAs of one staged (A^d tile, x window): m-tiles LO..7 (those below
// mtiles), k-steps outer so the live tiles' accumulators interleave; bs: this
// lane's B element of k-step 0 (k-step ks at + 4 ks rows (TR) / columns), xw:
// its x window element of m-tile 0, k-step 0 (m-tile mt at + 8 mt rows)
template <int LO, bool TR>
__device__ __forceinline__ void mma_live(double (&acc)[8][2], const double *bs, const double *xw, int mtiles)
{
#pragma unroll
    for (int ks = 0; ks < kMC / 4; ++ks) {
        const double b = TR ? bs[4 * ks * (kMR + 4)] : bs[4 * ks];
#pragma unroll
        for (int mt = LO; mt < 8; ++mt) {
            if (mt >= mtiles) continue;
            dmma884s(acc[mt][0], acc[mt][1], xw[8 * mt * kMS + 4 * ks], b);
        }
    }
}

// TR: the transposed product Y[k][c] += sum_r X[k - d][r] A^d[r][c] (A tile staged
// as [r][c], B fragment B[k = r][n = c]).
// grid.z > 1 (split-K of operators with few output rows): CTA z takes the
// input columns [z csz, (z + 1) csz) and writes its partial product to
// y + z ystride; k_sum_partials adds the partials in z order (deterministic).
template <bool TR>
__global__ void __launch_bounds__(kMT) k_toep_mma(const double *__restrict__ blocks, int64_t R, int64_t C,
                                                  int64_t n_steps, const double *__restrict__ x,
                                                  double *__restrict__ y, int64_t d_off, int64_t n_blocks,
                                                  int64_t csz, int64_t ystride)
{
    const int64_t n_in = TR ? R : C, n_out = TR ? C : R;
    int64_t c_begin = 0, c_end = n_in;
    if (gridDim.z > 1) {
        c_begin = (int64_t)blockIdx.z * csz;
        c_end = min(n_in, c_begin + csz);
        y += (int64_t)blockIdx.z * ystride;
    }
    // x window of a group of 32 blocks d in [db, db + 32): the rows k - d for the
    // tile's steps k_lo + j, i.e. x[k_lo - db - 32 + w], w = 0..95 (row of step j
    // at block d: w = j - (d - db) + 32)
    __shared__ __align__(16) double Xw[96][kMS];
    // A^d tile: [out 32][in 32] (row stride 36) or, transposed, [in 32][out 32] (stride 36)
    __shared__ __align__(16) double As[kMR * kMS > kMC * (kMR + 4) ? kMR * kMS : kMC * (kMR + 4)];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, gq = lane >> 2, tq = lane & 3;
    const int64_t r0 = (int64_t)blockIdx.x * kMR, k_lo = (int64_t)blockIdx.y * 64;
    const int nst = (int)min((int64_t)64, n_steps - k_lo), mtiles = (nst + 7) >> 3;
    double acc[8][2];
#pragma unroll
    for (int mt = 0; mt < 8; ++mt) acc[mt][0] = acc[mt][1] = 0.0;
    const int64_t dmax = min(k_lo + nst - 1, d_off + n_blocks - 1);
    for (int64_t c0 = c_begin; c0 < c_end; c0 += kMC) {
        for (int64_t db = d_off; db <= dmax; db += 32) {
            __syncthreads();
            for (int i = tid; i < 96 * kMC; i += kMT) {
                const int w = i / kMC, cc = i % kMC;
                const int64_t xr = k_lo - db - 32 + w;
                Xw[w][cc] = (xr >= 0 && xr < k_lo + nst && c0 + cc < n_in) ? __ldg(x + xr * n_in + c0 + cc) : 0.0;
            }
            const int64_t de = min(dmax, db + 31);
            // A^d tiles pass through registers: the loads of tile d + 1 are issued
            // before the DMMAs of tile d, so HBM latency overlaps the tensor work
            constexpr int PT = kMR * kMC / kMT;   // elements per thread
            auto fetch = [&](int64_t d, double (&v)[PT]) {
                const double *Ad = blocks + (d - d_off) * R * C;
#pragma unroll
                for (int u = 0; u < PT; ++u) {
                    const int i = tid + kMT * u;
                    if (TR) {   // rows c0 + ii of A, 32 output columns r0.. (coalesced along the row)
                        const int ii = i / kMR, oo = i % kMR;
                        v[u] = (c0 + ii < n_in && r0 + oo < n_out) ? __ldg(Ad + (c0 + ii) * C + r0 + oo) : 0.0;
                    } else {
                        const int rr = i / kMC, cc = i % kMC;
                        v[u] = (r0 + rr < R && c0 + cc < C) ? __ldg(Ad + (r0 + rr) * C + c0 + cc) : 0.0;
                    }
                }
            };
            double nxt[PT];
            fetch(db, nxt);
            for (int64_t d = db; d <= de; ++d) {
                __syncthreads();
#pragma unroll
                for (int u = 0; u < PT; ++u) {
                    const int i = tid + kMT * u;
                    if (TR) As[(i / kMR) * (kMR + 4) + i % kMR] = nxt[u];
                    else As[(i / kMC) * kMS + i % kMC] = nxt[u];
                }
                __syncthreads();
                if (d < de) fetch(d + 1, nxt);
                const int dl = (int)(d - k_lo);      // steps j < dl of the tile have no term (k < d)
                const int wo = 32 - (int)(d - db);   // window row of step j: j + wo
                // m-tiles with every step below dl are skipped: a predicated DMMA
                // still takes its tensor-pipe slot, so the live range [mt_lo, 8)
                // selects a loop whose start is a compile-time constant (the live
                // tiles' DMMAs interleave, independent accumulators)
                const int mt_lo = dl > 0 ? dl >> 3 : 0;
                const double *bs = TR ? &As[tq * (kMR + 4) + 8 * warp + gq] : &As[(8 * warp + gq) * kMS + tq];
                const double *xw = &Xw[gq + wo][tq];
                switch (mt_lo) {
                case 0: mma_live<0, TR>(acc, bs, xw, mtiles); break;
                case 1: mma_live<1, TR>(acc, bs, xw, mtiles); break;
                case 2: mma_live<2, TR>(acc, bs, xw, mtiles); break;
                case 3: mma_live<3, TR>(acc, bs, xw, mtiles); break;
                case 4: mma_live<4, TR>(acc, bs, xw, mtiles); break;
                case 5: mma_live<5, TR>(acc, bs, xw, mtiles); break;
                case 6: mma_live<6, TR>(acc, bs, xw, mtiles); break;
                default: mma_live<7, TR>(acc, bs, xw, mtiles); break;
                }
            }
        }
    }
#pragma unroll
    for (int mt = 0; mt < 8; ++mt) {
        const int j = 8 * mt + gq;
        if (j >= nst) continue;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int64_t r = r0 + 8 * warp + 2 * tq + h;
            if (r < n_out) y[(k_lo + j) * n_out + r] = acc[mt][h];
        }
    }
}

static int launch_toep_mma(const double *blocks, int64_t R, int64_t C, int tr, int64_t n_steps, const double *x,
                           double *y, int64_t d_off, int64_t n_blocks, cudaStream_t st, const char *what,
                           int64_t groups = 1, int64_t csz = 0)
{
    dim3 g((unsigned)cdiv(tr ? C : R, kMR), (unsigned)cdiv(n_steps, 64), (unsigned)groups);
    const int64_t ystride = n_steps * (tr ? C : R);
    if (tr) k_toep_mma<true><<<g, kMT, 0, st>>>(blocks, R, C, n_steps, x, y, d_off, n_blocks, csz, ystride);
    else k_toep_mma<false><<<g, kMT, 0, st>>>(blocks, R, C, n_steps, x, y, d_off, n_blocks, csz, ystride);
    return cuda_check(cudaGetLastError(), what);
}

__global__ void k_sum_partials(const double *__restrict__ part, int64_t groups, int64_t n, double *__restrict__ y)
{
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        double v = part[i];
        for (int64_t z = 1; z < groups; ++z) v += part[z * n + i];
        y[i] = v;
    }
}

// split-K of the tensor-core product for operators with few output rows
// (< kMmaMinRows, whose row tiles alone cannot fill the GPU): groups of
// 32-column chunks of the input index, about 12 groups; the split depends on
// the input length only, so row shards of an operator (RowShardedToeplitz)
// sum in the same order as the whole operator.  Returns the group count and
// the columns per group.
// Large operators (>= kMmaMinRows rows) split too, in groups of 64 chunks
// (2048 input columns): the row tiles alone give one CTA wave or less
// (12288 rows: 384 CTAs over 148 SMs, 2.6 per SM -- the SMs with 3 set the
// time); 12288 columns -> 6 groups, 2304 CTAs.  Again a function of the
// input length only (within the large-operator regime).
static int64_t toep_groups(int64_t n_in, int64_t n_out, int64_t n_steps, int64_t *csz)
{
    (void)n_steps;
    const int64_t chunks = cdiv(n_in, kMC);
    *csz = chunks * kMC;
    if (chunks < 2) return 1;
    if (n_out >= kMmaMinRows) {
        static const int64_t per_big = getenv("HB_TOEP_CHUNKS_BIG") ? atoll(getenv("HB_TOEP_CHUNKS_BIG")) : 64;
        if (per_big <= 0 || chunks <= per_big) return 1;
        const int64_t g = cdiv(chunks, per_big), per = cdiv(chunks, g);
        *csz = per * kMC;
        return cdiv(chunks, per);
    }
    static const int64_t target = getenv("HB_TOEP_GROUPS") ? atoll(getenv("HB_TOEP_GROUPS")) : 12;
    const int64_t per = cdiv(chunks, std::max<int64_t>(1, target));
    *csz = per * kMC;
    return cdiv(chunks, per);
}

extern "C" size_t hb_toeplitz_apply_workspace(int64_t n_blocks, int64_t R, int64_t C, int transpose,
                                              int diagonal_only, int64_t n_steps)
{
    if (diagonal_only || n_blocks < 1 || R < 1 || C < 1 || n_steps < 1) return 0;
    const int64_t n_out = transpose ? C : R, n_in = transpose ? R : C;
    int64_t csz;
    const int64_t groups = toep_groups(n_in, n_out, n_steps, &csz);
    return groups > 1 ? (size_t)groups * (size_t)(n_steps * n_out) * sizeof(double) : 0;
}

extern "C" int hb_toeplitz_apply_ws(int64_t n_blocks, int64_t R, int64_t C, const double *blocks_dev, int transpose,
                                    int diagonal_only, int64_t n_steps, const double *x_dev, double *y_dev,
                                    void *workspace_dev, size_t workspace_bytes, void *stream)
{
    const size_t need = hb_toeplitz_apply_workspace(n_blocks, R, C, transpose, diagonal_only, n_steps);
    if (need == 0 || !workspace_dev || workspace_bytes < need || (!diagonal_only && n_steps > n_blocks) || !blocks_dev ||
        !x_dev || !y_dev)
        return hb_toeplitz_apply(n_blocks, R, C, blocks_dev, transpose, diagonal_only, n_steps, x_dev, y_dev, stream);
    // tensor-core product split over groups of input columns into partials, summed in group order
    const int64_t n_out = transpose ? C : R, n_in = transpose ? R : C;
    int64_t csz;
    const int64_t groups = toep_groups(n_in, n_out, n_steps, &csz);
    double *part = (double *)workspace_dev;
    cudaStream_t st = (cudaStream_t)stream;
    int rc = launch_toep_mma(blocks_dev, R, C, transpose, n_steps, x_dev, part, 0, n_blocks, st,
                             "hb_toeplitz_apply_ws", groups, csz);
    if (rc) return rc;
    const int64_t n = n_steps * n_out;
    k_sum_partials<<<(unsigned)std::min<int64_t>(cdiv(n, 256), 148 * 8), 256, 0, st>>>(part, groups, n, y_dev);
    return cuda_check(cudaGetLastError(), "hb_toeplitz_apply_ws");
}

extern "C" int hb_toeplitz_apply(int64_t n_blocks, int64_t R, int64_t C, const double *blocks_dev, int transpose,
                                 int diagonal_only, int64_t n_steps, const double *x_dev, double *y_dev,
                                 void *stream)
{
    if (n_blocks < 1 || R < 1 || C < 1 || n_steps < 1 || !blocks_dev || !x_dev || !y_dev) {
        set_error("hb_toeplitz_apply: bad arguments");
        return HB_ERR_INVALID;
    }
    if (!diagonal_only && n_steps > n_blocks) {
        set_error("hb_toeplitz_apply: more time steps (%lld) than stored blocks (%lld)", (long long)n_steps,
                  (long long)n_blocks);
        return HB_ERR_INVALID;
    }
    const int64_t n_out = transpose ? C : R;
    if (!diagonal_only && n_out >= kMmaMinRows)   // tensor-core GEMMs
        return launch_toep_mma(blocks_dev, R, C, transpose, n_steps, x_dev, y_dev, 0, n_blocks, (cudaStream_t)stream,
                               "hb_toeplitz_apply");
    if (!transpose && !diagonal_only && n_steps <= kRowsMaxSteps) {   // warp per (row, kMK-step tile)
        const int64_t warps = n_out * cdiv(n_steps, kMK);
        k_toep_rows<<<(unsigned)cdiv(warps * 32, 256), 256, 0, (cudaStream_t)stream>>>(blocks_dev, R, C, n_steps,
                                                                                      x_dev, y_dev, 0, n_blocks);
        return cuda_check(cudaGetLastError(), "hb_toeplitz_apply");
    }
    dim3 g((unsigned)cdiv(n_out, kTR), (unsigned)cdiv(n_steps, kTK));
    k_toeplitz<<<g, 256, 0, (cudaStream_t)stream>>>(blocks_dev, R, C, transpose, diagonal_only, n_steps, 0, 0, 0,
                                                    n_blocks, x_dev, y_dev, 0);
    return cuda_check(cudaGetLastError(), "hb_toeplitz_apply");
}

extern "C" int hb_toeplitz_apply_range(int64_t d_off, int64_t n_blocks, int64_t R, int64_t C, const double *blocks_dev,
                                       int transpose, int64_t n_steps, const double *x_dev, double *y_dev,
                                       void *stream)
{
    if (d_off < 0 || n_blocks < 1 || R < 1 || C < 1 || n_steps < 1 || !blocks_dev || !x_dev || !y_dev) {
        set_error("hb_toeplitz_apply_range: bad arguments");
        return HB_ERR_INVALID;
    }
    const int64_t n_out = transpose ? C : R;
    if (n_out >= kMmaMinRows)
        return launch_toep_mma(blocks_dev, R, C, transpose, n_steps, x_dev, y_dev, d_off, n_blocks,
                               (cudaStream_t)stream, "hb_toeplitz_apply_range");
    if (!transpose && n_steps <= kRowsMaxSteps) {
        const int64_t warps = n_out * cdiv(n_steps, kMK);
        k_toep_rows<<<(unsigned)cdiv(warps * 32, 256), 256, 0, (cudaStream_t)stream>>>(blocks_dev, R, C, n_steps,
                                                                                      x_dev, y_dev, d_off, n_blocks);
        return cuda_check(cudaGetLastError(), "hb_toeplitz_apply_range");
    }
    dim3 g((unsigned)cdiv(n_out, kTR), (unsigned)cdiv(n_steps, kTK));
    k_toeplitz<<<g, 256, 0, (cudaStream_t)stream>>>(blocks_dev, R, C, transpose, 0, n_steps, 0, 0, d_off, n_blocks,
                                                    x_dev, y_dev, 0);
    return cuda_check(cudaGetLastError(), "hb_toeplitz_apply_range");
}

extern "C" int hb_forward_subst_step(int64_t n_blocks, int64_t R, int64_t C, const double *blocks_dev, int transpose,
                                     int64_t k, const double *x_dev, double *acc_dev, void *stream)
{
    if (n_blocks < 1 || R < 1 || C < 1 || k < 0 || k >= n_blocks || !blocks_dev || !x_dev || !acc_dev) {
        set_error("hb_forward_subst_step: bad arguments");
        return HB_ERR_INVALID;
    }
    if (k == 0) return HB_OK;
    const int64_t n_out = transpose ? C : R;
    // one output time (k); y row offset so that y + k * n_out == acc
    dim3 g((unsigned)cdiv(n_out, kTR), 1);
    k_toeplitz<<<g, 256, 0, (cudaStream_t)stream>>>(blocks_dev, R, C, transpose, 0, k + 1, k, 1, 0, n_blocks, x_dev,
                                                    acc_dev - k * n_out, 1);
    return cuda_check(cudaGetLastError(), "hb_forward_subst_step");
}

extern "C" int hb_forward_solve(int64_t n_blocks, int64_t n, const double *blocks_dev, int transpose,
                                int diagonal_only, int64_t n_steps, const double *inv_dev, const double *rhs_dev,
                                double *x_dev, double *h_work_dev, void *stream)
{
    if (n_blocks < 1 || n < 1 || n_steps < 1 || !blocks_dev || !inv_dev || !rhs_dev || !x_dev || !h_work_dev ||
        (!diagonal_only && n_steps > n_blocks)) {
        set_error("hb_forward_solve: bad arguments");
        return HB_ERR_INVALID;
    }
    cudaStream_t st = (cudaStream_t)stream;
    const unsigned g_rows = (unsigned)cdiv(n, 8 / kHW), g_cols = (unsigned)cdiv(n, 32);
    const unsigned g_hist = (unsigned)cdiv(n, 8 / kHW);
    for (int64_t k = 0; k < n_steps; ++k) {
        const bool hist = !diagonal_only && k > 0;
        if (hist) {
            if (transpose) k_hist_cols<<<g_cols, 256, 0, st>>>(blocks_dev, n, k, x_dev, h_work_dev);
            else k_hist_rows<<<g_hist, 256, 0, st>>>(blocks_dev, n, n, n_blocks, k, x_dev, h_work_dev);
        }
        k_inv_apply<<<g_rows, 256, 0, st>>>(inv_dev, n, rhs_dev + k * n, h_work_dev, hist ? 1 : 0, x_dev + k * n);
    }
    return cuda_check(cudaGetLastError(), "hb_forward_solve");
}

extern "C" size_t hb_forward_solve_workspace(int64_t n) { return n < 1 ? 0 : (size_t)(kFT + 1) * (size_t)n * sizeof(double); }

extern "C" int hb_forward_solve_ws(int64_t n_blocks, int64_t n, const double *blocks_dev, int transpose,
                                   int diagonal_only, int64_t n_steps, const double *inv_dev, const double *rhs_dev,
                                   double *x_dev, void *workspace_dev, size_t workspace_bytes, void *stream)
{
    if (n_blocks < 1 || n < 1 || n_steps < 1 || !blocks_dev || !inv_dev || !rhs_dev || !x_dev || !workspace_dev ||
        workspace_bytes < hb_forward_solve_workspace(n) || (!diagonal_only && n_steps > n_blocks)) {
        set_error("hb_forward_solve_ws: bad arguments");
        return HB_ERR_INVALID;
    }
    double *h = (double *)workspace_dev, *H = h + n;
    if (transpose || diagonal_only)   // the per-step form (transposed history kernel / no history)
        return hb_forward_solve(n_blocks, n, blocks_dev, transpose, diagonal_only, n_steps, inv_dev, rhs_dev, x_dev,
                                h, stream);
    cudaStream_t st = (cudaStream_t)stream;
    const unsigned g_hist = (unsigned)cdiv(n, 8 / kHW);
    for (int64_t k0 = 0; k0 < n_steps; k0 += kFT) {
        const int nk = (int)std::min<int64_t>(kFT, n_steps - k0);
        if (k0 > 0) k_hist_far<<<g_hist, 256, 0, st>>>(blocks_dev, n, n, n_blocks, k0, nk, x_dev, H);
        for (int64_t k = k0; k < k0 + nk; ++k) {
            const int64_t dn = std::min(k - k0, n_blocks - 1);
            const bool hist = k > 0;
            if (hist)
                k_hist_near<<<g_hist, 256, 0, st>>>(blocks_dev, n, n, k, dn, x_dev,
                                                    k0 > 0 ? H + (k - k0) * n : nullptr, h);
            k_inv_apply_row<<<(unsigned)n, 256, 0, st>>>(inv_dev, n, rhs_dev + k * n, h, hist ? 1 : 0,
                                                         x_dev + k * n);
        }
    }
    return cuda_check(cudaGetLastError(), "hb_forward_solve_ws");
}

extern "C" int hb_forward_history(int64_t n_blocks, int64_t R, int64_t C, const double *blocks_dev, int64_t k,
                                  const double *x_dev, double *h_dev, void *stream)
{
    if (n_blocks < 1 || R < 1 || C < 1 || k < 0 || !blocks_dev || !x_dev || !h_dev) {
        set_error("hb_forward_history: bad arguments");
        return HB_ERR_INVALID;
    }
    k_hist_rows<<<(unsigned)cdiv(R, 8 / kHW), 256, 0, (cudaStream_t)stream>>>(blocks_dev, R, C, n_blocks, k, x_dev,
                                                                            h_dev);
    return cuda_check(cudaGetLastError(), "hb_forward_history");
}

extern "C" int hb_forward_history_far(int64_t n_blocks, int64_t R, int64_t C, const double *blocks_dev, int64_t k0,
                                      int64_t nk, const double *x_dev, double *H_dev, void *stream)
{
    if (n_blocks < 1 || R < 1 || C < 1 || k0 < 1 || nk < 1 || nk > kFT || !blocks_dev || !x_dev || !H_dev) {
        set_error("hb_forward_history_far: bad arguments");
        return HB_ERR_INVALID;
    }
    k_hist_far<<<(unsigned)cdiv(R, 8 / kHW), 256, 0, (cudaStream_t)stream>>>(blocks_dev, R, C, n_blocks, k0, (int)nk,
                                                                           x_dev, H_dev);
    return cuda_check(cudaGetLastError(), "hb_forward_history_far");
}

extern "C" int hb_forward_history_near(int64_t n_blocks, int64_t R, int64_t C, const double *blocks_dev, int64_t k,
                                       int64_t k0, const double *x_dev, const double *Hk_dev, double *h_dev,
                                       void *stream)
{
    if (n_blocks < 1 || R < 1 || C < 1 || k < 1 || k0 < 0 || k0 > k || !blocks_dev || !x_dev || !h_dev) {
        set_error("hb_forward_history_near: bad arguments");
        return HB_ERR_INVALID;
    }
    if (k - k0 >= kFT) {
        set_error("hb_forward_history_near: k - k0 must be below the tile length 8");
        return HB_ERR_INVALID;
    }
    k_hist_near<<<(unsigned)cdiv(R, 8 / kHW), 256, 0, (cudaStream_t)stream>>>(
        blocks_dev, R, C, k, std::min(k - k0, n_blocks - 1), x_dev, Hk_dev, h_dev);
    return cuda_check(cudaGetLastError(), "hb_forward_history_near");
}

extern "C" int hb_inv_apply(int64_t n, const double *inv_dev, const double *rhs_dev, const double *h_dev,
                            double *x_dev, void *stream)
{
    if (n < 1 || !inv_dev || !rhs_dev || !x_dev) {
        set_error("hb_inv_apply: bad arguments");
        return HB_ERR_INVALID;
    }
    k_inv_apply_row<<<(unsigned)n, 256, 0, (cudaStream_t)stream>>>(inv_dev, n, rhs_dev, h_dev,
                                                                             h_dev ? 1 : 0, x_dev);
    return cuda_check(cudaGetLastError(), "hb_inv_apply");
}
