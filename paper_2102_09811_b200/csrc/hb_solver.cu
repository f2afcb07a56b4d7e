// hb_solver.cu -- block lower-triangular Toeplitz products for the solve.
//
// Replaces the numpy loops of heatbem/solver.py:47-73 (apply_toeplitz) and
// :178-182 (history sums of forward_block_solve).  One CTA owns a tile of 16
// output rows x 16 time steps and walks the (d, column) space in 32-wide
// chunks staged through shared memory; every output is a fixed-order sum
// (d ascending, column ascending), so results are bitwise deterministic.
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

}  // namespace hb

using namespace hb;

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
