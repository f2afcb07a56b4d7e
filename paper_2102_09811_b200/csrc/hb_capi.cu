// hb_capi.cu -- C-ABI glue: error state, version, FP64 throughput probe,
// and the curl combination D = D2 + alpha^2 sum_o T_o^T V T_o.
#include <cstdarg>
#include <cstdio>

#include "hb_common.cuh"

namespace hb {

static thread_local char g_err[512] = "";

void set_error(const char *fmt, ...)
{
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
}

int cuda_check(cudaError_t err, const char *what)
{
    if (err == cudaSuccess) return HB_OK;
    set_error("%s: %s (%s)", what, cudaGetErrorString(err), cudaGetErrorName(err));
    return HB_ERR_CUDA;
}

// 8 independent DFMA chains per thread; nothing else in the loop body.
__global__ void __launch_bounds__(256) k_fp64_probe(int64_t iters, double *sink)
{
    double a[8];
    const double m = 1.0 + 1e-9 * threadIdx.x, c = 1e-12;
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = 1.0 + k * 1e-3 + blockIdx.x * 1e-7;
    for (int64_t i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) a[k] = fma(a[k], m, c);
    }
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += a[k];
    if (s == 12345.678) sink[blockIdx.x] = s;   // never true; keeps the chains live
}

// D[d][m][n] = D2[d][m][n] + a2 * sum_{(e,i) in star(m)} sum_{(f,j) in star(n)}
//              (curl_{e,i} . curl_{f,j}) V[d][e][f], computed for n >= m and mirrored
__global__ void __launch_bounds__(256) k_curl_combine(hb_mesh_desc M, double a2, const double *curls,
                                                      const double *V, const double *D2, double *D)
{
    const int64_t m = blockIdx.x, d = blockIdx.y;
    const int64_t N = M.N_x, E = M.E_x;
    const double *Vd = V + d * E * E;
    const double *D2d = D2 + d * N * N;
    double *Dd = D + d * N * N;
    const int64_t sm0 = __ldg(M.star_indptr_dev + m), sm1 = __ldg(M.star_indptr_dev + m + 1);
    for (int64_t n = m + threadIdx.x; n < N; n += blockDim.x) {
        const int64_t sn0 = __ldg(M.star_indptr_dev + n), sn1 = __ldg(M.star_indptr_dev + n + 1);
        double acc = 0.0;
        for (int64_t a = sm0; a < sm1; ++a) {
            const int64_t e = __ldg(M.star_elem_dev + a), i = __ldg(M.star_local_dev + a);
            const double c0 = __ldg(curls + 9 * e + 3 * i), c1 = __ldg(curls + 9 * e + 3 * i + 1),
                         c2 = __ldg(curls + 9 * e + 3 * i + 2);
            const double *Ve = Vd + e * E;
            for (int64_t b = sn0; b < sn1; ++b) {
                const int64_t f = __ldg(M.star_elem_dev + b), j = __ldg(M.star_local_dev + b);
                const double dot = c0 * __ldg(curls + 9 * f + 3 * j) + c1 * __ldg(curls + 9 * f + 3 * j + 1) +
                                   c2 * __ldg(curls + 9 * f + 3 * j + 2);
                acc = fma(dot, __ldg(Ve + f), acc);
            }
        }
        const double val = D2d[m * N + n] + a2 * acc;
        Dd[m * N + n] = val;
        Dd[n * N + m] = val;
    }
}

}  // namespace hb

using namespace hb;

extern "C" int hb_version(void) { return 1000; }   // 1.0.0

extern "C" const char *hb_last_error(void) { return g_err; }

extern "C" int hb_fp64_probe(int64_t grid, int64_t iters, double *sink_dev, void *stream)
{
    if (grid < 1 || iters < 1 || !sink_dev) { set_error("hb_fp64_probe: bad arguments"); return HB_ERR_INVALID; }
    k_fp64_probe<<<(unsigned)grid, 256, 0, (cudaStream_t)stream>>>(iters, sink_dev);
    return cuda_check(cudaGetLastError(), "hb_fp64_probe");
}

extern "C" int hb_curl_combine(const hb_mesh_desc *mesh, int64_t n_blocks, double alpha, const double *curls_dev,
                               const double *V_dev, const double *D2_dev, double *D_dev, void *stream)
{
    if (!mesh || n_blocks < 1 || !curls_dev || !V_dev || !D2_dev || !D_dev) {
        set_error("hb_curl_combine: bad arguments");
        return HB_ERR_INVALID;
    }
    dim3 g((unsigned)mesh->N_x, (unsigned)n_blocks);
    k_curl_combine<<<g, 256, 0, (cudaStream_t)stream>>>(*mesh, alpha * alpha, curls_dev, V_dev, D2_dev, D_dev);
    return cuda_check(cudaGetLastError(), "hb_curl_combine");
}
