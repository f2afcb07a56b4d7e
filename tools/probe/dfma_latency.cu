// DFMA dependent-issue latency and per-warp throughput on one SM sub-partition:
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dfma_latency dfma_latency.cu
#include <cstdio>
#include <cuda_runtime.h>
template <int CH>
__global__ void k(double *out, long long *cyc, int iters, double a, double b)
{
    double v[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) v[c] = threadIdx.x + c;
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 8; ++u)
#pragma unroll
            for (int c = 0; c < CH; ++c) v[c] = fma(v[c], a, b);
    }
    const long long t1 = clock64();
    double s = 0;
#pragma unroll
    for (int c = 0; c < CH; ++c) s += v[c];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
template <int CH>
void run(int threads)
{
    double *out; long long *cyc, h;
    cudaMalloc(&out, 1024 * sizeof(double)); cudaMalloc(&cyc, 8);
    const int iters = 4096;
    k<CH><<<1, threads>>>(out, cyc, iters, 0.999, 1e-3);
    k<CH><<<1, threads>>>(out, cyc, iters, 0.999, 1e-3);
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    const double per = (double)h / (iters * 8.0);
    printf("chains %d threads %4d (warps/SMSP %.2f): %.2f cycles per round of %d DFMA/warp -> %.2f cycles/DFMA-warp-instr per SMSP\n",
           CH, threads, threads / 128.0, per, CH, per / (CH * (threads / 128.0 < 1 ? 1 : threads / 128.0)));
    cudaFree(out); cudaFree(cyc);
}
int main()
{
    run<1>(32); run<2>(32); run<4>(32); run<8>(32);
    run<1>(128); run<2>(128); run<1>(256); run<2>(256); run<1>(512); run<2>(512); run<4>(512); run<2>(1024);
    return 0;
}
