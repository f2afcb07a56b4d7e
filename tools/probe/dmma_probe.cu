// DMMA (mma.sync m8n8k4 f64) probe on sm_100a: fragment layout check and
// throughput.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma_probe dmma_probe.cu
#include <cstdio>
#include <cmath>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double &d0, double &d1, double a, double b)
{
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

// layout: A[8][4] row-major, B[4][8]; lane l holds a = A[l/4][l%4], b = B[l%4][l/4];
// D[l/4][2*(l%4)+i] = d_i
__global__ void k_layout(const double *A, const double *B, double *D)
{
    const int l = threadIdx.x;
    double d0 = 0, d1 = 0;
    dmma(d0, d1, A[(l / 4) * 4 + l % 4], B[(l % 4) * 8 + l / 4]);
    D[(l / 4) * 8 + 2 * (l % 4)] = d0;
    D[(l / 4) * 8 + 2 * (l % 4) + 1] = d1;
}

__global__ void k_tput(int iters, double *sink)
{
    const int l = threadIdx.x & 31;
    double a = 1.0 + 1e-9 * l, b = 1.0 - 1e-9 * l;
    double c[8][2];
    for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0.0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) dmma(c[i][0], c[i][1], a, b);
    }
    double s = 0;
    for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
    if (s == 12345.0) sink[threadIdx.x] = s;
}

int main()
{
    double hA[32], hB[32], hD[64], ref[64];
    for (int i = 0; i < 32; ++i) { hA[i] = 1 + i; hB[i] = 0.5 * i - 3; }
    for (int r = 0; r < 8; ++r)
        for (int c = 0; c < 8; ++c) {
            double s = 0;
            for (int k = 0; k < 4; ++k) s += hA[r * 4 + k] * hB[k * 8 + c];
            ref[r * 8 + c] = s;
        }
    double *dA, *dB, *dD, *sink;
    cudaMalloc(&dA, 256); cudaMalloc(&dB, 256); cudaMalloc(&dD, 512); cudaMalloc(&sink, 4096);
    cudaMemcpy(dA, hA, 256, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, hB, 256, cudaMemcpyHostToDevice);
    k_layout<<<1, 32>>>(dA, dB, dD);
    cudaMemcpy(hD, dD, 512, cudaMemcpyDeviceToHost);
    double err = 0;
    for (int i = 0; i < 64; ++i) err = fmax(err, fabs(hD[i] - ref[i]));
    printf("layout max err %g\n", err);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int warps : {4, 8, 16}) {
        const int iters = 20000, grid = sms * 4;
        k_tput<<<grid, warps * 32>>>(100, sink);
        cudaEvent_t s, e;
        cudaEventCreate(&s); cudaEventCreate(&e);
        cudaEventRecord(s);
        k_tput<<<grid, warps * 32>>>(iters, sink);
        cudaEventRecord(e);
        cudaEventSynchronize(e);
        float ms = 0;
        cudaEventElapsedTime(&ms, s, e);
        const double flops = 2.0 * 256 * 8 * (double)iters * grid * warps;
        printf("warps/CTA %d (4 CTAs/SM): %.2f TFLOP/s\n", warps, flops / (ms * 1e-3) / 1e12);
    }
    return 0;
}
