// FP64 MMA throughput probe (B200): m8n8k4 / m16n8k4 / m16n8k8 with 8
// independent accumulators per warp and register operands, and m8n8k4 with
// its A operand loaded from shared memory per instruction (as k_toep_mma).
#include <cstdio>
#include <cuda_runtime.h>
template <int SHAPE>
__global__ void k(double *out, int iters)
{
    __shared__ double sm[8][32 * 9];
    for (int i = threadIdx.x; i < 8 * 32 * 9; i += blockDim.x) (&sm[0][0])[i] = i * 1e-6;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    double a0 = threadIdx.x * 1e-3, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, b0 = 0.5, b1 = 0.25;
    double c[8][4];
    for (int i = 0; i < 8; ++i) for (int j = 0; j < 4; ++j) c[i][j] = 0.0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (SHAPE == 0)
                asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                             : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a0), "d"(b0));
            else if (SHAPE == 1)
                asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
                             : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3]) : "d"(a0), "d"(a1), "d"(b0));
            else if (SHAPE == 2)
                asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                             : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3]) : "d"(a0), "d"(a1), "d"(a2), "d"(a3), "d"(b0), "d"(b1));
            else {   // A operand from shared memory, one LDS per MMA
                const double a = sm[i][(lane * 9 + (it & 7)) % (32 * 9)];
                asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                             : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b0));
            }
        }
    }
    double s = 0;
    for (int i = 0; i < 8; ++i) for (int j = 0; j < 4; ++j) s += c[i][j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main()
{
    double *o; cudaMalloc(&o, 148 * 8 * 1024 * 8);
    const int iters = 20000;
    const long fma_per_inst[4] = {8 * 8 * 4, 16 * 8 * 4, 16 * 8 * 8, 8 * 8 * 4};
    for (int sh = 0; sh < 4; ++sh) {
        for (int warps : {4, 8, 16}) {
            cudaEvent_t s, e; cudaEventCreate(&s); cudaEventCreate(&e);
            auto run = [&]() {
                if (sh == 0) k<0><<<148 * 4, 32 * warps>>>(o, iters);
                if (sh == 1) k<1><<<148 * 4, 32 * warps>>>(o, iters);
                if (sh == 2) k<2><<<148 * 4, 32 * warps>>>(o, iters);
                if (sh == 3) k<3><<<148 * 4, 32 * warps>>>(o, iters);
            };
            run(); cudaDeviceSynchronize();
            cudaEventRecord(s); run(); cudaEventRecord(e); cudaEventSynchronize(e);
            float ms; cudaEventElapsedTime(&ms, s, e);
            double flop = 2.0 * fma_per_inst[sh] * 8.0 * iters * (148.0 * 4 * warps);
            printf("shape %d warps/CTA %d: %.2f TFLOP/s (%s)\n", sh, warps, flop / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}
