// hb_capi.cu -- C-ABI glue: error state, version, FP64 throughput probe,
// and the curl combination D = D2 + alpha^2 sum_o T_o^T V T_o.
#include <algorithm>
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

// D = D2 + a2 * sum_{(e,i) in star(m)} sum_{(f,j) in star(n)} (curl_ei . curl_fj) V[e][f]
// in two stages per block d:
//   W[e][o][n] = sum_{(f,j) in star(n)} curl_fj[o] V[e][f]    (row e of V staged in smem)
//   D[m][n]    = D2[m][n] + a2 sum_{(e,i) in star(m)} sum_o curl_ei[o] W[e][o][n]
// the second stage runs on 32x32 tile pairs (ti <= tj), computes n >= m and
// writes the mirror through shared memory (exact symmetry, coalesced).
// D = D2 + a^2 sum_k T_k^T V T_k, one CTA per (node tile ti <= node tile tj)
// and a range of blocks d.  The elements of the stars of a 32-node tile form
// a sorted list (mesh plan: tile_eptr/tile_elem, star_pos = position of each
// star entry in its node's tile list); the CTA stages V[rows of ti][cols of tj]
// in shared memory 32 rows at a time and forms, entirely on chip,
//   W_k[e][n] = sum_{(f,j) in star(n)} c_k(f,j) V[e][f]            (T stage)
//   D[m][n]  += sum_{(e,i) in star(m), e in chunk} sum_k c_k(e,i) W_k[e][n]
// in the star orders (node stars are element-sorted, chunks ascending), so
// the sums are those of the two-pass W formulation without its E_x x 3N_x
// intermediate in HBM.  Upper tiles only; the lower triangle is mirrored.
constexpr int kCT = 32;    // nodes per tile
constexpr int kRC = 32;    // staged V rows per chunk (one per lane)
constexpr int kMaxJ = 8;   // column elements per tile <= 32 kMaxJ
#ifndef HB_CURL_WARPS
#define HB_CURL_WARPS 16   // warps per CTA sharing one tile pair's shared-memory stages (latency hiding)
#endif
constexpr int kCW = HB_CURL_WARPS, kCQ = kCT / kCW;   // output rows per warp in the D stage

struct CurlArgs {
    hb_mesh_desc M;
    double a2;
    const double *curls, *V, *D2;
    double *D;
    int64_t n_blocks;
    int dpc, ldv, smax, emax;
    // D2 as the sum of nparts full-size partials (row-parallel ranks' p1 x p1
    // contributions, read over NVLink peer memory): parts[p] + (part_doff + d) N^2
    int nparts;
    const double *const *parts;
    int64_t part_doff;
};

// D2[d][m][n] of the combine: the contiguous D2 blocks, or the partials summed
// in part order (deterministic)
__device__ __forceinline__ double curl_d2(const CurlArgs &C, int64_t d, int64_t idx)
{
    if (C.nparts == 0) return C.D2[d * C.M.N_x * C.M.N_x + idx];
    const int64_t off = (C.part_doff + d) * C.M.N_x * C.M.N_x + idx;
    double s = C.parts[0][off];
    for (int p = 1; p < C.nparts; ++p) s += C.parts[p][off];
    return s;
}

// star entry of a tile: curl vector of (element, local hat) and the element's
// position in the tile's element list (two 16-byte broadcast loads)
struct __align__(16) CurlEnt {
    double c0, c1, c2;
    int pos, pad;
};

__global__ void __launch_bounds__(32 * kCW) k_curl_tile(const CurlArgs C)
{
    extern __shared__ __align__(16) double csm[];
    const int64_t N = C.M.N_x, E = C.M.E_x;
    const int64_t nt = cdiv(N, kCT);
    int64_t ti = 0, rem = blockIdx.x;
    while (rem >= nt - ti) { rem -= nt - ti; ++ti; }
    const int64_t tj = ti + rem;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

    double *Vs = csm;                                   // [kRC][ldv]
    double *Ts = Vs + kRC * C.ldv;                      // [3][kCT][33]: Ts[k][n][r]
    double *Dt = Ts + 3 * kCT * 33;                     // [32][33]
    CurlEnt *cE = (CurlEnt *)(Dt + 32 * 33);            // [smax] star entries of tile tj
    CurlEnt *rE = cE + C.smax;                          // [smax] star entries of tile ti
    int64_t *rowE = (int64_t *)(rE + C.smax);           // [emax] elements of ti
    int *cPtr = (int *)(rowE + C.emax);                 // [33]
    int *rPtr = cPtr + 33;                              // [33]

    const int64_t nn0 = tj * kCT, mm0 = ti * kCT;
    const int nnc = (int)(N - nn0 < kCT ? N - nn0 : (int64_t)kCT), nmr = (int)(N - mm0 < kCT ? N - mm0 : (int64_t)kCT);
    const int64_t B0 = C.M.curl_tile_eptr_dev[tj], B = C.M.curl_tile_eptr_dev[tj + 1] - B0;
    const int64_t A0 = C.M.curl_tile_eptr_dev[ti], A = C.M.curl_tile_eptr_dev[ti + 1] - A0;
    const int64_t cs0 = C.M.star_indptr_dev[nn0], rs0 = C.M.star_indptr_dev[mm0];
    int64_t coff[kMaxJ];                                // this lane's column elements
#pragma unroll
    for (int j = 0; j < kMaxJ; ++j) {
        const int c = lane + 32 * j;
        coff[j] = c < B ? C.M.curl_tile_elem_dev[B0 + c] : 0;
    }
    for (int i = tid; i < A; i += blockDim.x) rowE[i] = C.M.curl_tile_elem_dev[A0 + i];
    for (int i = tid; i <= kCT; i += blockDim.x) {
        cPtr[i] = (int)(C.M.star_indptr_dev[nn0 + min(i, nnc)] - cs0);
        rPtr[i] = (int)(C.M.star_indptr_dev[mm0 + min(i, nmr)] - rs0);
    }
    __syncthreads();
    for (int i = tid; i < cPtr[kCT]; i += blockDim.x) {
        const int64_t s = cs0 + i, f = C.M.star_elem_dev[s], j = C.M.star_local_dev[s];
        cE[i] = CurlEnt{C.curls[9 * f + 3 * j], C.curls[9 * f + 3 * j + 1], C.curls[9 * f + 3 * j + 2],
                        C.M.curl_star_pos_dev[s], 0};
    }
    for (int i = tid; i < rPtr[kCT]; i += blockDim.x) {
        const int64_t s = rs0 + i, e = C.M.star_elem_dev[s], l = C.M.star_local_dev[s];
        rE[i] = CurlEnt{C.curls[9 * e + 3 * l], C.curls[9 * e + 3 * l + 1], C.curls[9 * e + 3 * l + 2],
                        C.M.curl_star_pos_dev[s], 0};
    }
    __syncthreads();

    const int64_t d_lo = (int64_t)blockIdx.y * C.dpc, d_hi = (C.n_blocks < d_lo + C.dpc ? C.n_blocks : d_lo + C.dpc);
    const double *vrow = Vs + lane * C.ldv;
    for (int64_t d = d_lo; d < d_hi; ++d) {
        const double *Vd = C.V + d * E * E;
        double acc[kCQ];
        int sp[kCQ];
#pragma unroll
        for (int q = 0; q < kCQ; ++q) {
            acc[q] = 0.0;
            sp[q] = rPtr[min(warp + kCW * q, kCT)];
        }
        for (int r0 = 0; r0 < (int)A; r0 += kRC) {
            const int rc = (int)A - r0 < kRC ? (int)A - r0 : kRC;
            // gather the chunk with async copies: all of its loads in flight at once
            for (int r = warp; r < rc; r += kCW) {
                const double *Vr = Vd + rowE[r0 + r] * E;
                const unsigned sa = (unsigned)__cvta_generic_to_shared(Vs + r * C.ldv + lane);
#pragma unroll
                for (int j = 0; j < kMaxJ; ++j)
                    if (lane + 32 * j < B)
                        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa + 256 * j),
                                     "l"(Vr + coff[j]) : "memory");
            }
            asm volatile("cp.async.wait_all;\n" ::: "memory");
            __syncthreads();
            // T stage: warp per node (uniform star loop, broadcast entries), lane per staged row
            // (rows >= rc compute unused values)
            for (int nl = warp; nl < nnc; nl += kCW) {
                double w0 = 0.0, w1 = 0.0, w2 = 0.0;
                for (int s = cPtr[nl]; s < cPtr[nl + 1]; ++s) {
                    const CurlEnt ce = cE[s];
                    const double v = vrow[ce.pos];
                    w0 = fma(ce.c0, v, w0);
                    w1 = fma(ce.c1, v, w1);
                    w2 = fma(ce.c2, v, w2);
                }
                Ts[(0 * kCT + nl) * 33 + lane] = w0;
                Ts[(1 * kCT + nl) * 33 + lane] = w1;
                Ts[(2 * kCT + nl) * 33 + lane] = w2;
            }
            __syncthreads();
            // D stage: warp per output row m, lane per column n; the row's star
            // entries in this chunk are the next ones (element-sorted stars)
            const int rend = r0 + rc;
#pragma unroll
            for (int q = 0; q < kCQ; ++q) {
                const int ml = warp + kCW * q;
                if (ml < nmr) {
                    const int se = rPtr[ml + 1];
                    int s = sp[q];
                    for (; s < se; ++s) {
                        const CurlEnt re = rE[s];
                        if (re.pos >= rend) break;
                        const int pr = re.pos - r0;
                        acc[q] = fma(re.c0, Ts[(0 * kCT + lane) * 33 + pr], acc[q]);
                        acc[q] = fma(re.c1, Ts[(1 * kCT + lane) * 33 + pr], acc[q]);
                        acc[q] = fma(re.c2, Ts[(2 * kCT + lane) * 33 + pr], acc[q]);
                    }
                    sp[q] = s;
                }
            }
            __syncthreads();
        }

        double *Dd = C.D + d * N * N;
#pragma unroll
        for (int q = 0; q < kCQ; ++q) {
            const int ml = warp + kCW * q;
            const int64_t m = mm0 + ml, n = nn0 + lane;
            double val = 0.0;
            if (ml < nmr && lane < nnc && n >= m) {
                val = fma(C.a2, acc[q], curl_d2(C, d, m * N + n));
                Dd[m * N + n] = val;
            }
            Dt[ml * 33 + lane] = val;
        }
        __syncthreads();
        for (int r = warp; r < kCT; r += kCW) {   // D[n][m] = D[m][n] for n > m
            const int64_t n = nn0 + r, m = mm0 + lane;
            if (r < nnc && lane < nmr && n > m) Dd[n * N + m] = Dt[lane * 33 + r];
        }
        __syncthreads();
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

extern "C" size_t hb_curl_workspace(const hb_mesh_desc *mesh, int64_t blocks_per_pass)
{
    (void)mesh; (void)blocks_per_pass;
    return 0;   // the tile kernel keeps its intermediates on chip
}

static int curl_launch(const hb_mesh_desc *mesh, int64_t n_blocks, double alpha, const double *curls_dev,
                       const double *V_dev, const double *D2_dev, double *D_dev, int nparts,
                       const double *const *parts, int64_t part_doff, void *stream);

extern "C" int hb_curl_combine(const hb_mesh_desc *mesh, int64_t n_blocks, double alpha, const double *curls_dev,
                               const double *V_dev, const double *D2_dev, double *D_dev, void *workspace_dev,
                               size_t workspace_bytes, void *stream)
{
    (void)workspace_dev; (void)workspace_bytes;
    if (!mesh || n_blocks < 1 || !curls_dev || !V_dev || !D2_dev || !D_dev) {
        set_error("hb_curl_combine: bad arguments");
        return HB_ERR_INVALID;
    }
    return curl_launch(mesh, n_blocks, alpha, curls_dev, V_dev, D2_dev, D_dev, 0, nullptr, 0, stream);
}

extern "C" int hb_curl_combine_parts(const hb_mesh_desc *mesh, int64_t n_blocks, double alpha,
                                     const double *curls_dev, const double *V_dev, int64_t n_parts,
                                     const double *const *parts_dev, int64_t part_d_offset, double *D_dev,
                                     void *stream)
{
    if (!mesh || n_blocks < 1 || !curls_dev || !V_dev || n_parts < 1 || n_parts > 64 || !parts_dev || !D_dev ||
        part_d_offset < 0) {
        set_error("hb_curl_combine_parts: bad arguments");
        return HB_ERR_INVALID;
    }
    return curl_launch(mesh, n_blocks, alpha, curls_dev, V_dev, nullptr, D_dev, (int)n_parts, parts_dev,
                       part_d_offset, stream);
}

static int curl_launch(const hb_mesh_desc *mesh, int64_t n_blocks, double alpha, const double *curls_dev,
                       const double *V_dev, const double *D2_dev, double *D_dev, int nparts,
                       const double *const *parts, int64_t part_doff, void *stream)
{
    if (!mesh->curl_tile_eptr_dev || !mesh->curl_tile_elem_dev || !mesh->curl_star_pos_dev ||
        mesh->curl_tile_emax < 1 || mesh->curl_tile_smax < 1) {
        set_error("hb_curl_combine: mesh descriptor has no curl tile plan");
        return HB_ERR_INVALID;
    }
    CurlArgs C{};
    C.M = *mesh; C.a2 = alpha * alpha; C.curls = curls_dev; C.V = V_dev; C.D2 = D2_dev; C.D = D_dev;
    C.nparts = nparts; C.parts = parts; C.part_doff = part_doff;
    C.n_blocks = n_blocks;
    C.emax = (int)mesh->curl_tile_emax;
    C.smax = (int)mesh->curl_tile_smax;
    C.ldv = C.emax | 1;
    if (C.emax > 32 * kMaxJ) {
        set_error("hb_curl_combine: %d elements around a 32-node tile (max %d)", C.emax, 32 * kMaxJ);
        return HB_ERR_UNSUPPORTED;
    }
    const size_t smem = sizeof(double) * ((size_t)kRC * C.ldv + 3 * kCT * 33 + 32 * 33) +
                        sizeof(CurlEnt) * 2 * (size_t)C.smax + sizeof(int64_t) * (size_t)C.emax + sizeof(int) * 66;
    if (smem > 227 * 1024) {
        set_error("hb_curl_combine: node tiles too large for shared memory (%d elements)", C.emax);
        return HB_ERR_UNSUPPORTED;
    }
    if (smem > 48 * 1024) cudaFuncSetAttribute(k_curl_tile, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int dev = 0, nsm = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_curl_tile, 32 * kCW, smem);
    const int64_t nt = cdiv(mesh->N_x, kCT), npairs = nt * (nt + 1) / 2;
    // blocks per CTA: enough CTAs for ~4 waves, the rest loops on chip (plan reuse)
    const int64_t want = (int64_t)std::max(1, per_sm) * nsm * 4;
    C.dpc = (int)std::max<int64_t>(1, std::min<int64_t>(n_blocks, npairs * n_blocks / std::max<int64_t>(1, want)));
    const int64_t gy = cdiv(n_blocks, C.dpc);
    k_curl_tile<<<dim3((unsigned)npairs, (unsigned)gy), 32 * kCW, smem, (cudaStream_t)stream>>>(C);
    return cuda_check(cudaGetLastError(), "hb_curl_combine");
}

// ---------------------------------------------------------------------------
// CUDA IPC for row-parallel assembly (peer d-shard buffers)
// ---------------------------------------------------------------------------
#include <cuda.h>
#include <cstring>

namespace {
typedef CUresult (*PFN_ptrAttr)(void *, CUpointer_attribute, CUdeviceptr);
PFN_ptrAttr ptr_attr_fn()
{
    static PFN_ptrAttr fn = nullptr;
    if (!fn) {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPointByVersion("cuPointerGetAttribute", &p, 12000, cudaEnableDefault, &q) ==
                cudaSuccess && q == cudaDriverEntryPointSuccess)
            fn = (PFN_ptrAttr)p;
    }
    return fn;
}
}  // namespace

extern "C" int hb_ipc_export(const void *ptr_dev, void *handle64, int64_t *offset)
{
    if (!ptr_dev || !handle64 || !offset) { set_error("hb_ipc_export: bad arguments"); return HB_ERR_INVALID; }
    PFN_ptrAttr fn = ptr_attr_fn();
    if (!fn) { set_error("hb_ipc_export: cuPointerGetAttribute unavailable"); return HB_ERR_CUDA; }
    CUdeviceptr base = 0;
    if (fn(&base, CU_POINTER_ATTRIBUTE_RANGE_START_ADDR, (CUdeviceptr)ptr_dev) != CUDA_SUCCESS) {
        set_error("hb_ipc_export: not a device allocation");
        return HB_ERR_INVALID;
    }
    cudaIpcMemHandle_t h;
    int rc = cuda_check(cudaIpcGetMemHandle(&h, (void *)base), "cudaIpcGetMemHandle");
    if (rc) return rc;
    static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
    std::memcpy(handle64, &h, sizeof(h));
    *offset = (int64_t)((CUdeviceptr)ptr_dev - base);
    return HB_OK;
}

extern "C" int hb_ipc_import(const void *handle64, int64_t offset, void **ptr_dev)
{
    if (!handle64 || !ptr_dev || offset < 0) { set_error("hb_ipc_import: bad arguments"); return HB_ERR_INVALID; }
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle64, sizeof(h));
    void *base = nullptr;
    int rc = cuda_check(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
    if (rc) return rc;
    *ptr_dev = (char *)base + offset;
    return HB_OK;
}

extern "C" int hb_ipc_close(void *ptr_dev, int64_t offset)
{
    if (!ptr_dev) { set_error("hb_ipc_close: bad arguments"); return HB_ERR_INVALID; }
    return cuda_check(cudaIpcCloseMemHandle((char *)ptr_dev - offset), "cudaIpcCloseMemHandle");
}

// rows [r0, r1) of every block of a (n_blocks, R, C) float64 array, device ->
// page-locked host, as ONE strided copy on `stream` (row-slab streaming of an
// operator while the next slab is assembled)
extern "C" int hb_copy_row_slab_d2h(double *host_dst, const double *dev_src, int64_t n_blocks, int64_t R, int64_t C,
                                    int64_t r0, int64_t r1, void *stream)
{
    if (!host_dst || !dev_src || n_blocks < 1 || R < 1 || C < 1 || r0 < 0 || r1 > R || r1 <= r0) {
        set_error("hb_copy_row_slab_d2h: bad arguments");
        return HB_ERR_INVALID;
    }
    const size_t pitch = sizeof(double) * (size_t)(R * C), width = sizeof(double) * (size_t)((r1 - r0) * C);
    const size_t off = (size_t)(r0 * C);
    return cuda_check(cudaMemcpy2DAsync(host_dst + off, pitch, dev_src + off, pitch, width, (size_t)n_blocks,
                                        cudaMemcpyDeviceToHost, (cudaStream_t)stream),
                      "hb_copy_row_slab_d2h");
}
