// hb_data.cu -- boundary data on the device: L2 projection of heat-kernel
// data onto X00 / X10, the p1 mass solve, and the relative L2(Sigma) error.
//
// Replaces the host numpy steps before and after the solve:
//   project_to_space       heatbem/field.py:84-119 (tensor rule: triangle
//                          order 6, 4 Gauss points per time step; X10 with a
//                          dense Cholesky solve of the p1 mass matrix)
//   relative_error_sigma   heatbem/field.py:193-215
// for the data family the study driver uses (heatbem/field.py:20-44):
//   kind 0  G_alpha(x - src, t + shift)                (kernels.py:59-66)
//   kind 1  alpha dG_alpha/dn_x (x - src, t + shift)   (kernels.py:69-86)
// The X10 mass system is solved with Jacobi-preconditioned CG, one CTA per
// time step (the p1 mass matrix is well conditioned: cond ~ 10 on shape-
// regular meshes, so CG reaches the rounding floor in a few dozen steps);
// the matrix is applied matrix-free from the node stars.  All sums run in
// a fixed order: results are bitwise reproducible.
#include <algorithm>

#include "hb_common.cuh"

namespace hb {

namespace {

constexpr double kFourPi = 12.566370614359172;

// kernels.py:59-66 / 69-86, same operation order
__device__ __forceinline__ double datum_value(const hb_heat_datum &g, const double *x, const double *n, double t)
{
    const double dt = t + g.time_shift;
    if (!(dt > 0.0)) return 0.0;
    const double r0 = x[0] - g.src[0], r1 = x[1] - g.src[1], r2 = x[2] - g.src[2];
    const double rho2 = __dadd_rn(__dadd_rn(__dmul_rn(r0, r0), __dmul_rn(r1, r1)), __dmul_rn(r2, r2));
    const double e = exp(-rho2 / (4.0 * g.alpha * dt));
    if (g.kind == HB_DATUM_VALUE) return pow(kFourPi * g.alpha * dt, -1.5) * e;
    const double rn = __dadd_rn(__dadd_rn(__dmul_rn(r0, n[0]), __dmul_rn(r1, n[1])), __dmul_rn(r2, n[2]));
    return -rn / (16.0 * pow(kPi * g.alpha, 1.5) * pow(dt, 2.5)) * e;
}

// element loads: X00 -> out[i][e] = 2 sum_q tw_q sum_p qw_p g
//                X10 -> L[i][e][j] = sum_q tw_q 2 A_e sum_p qw_p hat_j(p) g
__global__ void __launch_bounds__(256) k_data_loads(const hb_data_desc D, const hb_heat_datum g, int space,
                                                    int64_t E_t, double step, double *__restrict__ out)
{
    const int64_t n_items = E_t * D.E_x;
    for (int64_t it = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; it < n_items;
         it += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = it / D.E_x, e = it % D.E_x;
        const double *pts = D.qpts_dev + e * D.nq * 3;
        const double *nrm = D.normals_dev + e * 3;
        double acc[3] = {0.0, 0.0, 0.0};
        for (int q = 0; q < D.n_tq; ++q) {
            const double t = (double)i * step + D.tq[q] * step;
            double s[3] = {0.0, 0.0, 0.0};
            for (int p = 0; p < D.nq; ++p) {
                const double v = datum_value(g, pts + 3 * p, nrm, t);
                if (space == 0) {
                    s[0] = fma(v, D.qw_dev[p], s[0]);
                } else {
                    const double w = D.qw_dev[p];
#pragma unroll
                    for (int j = 0; j < 3; ++j) s[j] = fma(v, w * D.hats_dev[3 * p + j], s[j]);
                }
            }
            if (space == 0) {
                acc[0] = fma(D.tw[q], s[0], acc[0]);
            } else {
                const double a2 = 2.0 * D.areas_dev[e];
#pragma unroll
                for (int j = 0; j < 3; ++j) acc[j] = fma(D.tw[q], a2 * s[j], acc[j]);
            }
        }
        if (space == 0) {
            out[it] = 2.0 * acc[0];
        } else {
#pragma unroll
            for (int j = 0; j < 3; ++j) out[it * 3 + j] = acc[j];
        }
    }
}

// X10 load vector b[i][n] = sum over n's star (ascending element) of L[i][e][j]
__global__ void __launch_bounds__(256) k_star_gather(const hb_data_desc D, int64_t E_t, const double *__restrict__ L,
                                                     double *__restrict__ b)
{
    const int64_t n_items = E_t * D.N_x;
    for (int64_t it = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; it < n_items;
         it += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = it / D.N_x, n = it % D.N_x;
        double s = 0.0;
        for (int64_t k = D.star_indptr_dev[n]; k < D.star_indptr_dev[n + 1]; ++k)
            s += L[(i * D.E_x + D.star_elem_dev[k]) * 3 + D.star_local_dev[k]];
        b[it] = s;
    }
}

// (M x)[n] = sum_{(e,j) in star(n)} A_e/12 (x[n] + x[a] + x[b] + x[c]), (a,b,c) = nodes of e
__device__ __forceinline__ double mass_row(const hb_data_desc &D, const double *x, int64_t n)
{
    double s = 0.0;
    const double xn = x[n];
    for (int64_t k = D.star_indptr_dev[n]; k < D.star_indptr_dev[n + 1]; ++k) {
        const int64_t e = D.star_elem_dev[k];
        const int64_t *tn = D.tri_nodes_dev + 3 * e;
        const double sum = (x[tn[0]] + x[tn[1]]) + x[tn[2]];
        s = fma(D.areas_dev[e] * (1.0 / 12.0), xn + sum, s);
    }
    return s;
}

__device__ __forceinline__ double mass_diag(const hb_data_desc &D, int64_t n)
{
    double s = 0.0;
    for (int64_t k = D.star_indptr_dev[n]; k < D.star_indptr_dev[n + 1]; ++k)
        s += D.areas_dev[D.star_elem_dev[k]] * (2.0 / 12.0);
    return s;
}

constexpr int kCgThreads = 1024;

// fixed-order CTA sum (deterministic)
__device__ __forceinline__ double cta_sum(double v, double *red)
{
    for (int o = 16; o >= 1; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) red[w] = v;
    __syncthreads();
    if (w == 0) {
        v = l < (int)(blockDim.x >> 5) ? red[l] : 0.0;
        for (int o = 16; o >= 1; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
        if (l == 0) red[32] = v;
    }
    __syncthreads();
    return red[32];
}

// Jacobi-PCG for M x_i = b_i, one CTA per time step i.  work: r, z/q, p
// vectors (3 N_x per step).  Stops when ||r|| <= tol ||b|| or after max_iter.
__global__ void __launch_bounds__(kCgThreads) k_mass_cg(const hb_data_desc D, const double *__restrict__ b_all,
                                                        double *__restrict__ x_all, double *__restrict__ work,
                                                        double tol, int64_t max_iter, int64_t *__restrict__ iters)
{
    __shared__ double red[33];
    const int64_t N = D.N_x, i = blockIdx.x;
    const double *b = b_all + i * N;
    double *x = x_all + i * N, *r = work + i * 3 * N, *q = r + N, *p = q + N;
    double bb = 0.0, rz = 0.0;
    for (int64_t n = threadIdx.x; n < N; n += blockDim.x) {
        const double bn = b[n], z = bn / mass_diag(D, n);
        x[n] = 0.0;
        r[n] = bn;
        p[n] = z;
        bb = fma(bn, bn, bb);
        rz = fma(bn, z, rz);
    }
    bb = cta_sum(bb, red);
    rz = cta_sum(rz, red);
    const double stop = tol * tol * bb;
    double rr = bb;
    int64_t it = 0;
    while (it < max_iter && rr > stop) {
        double pq = 0.0;
        for (int64_t n = threadIdx.x; n < N; n += blockDim.x) {
            const double v = mass_row(D, p, n);
            q[n] = v;
            pq = fma(p[n], v, pq);
        }
        pq = cta_sum(pq, red);
        const double a = rz / pq;
        double rz_new = 0.0, rr_new = 0.0;
        for (int64_t n = threadIdx.x; n < N; n += blockDim.x) {
            x[n] = fma(a, p[n], x[n]);
            const double rn = fma(-a, q[n], r[n]);
            r[n] = rn;
            const double z = rn / mass_diag(D, n);
            q[n] = z;
            rz_new = fma(rn, z, rz_new);
            rr_new = fma(rn, rn, rr_new);
        }
        rz_new = cta_sum(rz_new, red);
        rr = cta_sum(rr_new, red);
        const double beta = rz_new / rz;
        rz = rz_new;
        for (int64_t n = threadIdx.x; n < N; n += blockDim.x) p[n] = fma(beta, p[n], q[n]);
        __syncthreads();
        ++it;
    }
    if (threadIdx.x == 0 && iters) iters[i] = it;
}

// per (i, e): [num, den] of relative_error_sigma (field.py:193-215)
__global__ void __launch_bounds__(256) k_error_terms(const hb_data_desc D, const hb_heat_datum g, int64_t E_t,
                                                     double step, const double *__restrict__ coeff, int p1,
                                                     double *__restrict__ terms)
{
    const int64_t n_items = E_t * D.E_x;
    for (int64_t it = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; it < n_items;
         it += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = it / D.E_x, e = it % D.E_x;
        const double *pts = D.qpts_dev + e * D.nq * 3;
        const double *nrm = D.normals_dev + e * 3;
        double c[3];
        if (p1) {
#pragma unroll
            for (int j = 0; j < 3; ++j) c[j] = coeff[i * D.N_x + D.tri_nodes_dev[3 * e + j]];
        } else {
            c[0] = c[1] = c[2] = coeff[i * D.E_x + e];
        }
        const double a2 = 2.0 * D.areas_dev[e];
        double num = 0.0, den = 0.0;
        for (int q = 0; q < D.n_tq; ++q) {
            const double t = (double)i * step + D.tq[q] * step;
            double sn = 0.0, sd = 0.0;
            for (int p = 0; p < D.nq; ++p) {
                const double v = datum_value(g, pts + 3 * p, nrm, t);
                double dens = c[0];
                if (p1) {
                    const double *h = D.hats_dev + 3 * p;
                    dens = fma(c[2], h[2], fma(c[1], h[1], c[0] * h[0]));
                }
                const double aw = a2 * D.qw_dev[p], dv = v - dens;
                sn = fma(aw * dv, dv, sn);
                sd = fma(aw * v, v, sd);
            }
            num = fma(D.tw[q] * step, sn, num);
            den = fma(D.tw[q] * step, sd, den);
        }
        terms[2 * it] = num;
        terms[2 * it + 1] = den;
    }
}

// fixed-order reduction of n (num, den) pairs into out[2]
__global__ void __launch_bounds__(1024) k_reduce_pairs(const double *__restrict__ terms, int64_t n,
                                                       double *__restrict__ out)
{
    __shared__ double red[33];
    double a = 0.0, b = 0.0;
    for (int64_t k = threadIdx.x; k < n; k += blockDim.x) {
        a += terms[2 * k];
        b += terms[2 * k + 1];
    }
    a = cta_sum(a, red);
    b = cta_sum(b, red);
    if (threadIdx.x == 0) {
        out[0] = a;
        out[1] = b;
    }
}

bool desc_ok(const hb_data_desc *D)
{
    return D && D->E_x > 0 && D->N_x > 0 && D->nq > 0 && D->n_tq > 0 && D->n_tq <= 8 && D->qpts_dev &&
           D->qw_dev && D->hats_dev && D->areas_dev && D->normals_dev && D->tri_nodes_dev && D->star_indptr_dev &&
           D->star_elem_dev && D->star_local_dev;
}

unsigned grid_for(int64_t items)
{
    return (unsigned)std::min<int64_t>(cdiv(items, 256), 148 * 16);
}

}  // namespace

}  // namespace hb

using namespace hb;

extern "C" size_t hb_project_workspace(const hb_data_desc *D, int space, int64_t E_t)
{
    if (!desc_ok(D) || E_t < 1) return 0;
    if (space == 0) return 0;
    // element loads (E_t, E_x, 3), the load vector b (E_t, N_x), CG vectors (E_t, 3 N_x), iteration counts
    return sizeof(double) * (size_t)(E_t * D->E_x * 3 + E_t * D->N_x + E_t * 3 * D->N_x) + sizeof(int64_t) * E_t;
}

extern "C" int hb_project_data(const hb_data_desc *D, const hb_heat_datum *g, int space, int64_t E_t, double step,
                               double *out_dev, void *work_dev, size_t work_bytes, double tol, int64_t max_iter,
                               int64_t *max_iters_out, void *stream)
{
    if (!desc_ok(D) || !g || (space != 0 && space != 1) || E_t < 1 || !(step > 0.0) || !out_dev ||
        (g->kind != HB_DATUM_VALUE && g->kind != HB_DATUM_NORMAL_DERIV) || !(g->alpha > 0.0)) {
        set_error("hb_project_data: bad arguments");
        return HB_ERR_INVALID;
    }
    cudaStream_t st = (cudaStream_t)stream;
    if (space == 0) {
        k_data_loads<<<grid_for(E_t * D->E_x), 256, 0, st>>>(*D, *g, 0, E_t, step, out_dev);
        if (max_iters_out) *max_iters_out = 0;
        return cuda_check(cudaGetLastError(), "hb_project_data");
    }
    if (!work_dev || work_bytes < hb_project_workspace(D, space, E_t) || max_iter < 1 || !(tol > 0.0)) {
        set_error("hb_project_data: X10 needs %zu bytes of workspace and tol > 0, max_iter >= 1",
                  hb_project_workspace(D, space, E_t));
        return HB_ERR_WORKSPACE;
    }
    double *L = (double *)work_dev, *b = L + E_t * D->E_x * 3, *cg = b + E_t * D->N_x;
    int64_t *its = (int64_t *)(cg + E_t * 3 * D->N_x);
    k_data_loads<<<grid_for(E_t * D->E_x), 256, 0, st>>>(*D, *g, 1, E_t, step, L);
    k_star_gather<<<grid_for(E_t * D->N_x), 256, 0, st>>>(*D, E_t, L, b);
    k_mass_cg<<<(unsigned)E_t, kCgThreads, 0, st>>>(*D, b, out_dev, cg, tol, max_iter, its);
    int rc = cuda_check(cudaGetLastError(), "hb_project_data");
    if (rc || !max_iters_out) return rc;
    // iteration report: the caller asked for it, so synchronise the stream
    int64_t *h = new int64_t[E_t];
    rc = cuda_check(cudaMemcpyAsync(h, its, sizeof(int64_t) * E_t, cudaMemcpyDeviceToHost, st), "hb_project_data");
    if (!rc) rc = cuda_check(cudaStreamSynchronize(st), "hb_project_data");
    if (!rc) {
        int64_t m = 0;
        for (int64_t i = 0; i < E_t; ++i) m = std::max(m, h[i]);
        *max_iters_out = m;
    }
    delete[] h;
    return rc;
}

extern "C" int hb_p1_mass_solve(const hb_data_desc *D, int64_t E_t, const double *b_dev, double *x_dev, void *work_dev,
                                size_t work_bytes, double tol, int64_t max_iter, void *stream)
{
    if (!desc_ok(D) || E_t < 1 || !b_dev || !x_dev || !work_dev || max_iter < 1 || !(tol > 0.0) ||
        work_bytes < sizeof(double) * (size_t)(E_t * 3 * D->N_x)) {
        set_error("hb_p1_mass_solve: bad arguments (workspace: 3 E_t N_x doubles)");
        return HB_ERR_INVALID;
    }
    k_mass_cg<<<(unsigned)E_t, kCgThreads, 0, (cudaStream_t)stream>>>(*D, b_dev, x_dev, (double *)work_dev, tol,
                                                                        max_iter, nullptr);
    return cuda_check(cudaGetLastError(), "hb_p1_mass_solve");
}

extern "C" int hb_error_sigma(const hb_data_desc *D, const hb_heat_datum *g, int64_t E_t, double step,
                              const double *coeff_dev, int p1, double *out2_dev, void *work_dev, size_t work_bytes,
                              void *stream)
{
    if (!desc_ok(D) || !g || E_t < 1 || !(step > 0.0) || !coeff_dev || !out2_dev || !work_dev ||
        work_bytes < sizeof(double) * (size_t)(2 * E_t * D->E_x) ||
        (g->kind != HB_DATUM_VALUE && g->kind != HB_DATUM_NORMAL_DERIV)) {
        set_error("hb_error_sigma: bad arguments (workspace: 2 E_t E_x doubles)");
        return HB_ERR_INVALID;
    }
    cudaStream_t st = (cudaStream_t)stream;
    double *terms = (double *)work_dev;
    k_error_terms<<<grid_for(E_t * D->E_x), 256, 0, st>>>(*D, *g, E_t, step, coeff_dev, p1 ? 1 : 0, terms);
    k_reduce_pairs<<<1, 1024, 0, st>>>(terms, E_t * D->E_x, out2_dev);
    return cuda_check(cudaGetLastError(), "hb_error_sigma");
}
