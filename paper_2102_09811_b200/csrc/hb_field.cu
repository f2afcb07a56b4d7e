// hb_field.cu -- interior potentials (representation formula), sm_100a.
//
// Replaces heatbem/_field_numba.py:15-79 (_eval_potential).  For an
// evaluation point (x, t = k h + eps) the reference sums, per element e and
// quadrature node q,
//     s = sum_{m=0..k} c_m G(rho, m h + eps)      (+ dens[k] G(rho, 0) if cur)
//     c_m = dens[k-1-m] - dens[k-m] * [k-m < k or cur]
// and recomputes every G for every output time.  The G values depend on
// (x, eps, m) only, so points that share (x, eps) -- e.g. one spatial point
// at all time-step ends -- share them: one warp owns such a group, its lanes
// first evaluate G(m), m = 0..kmax, once per (e, q) into shared memory, then
// each lane contracts them with its own output time's density differences.
// The reference's evaluation order of the sums (m innermost, then q, then e)
// is kept, and c_m is formed exactly as the reference forms it.
#include <algorithm>

#include "hb_common.cuh"

namespace hb {

// heatbem/_assembly_numba.py:25-32 (delta branch first, then rho branch)
__device__ __forceinline__ double dev_g_dtau(double rho, double delta, double a, double deps, double reps)
{
    if (delta <= deps) return 1.0 / (4.0 * kPi * a * rho);
    if (rho <= reps) return 1.0 / (4.0 * sqrt((kPi * kPi * kPi) * (a * a * a) * delta));
    const double x = rho / (2.0 * sqrt(a * delta));
    return erf(x) / (4.0 * kPi * a * rho);
}

// heatbem/_assembly_numba.py:48-59 (rho branch first)
__device__ __forceinline__ double dev_dn_g_dtau(double rn, double rho, double delta, double a, double deps,
                                                double reps)
{
    if (rho <= reps) return 0.0;
    if (delta <= deps) return rn / (4.0 * kPi * (rho * rho * rho));
    const double x = rho / (2.0 * sqrt(a * delta));
    const double inner = erf(x) / rho - exp(-x * x) / sqrt(kPi * a * delta);
    return (rn / (rho * rho)) * inner / (4.0 * kPi);
}

struct PotArgs {
    int kind;
    int64_t n_groups, E_t, E_x, nq;
    const double *gx;          // (n_groups, 3)
    const double *geps;        // (n_groups,)
    const int64_t *gptr;       // (n_groups+1,) outputs of each group
    const int64_t *k;          // (n_out,) completed intervals per output
    const uint8_t *cur;        // (n_out,)
    const int64_t *out_idx;    // (n_out,) position in the caller's point list
    const double *dens, *qpts, *qw, *areas, *normals;
    double step, alpha, d_eps, r_eps;
    double *out;
    int kcap;                  // smem capacity of the G / density arrays
};

constexpr int kPotWarps = 4;
constexpr int kOutPerLane = 2;

__global__ void __launch_bounds__(kPotWarps * 32) k_potential(const PotArgs P)
{
    extern __shared__ __align__(16) double psm[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double *Gs = psm + warp * 3 * P.kcap;      // G(m), m = 0..kmax
    double *Ds = Gs + P.kcap;                  // dens[j], j = 0..kmax (j < E_t)
    double *G0 = Ds + P.kcap;                  // G(rho, 0) for the current-interval term
    for (int64_t g = (int64_t)blockIdx.x * kPotWarps + warp; g < P.n_groups; g += (int64_t)gridDim.x * kPotWarps) {
        const double px = P.gx[3 * g], py = P.gx[3 * g + 1], pz = P.gx[3 * g + 2];
        const double eps = P.geps[g];
        const int64_t o0 = P.gptr[g], o1 = P.gptr[g + 1];
        for (int64_t ob = o0; ob < o1; ob += 32 * kOutPerLane) {
            // this lane's outputs: ob + lane and ob + 63 - lane (pairs a short
            // history with a long one when the caller sorted k ascending)
            int64_t oi[kOutPerLane];
            int kk[kOutPerLane];
            bool cu[kOutPerLane], ok[kOutPerLane];
            int kmax = 0;
            for (int r = 0; r < kOutPerLane; ++r) {
                oi[r] = ob + (r == 0 ? lane : 32 * kOutPerLane - 1 - lane);
                ok[r] = oi[r] < o1;
                kk[r] = ok[r] ? (int)P.k[oi[r]] : 0;
                cu[r] = ok[r] ? P.cur[oi[r]] != 0 : false;
                kmax = max(kmax, kk[r]);
            }
            for (int o = 16; o >= 1; o >>= 1) kmax = max(kmax, __shfl_xor_sync(kFull, kmax, o));
            double acc[kOutPerLane];
            for (int r = 0; r < kOutPerLane; ++r) acc[r] = 0.0;
            for (int64_t e = 0; e < P.E_x; ++e) {
                const double nyx = __ldg(P.normals + 3 * e), nyy = __ldg(P.normals + 3 * e + 1),
                             nyz = __ldg(P.normals + 3 * e + 2);
                double el[kOutPerLane];
                for (int r = 0; r < kOutPerLane; ++r) el[r] = 0.0;
                for (int64_t q = 0; q < P.nq; ++q) {
                    const double *y = P.qpts + 3 * (e * P.nq + q);
                    const double rx = px - __ldg(y), ry = py - __ldg(y + 1), rz = pz - __ldg(y + 2);
                    const double rho = sqrt(rx * rx + ry * ry + rz * rz);
                    const double rn = rx * nyx + ry * nyy + rz * nyz;
                    for (int m = lane; m <= kmax; m += 32) {
                        const double gap = (double)m * P.step + eps;
                        Gs[m] = P.kind == 0 ? dev_g_dtau(rho, gap, P.alpha, P.d_eps, P.r_eps)
                                            : dev_dn_g_dtau(rn, rho, gap, P.alpha, P.d_eps, P.r_eps);
                        Ds[m] = m < P.E_t ? __ldg(P.dens + ((int64_t)m * P.E_x + e) * P.nq + q) : 0.0;
                    }
                    if (lane == 0)
                        G0[0] = P.kind == 0 ? dev_g_dtau(rho, 0.0, P.alpha, P.d_eps, P.r_eps)
                                            : dev_dn_g_dtau(rn, rho, 0.0, P.alpha, P.d_eps, P.r_eps);
                    __syncwarp();
                    const double w = __ldg(P.qw + q);
                    for (int r = 0; r < kOutPerLane; ++r) {
                        if (!ok[r]) continue;
                        const int k = kk[r];
                        double s = 0.0;
                        for (int m = 0; m <= k; ++m) {
                            const int hi = k - 1 - m, lo = k - m;
                            double c = (hi >= 0 && hi < P.E_t) ? Ds[hi] : 0.0;
                            if (lo >= 0 && lo < P.E_t && (lo < k || cu[r])) c -= Ds[lo];
                            if (c == 0.0) continue;
                            s = fma(c, Gs[m], s);
                        }
                        if (cu[r] && k >= 0 && k < P.E_t) s = fma(Ds[k], G0[0], s);
                        el[r] = fma(w, s, el[r]);
                    }
                    __syncwarp();
                }
                const double a2 = 2.0 * __ldg(P.areas + e);
                for (int r = 0; r < kOutPerLane; ++r) acc[r] = fma(a2, el[r], acc[r]);
            }
            for (int r = 0; r < kOutPerLane; ++r)
                if (ok[r]) P.out[P.out_idx[oi[r]]] = acc[r];
        }
    }
}

}  // namespace hb

using namespace hb;

// Outputs sharing (x, eps) form one group (gptr); k ascending within a group.
extern "C" int hb_potential(int kind, int64_t n_groups, int64_t E_t, int64_t E_x, int64_t nq,
                                    const double *gx_dev, const double *geps_dev, const int64_t *gptr_dev,
                                    const int64_t *k_dev, const uint8_t *cur_dev, const int64_t *out_idx_dev,
                                    int64_t kmax, const double *dens_dev, const double *qpts_dev,
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
    P.dens = dens_dev; P.qpts = qpts_dev; P.qw = qw_dev; P.areas = areas_dev; P.normals = normals_dev;
    P.step = step; P.alpha = alpha; P.d_eps = d_eps; P.r_eps = r_eps; P.out = out_dev;
    P.kcap = (int)std::max<int64_t>(kmax + 1, E_t + 1);
    const size_t sm = (size_t)kPotWarps * 3 * P.kcap * sizeof(double);
    if (sm > 200 * 1024) { set_error("hb_potential: time history too long (%lld)", (long long)kmax); return HB_ERR_INVALID; }
    if (sm > 48 * 1024) cudaFuncSetAttribute(k_potential, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    int dev = 0, nsm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    const int64_t grid = std::min<int64_t>(cdiv(n_groups, kPotWarps), (int64_t)nsm * 16);
    k_potential<<<(unsigned)grid, kPotWarps * 32, sm, (cudaStream_t)stream>>>(P);
    return cuda_check(cudaGetLastError(), "hb_potential");
}

