/*
 * oracle/heatbem_oracle.c -- CPU ORACLE, TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference's jitted hot loops so the parity
 * tests (tests/), __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference leg have a checker that runs without the reference tree
 * (which is absent on the GPU box).  Nothing in paper_2102_09811_b200/ may
 * link or call this file; the product path is the CUDA library.
 *
 * Pinned against the reference: tests/golden/ holds vectors produced by the
 * reference itself (oracle/gen_golden.py, numba + glibc libm in this
 * container); tests/test_oracle_golden.py checks this file against them,
 * bit for bit.
 *
 * Followed, function by function:
 *   scalar kernels      <- heatbem/_assembly_numba.py:25-104
 *   pass_row / *_pass   <- heatbem/_assembly_numba.py:111-272 (_toeplitz_pass)
 *   scatter_add         <- heatbem/_assembly_numba.py:275-285 (_scatter_add)
 *   plan_targets        <- heatbem/assembly.py:72-89 (AssemblyPlan.targets)
 *   *_assemble          <- heatbem/assembly.py:208-239 (_assemble_operator loop
 *                          and the symmetric mirror)
 *   *_potential         <- heatbem/_field_numba.py:15-79 (_eval_potential)
 *
 * Arithmetic is written in the reference's evaluation order and compiled
 * with -ffp-contract=off so every product/sum rounds exactly as numba's
 * (non-fastmath) LLVM code does; erf/exp come from the host glibc libm, as
 * in numba (math.erf -> extern erf, math.exp -> llvm.exp -> libm exp).
 * numba lowers integer powers x**3 to repeated multiplication.
 *
 * heatbem_oracle_q.c includes this file with HB_REAL = __float128
 * (libquadmath): the SAME quadrature evaluated in 113-bit arithmetic.  It is
 * the "exact" value against which the rounding error of the reference and
 * of the GPU are both measured (the conditioning-aware gate of SURVEY 8(c)).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#ifndef HB_REAL
#define HB_REAL double
#define HB_ERF erf
#define HB_EXP exp
#define HB_SQRT sqrt
#define HB_PI 3.141592653589793
#define HB_SYM(name) name
#define HB_WITH_PASS 1
#endif
typedef HB_REAL real;
#define PI ((real)HB_PI)

static inline real cube(real x) { return x * x * x; }

/* _assembly_numba.py:25-32 */
static inline real g_dtau(real rho, real delta, real a, real deps, real reps)
{
    if (delta <= deps) return 1.0 / (4.0 * PI * a * rho);
    if (rho <= reps) return 1.0 / (4.0 * HB_SQRT(cube(PI) * cube(a) * delta));
    real x = rho / (2.0 * HB_SQRT(a * delta));
    return HB_ERF(x) / (4.0 * PI * a * rho);
}

/* _assembly_numba.py:35-45 */
static inline real g_dtaudt(real rho, real delta, real a, real deps, real reps)
{
    if (delta <= deps) return rho / (8.0 * PI * a * a);
    if (rho <= reps) return HB_SQRT(delta) / (2.0 * HB_SQRT(cube(PI) * cube(a)));
    real x = rho / (2.0 * HB_SQRT(a * delta));
    real t1 = (rho / (2.0 * a * a) + delta / (a * rho)) * HB_ERF(x);
    real t2 = HB_SQRT(delta) / HB_SQRT(PI * cube(a)) * HB_EXP(-x * x);
    return (t1 + t2) / (4.0 * PI);
}

/* _assembly_numba.py:48-59 */
static inline real dn_g_dtau(real rn, real rho, real delta, real a, real deps, real reps)
{
    if (rho <= reps) return 0.0;
    if (delta <= deps) return rn / (4.0 * PI * cube(rho));
    real x = rho / (2.0 * HB_SQRT(a * delta));
    real inner = HB_ERF(x) / rho - HB_EXP(-x * x) / HB_SQRT(PI * a * delta);
    return (rn / (rho * rho)) * inner / (4.0 * PI);
}

/* _assembly_numba.py:62-76 */
static inline real dn_g_dtaudt(real rn, real rho, real delta, real a, real deps, real reps)
{
    if (rho <= reps) return 0.0;
    if (delta <= deps) return -rn / (8.0 * PI * a * rho);
    real x = rho / (2.0 * HB_SQRT(a * delta));
    real inner = (1.0 / (2.0 * a) - delta / (rho * rho)) * HB_ERF(x)
               + HB_SQRT(delta) / (rho * HB_SQRT(PI * a)) * HB_EXP(-x * x);
    return -(rn / rho) * inner / (4.0 * PI);
}

/* _assembly_numba.py:79-87 */
static inline real op_value(int op, real rx, real ry, real rz, real nyx, real nyy, real nyz,
                            real delta, real a, real deps, real reps)
{
    real rho = HB_SQRT(rx * rx + ry * ry + rz * rz);
    if (op == 0) return g_dtaudt(rho, delta, a, deps, reps);
    if (op == 1) {
        real rn = rx * nyx + ry * nyy + rz * nyz;
        return dn_g_dtaudt(rn, rho, delta, a, deps, reps);
    }
    return a * g_dtau(rho, delta, a, deps, reps);
}

/* _assembly_numba.py:90-104: combined d = 0 kernel (i_t = 0 only) */
static inline real op_comb0(int op, real rx, real ry, real rz, real nyx, real nyy, real nyz,
                            real a, real h, real deps, real reps)
{
    real rho = HB_SQRT(rx * rx + ry * ry + rz * rz);
    if (op == 0) return h * g_dtau(rho, 0.0, a, deps, reps) + g_dtaudt(rho, 0.0, a, deps, reps);
    if (op == 1) {
        real rn = rx * nyx + ry * nyy + rz * nyz;
        return h * dn_g_dtau(rn, rho, 0.0, a, deps, reps) + dn_g_dtaudt(rn, rho, 0.0, a, deps, reps);
    }
    return a * g_dtau(rho, 0.0, a, deps, reps);
}

typedef struct {
    int op, test_p1, trial_p1, symmetric;
    int64_t E_x, N_x;
    double alpha, h_t, d_eps, r_eps;
    const int64_t *tri_nodes;   /* (E_x,3) */
    const double *verts_tri;    /* (E_x,3,3) */
    const double *normals, *centroids, *diameters, *areas;
    const double *reg_hats, *reg_w, *reg_pts; int64_t n_reg;
    const double *near_hats, *near_w, *near_pts; int64_t n_near;
    const int64_t *tn_indptr, *tn_idx, *tn_case, *tn_permt, *tn_perms;
    const int64_t *duf_off; const double *duf_t, *duf_s, *duf_w;
} problem_t;

/* one (test e, trial f) pair of _toeplitz_pass (_assembly_numba.py:138-266):
 * lm/lmc = the staged 3x3 local values before the jacobian, jac returned */
static real pair_eval(const problem_t *P, int64_t e, int64_t f, real delta, int need_comb,
                      real lm[3][3], real lmc[3][3])
{
    const int n_t = P->test_p1 ? 3 : 1, n_s = P->trial_p1 ? 3 : 1;
    const int op = P->op;
    const real a = P->alpha, deps = P->d_eps, reps = P->r_eps, h = P->h_t;
    real ht[3] = {1.0, 0.0, 0.0}, hs[3] = {1.0, 0.0, 0.0};
    const real nxx = P->normals[3 * e], nxy = P->normals[3 * e + 1], nxz = P->normals[3 * e + 2];
    const int64_t t_lo = P->tn_indptr[e], t_hi = P->tn_indptr[e + 1];
    {
        int64_t tpos = -1, lo = t_lo, hi = t_hi;
        while (lo < hi) {
            int64_t mid = (lo + hi) / 2, v = P->tn_idx[mid];
            if (v < f) lo = mid + 1;
            else if (v > f) hi = mid;
            else { tpos = mid; break; }
        }
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j) { lm[i][j] = 0.0; lmc[i][j] = 0.0; }
        const real nyx = P->normals[3 * f], nyy = P->normals[3 * f + 1], nyz = P->normals[3 * f + 2];
        if (tpos >= 0) {
            /* touching pair: Duffy rule on permuted charts */
            const int64_t cs = P->tn_case[tpos];
            const int64_t *pt = P->tn_permt + 3 * tpos, *ps = P->tn_perms + 3 * tpos;
            const double *ve = P->verts_tri + 9 * e, *vf = P->verts_tri + 9 * f;
            real A[3][3], B[3][3];
            for (int k = 0; k < 3; ++k)
                for (int c = 0; c < 3; ++c) { A[k][c] = ve[3 * pt[k] + c]; B[k][c] = vf[3 * ps[k] + c]; }
            for (int64_t q = P->duf_off[cs]; q < P->duf_off[cs + 1]; ++q) {
                const real ut = P->duf_t[2 * q], vt = P->duf_t[2 * q + 1];
                const real us = P->duf_s[2 * q], vs = P->duf_s[2 * q + 1];
                real X[3], Y[3];
                for (int c = 0; c < 3; ++c) {
                    X[c] = A[0][c] + ut * (A[1][c] - A[0][c]) + vt * (A[2][c] - A[0][c]);
                    Y[c] = B[0][c] + us * (B[1][c] - B[0][c]) + vs * (B[2][c] - B[0][c]);
                }
                const real rx = X[0] - Y[0], ry = X[1] - Y[1], rz = X[2] - Y[2];
                const real w = P->duf_w[q];
                const real val = w * op_value(op, rx, ry, rz, nyx, nyy, nyz, delta, a, deps, reps);
                if (P->test_p1) { ht[0] = 1.0 - ut - vt; ht[1] = ut; ht[2] = vt; }
                if (P->trial_p1) { hs[0] = 1.0 - us - vs; hs[1] = us; hs[2] = vs; }
                const real cv = need_comb ? w * op_comb0(op, rx, ry, rz, nyx, nyy, nyz, a, h, deps, reps) : 0.0;
                for (int i = 0; i < n_t; ++i) {
                    const int64_t oi = P->test_p1 ? pt[i] : i;
                    for (int j = 0; j < n_s; ++j) {
                        const int64_t oj = P->trial_p1 ? ps[j] : j;
                        const real hij = ht[i] * hs[j];
                        lm[oi][oj] += val * hij;
                        if (need_comb) lmc[oi][oj] += cv * hij;
                    }
                }
            }
        } else {
            /* separated pair: regular product rule, bumped when close.  The
             * classification stays in double: it is the reference's exact
             * IEEE test (_assembly_numba.py:218-223) in both builds. */
            const double dcx = P->centroids[3 * e] - P->centroids[3 * f];
            const double dcy = P->centroids[3 * e + 1] - P->centroids[3 * f + 1];
            const double dcz = P->centroids[3 * e + 2] - P->centroids[3 * f + 2];
            const double dist = sqrt(dcx * dcx + dcy * dcy + dcz * dcz);
            const double de = P->diameters[e], df = P->diameters[f];
            const double dmax = de > df ? de : df;   /* Python max(a, b) */
            const double *hats, *wq, *pts; int64_t nq;
            if (dist < 2.0 * dmax) { hats = P->near_hats; wq = P->near_w; pts = P->near_pts; nq = P->n_near; }
            else { hats = P->reg_hats; wq = P->reg_w; pts = P->reg_pts; nq = P->n_reg; }
            for (int64_t p = 0; p < nq; ++p) {
                const double *xp = pts + 3 * (e * nq + p);
                for (int64_t q = 0; q < nq; ++q) {
                    const double *yq = pts + 3 * (f * nq + q);
                    const real rx = (real)xp[0] - yq[0], ry = (real)xp[1] - yq[1], rz = (real)xp[2] - yq[2];
                    const real w = (real)wq[p] * wq[q];
                    const real val = w * op_value(op, rx, ry, rz, nyx, nyy, nyz, delta, a, deps, reps);
                    const real cv = need_comb ? w * op_comb0(op, rx, ry, rz, nyx, nyy, nyz, a, h, deps, reps) : 0.0;
                    if (P->test_p1) { ht[0] = hats[3 * p]; ht[1] = hats[3 * p + 1]; ht[2] = hats[3 * p + 2]; }
                    if (P->trial_p1) { hs[0] = hats[3 * q]; hs[1] = hats[3 * q + 1]; hs[2] = hats[3 * q + 2]; }
                    for (int i = 0; i < n_t; ++i)
                        for (int j = 0; j < n_s; ++j) {
                            const real hij = ht[i] * hs[j];
                            lm[i][j] += val * hij;
                            if (need_comb) lmc[i][j] += cv * hij;
                        }
                }
            }
        }
        real jac = 4.0 * (real)P->areas[e] * P->areas[f];
        if (P->symmetric && e == f) jac *= 0.5;
        if (op == 2) jac *= nxx * nyx + nxy * nyy + nxz * nyz;
        return jac;
    }
}

/* the per-test-element body of _toeplitz_pass (_assembly_numba.py:126-272),
 * accumulating into loc_e / locc_e = (n_t, C) slices */
static void pass_row(const problem_t *P, int64_t e, real delta, int need_comb, real *loc_e, real *locc_e)
{
    const int64_t E_x = P->E_x;
    const int n_t = P->test_p1 ? 3 : 1, n_s = P->trial_p1 ? 3 : 1;
    const int64_t C = P->trial_p1 ? P->N_x : E_x;
    real lm[3][3], lmc[3][3];
    for (int64_t f = P->symmetric ? e : 0; f < E_x; ++f) {
        const real jac = pair_eval(P, e, f, delta, need_comb, lm, lmc);
        for (int i = 0; i < n_t; ++i)
            for (int j = 0; j < n_s; ++j) {
                const int64_t col = P->trial_p1 ? P->tri_nodes[3 * f + j] : f;
                loc_e[i * C + col] += jac * lm[i][j];
                if (need_comb) locc_e[i * C + col] += jac * lmc[i][j];
            }
    }
}

#define HB_PROBLEM_ARGS \
    int op, int test_p1, int trial_p1, int symmetric, int64_t E_x, int64_t N_x, \
    double alpha, double h_t, double d_eps, double r_eps, \
    const int64_t *tri_nodes, const double *verts_tri, const double *normals, \
    const double *centroids, const double *diameters, const double *areas, \
    const double *reg_hats, const double *reg_w, const double *reg_pts, int64_t n_reg, \
    const double *near_hats, const double *near_w, const double *near_pts, int64_t n_near, \
    const int64_t *tn_indptr, const int64_t *tn_idx, const int64_t *tn_case, \
    const int64_t *tn_permt, const int64_t *tn_perms, \
    const int64_t *duf_off, const double *duf_t, const double *duf_s, const double *duf_w

#define HB_PROBLEM_INIT { op, test_p1, trial_p1, symmetric, E_x, N_x, alpha, h_t, d_eps, r_eps, \
    tri_nodes, verts_tri, normals, centroids, diameters, areas, reg_hats, reg_w, reg_pts, n_reg, \
    near_hats, near_w, near_pts, n_near, tn_indptr, tn_idx, tn_case, tn_permt, tn_perms, \
    duf_off, duf_t, duf_s, duf_w }

static void set_threads(int n)
{
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}

/* one pass for the listed test rows (rows == NULL: all), into real staging
 * rows (n_rows, n_t, C) indexed by position in `rows` */
static void run_pass(const problem_t *P, real delta, int need_comb, const int64_t *rows, int64_t n_rows,
                     real *loc, real *locc, int n_threads)
{
    const int64_t n = rows ? n_rows : P->E_x;
    const int64_t stride = (P->test_p1 ? 3 : 1) * (P->trial_p1 ? P->N_x : P->E_x);
    set_threads(n_threads);
    #pragma omp parallel for schedule(dynamic, 1)
    for (int64_t k = 0; k < n; ++k) {
        const int64_t e = rows ? rows[k] : k;
        pass_row(P, e, delta, need_comb, loc + k * stride, locc + k * stride);
    }
}

/* _scatter_add (_assembly_numba.py:275-285) */
static void scatter_add(const real *loc, const int64_t *tri_nodes, int test_p1, real factor, real *block,
                        int64_t E_x, int64_t C)
{
    const int n_t = test_p1 ? 3 : 1;
    for (int64_t e = 0; e < E_x; ++e)
        for (int i = 0; i < n_t; ++i) {
            const int64_t row = test_p1 ? tri_nodes[3 * e + i] : e;
            const real *src = loc + (e * n_t + i) * C;
            real *dst = block + row * C;
            for (int64_t c = 0; c < C; ++c) dst[c] += factor * src[c];
        }
}

/* AssemblyPlan.targets (assembly.py:72-89) */
static int plan_targets(int64_t n_blocks, int64_t i_t, int64_t *d, double *mult, int *comb)
{
    int n = 0;
    if (i_t == 0) {
        d[n] = 0; mult[n] = 1.0; comb[n] = 1; ++n;
        if (n_blocks > 1) { d[n] = 1; mult[n] = -1.0; comb[n] = 0; ++n; }
        return n;
    }
    if (i_t - 1 <= n_blocks - 1) { d[n] = i_t - 1; mult[n] = -1.0; comb[n] = 0; ++n; }
    if (i_t <= n_blocks - 1) { d[n] = i_t; mult[n] = 2.0; comb[n] = 0; ++n; }
    if (i_t + 1 <= n_blocks - 1) { d[n] = i_t + 1; mult[n] = -1.0; comb[n] = 0; ++n; }
    return n;
}

#if HB_WITH_PASS
/* One pass at delta (drop-in of _toeplitz_pass), double staging. */
int hb_oracle_pass(HB_PROBLEM_ARGS, double delta, int need_comb, const int64_t *rows, int64_t n_rows,
                   double *loc, double *loc_comb, int n_threads)
{
    const problem_t P = HB_PROBLEM_INIT;
    run_pass(&P, delta, need_comb, rows, n_rows, loc, loc_comb, n_threads);
    return 0;
}
#endif

/* The whole _assemble_operator loop (assembly.py:208-239): E_t + 1 passes,
 * fixed-order scatter, symmetric mirror.  blocks: (E_t, R, C). */
int HB_SYM(hb_oracle_assemble)(HB_PROBLEM_ARGS, int64_t E_t, double step, double *blocks, int n_threads)
{
    const problem_t P = HB_PROBLEM_INIT;
    const int64_t R = test_p1 ? N_x : E_x, C = trial_p1 ? N_x : E_x;
    const int64_t n_t = test_p1 ? 3 : 1;
    const size_t loc_n = (size_t)E_x * n_t * C, blk_n = (size_t)E_t * R * C;
    real *loc = calloc(loc_n, sizeof(real));
    real *locc = calloc(loc_n, sizeof(real));
    real *acc = calloc(blk_n, sizeof(real));
    real *tmp = symmetric ? malloc((size_t)R * C * sizeof(real)) : NULL;
    if (!loc || !locc || !acc || (symmetric && !tmp)) { free(loc); free(locc); free(acc); free(tmp); return -1; }
    for (int64_t i_t = 0; i_t <= E_t; ++i_t) {
        const int need_comb = i_t == 0;
        memset(loc, 0, loc_n * sizeof(real));
        run_pass(&P, (real)((double)i_t * step), need_comb, NULL, 0, loc, locc, n_threads);
        int64_t d[3]; double mult[3]; int comb[3];
        const int nt = plan_targets(E_t, i_t, d, mult, comb);
        for (int k = 0; k < nt; ++k)
            scatter_add(comb[k] ? locc : loc, tri_nodes, test_p1, mult[k], acc + d[k] * R * C, E_x, C);
    }
    for (int64_t dd = 0; dd < E_t; ++dd) {
        real *B = acc + dd * R * C;
        if (symmetric) {   /* blocks[d] = blocks[d] + blocks[d].T */
            for (int64_t i = 0; i < R; ++i)
                for (int64_t j = 0; j < C; ++j) tmp[i * C + j] = B[i * C + j] + B[j * C + i];
            memcpy(B, tmp, (size_t)R * C * sizeof(real));
        }
        for (size_t i = 0; i < (size_t)R * C; ++i) blocks[dd * R * C + i] = (double)B[i];
    }
    free(loc); free(locc); free(acc); free(tmp);
    return 0;
}

/* Rows of a p0-test operator (V p0p0 or K) for meshes too large for a full
 * oracle assembly: the same pair values, the same i_t-ordered scatter.  For
 * symmetric ops the entry (e, f) of B + B^T is U[e][f] + U[f][e] where U is
 * the upper (f >= e) staging, so pairs are evaluated in the (min, max)
 * orientation the reference uses.  out: (E_t, n_rows, C). */
int HB_SYM(hb_oracle_rows)(HB_PROBLEM_ARGS, int64_t E_t, double step, const int64_t *rows, int64_t n_rows,
                           double *out, int n_threads)
{
    if (test_p1) return -2;
    const problem_t P = HB_PROBLEM_INIT;
    const int64_t C = trial_p1 ? N_x : E_x;
    const size_t rs = (size_t)n_rows * C;
    real *U = calloc((size_t)E_t * rs, sizeof(real));
    real *Ucol = symmetric ? calloc((size_t)E_t * rs, sizeof(real)) : NULL;  /* Ucol[d][k][f] = U[f][rows[k]] */
    if (!U || (symmetric && !Ucol)) { free(U); free(Ucol); return -1; }
    set_threads(n_threads);
    #pragma omp parallel for schedule(dynamic, 1)
    for (int64_t r = 0; r < n_rows; ++r) {
        const int64_t e = rows[r];
        real *loc = calloc(C, sizeof(real)), *locc = calloc(C, sizeof(real));
        real *cl = calloc(C, sizeof(real)), *clc = calloc(C, sizeof(real));
        real lm[3][3], lmc[3][3];
        for (int64_t i_t = 0; i_t <= E_t; ++i_t) {
            const int need_comb = i_t == 0;
            const real delta = (real)((double)i_t * step);
            memset(loc, 0, C * sizeof(real));
            memset(cl, 0, C * sizeof(real));
            for (int64_t f = symmetric ? e : 0; f < E_x; ++f) {
                const real jac = pair_eval(&P, e, f, delta, need_comb, lm, lmc);
                for (int j = 0; j < (trial_p1 ? 3 : 1); ++j) {
                    const int64_t col = trial_p1 ? tri_nodes[3 * f + j] : f;
                    loc[col] += jac * lm[0][j];
                    if (need_comb) locc[col] += jac * lmc[0][j];
                }
            }
            if (symmetric)   /* column e of the upper staging: pairs (f, e), f < e */
                for (int64_t f = 0; f < e; ++f) {
                    const real jac = pair_eval(&P, f, e, delta, need_comb, lm, lmc);
                    cl[f] += jac * lm[0][0];
                    if (need_comb) clc[f] += jac * lmc[0][0];
                }
            int64_t d[3]; double mult[3]; int comb[3];
            const int nt = plan_targets(E_t, i_t, d, mult, comb);
            for (int k = 0; k < nt; ++k) {
                real *u = U + d[k] * rs + r * C;
                const real *src = comb[k] ? locc : loc;
                for (int64_t c = 0; c < C; ++c) u[c] += mult[k] * src[c];
                if (symmetric) {
                    real *uc = Ucol + d[k] * rs + r * C;
                    const real *cs = comb[k] ? clc : cl;
                    for (int64_t c = 0; c < C; ++c) uc[c] += mult[k] * cs[c];
                }
            }
        }
        free(loc); free(locc); free(cl); free(clc);
    }
    for (int64_t dd = 0; dd < E_t; ++dd)
        for (int64_t r = 0; r < n_rows; ++r)
            for (int64_t f = 0; f < C; ++f) {
                const size_t i = dd * rs + r * C + f;
                if (!symmetric) { out[i] = (double)U[i]; continue; }
                /* B[e][f] = U[e][f] + U[f][e]: for f > e the second term is
                 * the (never written) lower staging = +0, for f < e the
                 * first; the diagonal is U[e][e] + U[e][e] */
                const int64_t e = rows[r];
                const real uef = f >= e ? U[i] : 0.0, ufe = f <= e ? (f == e ? U[i] : Ucol[i]) : 0.0;
                out[i] = (double)(uef + ufe);
            }
    free(U); free(Ucol);
    return 0;
}

/* D = D2 + alpha^2 sum_{e in star(m), f in star(n)} (curl_e,m . curl_f,n) V[e][f]
 * (heatbem/assembly.py:289-334 as a dense restatement; used by the quad build
 * for the exact D -- the double build's D goes through scipy exactly as the
 * reference does, oracle.curl_combine).  V given in the same precision. */
int HB_SYM(hb_oracle_curl_combine)(int64_t n_blocks, int64_t E_x, int64_t N_x, double alpha,
                                   const int64_t *tri_nodes, const double *curls,
                                   const double *V, const double *D2, double *D, int n_threads)
{
    set_threads(n_threads);
    const real a2 = (real)alpha * alpha;
    int bad = 0;
    #pragma omp parallel for schedule(dynamic, 1)
    for (int64_t d = 0; d < n_blocks; ++d) {
        real *acc = calloc((size_t)N_x * N_x, sizeof(real));
        if (!acc) { bad = 1; continue; }
        const double *Vd = V + d * E_x * E_x;
        for (int64_t e = 0; e < E_x; ++e)
            for (int i = 0; i < 3; ++i) {
                const int64_t m = tri_nodes[3 * e + i];
                const double *ce = curls + 9 * e + 3 * i;
                for (int64_t f = 0; f < E_x; ++f) {
                    const real v = Vd[e * E_x + f];
                    for (int j = 0; j < 3; ++j) {
                        const int64_t n = tri_nodes[3 * f + j];
                        const double *cf = curls + 9 * f + 3 * j;
                        const real dot = (real)ce[0] * cf[0] + (real)ce[1] * cf[1] + (real)ce[2] * cf[2];
                        acc[m * N_x + n] += dot * v;
                    }
                }
            }
        for (int64_t i = 0; i < N_x * N_x; ++i)
            D[d * N_x * N_x + i] = (double)((real)D2[d * N_x * N_x + i] + a2 * acc[i]);
        free(acc);
    }
    return bad ? -1 : 0;
}

/* _field_numba._eval_potential (_field_numba.py:15-79) */
int HB_SYM(hb_oracle_potential)(int kind, const double *points, const int64_t *k_arr, const double *eps_arr,
                                const uint8_t *cur_arr, const double *dens, const double *qpts, const double *qw,
                                const double *areas, const double *normals, int64_t n_pts, int64_t E_t,
                                int64_t E_x, int64_t nq, double h_t, double alpha, double d_eps, double r_eps,
                                double *out, int n_threads)
{
    set_threads(n_threads);
    #pragma omp parallel for schedule(dynamic, 1)
    for (int64_t p = 0; p < n_pts; ++p) {
        const int64_t k = k_arr[p];
        const real eps = eps_arr[p];
        const int use_cur = cur_arr[p] != 0;
        const real px = points[3 * p], py = points[3 * p + 1], pz = points[3 * p + 2];
        const real a = alpha, de = d_eps, re = r_eps;
        real acc = 0.0;
        for (int64_t e = 0; e < E_x; ++e) {
            const real nyx = normals[3 * e], nyy = normals[3 * e + 1], nyz = normals[3 * e + 2];
            real el = 0.0;
            for (int64_t q = 0; q < nq; ++q) {
                const double *y = qpts + 3 * (e * nq + q);
                const real rx = px - y[0], ry = py - y[1], rz = pz - y[2];
                const real rho = HB_SQRT(rx * rx + ry * ry + rz * rz);
                const real rn = rx * nyx + ry * nyy + rz * nyz;
                real s = 0.0;
                for (int64_t m = 0; m <= k; ++m) {
                    const int64_t hi = k - 1 - m, lo = k - m;
                    real c = (hi >= 0 && hi < E_t) ? (real)dens[(hi * E_x + e) * nq + q] : 0.0;
                    if (lo >= 0 && lo < E_t && (lo < k || use_cur)) c -= dens[(lo * E_x + e) * nq + q];
                    if (c == 0.0) continue;
                    const real gap = (real)((double)m * h_t) + eps;
                    const real g = kind == 0 ? g_dtau(rho, gap, a, de, re) : dn_g_dtau(rn, rho, gap, a, de, re);
                    s += c * g;
                }
                if (use_cur && k >= 0 && k < E_t) {
                    const real g0 = kind == 0 ? g_dtau(rho, 0.0, a, de, re) : dn_g_dtau(rn, rho, 0.0, a, de, re);
                    s += dens[(k * E_x + e) * nq + q] * g0;
                }
                el += (real)qw[q] * s;
            }
            acc += 2.0 * (real)areas[e] * el;
        }
        out[p] = (double)acc;
    }
    return 0;
}

#if HB_WITH_PASS
int hb_oracle_max_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
#endif
