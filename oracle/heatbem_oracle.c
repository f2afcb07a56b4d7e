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
 * container); tests/test_oracle_golden.py checks this file against them.
 *
 * Followed, function by function:
 *   scalar kernels   <- heatbem/_assembly_numba.py:25-104
 *   hb_oracle_pass   <- heatbem/_assembly_numba.py:111-272 (_toeplitz_pass)
 *   scatter          <- heatbem/_assembly_numba.py:275-285 (_scatter_add)
 *   hb_oracle_assemble <- heatbem/assembly.py:178-242 (_assemble_operator loop,
 *                       AssemblyPlan.targets assembly.py:72-89, mirror :237-239)
 *   hb_oracle_potential <- heatbem/_field_numba.py:15-79
 *
 * Arithmetic is written in the reference's evaluation order and compiled
 * with -ffp-contract=off so every product/sum rounds exactly as numba's
 * (non-fastmath) LLVM code does; erf/exp come from the host glibc libm, as
 * in numba (math.erf -> extern erf, math.exp -> llvm.exp -> libm exp).
 * Integer powers x**3 are lowered by numba to repeated multiplication.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define PI 3.141592653589793

static inline double cube(double x) { return x * x * x; }

/* _assembly_numba.py:25-32 */
static inline double g_dtau(double rho, double delta, double a, double deps, double reps)
{
    if (delta <= deps) return 1.0 / (4.0 * PI * a * rho);
    if (rho <= reps) return 1.0 / (4.0 * sqrt(cube(PI) * cube(a) * delta));
    double x = rho / (2.0 * sqrt(a * delta));
    return erf(x) / (4.0 * PI * a * rho);
}

/* _assembly_numba.py:35-45 */
static inline double g_dtaudt(double rho, double delta, double a, double deps, double reps)
{
    if (delta <= deps) return rho / (8.0 * PI * a * a);
    if (rho <= reps) return sqrt(delta) / (2.0 * sqrt(cube(PI) * cube(a)));
    double x = rho / (2.0 * sqrt(a * delta));
    double t1 = (rho / (2.0 * a * a) + delta / (a * rho)) * erf(x);
    double t2 = sqrt(delta) / sqrt(PI * cube(a)) * exp(-x * x);
    return (t1 + t2) / (4.0 * PI);
}

/* _assembly_numba.py:48-59 */
static inline double dn_g_dtau(double rn, double rho, double delta, double a,
                               double deps, double reps)
{
    if (rho <= reps) return 0.0;
    if (delta <= deps) return rn / (4.0 * PI * cube(rho));
    double x = rho / (2.0 * sqrt(a * delta));
    double inner = erf(x) / rho - exp(-x * x) / sqrt(PI * a * delta);
    return (rn / (rho * rho)) * inner / (4.0 * PI);
}

/* _assembly_numba.py:62-76 */
static inline double dn_g_dtaudt(double rn, double rho, double delta, double a,
                                 double deps, double reps)
{
    if (rho <= reps) return 0.0;
    if (delta <= deps) return -rn / (8.0 * PI * a * rho);
    double x = rho / (2.0 * sqrt(a * delta));
    double inner = (1.0 / (2.0 * a) - delta / (rho * rho)) * erf(x)
                 + sqrt(delta) / (rho * sqrt(PI * a)) * exp(-x * x);
    return -(rn / rho) * inner / (4.0 * PI);
}

/* _assembly_numba.py:79-87 */
static inline double op_value(int op, double rx, double ry, double rz,
                              double nyx, double nyy, double nyz,
                              double delta, double a, double deps, double reps)
{
    double rho = sqrt(rx * rx + ry * ry + rz * rz);
    if (op == 0) return g_dtaudt(rho, delta, a, deps, reps);
    if (op == 1) {
        double rn = rx * nyx + ry * nyy + rz * nyz;
        return dn_g_dtaudt(rn, rho, delta, a, deps, reps);
    }
    return a * g_dtau(rho, delta, a, deps, reps);
}

/* _assembly_numba.py:90-104: combined d = 0 kernel (i_t = 0 only) */
static inline double op_comb0(int op, double rx, double ry, double rz,
                              double nyx, double nyy, double nyz,
                              double a, double h, double deps, double reps)
{
    double rho = sqrt(rx * rx + ry * ry + rz * rz);
    if (op == 0) return h * g_dtau(rho, 0.0, a, deps, reps) + g_dtaudt(rho, 0.0, a, deps, reps);
    if (op == 1) {
        double rn = rx * nyx + ry * nyy + rz * nyz;
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
} hb_oracle_problem;

/* the per-test-element body of _toeplitz_pass (_assembly_numba.py:126-272),
 * writing into loc_e / locc_e = (n_t, C) slices */
static void pass_row(const hb_oracle_problem *P, int64_t e, double delta, int need_comb,
                     double *loc_e, double *locc_e)
{
    const int64_t E_x = P->E_x;
    const int n_t = P->test_p1 ? 3 : 1, n_s = P->trial_p1 ? 3 : 1;
    const int64_t C = P->trial_p1 ? P->N_x : E_x;
    const int op = P->op;
    const double a = P->alpha, deps = P->d_eps, reps = P->r_eps, h = P->h_t;
    double lm[3][3], lmc[3][3];
    double ht[3] = {1.0, 0.0, 0.0}, hs[3] = {1.0, 0.0, 0.0};
    const double nxx = P->normals[3 * e], nxy = P->normals[3 * e + 1], nxz = P->normals[3 * e + 2];
    const int64_t t_lo = P->tn_indptr[e], t_hi = P->tn_indptr[e + 1];
    const int64_t f0 = P->symmetric ? e : 0;
    for (int64_t f = f0; f < E_x; ++f) {
        int64_t tpos = -1, lo = t_lo, hi = t_hi;
        while (lo < hi) {
            int64_t mid = (lo + hi) / 2, v = P->tn_idx[mid];
            if (v < f) lo = mid + 1;
            else if (v > f) hi = mid;
            else { tpos = mid; break; }
        }
        memset(lm, 0, sizeof lm);
        memset(lmc, 0, sizeof lmc);
        const double nyx = P->normals[3 * f], nyy = P->normals[3 * f + 1], nyz = P->normals[3 * f + 2];
        if (tpos >= 0) {
            const int64_t cs = P->tn_case[tpos];
            const int64_t *pt = P->tn_permt + 3 * tpos, *ps = P->tn_perms + 3 * tpos;
            const double *ve = P->verts_tri + 9 * e, *vf = P->verts_tri + 9 * f;
            double A[3][3], B[3][3];
            for (int k = 0; k < 3; ++k)
                for (int c = 0; c < 3; ++c) { A[k][c] = ve[3 * pt[k] + c]; B[k][c] = vf[3 * ps[k] + c]; }
            for (int64_t q = P->duf_off[cs]; q < P->duf_off[cs + 1]; ++q) {
                const double ut = P->duf_t[2 * q], vt = P->duf_t[2 * q + 1];
                const double us = P->duf_s[2 * q], vs = P->duf_s[2 * q + 1];
                double X[3], Y[3];
                for (int c = 0; c < 3; ++c) {
                    X[c] = A[0][c] + ut * (A[1][c] - A[0][c]) + vt * (A[2][c] - A[0][c]);
                    Y[c] = B[0][c] + us * (B[1][c] - B[0][c]) + vs * (B[2][c] - B[0][c]);
                }
                const double rx = X[0] - Y[0], ry = X[1] - Y[1], rz = X[2] - Y[2];
                const double w = P->duf_w[q];
                const double val = w * op_value(op, rx, ry, rz, nyx, nyy, nyz, delta, a, deps, reps);
                if (P->test_p1) { ht[0] = 1.0 - ut - vt; ht[1] = ut; ht[2] = vt; }
                if (P->trial_p1) { hs[0] = 1.0 - us - vs; hs[1] = us; hs[2] = vs; }
                const double cv = need_comb
                    ? w * op_comb0(op, rx, ry, rz, nyx, nyy, nyz, a, h, deps, reps) : 0.0;
                for (int i = 0; i < n_t; ++i) {
                    const int64_t oi = P->test_p1 ? pt[i] : i;
                    for (int j = 0; j < n_s; ++j) {
                        const int64_t oj = P->trial_p1 ? ps[j] : j;
                        const double hij = ht[i] * hs[j];
                        lm[oi][oj] += val * hij;
                        if (need_comb) lmc[oi][oj] += cv * hij;
                    }
                }
            }
        } else {
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
                    const double rx = xp[0] - yq[0], ry = xp[1] - yq[1], rz = xp[2] - yq[2];
                    const double w = wq[p] * wq[q];
                    const double val = w * op_value(op, rx, ry, rz, nyx, nyy, nyz, delta, a, deps, reps);
                    const double cv = need_comb
                        ? w * op_comb0(op, rx, ry, rz, nyx, nyy, nyz, a, h, deps, reps) : 0.0;
                    if (P->test_p1) { ht[0] = hats[3 * p]; ht[1] = hats[3 * p + 1]; ht[2] = hats[3 * p + 2]; }
                    if (P->trial_p1) { hs[0] = hats[3 * q]; hs[1] = hats[3 * q + 1]; hs[2] = hats[3 * q + 2]; }
                    for (int i = 0; i < n_t; ++i)
                        for (int j = 0; j < n_s; ++j) {
                            const double hij = ht[i] * hs[j];
                            lm[i][j] += val * hij;
                            if (need_comb) lmc[i][j] += cv * hij;
                        }
                }
            }
        }
        double jac = 4.0 * P->areas[e] * P->areas[f];
        if (P->symmetric && e == f) jac *= 0.5;
        if (op == 2) jac *= nxx * nyx + nxy * nyy + nxz * nyz;
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

/* One pass at delta for the listed test elements (rows == NULL: all).
 * loc / loc_comb are (n_rows, n_t, C), indexed by position in `rows`.
 * Restates _toeplitz_pass (_assembly_numba.py:111-272). */
int hb_oracle_pass(HB_PROBLEM_ARGS, double delta, int need_comb,
                   const int64_t *rows, int64_t n_rows,
                   double *loc, double *loc_comb, int n_threads)
{
    const hb_oracle_problem P = HB_PROBLEM_INIT;
    const int64_t n = rows ? n_rows : E_x;
    const int64_t stride = (test_p1 ? 3 : 1) * (trial_p1 ? N_x : E_x);
    set_threads(n_threads);
    #pragma omp parallel for schedule(dynamic, 1)
    for (int64_t k = 0; k < n; ++k) {
        const int64_t e = rows ? rows[k] : k;
        pass_row(&P, e, delta, need_comb, loc + k * stride, loc_comb + k * stride);
    }
    return 0;
}

/* _scatter_add (_assembly_numba.py:275-285) */
static void scatter_add(const double *loc, const int64_t *tri_nodes, int test_p1,
                        double factor, double *block, int64_t E_x, int64_t C)
{
    const int n_t = test_p1 ? 3 : 1;
    for (int64_t e = 0; e < E_x; ++e)
        for (int i = 0; i < n_t; ++i) {
            const int64_t row = test_p1 ? tri_nodes[3 * e + i] : e;
            const double *src = loc + (e * n_t + i) * C;
            double *dst = block + row * C;
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

/* The whole _assemble_operator loop (assembly.py:208-239): E_t + 1 passes,
 * fixed-order scatter, symmetric mirror.  blocks: (E_t, R, C), zeroed here. */
int hb_oracle_assemble(HB_PROBLEM_ARGS, int64_t E_t, double step, double *blocks, int n_threads)
{
    const int64_t R = test_p1 ? N_x : E_x, C = trial_p1 ? N_x : E_x;
    const int64_t n_t = test_p1 ? 3 : 1;
    const size_t loc_n = (size_t)E_x * n_t * C;
    double *loc = malloc(loc_n * sizeof(double));
    double *locc = malloc(loc_n * sizeof(double));
    if (!loc || !locc) { free(loc); free(locc); return -1; }
    memset(blocks, 0, (size_t)E_t * R * C * sizeof(double));
    memset(locc, 0, loc_n * sizeof(double));
    for (int64_t i_t = 0; i_t <= E_t; ++i_t) {
        const int need_comb = i_t == 0;
        memset(loc, 0, loc_n * sizeof(double));
        hb_oracle_pass(op, test_p1, trial_p1, symmetric, E_x, N_x, alpha, step, d_eps, r_eps,
                       tri_nodes, verts_tri, normals, centroids, diameters, areas,
                       reg_hats, reg_w, reg_pts, n_reg, near_hats, near_w, near_pts, n_near,
                       tn_indptr, tn_idx, tn_case, tn_permt, tn_perms,
                       duf_off, duf_t, duf_s, duf_w,
                       (double)i_t * step, need_comb, NULL, 0, loc, locc, n_threads);
        int64_t d[3]; double mult[3]; int comb[3];
        const int nt = plan_targets(E_t, i_t, d, mult, comb);
        for (int k = 0; k < nt; ++k)
            scatter_add(comb[k] ? locc : loc, tri_nodes, test_p1, mult[k],
                        blocks + d[k] * R * C, E_x, C);
    }
    if (symmetric) {
        /* blocks[d] = blocks[d] + blocks[d].T (element-wise, into a copy) */
        double *tmp = malloc((size_t)R * C * sizeof(double));
        if (!tmp) { free(loc); free(locc); return -1; }
        for (int64_t dd = 0; dd < E_t; ++dd) {
            double *B = blocks + dd * R * C;
            for (int64_t i = 0; i < R; ++i)
                for (int64_t j = 0; j < C; ++j) tmp[i * C + j] = B[i * C + j] + B[j * C + i];
            memcpy(B, tmp, (size_t)R * C * sizeof(double));
        }
        free(tmp);
    }
    free(loc);
    free(locc);
    return 0;
}

/* Rows [of a p0-test operator] of all E_t blocks, for meshes too large for a
 * full oracle assembly: same passes, same i_t-ordered scatter, and the mirror
 * entries (f < e) taken from pair (f, e) as the reference's B + B^T does.
 * out: (E_t, n_rows, C).  Only p0 test (V p0p0, K). */
int hb_oracle_rows(HB_PROBLEM_ARGS, int64_t E_t, double step, const int64_t *rows, int64_t n_rows,
                   double *out, int n_threads)
{
    if (test_p1) return -2;
    const int64_t C = trial_p1 ? N_x : E_x;
    /* upper part U[e, :] for the requested rows, and for symmetric ops the
     * column U[:, e] restricted to f < e, i.e. rows f of the pass */
    const size_t rs = (size_t)n_rows * C;
    double *loc = malloc(rs * sizeof(double)), *locc = malloc(rs * sizeof(double));
    double *U = calloc((size_t)E_t * rs, sizeof(double));
    double *Ucol = NULL, *colloc = NULL, *collocc = NULL;
    int64_t *allrows = NULL;
    if (!loc || !locc || !U) goto fail;
    if (symmetric) {
        /* column e of U needs pass rows f < e; compute the full pass for all
         * f (cost of the full pass; acceptable for an oracle) */
        Ucol = calloc((size_t)E_t * rs, sizeof(double));   /* Ucol[d][k][f] = U[f][rows[k]] */
        colloc = malloc((size_t)E_x * C * sizeof(double));
        collocc = malloc((size_t)E_x * C * sizeof(double));
        if (!Ucol || !colloc || !collocc) goto fail;
    }
    memset(locc, 0, rs * sizeof(double));
    if (collocc) memset(collocc, 0, (size_t)E_x * C * sizeof(double));
    for (int64_t i_t = 0; i_t <= E_t; ++i_t) {
        const int need_comb = i_t == 0;
        const double delta = (double)i_t * step;
        int64_t d[3]; double mult[3]; int comb[3];
        const int nt = plan_targets(E_t, i_t, d, mult, comb);
        if (!symmetric) {
            memset(loc, 0, rs * sizeof(double));
            hb_oracle_pass(op, test_p1, trial_p1, symmetric, E_x, N_x, alpha, step, d_eps, r_eps,
                           tri_nodes, verts_tri, normals, centroids, diameters, areas,
                           reg_hats, reg_w, reg_pts, n_reg, near_hats, near_w, near_pts, n_near,
                           tn_indptr, tn_idx, tn_case, tn_permt, tn_perms,
                           duf_off, duf_t, duf_s, duf_w,
                           delta, need_comb, rows, n_rows, loc, locc, n_threads);
            for (int k = 0; k < nt; ++k) {
                const double *src = comb[k] ? locc : loc;
                double *dst = U + d[k] * rs;
                for (size_t i = 0; i < rs; ++i) dst[i] += mult[k] * src[i];
            }
        } else {
            memset(colloc, 0, (size_t)E_x * C * sizeof(double));
            hb_oracle_pass(op, test_p1, trial_p1, symmetric, E_x, N_x, alpha, step, d_eps, r_eps,
                           tri_nodes, verts_tri, normals, centroids, diameters, areas,
                           reg_hats, reg_w, reg_pts, n_reg, near_hats, near_w, near_pts, n_near,
                           tn_indptr, tn_idx, tn_case, tn_permt, tn_perms,
                           duf_off, duf_t, duf_s, duf_w,
                           delta, need_comb, NULL, 0, colloc, collocc, n_threads);
            for (int k = 0; k < nt; ++k) {
                const double *src = comb[k] ? collocc : colloc;
                for (int64_t r = 0; r < n_rows; ++r) {
                    const int64_t e = rows[r];
                    double *u = U + d[k] * rs + r * C, *uc = Ucol + d[k] * rs + r * C;
                    for (int64_t f = 0; f < C; ++f) {
                        u[f] += mult[k] * src[e * C + f];    /* U[e][f]  */
                        uc[f] += mult[k] * src[f * C + e];   /* U[f][e]  */
                    }
                }
            }
        }
    }
    for (int64_t dd = 0; dd < E_t; ++dd)
        for (int64_t r = 0; r < n_rows; ++r)
            for (int64_t f = 0; f < C; ++f) {
                const size_t i = dd * rs + r * C + f;
                out[i] = symmetric ? U[i] + Ucol[i] : U[i];
            }
    free(loc); free(locc); free(U); free(Ucol); free(colloc); free(collocc); free(allrows);
    return 0;
fail:
    free(loc); free(locc); free(U); free(Ucol); free(colloc); free(collocc); free(allrows);
    return -1;
}

/* _field_numba._eval_potential (_field_numba.py:15-79) */
int hb_oracle_potential(int kind, const double *points, const int64_t *k_arr,
                        const double *eps_arr, const uint8_t *cur_arr,
                        const double *dens, const double *qpts, const double *qw,
                        const double *areas, const double *normals,
                        int64_t n_pts, int64_t E_t, int64_t E_x, int64_t nq,
                        double h_t, double alpha, double d_eps, double r_eps,
                        double *out, int n_threads)
{
    set_threads(n_threads);
    #pragma omp parallel for schedule(dynamic, 1)
    for (int64_t p = 0; p < n_pts; ++p) {
        const int64_t k = k_arr[p];
        const double eps = eps_arr[p];
        const int use_cur = cur_arr[p] != 0;
        const double px = points[3 * p], py = points[3 * p + 1], pz = points[3 * p + 2];
        double acc = 0.0;
        for (int64_t e = 0; e < E_x; ++e) {
            const double nyx = normals[3 * e], nyy = normals[3 * e + 1], nyz = normals[3 * e + 2];
            double el = 0.0;
            for (int64_t q = 0; q < nq; ++q) {
                const double *y = qpts + 3 * (e * nq + q);
                const double rx = px - y[0], ry = py - y[1], rz = pz - y[2];
                const double rho = sqrt(rx * rx + ry * ry + rz * rz);
                const double rn = rx * nyx + ry * nyy + rz * nyz;
                double s = 0.0;
                for (int64_t m = 0; m <= k; ++m) {
                    const int64_t hi = k - 1 - m, lo = k - m;
                    double c = (hi >= 0 && hi < E_t) ? dens[(hi * E_x + e) * nq + q] : 0.0;
                    if (lo >= 0 && lo < E_t && (lo < k || use_cur)) c -= dens[(lo * E_x + e) * nq + q];
                    if (c == 0.0) continue;
                    const double gap = (double)m * h_t + eps;
                    const double g = kind == 0 ? g_dtau(rho, gap, alpha, d_eps, r_eps)
                                               : dn_g_dtau(rn, rho, gap, alpha, d_eps, r_eps);
                    s += c * g;
                }
                if (use_cur && k >= 0 && k < E_t) {
                    const double g0 = kind == 0 ? g_dtau(rho, 0.0, alpha, d_eps, r_eps)
                                                : dn_g_dtau(rn, rho, 0.0, alpha, d_eps, r_eps);
                    s += dens[(k * E_x + e) * nq + q] * g0;
                }
                el += qw[q] * s;
            }
            acc += 2.0 * areas[e] * el;
        }
        out[p] = acc;
    }
    return 0;
}

int hb_oracle_max_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
