/*
 * heatbem_b200.h -- C ABI of the B200 (sm_100a) space-time heat BEM library.
 *
 * Plain pointers and sizes only.  Every array argument named *_dev is a
 * device pointer the caller owns (PyTorch allocates them); the library keeps
 * no allocations between calls.  All entry points are stream-ordered on the
 * cudaStream_t passed as `stream` (NULL = legacy default stream), return 0
 * on success or a negative HB_ERR_* code, and never abort; the message of
 * the last failure on the calling thread is available from hb_last_error().
 *
 * Reference interfaces replaced (file:line in the heatbem reference):
 *   hb_assemble              heatbem/assembly.py:178-242 (_assemble_operator:
 *                            the E_t+1 _toeplitz_pass calls of
 *                            _assembly_numba.py:111-272, the _scatter_add
 *                            of _assembly_numba.py:275-285 and the symmetric
 *                            mirror of assembly.py:237-239) -- one call
 *                            builds blocks [d_begin, d_end) of V, V11, K or D2.
 *   hb_curl_combine          heatbem/assembly.py:314-334
 *                            (hypersingular_from_single_layer).
 *   hb_potential             heatbem/_field_numba.py:15-79 (_eval_potential)
 *                            plus the per-point loop of field.py:147-167.
 *   hb_toeplitz_apply        heatbem/solver.py:47-73 (apply_toeplitz).
 *   hb_forward_subst_step    heatbem/solver.py:178-182 (history update of
 *                            forward_block_solve).
 *   hb_project_data          heatbem/field.py:84-119 (project_to_space) for
 *                            heat-kernel data; hb_p1_mass_solve its X10 mass
 *                            solve; hb_error_sigma field.py:193-215.
 */
#ifndef HEATBEM_B200_H
#define HEATBEM_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HB_OK 0
#define HB_ERR_INVALID (-1)     /* bad argument / inconsistent sizes        */
#define HB_ERR_CUDA (-2)        /* CUDA launch or runtime failure           */
#define HB_ERR_WORKSPACE (-3)   /* workspace too small for one row chunk    */
#define HB_ERR_UNSUPPORTED (-4) /* op / space combination not implemented   */

/* operator codes, as heatbem/assembly.py:21 */
#define HB_OP_SINGLE_LAYER 0    /* G^{dtau dt}                              */
#define HB_OP_DOUBLE_LAYER 1    /* alpha dG^{dtau dt}/dn_y                  */
#define HB_OP_HYPERSINGULAR2 2  /* alpha G^{dtau} n_x.n_y                   */

int hb_version(void);
const char *hb_last_error(void);

/* Mesh, rule tables and adjacency: every array is what
 * heatbem/assembly.py:201-206 hands to _toeplitz_pass, plus three
 * host-built index lists (singular work list, node stars). */
typedef struct {
    int64_t E_x, N_x;
    const int64_t *tri_nodes_dev;   /* (E_x,3)                              */
    const double *verts_tri_dev;    /* (E_x,3,3)                            */
    const double *normals_dev;      /* (E_x,3)                              */
    const double *centroids_dev;    /* (E_x,3)                              */
    const double *diameters_dev;    /* (E_x,)                               */
    const double *areas_dev;        /* (E_x,)                               */
    const double *reg_hats_dev, *reg_w_dev, *reg_pts_dev;    /* (nr,3) (nr,) (E_x,nr,3) */
    int64_t n_reg;
    const double *near_hats_dev, *near_w_dev, *near_pts_dev; /* (nn,3) (nn,) (E_x,nn,3) */
    int64_t n_near;
    const int64_t *tn_indptr_dev;   /* (E_x+1,) touching CSR                */
    const int64_t *tn_idx_dev;      /* (nnz,) trial element, sorted per row */
    const int64_t *tn_case_dev;     /* (nnz,) 0 identical 1 edge 2 vertex   */
    const int64_t *tn_permt_dev;    /* (nnz,3)                              */
    const int64_t *tn_perms_dev;    /* (nnz,3)                              */
    const int64_t *duf_off_dev;     /* (4,) offsets into the Duffy table    */
    const double *duf_t_dev, *duf_s_dev, *duf_w_dev;         /* (nd,2) (nd,2) (nd,) */
    /* singular work list: CSR positions to evaluate, sorted by test row;
     * for symmetric ops only positions with tn_idx >= row.
     * sing_rowptr (E_x+1,) delimits each row's slice of sing_pos. */
    const int64_t *sing_pos_dev;
    const int64_t *sing_rowptr_dev;
    int64_t sing_max_per_row;
    const int64_t *sing_row_dev;    /* (nnz,) test row of each CSR position */
    /* node stars: for node n, (element, local vertex) pairs sorted by
     * element in star_elem/star_local[star_indptr[n] : star_indptr[n+1]] */
    const int64_t *star_indptr_dev, *star_elem_dev, *star_local_dev;
    int64_t star_max;               /* max star size                        */
    /* curl-combine plan over 32-node tiles t = 0..ceil(N_x/32)-1: the sorted
     * distinct elements of the tile's node stars are
     * curl_tile_elem[curl_tile_eptr[t] .. curl_tile_eptr[t+1]); star entry s
     * (node n) sits at curl_star_pos[s] in the list of n's tile. */
    const int64_t *curl_tile_eptr_dev, *curl_tile_elem_dev;
    const int32_t *curl_star_pos_dev;
    int64_t curl_tile_emax;         /* max elements per tile                */
    int64_t curl_tile_smax;         /* max star entries per tile            */
} hb_mesh_desc;

/* Optional per-call statistics (host memory).  When hb_assembly_desc.stats
 * is non-NULL, hb_assemble brackets every pair-kernel and finalize launch
 * with CUDA events on `stream`, synchronises the stream before returning
 * and ADDS the elapsed times and launch counts here. */
typedef struct {
    double pair_ms;                 /* k_pairs launches (regular + singular) */
    double finalize_ms;             /* staging -> blocks (+ symmetrize)      */
    int64_t pair_launches;
    int64_t launches;               /* all kernels launched by the call      */
} hb_assembly_stats;

typedef struct {
    int op;                         /* HB_OP_*                              */
    int test_p1, trial_p1, symmetric;
    int64_t E_t;                    /* number of time steps (blocks)        */
    double step;                    /* h_t = T / E_t (TimeGrid.step)        */
    double alpha, d_eps, r_eps;     /* KernelParams.alpha/delta_eps/rho_eps */
    int64_t d_begin, d_end;         /* blocks produced: [d_begin, d_end)    */
    double *blocks_dev;             /* (d_end-d_begin, R, C) row-major      */
    void *workspace_dev;            /* staging, >= hb_assemble_min_workspace */
    size_t workspace_bytes;
    hb_assembly_stats *stats;       /* optional (NULL: no timing, no sync)  */
    /* Row-parallel assembly.  Test rows [row_begin, row_end)
     * only (row_end <= row_begin: all rows); with block_ptrs_dev != NULL
     * (device array of d_end - d_begin pointers) block d is written at
     * block_ptrs_dev[d - d_begin] -- e.g. the d-owner's memory on another
     * GPU (CUDA IPC, hb_ipc_*) -- instead of blocks_dev.  Every entry of a
     * block is written by exactly one row range (V: direct and mirrored
     * entries of its rows), so ranks splitting the rows fill the d-sharded
     * blocks bitwise as one GPU would.  p1 x p1 operators accumulate over
     * element rows: a row range gives the (symmetrised) contribution of those
     * rows -- partial sums to be added across ranks (distributed.py: NCCL
     * reduce-scatter); contiguous blocks only. */
    int64_t row_begin, row_end;
    double *const *block_ptrs_dev;
    /* Row-sharded destination (the solve operator's layout, SURVEY 8(e):
     * rank k holds rows [bounds[k], bounds[k+1]) of every block).  With
     * n_row_shards > 0 (p0 test functions only; exclusive with
     * block_ptrs_dev) entry (d, r, c) is written at
     *   row_shard_ptrs_dev[k] + ((d - d_begin) (bounds[k+1] - bounds[k])
     *                            + r - bounds[k]) C + c,
     * bounds = row_shard_bounds_dev (n_row_shards + 1 ascending device
     * int64 values, bounds[0] = 0, bounds[n] = R), pointers typically the
     * peers' shards mapped with hb_ipc_import.  The finalize stores ARE the
     * exchange: V's mirrored entries land in the owner of their row, so
     * ranks splitting the pair work by any row ranges fill the row shards
     * bitwise as one GPU fills the whole blocks. */
    int64_t n_row_shards;
    const int64_t *row_shard_bounds_dev;
    double *const *row_shard_ptrs_dev;
} hb_assembly_desc;

/* bytes of staging for one test-row chunk (the minimum) and for all rows */
size_t hb_assemble_min_workspace(const hb_mesh_desc *mesh, const hb_assembly_desc *a);
size_t hb_assemble_full_workspace(const hb_mesh_desc *mesh, const hb_assembly_desc *a);

/* Fused single layer + hypersingular operator (heatbem assembly.py:337-361,
 * assemble_hypersingular without a given single_layer; replaces the
 * assemble_single_layer + hypersingular_from_single_layer sequence,
 * assembly.py:314-334).  d2 describes D2 (op HB_OP_HYPERSINGULAR2, p1 x p1,
 * symmetric, all rows, contiguous blocks); its blocks_dev receives
 * D = D2 + alpha^2 sum_o T_o^T V T_o, its workspace holds the staging of
 * BOTH operators for a test-row chunk (>= hb_assemble_vd_min_workspace).
 * V and D2 are assembled in the same row chunks and the p1 x p1 finalize
 * adds alpha^2 (curl_ei . curl_fj) V_ef to each pair (e, f >= e) as it
 * accumulates D2, so V is never re-read for the curl transform.
 * V_blocks_dev (nullable): V of the same blocks, p0 x p0 -- bitwise the
 * blocks hb_assemble gives.  curls_dev: (E_x, 3, 3) surface curls,
 * curl of hat i on e = (v_{i+1} - v_{i+2}) / (2 area_e).
 * The memory-lean path (D without V's blocks: NULL V_blocks_dev); when V is
 * kept anyway, hb_assemble + hb_curl_combine on separate streams is faster
 * (the fused finalize loads twice as much as the plain p1 x p1 one). */
size_t hb_assemble_vd_min_workspace(const hb_mesh_desc *mesh, const hb_assembly_desc *d2);
size_t hb_assemble_vd_full_workspace(const hb_mesh_desc *mesh, const hb_assembly_desc *d2);
int hb_assemble_vd(const hb_mesh_desc *mesh, const hb_assembly_desc *d2, double *V_blocks_dev,
                   const double *curls_dev, void *stream);

/* Assemble blocks [d_begin, d_end) of one operator.  Writes every entry of
 * blocks_dev; results are bitwise deterministic run to run and independent
 * of d_begin/d_end (so d-sharded ranks reproduce the 1-GPU blocks). */
int hb_assemble(const hb_mesh_desc *mesh, const hb_assembly_desc *a, void *stream);

/* Whole forward substitution (solver.py:165-184) for square blocks
 * (n x n): x[k] = inv (rhs[k] - sum_{d=1..k} A^d x[k-d]), k = 0..n_steps-1,
 * with inv = (A^0)^{-1} (or of A^0^T when transposed) supplied by the caller;
 * h_work: n doubles.  Fixed-order sums: deterministic. */
int hb_forward_solve(int64_t n_blocks, int64_t n, const double *blocks_dev, int transpose, int diagonal_only,
                     int64_t n_steps, const double *inv_dev, const double *rhs_dev, double *x_dev,
                     double *h_work_dev, void *stream);

/* The same substitution blocked in tiles of 8 steps: per tile, the history
 * terms from earlier tiles of all 8 steps in one pass over the blocks (each
 * block read once per tile), then per step only the near terms d < 8 and the
 * inverse apply -- about E_t^2 / 16 block reads instead of E_t^2 / 2.
 * workspace: hb_forward_solve_workspace(n) bytes of device memory.  The
 * transposed and diagonal-only forms run the per-step path. */
size_t hb_forward_solve_workspace(int64_t n);
/* The two history kernels of the blocked substitution on R rows (a row
 * shard) x C columns, the same per-row sums as hb_forward_solve_ws:
 * _far: H[i][r] = sum_d A^d(r, :) x[k0 + i - d] over 0 <= k0 + i - d < k0,
 *       i < nk <= 8, k0 >= 1 (H: nk x R);
 * _near: h[r] = Hk[r] (if Hk) + sum_{d=1..min(k-k0, n_blocks-1)} A^d(r, :) x[k-d],
 *       k0 <= k < k0 + 8 (the near terms of step k of its tile). */
int hb_forward_history_far(int64_t n_blocks, int64_t R, int64_t C, const double *blocks_dev, int64_t k0, int64_t nk,
                           const double *x_dev, double *H_dev, void *stream);
int hb_forward_history_near(int64_t n_blocks, int64_t R, int64_t C, const double *blocks_dev, int64_t k, int64_t k0,
                            const double *x_dev, const double *Hk_dev, double *h_dev, void *stream);
int hb_forward_solve_ws(int64_t n_blocks, int64_t n, const double *blocks_dev, int transpose, int diagonal_only,
                        int64_t n_steps, const double *inv_dev, const double *rhs_dev, double *x_dev,
                        void *workspace_dev, size_t workspace_bytes, void *stream);

/* CUDA IPC for row-parallel assembly: export a device pointer (anywhere
 * inside an allocation) as a 64-byte handle of its allocation plus the byte
 * offset; import opens the handle in this process (peer access enabled
 * lazily) and returns the pointer; close releases an imported allocation
 * (pass the pointer import returned). */
int hb_ipc_export(const void *ptr_dev, void *handle64, int64_t *offset);
int hb_ipc_import(const void *handle64, int64_t offset, void **ptr_dev);
int hb_ipc_close(void *ptr_dev, int64_t offset);

/* Pair classes exactly as the assembly kernels see them, for test rows
 * [e0, e1) and every trial element: out[(e-e0)*E_x + f] = 0 separated far,
 * 1 separated near (bumped rule), 2 identical, 3 common edge, 4 common
 * vertex -- the reference's _touching_csr + near test
 * (assembly.py:119-144, _assembly_numba.py:139-151,217-223). */
int hb_pair_classes(const hb_mesh_desc *mesh, int64_t e0, int64_t e1, int8_t *out_dev, void *stream);

/* D = D2 + alpha^2 sum_o T_o^T V T_o per block (curl of the hat functions,
 * heatbem/assembly.py:289-334).  V: (nb, E_x, E_x), D2 and D: (nb, N_x, N_x);
 * D may alias D2.  curls_dev: (E_x, 3, 3) surface curls per local hat.
 * Needs the mesh's curl tile plan; hb_curl_workspace returns 0 (the
 * workspace arguments are kept for ABI stability and may be NULL). */
size_t hb_curl_workspace(const hb_mesh_desc *mesh, int64_t blocks_per_pass);
int hb_curl_combine(const hb_mesh_desc *mesh, int64_t n_blocks, double alpha,
                    const double *curls_dev, const double *V_dev, const double *D2_dev,
                    double *D_dev, void *workspace_dev, size_t workspace_bytes, void *stream);

/* hb_curl_combine with D2 given as the sum of n_parts full-size partials
 * (parts_dev: device array of n_parts pointers to (n_blocks_total, N, N)
 * blocks; block d of this call is block part_d_offset + d of every part),
 * summed in part order -- the row-parallel ranks' p1 x p1 partials read over
 * NVLink peer memory (hb_ipc_import): the cross-rank sum of D2 and the curl
 * transform in one kernel, no collective (distributed.hypersingular_rows_peer). */
int hb_curl_combine_parts(const hb_mesh_desc *mesh, int64_t n_blocks, double alpha, const double *curls_dev,
                          const double *V_dev, int64_t n_parts, const double *const *parts_dev,
                          int64_t part_d_offset, double *D_dev, void *stream);

/* Interior potential, heatbem/_field_numba.py:15-79 (kind 0: single layer,
 * kind 1: double layer).  Evaluation outputs are grouped by spatial point and
 * time offset: group g = (gx[g], geps[g]) owns outputs gptr[g]..gptr[g+1]-1,
 * output o has k[o] completed intervals (ascending within a group), the
 * current-interval flag cur[o] (eps > 0 and k < E_t) and is written to
 * out[out_idx[o]].  The kernel values of a group are evaluated once per
 * (element, node, gap) and shared by all its output times.
 * dens_t_dev: (E_x, nq, E_t) density at the spatial quadrature nodes, time
 * fastest (the reference's (E_t, E_x, nq) array transposed);
 * qpts_dev: (E_x, nq, 3); qw_dev (nq,); kmax = max k over all outputs. */
int hb_potential(int kind, int64_t n_groups, int64_t E_t, int64_t E_x, int64_t nq,
                 const double *gx_dev, const double *geps_dev, const int64_t *gptr_dev,
                 const int64_t *k_dev, const uint8_t *cur_dev, const int64_t *out_idx_dev, int64_t kmax,
                 const double *dens_t_dev, const double *qpts_dev, const double *qw_dev,
                 const double *areas_dev, const double *normals_dev,
                 double step, double alpha, double d_eps, double r_eps, double *out_dev, void *stream);

/* Representation formula on a space-time grid (heatbem/field.py:184-190 for
 * the EvalPoints (x_i, k_j h), eps = 0): out[i][j] = V~q - W g at point x_i
 * (n_points, 3) and time k_j h (k ascending, kmax <= 64).  Both potentials in
 * one pass: the kernel values share x, the branch regions and the middle-
 * region piece.  dens_single (p0 q) and dens_double (p1 g interpolated) at the
 * quadrature nodes, (E_x, nq, E_t) time fastest, as for hb_potential. */
int hb_represent_grid(int64_t n_points, int64_t n_times, int64_t E_t, int64_t E_x, int64_t nq,
                      const double *x_dev, const int64_t *k_dev, int64_t kmax,
                      const double *dens_single_dev, const double *dens_double_dev,
                      const double *qpts_dev, const double *qw_dev, const double *areas_dev,
                      const double *normals_dev, double step, double alpha, double d_eps, double r_eps,
                      double *out_dev, void *stream);

/* hb_represent_grid for a p0 single-layer density and a p1 double-layer
 * density with the time contraction done once per ELEMENT: the kernel values
 * of the element's nq nodes are summed (weights 2 A qw and 2 A qw hat_i) before
 * the Toeplitz products, which then run on the FP64 tensor cores -- 4 products
 * per element instead of 2 nq.  dens_elem (E_x, E_t): the p0 density per
 * element; dens_vert (E_x, 3, E_t): the p1 density at each element's vertices
 * (tri_nodes order); hats (nq, 3) at the quadrature nodes; time fastest.
 * eps in [0, step): the outputs are u(x_i, k_j h + eps) -- eps > 0 is the
 * reference's current-interval case (_field_numba.py:53-76) and requires
 * k_j >= 1 (k_j = 0 outputs are written as NaN; field.py routes such points
 * through hb_potential).  kmax <= 64 for eps > 0; at time-step ends (eps = 0)
 * kmax <= 512: histories longer than 64 steps run one launch per block of 64
 * output steps, each contracting the gap windows below it as full Toeplitz
 * tiles (the reference's _eval_potential handles any k, _field_numba.py:33-76;
 * longer histories still go through hb_potential). */
int hb_represent_grid_elem(int64_t n_points, int64_t n_times, int64_t E_t, int64_t E_x, int64_t nq,
                           const double *x_dev, const int64_t *k_dev, int64_t kmax,
                           const double *dens_elem_dev, const double *dens_vert_dev, const double *hats_dev,
                           const double *qpts_dev, const double *qw_dev, const double *areas_dev,
                           const double *normals_dev, double step, double alpha, double d_eps, double r_eps,
                           double eps, double *out_dev, void *stream);

/* y^k = sum_{d<=k} A^d x^{k-d} (heatbem/solver.py:47-73).  blocks
 * (n_blocks, R, C) row-major; transpose applies A^d^T (input length R,
 * output length C); diagonal_only uses A^0 for every k (mass matrix).
 * x (n_steps, n_in), y (n_steps, n_out), n_steps <= n_blocks unless
 * diagonal_only. */
int hb_toeplitz_apply(int64_t n_blocks, int64_t R, int64_t C, const double *blocks_dev,
                      int transpose, int diagonal_only, int64_t n_steps,
                      const double *x_dev, double *y_dev, void *stream);

/* hb_toeplitz_apply with a caller workspace: operators with few output rows
 * split the tensor-core product over groups of blocks d (partial products
 * in the workspace, summed in group order -- deterministic) so that the GPU
 * is full; bytes needed from hb_toeplitz_apply_workspace (0: no split, the
 * plain hb_toeplitz_apply runs). */
size_t hb_toeplitz_apply_workspace(int64_t n_blocks, int64_t R, int64_t C, int transpose, int diagonal_only,
                                   int64_t n_steps);
int hb_toeplitz_apply_ws(int64_t n_blocks, int64_t R, int64_t C, const double *blocks_dev,
                         int transpose, int diagonal_only, int64_t n_steps, const double *x_dev,
                         double *y_dev, void *workspace_dev, size_t workspace_bytes, void *stream);

/* Partial product of a d-sharded operator: y^k = sum over the LOCAL blocks
 * d in [d_off, d_off + n_blocks), d <= k, of A^d x^{k-d}; summing y over the
 * ranks (one all-reduce) gives apply_toeplitz of the full operator. */
int hb_toeplitz_apply_range(int64_t d_off, int64_t n_blocks, int64_t R, int64_t C, const double *blocks_dev,
                            int transpose, int64_t n_steps, const double *x_dev, double *y_dev, void *stream);

/* Forward-substitution history of heatbem/solver.py:178-182 for step k:
 * acc -= sum_{d=1..k} A^d x^{k-d}, x holding the solved steps 0..k-1. */
int hb_forward_subst_step(int64_t n_blocks, int64_t R, int64_t C, const double *blocks_dev,
                          int transpose, int64_t k, const double *x_dev, double *acc_dev,
                          void *stream);

/* Row-sharded forward substitution (solver.py:178-182 on one rank's rows):
 * h[r] = sum_{d=1..min(k, n_blocks-1)} A^d(r, :) x[k-d] for the R local rows
 * of blocks (n_blocks, R, C); x (>= k, C) holds the solved steps (all
 * columns, replicated); h (R,).  k = 0 writes zeros.  Fixed-order sums. */
int hb_forward_history(int64_t n_blocks, int64_t R, int64_t C, const double *blocks_dev, int64_t k,
                       const double *x_dev, double *h_dev, void *stream);

/* x = inv (rhs - h) (h may be NULL: x = inv rhs); inv (n, n) row-major: the
 * (A^0)^{-1} step of forward_block_solve (solver.py:183). */
int hb_inv_apply(int64_t n, const double *inv_dev, const double *rhs_dev, const double *h_dev,
                 double *x_dev, void *stream);

/* Rows [r0, r1) of every block of a (n_blocks, R, C) float64 device array
 * copied into the same positions of a page-locked host array of that shape:
 * one strided asynchronous copy on `stream` (row-slab streaming of V / K,
 * assembly.py _assemble_streamed). */
int hb_copy_row_slab_d2h(double *host_dst, const double *dev_src, int64_t n_blocks, int64_t R, int64_t C,
                         int64_t r0, int64_t r1, void *stream);

/* ---- boundary data (heatbem/field.py:84-119 project_to_space, :193-215
 * relative_error_sigma) for the heat-kernel data family of the study driver
 * (ManufacturedSolution, field.py:20-44):
 *   HB_DATUM_VALUE         G_alpha(x - src, t + time_shift)        kernels.py:59-66
 *   HB_DATUM_NORMAL_DERIV  alpha dG_alpha/dn_x (x - src, t + shift) kernels.py:69-86
 * (zero for t + shift <= 0).  Tensor rule: the order-6 triangle rule
 * (qpts (E_x,nq,3), qw (nq,), hats (nq,3)) x n_tq <= 8 Gauss points per step
 * (tq, tw on [0,1]); t = i h + tq h as TimeGrid.node(i) + q h. */
#define HB_DATUM_VALUE 0
#define HB_DATUM_NORMAL_DERIV 1
typedef struct {
    int kind;
    double src[3];
    double alpha;
    double time_shift;
} hb_heat_datum;

typedef struct {
    int64_t E_x, N_x, nq;
    const double *qpts_dev, *qw_dev, *hats_dev;
    const double *areas_dev, *normals_dev;
    const int64_t *tri_nodes_dev;
    const int64_t *star_indptr_dev, *star_elem_dev, *star_local_dev;   /* node stars, as hb_mesh_desc */
    int64_t n_tq;
    double tq[8], tw[8];
} hb_data_desc;

/* L2(Sigma_h) projection of the datum: space 0 (X00) -> out (E_t, E_x),
 * space 1 (X10) -> out (E_t, N_x), the p1 mass system solved per time step by
 * Jacobi-PCG to ||r|| <= tol ||b|| (max_iter steps at most; the reference
 * factorises the dense mass matrix, field.py:106-118).  X10 needs
 * hb_project_workspace bytes; max_iters_out (optional, host) receives the
 * largest CG iteration count and makes the call synchronous. */
size_t hb_project_workspace(const hb_data_desc *data, int space, int64_t E_t);
int hb_project_data(const hb_data_desc *data, const hb_heat_datum *g, int space, int64_t E_t, double step,
                    double *out_dev, void *work_dev, size_t work_bytes, double tol, int64_t max_iter,
                    int64_t *max_iters_out, void *stream);
/* x_i = M^{-1} b_i for the p1 mass matrix (field.py:73-81), i < E_t; b, x
 * (E_t, N_x); workspace 3 E_t N_x doubles. */
int hb_p1_mass_solve(const hb_data_desc *data, int64_t E_t, const double *b_dev, double *x_dev, void *work_dev,
                     size_t work_bytes, double tol, int64_t max_iter, void *stream);
/* out2 = [sum w h 2A qw (g - u_h)^2, sum w h 2A qw g^2] over all steps,
 * elements and nodes (relative error = sqrt(out2[0] / out2[1])); coeff
 * (E_t, N_x) if p1 else (E_t, E_x); workspace 2 E_t E_x doubles.
 * Fixed-order sums (deterministic). */
int hb_error_sigma(const hb_data_desc *data, const hb_heat_datum *g, int64_t E_t, double step,
                   const double *coeff_dev, int p1, double *out2_dev, void *work_dev, size_t work_bytes,
                   void *stream);

/* FP64 DFMA throughput probe used for the roofline denominator:
 * runs `iters` dependent-chain iterations of 8 independent DFMA streams per
 * thread over grid x 256 threads; flops = grid*256*iters*8*2. */
int hb_fp64_probe(int64_t grid, int64_t iters, double *sink_dev, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* HEATBEM_B200_H */
