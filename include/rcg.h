/*
 * rcg.h — C ABI of the B200-native augmented-PCG / Ritz-recycling hot path.
 *
 * The reference ("recycg", /root/reference/pkg/src/recycg) is pure Python; its
 * drop-in seams are the module-level functions that run_sequence resolves at
 * call time.  Each entry point below replaces one of them;
 * the Python package paper_1301_7530_b200 binds these with ctypes under the
 * reference's own names (INTEGRATION.md shows the binding).
 *
 * Conventions
 *  - every pointer argument is a DEVICE pointer unless its name ends in _host;
 *  - dense matrices are column-major with an explicit leading dimension
 *    (each column — one Krylov / augmentation vector — is contiguous);
 *  - every call is asynchronous on the context's stream unless documented to
 *    synchronize; calls on one context are not thread-safe, distinct contexts
 *    are independent (no global mutable state: reference SPEC.md:179-180);
 *  - return value: RCG_OK or an error code; rcg_last_error(ctx) has the text.
 *  - reductions are deterministic (fixed-order two-stage trees, no fp64
 *    atomics), so repeated runs are bitwise identical (reference
 *    tests/test_cli.py:129-136 determinism contract).
 */
#ifndef RCG_H
#define RCG_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum rcg_status {
  RCG_OK = 0,
  RCG_ERR_CONTRACT = 1,       /* ContractViolation (core.py:18-19)          */
  RCG_ERR_RANK_DEFICIENT = 2, /* RankDeficient(column) (core.py:22-27)      */
  RCG_ERR_NUMERICAL = 3,      /* NumericalFailure (core.py:30-31)           */
  RCG_ERR_CUDA = 4,
  RCG_ERR_OOM = 5
};

/* numerical-failure kinds reported by rcg_trace_view.failure */
enum rcg_failure {
  RCG_FAIL_NONE = 0,
  RCG_FAIL_RZ = 1,  /* "(r, z) <= 0: preconditioner or operator not SPD"  solver.py:229-230,:279-280 */
  RCG_FAIL_WAW = 2  /* "(w, A w) <= 0: operator not SPD on search space"  solver.py:244-245 */
};

typedef struct rcg_ctx rcg_ctx;
typedef struct rcg_trace rcg_trace;

/* CSR operator, full symmetric pattern (SparseSpdMatrix, core.py:34-111).
 * row_offsets is int32 when row_offsets_64 == 0, else int64; col_indices int32.
 * Optional SpMV stream copies (the CSR arrays stay valid and are used by the
 * setup kernels): dia_count > 0 selects the symmetric block-DIA copy (grid
 * operators; on a row slab together with the rem_* ghost-column remainder);
 * else block == 3 selects the 3x3 block copy in bsr_* (built by
 * rcg_csr_block3_build, optionally sliced): one column index per 9 values,
 * ~29% fewer bytes for vector-valued FEM operators (BASELINE configs 2/3/5). */
typedef struct {
  int64_t n;
  int64_t nnz;
  const void* row_offsets;
  int32_t row_offsets_64;
  int32_t block;                    /* 0 = scalar CSR only, 3 = bsr_* valid */
  const int32_t* col_indices;
  const double* values;
  const int32_t* bsr_row_offsets;   /* [n/3 + 1] block-row offsets (blocks)   */
  const int32_t* bsr_col_indices;   /* [nnz/9]   block column indices         */
  const double* bsr_values;         /* [nnz]     9 per block, row-major       */
  int32_t bsr_slice;                /* 0 = plain BSR above; 32 = sliced (SELL-32
                                       over block rows): bsr_row_offsets holds
                                       [ceil(n/96)+1] chunk slot offsets,
                                       bsr_col_indices [32*slots] (-1 = pad),
                                       bsr_values [288*slots] */
  int32_t dia_count;                /* > 0: symmetric block-diagonal (DIA) copy */
  int32_t dia_block;                /* DIA unit: 1 (scalar) or 3 (3x3 blocks)  */
  int32_t rem_rows;                 /* row slabs with a DIA copy: number of rows that
                                       have ghost-column entries (0 = none)     */
  const int64_t* dia_offsets;       /* [dia_count] upper block-diagonal offsets,
                                       ascending, dia_offsets[0] = 0 (device) */
  const double* dia_values;         /* dia_count * b*b * 32*ceil(n/b/32)
                                       doubles; b = 3: entry q = i*b + jj of
                                       block (p, p + off_d) at
                                       ((d*T + p/32)*9 + q)*32 + p%32,
                                       T = ceil(n/96); b = 1: A(p, p + off_d)
                                       at d*n + p; 0 = absent */
  /* Row slabs (sharded operators, columns >= n are ghost entries): the DIA copy
   * covers the local-local block (a principal submatrix of a symmetric DIA
   * operator is one too); the ghost-column entries are kept as an entry-major
   * (ELL) list over the rows that have any and added by a second, small kernel
   * (spmv.cu rem_body). */
  const int32_t* rem_row_ids;       /* [rem_rows] local row of each listed row    */
  const int32_t* rem_col_indices;   /* [rem_width * rem_rows] extended column
                                       index of entry e of listed row s at
                                       e * rem_rows + s (pads: any valid index)  */
  const double* rem_values;         /* same layout; pads are 0                    */
  int32_t rem_width;                /* entries per listed row (max over them)     */
  int32_t pad2;
} rcg_csr;

/* Deflation operator P = I - C G^{-1} (AC)^T, G = C^T A C (DeflationOperator,
 * solver.py:63-97).  C and AC are n x n_c column-major (ld >= n); L is the
 * lower Cholesky factor of G and Ginv = G^{-1}, both n_c x n_c (ld = n_c). */
typedef struct {
  int64_t n;
  int64_t n_c;
  const double* C;
  int64_t ldc;
  const double* AC;
  int64_t ldac;
  const double* L;
  const double* Ginv;
} rcg_deflation;

/* SolveConfig (solver.py:125-139) plus the launch batch (iterations queued
 * between two host polls of the device-side convergence flag; 0 = auto) and
 * krylov_cap (extension, 0 = none): keep only z_0..z_{cap-1} — Ritz
 * extraction then runs on the leading cap x cap Lanczos block (SURVEY.md
 * §8(c) "capped variants"; config 5 "stored Krylov basis up to 400 vecs"). */
typedef struct {
  double tol;
  int64_t max_iters;
  int32_t reorthogonalize;
  int32_t trace_capture;
  int32_t store_directions;
  int32_t batch;
  int64_t krylov_cap;
} rcg_solve_cfg;

/* Read-only view of a finished solve (SolveTrace, solver.py:142-162). */
typedef struct {
  int64_t n;
  int64_t iterations;      /* m                                              */
  int64_t n_betas;         /* m-1 if converged, m if stopped by max_iters    */
  int32_t converged;
  int32_t failure;         /* enum rcg_failure                               */
  int32_t early_exit;      /* loop skipped: ||r0|| <= 1e-13 ||b|| (solver.py:217-219) */
  int32_t pad_;
  double r0_norm;
  double b_norm;
  const double* alphas;         /* [m]   device */
  const double* betas;          /* [m]   device */
  const double* rz_inner;       /* [m]   device */
  const double* residual_norms; /* [m+1] device */
  const double* Z;              /* z_0..z_{min(m,cap)-1} (trace_capture), ld  */
  const double* W;              /* w_0..w_{m-1} (reorth or store_directions)  */
  const double* AW;             /* A w_j        (reorth)                      */
  const double* R;              /* r_0..r_{m-1} (store_directions)            */
  const double* waw;            /* (w_j, A w_j) [m] (reorth)                  */
  int64_t ld;
  double device_seconds;        /* GPU time of the iteration loop            */
} rcg_trace_view;

/* Row-sharded execution (one process per GPU).  Rank `rank`
 * owns n_local contiguous rows; the CSR it passes has local column indices
 * 0..n_local-1 for owned columns and n_local.. for ghost columns, grouped by
 * owner rank.  Every SpMV-input vector has room for n_ghost entries after its
 * n_local owned entries (leading dimensions count them).  send_idx lists, per
 * peer (send_off[q]..send_off[q+1]), the local entries that peer q reads;
 * ghosts from peer q land at n_local + recv_off[q]. */
typedef struct {
  int32_t nranks;
  int32_t rank;
  int64_t n_local;
  int64_t n_ghost;
  const int32_t* send_idx;   /* device [send_off[nranks]] */
  const int64_t* send_off;   /* HOST   [nranks + 1]       */
  const int64_t* recv_off;   /* HOST   [nranks + 1]       */
  double* send_buf;          /* device [send_off[nranks]] */
} rcg_halo;

/* ---- context ------------------------------------------------------------ */
int rcg_ctx_create(int device, void* cuda_stream, rcg_ctx** out);
void rcg_ctx_destroy(rcg_ctx* ctx);
int rcg_ctx_set_stream(rcg_ctx* ctx, void* cuda_stream);
const char* rcg_last_error(const rcg_ctx* ctx);
int rcg_version(void);
int rcg_num_kernel_launches(const rcg_ctx* ctx, int64_t* out_host); /* launches issued by ctx */
/* Debug (RCG_POOL_GUARD=1 runs): re-verify every live pool buffer's canary zone and
   return the number of write-past-the-end violations seen so far (0 when the guard is off). */
int64_t rcg_debug_guard_violations(void);

/* Live per-kernel-class timing of the solve loop: when enabled, every
 * iteration kernel is bracketed by CUDA events on the ctx stream and its
 * ALGORITHMIC bytes (each operand touched once) are accounted.  Classes: */
enum rcg_kclass {
  RCG_K_SPMV = 0,      /* K1: Aw = A w, (w, Aw)                         */
  RCG_K_UPDATE = 1,    /* K2: x, r update, ||r||^2                     */
  RCG_K_COARSE = 2,    /* coarse solve (n_c > 64)                      */
  RCG_K_PRECOND = 3,   /* K3: z = P M^-1 r, (r, z), AW^T [z w] partials */
  RCG_K_COLREDUCE = 4, /* K4: reorth partial reduction                  */
  RCG_K_WUPDATE = 5,   /* K5: w = z + beta w - W c                      */
  RCG_K_ACTR = 6,      /* K2b: AC^T (M^-1 r), projector GEMV-T (n_c > 0) */
  RCG_K_HALO = 7,      /* sharded: ghost exchange of w_j (pack, NCCL send/recv, unpack) */
  RCG_K_ALLREDUCE = 8, /* sharded: packed fp64 allreduces of the reduction slots */
  RCG_K_NUM = 9
};
typedef struct {
  int64_t launches;
  double seconds;
  double bytes;
} rcg_kernel_stat;
int rcg_ctx_set_profiling(rcg_ctx* ctx, int enable);
int rcg_ctx_kernel_stats(const rcg_ctx* ctx, rcg_kernel_stat* out_host, int n); /* n <= RCG_K_NUM */
int rcg_ctx_reset_stats(rcg_ctx* ctx);

/* NCCL communicator for sharded runs.  nccl_lib may be NULL (the copy
 * already loaded in the process, else libnccl.so.2 from the loader path). */
int rcg_comm_unique_id(const char* nccl_lib, void* id_out_host /* 128 bytes */);
int rcg_comm_init(rcg_ctx* ctx, const char* nccl_lib, const void* id_host, int nranks, int rank);
int rcg_comm_destroy(rcg_ctx* ctx);
int rcg_allreduce_sum(rcg_ctx* ctx, double* buf, int64_t count);
int rcg_halo_exchange(rcg_ctx* ctx, const rcg_halo* halo, double* vec);
/* Single-process loopback transport (validation of the sharded path on one
 * GPU): `nranks` host threads, each with its own context and stream, act as
 * ranks; collectives use device copies ordered by CUDA events. */
int rcg_loop_group_create(int nranks, void** group_out_host);
void rcg_loop_group_destroy(void* group);
int rcg_comm_init_loopback(rcg_ctx* ctx, void* group, int rank);

/* ---- operators (core.py) ------------------------------------------------- */
/* y = A x  (spmv, core.py:114-119 / SparseSpdMatrix.__matmul__ core.py:110-111) */
int rcg_spmv(rcg_ctx* ctx, const rcg_csr* A, const double* x, double* y);
/* Y = A X for k column-major columns (A @ C in build_deflation, solver.py:113) */
int rcg_spmm(rcg_ctx* ctx, const rcg_csr* A, const double* X, int64_t ldx,
             int64_t k, double* Y, int64_t ldy);
/* diag(A) and 1/diag(A) (SparseSpdMatrix.diagonal core.py:103-104,
 * Preconditioner.jacobi solver.py:39-41); either output may be NULL.
 * Returns RCG_ERR_CONTRACT if a diagonal entry is missing. */
int rcg_csr_diagonal(rcg_ctx* ctx, const rcg_csr* A, double* diag, double* inv_diag);
/* Does A (scalar CSR) have exact 3x3 block structure (n % 3 == 0, rows
 * 3p..3p+2 share one column pattern made of aligned column triples)?
 * Synchronizes; *is_block3_host = 0/1. */
int rcg_csr_block3_analyze(rcg_ctx* ctx, const rcg_csr* A, int32_t* is_block3_host);
/* Build the 3x3 BSR copy: bro[n/3+1], bci[nnz/9], bval[nnz]. */
int rcg_csr_block3_build(rcg_ctx* ctx, const rcg_csr* A, int32_t* bro, int32_t* bci, double* bval);
/* Sliced 3x3 blocks from a plain BSR operator (A->block == 3, bsr_slice == 0):
 * plan writes chunk_offsets[ceil(n/96)+1] (device) and the slot count
 * (synchronizes); build fills sci[32*slots], sval[288*slots].  The result is
 * used by setting bsr_row_offsets/col_indices/values to these arrays and
 * bsr_slice = 32. */
int rcg_csr_block3_slice_plan(rcg_ctx* ctx, const rcg_csr* A, int32_t* chunk_offsets, int64_t* slots_host);
int rcg_csr_block3_slice_build(rcg_ctx* ctx, const rcg_csr* A, const int32_t* chunk_offsets,
                               int32_t* sci, double* sval);
/* ---- device assembly of the BASELINE operators (problems.py) -------------- */
/* Structured FD diffusion with harmonic face means and Dirichlet faces
 * (_assemble_diffusion, /root/reference/pkg/src/recycg/problems.py:115-156),
 * cells row-major over dims[0..ndim) (ndim 1..3).  rows: ro64[n+1] gets the
 * int64 row offsets, *nnz_host the entry count (synchronizes).  fill: column
 * indices, values and (ro32 != NULL) an int32 copy of the offsets; the bytes
 * equal the host assembler's (problems.py:assemble_diffusion). */
int rcg_gen_diffusion_rows(rcg_ctx* ctx, const int64_t* dims, int32_t ndim, int64_t* ro64, int64_t* nnz_host);
int rcg_gen_diffusion_fill(rcg_ctx* ctx, const int64_t* dims, int32_t ndim, const double* coeff,
                           const int64_t* ro64, int32_t* ro32, int32_t* ci, double* va);
/* Q1 hex elasticity on nelem^3 elements, face x = 0 clamped (problems.py:
 * elasticity_q1; no reference generator exists).  Ke: the 24x24 element
 * stiffness at E = 1 (row-major, device); E: nelem^3 per-element moduli
 * [ex][ey][ez] (device) or NULL for E = 1. */
int rcg_gen_elasticity_rows(rcg_ctx* ctx, int64_t nelem, int64_t* ro64, int64_t* nnz_host);
int rcg_gen_elasticity_fill(rcg_ctx* ctx, int64_t nelem, const double* Ke, const double* E,
                            const int64_t* ro64, int32_t* ro32, int32_t* ci, double* va);
/* Symmetric block-diagonal (DIA) copy for grid operators whose entries lie on
 * a few block diagonals (5/7-point stencils with b = 1, Q1 elasticity with
 * b = 3): only the upper diagonals are stored, A(p, p - o) = A(p - o, p)^T
 * is read from the row p - o (both streams coalesced, no column indices).
 * analyze: the distinct block offsets of the longest row, verified against
 * every entry; *nd_host = their count (0: not DIA-structured; at most 64),
 * offs_host[0..nd) ascending (synchronizes).
 * build: offs = the upper offsets (>= 0, ascending, device), nd_up of them;
 * fills U (nd_up * b*b * 32*ceil(n/b/32) doubles, layout at dia_values) and
 * checks exact symmetry (values and pattern):
 * *symmetric_host = 1 when the copy reproduces A, else 0 (do not use it). */
int rcg_csr_dia_analyze(rcg_ctx* ctx, const rcg_csr* A, int32_t b, int64_t* offs_host, int32_t* nd_host);
int rcg_csr_dia_build(rcg_ctx* ctx, const rcg_csr* A, int32_t b, const int64_t* offs, int32_t nd_up, double* U,
                      int32_t* symmetric_host);
/* elementwise y = inv_diag * x (Preconditioner.apply, solver.py:50-54) */
int rcg_diag_apply(rcg_ctx* ctx, int64_t n, const double* inv_diag, const double* x, double* y);

/* ---- dense small kernels -------------------------------------------------- */
/* G = X^T Y (a x b, ld = a); symmetrize != 0 -> G = 0.5 (G + G^T) (a == b) */
int rcg_gemm_tn(rcg_ctx* ctx, int64_t n, int64_t a, int64_t b, const double* X,
                int64_t ldx, const double* Y, int64_t ldy, double* G, int32_t symmetrize);
/* Y = X Q  (X: n x m ld ldx; Q: m x s ld ldq; Y: n x s ld ldy) */
int rcg_gemm_nn(rcg_ctx* ctx, int64_t n, int64_t m, int64_t s, const double* X,
                int64_t ldx, const double* Q, int64_t ldq, double* Y, int64_t ldy);
/* Guarded Cholesky (dense_cholesky, core.py:195-243): pivot d_j <= pivot_rtol *
 * max(d_<j), d_j <= 0 or non-finite -> RCG_ERR_RANK_DEFICIENT, *bad_col_host = j.
 * Also writes Ginv = G^{-1} when Ginv != NULL.  Synchronizes. */
int rcg_dense_cholesky(rcg_ctx* ctx, const double* G, int64_t n, double pivot_rtol,
                       double* L, double* Ginv, int64_t* bad_col_host);

/* ---- deflation (solver.py:63-117) ---------------------------------------- */
/* AC = A C; G = sym(C^T AC); L = chol(G) with pivot_rtol 1e-12; Ginv = G^{-1}.
 * RCG_ERR_RANK_DEFICIENT with *bad_col_host on a guarded pivot.  Synchronizes. */
int rcg_deflation_build(rcg_ctx* ctx, const rcg_csr* A, const double* C, int64_t ldc,
                        int64_t n_c, double* AC, int64_t ldac, double* L, double* Ginv,
                        int64_t* bad_col_host);
/* out = P x (DeflationOperator.project, solver.py:84-91) */
int rcg_project(rcg_ctx* ctx, const rcg_deflation* D, const double* x, double* out);
/* x0 = C G^{-1} C^T b (DeflationOperator.initial_guess, solver.py:93-97) */
int rcg_initial_guess(rcg_ctx* ctx, const rcg_deflation* D, const double* b, double* x0);

/* ---- APCG solve (apcg_solve, solver.py:193-290) --------------------------- */
/* inv_diag == NULL -> identity preconditioner.  x receives the solution.
 * On RCG_OK or RCG_ERR_NUMERICAL a trace is returned in *trace_out (free with
 * rcg_trace_free); the NumericalFailure kind is in its view.  Synchronizes. */
int rcg_apcg_solve(rcg_ctx* ctx, const rcg_csr* A, const double* inv_diag,
                   const rcg_deflation* D, const double* b, double* x,
                   const rcg_solve_cfg* cfg, rcg_trace** trace_out);
/* Sharded variant: A holds this rank's rows (local/ghost column numbering
 * above), b/x/inv_diag are local slices, C/AC in D are local row blocks whose
 * leading dimension has room for the ghosts.  Reductions are allreduced, so
 * every rank sees the same alpha/beta/convergence and the same trace
 * coefficients; histories are local row blocks. */
int rcg_apcg_solve_sharded(rcg_ctx* ctx, const rcg_csr* A, const double* inv_diag,
                           const rcg_deflation* D, const double* b, double* x,
                           const rcg_solve_cfg* cfg, const rcg_halo* halo, rcg_trace** trace_out);
int rcg_deflation_build_sharded(rcg_ctx* ctx, const rcg_csr* A, double* C, int64_t ldc,
                                int64_t n_c, double* AC, int64_t ldac, double* L, double* Ginv,
                                const rcg_halo* halo, int64_t* bad_col_host);
int rcg_trace_get_view(const rcg_trace* trace, rcg_trace_view* out_host);
void rcg_trace_free(rcg_trace* trace);

/* ---- Ritz extraction / selection (ritz.py:61-138, recycle.py:157-175) ----- */
/* Lanczos tridiagonal d[m], e[m-1] from CG coefficients (lanczos_tridiag,
 * ritz.py:61-78).  RCG_ERR_NUMERICAL if some beta < 0.  Synchronizes. */
int rcg_lanczos_tridiag(rcg_ctx* ctx, const double* alphas, const double* betas,
                        int64_t m, double* d, double* e);
/* All eigenvalues of the symmetric tridiagonal (d, e), descending
 * (tridiag_eig values, core.py:169-177) by Sturm bisection. */
int rcg_tridiag_eigvals(rcg_ctx* ctx, const double* d, const double* e, int64_t m,
                        double* values_desc);
/* Eigenvectors for k requested descending indices idx[k] (device int64) of
 * (d, e) whose eigenvalues values_desc are given: Q is m x k (ld m).
 * Inverse iteration with in-cluster reorthogonalization. */
int rcg_tridiag_eigvecs(rcg_ctx* ctx, const double* d, const double* e, int64_t m,
                        const double* values_desc, const int64_t* idx, int64_t k,
                        double* Q);
/* Stagnation selection (select_converged, ritz.py:103-138) on device:
 * mask[m] (uint8) from cur[m], prev[m-1] (both descending). */
int rcg_select_converged(rcg_ctx* ctx, const double* cur, const double* prev, int64_t m,
                         double epsilon, uint8_t* mask);
/* One call for select_spectrum's numeric part (recycle.py:157-175 minus the
 * cluster filter): tridiagonal from (alphas, betas), Ritz values of H_m and
 * H_{m-1}, and the stagnation mask.  values[m], prev[max(m-1,1)], mask[m].
 * Synchronizes (RCG_ERR_NUMERICAL on beta < 0). */
int rcg_ritz_select(rcg_ctx* ctx, const double* alphas, const double* betas, int64_t m,
                    double epsilon, double* d_work, double* e_work,
                    double* values, double* prev, uint8_t* mask);
/* Cluster filter (replaces ritz.py:141-183, cluster_filter): the central
 * dense cluster of the m Ritz values (device array, descending) as the value
 * index range [range_host[0], range_host[1]]; the filter keeps the indices
 * outside it.  Same scores and tie order as the reference (best three-segment
 * constant fit of the gaps; ties -> larger cluster, smaller gap level, smaller
 * start).  m < max(2, min_cluster): empty range {m, m-1}.  min_cluster < 1:
 * RCG_ERR_CONTRACT.  Synchronizes. */
int rcg_cluster_filter(rcg_ctx* ctx, const double* values, int64_t m, int64_t min_cluster,
                       int64_t* range_host);
/* Ritz vectors y_i = V q_{idx_i} with V = [(-1)^j z_j / sqrt(rz_j)] (ritz.py:
 * 81-100), scaled by 1/sqrt(|theta_i|) when scale_by_theta != 0 (the SRKS
 * block, recycle.py:151), written to Y (n x k, ld ldy).  Forms only the k
 * requested columns: one skinny Z x Qtilde GEMM. */
int rcg_ritz_vectors(rcg_ctx* ctx, const double* alphas, const double* betas,
                     const double* rz, int64_t m, const double* Z, int64_t ldz,
                     int64_t n, const double* values_desc, const int64_t* idx,
                     int64_t k, int32_t scale_by_theta, double* Y, int64_t ldy);

/* ---- TRKS block (update_basis_trks, recycle.py:127-140) ------------------ */
/* column 2-norms of X (n x k) into norms[k] */
int rcg_column_norms(rcg_ctx* ctx, int64_t n, int64_t k, const double* X, int64_t ldx,
                     double* norms);
/* sharded: 2-norms of the global columns (local sums of squares allreduced) */
int rcg_column_norms_sharded(rcg_ctx* ctx, int64_t n_local, int64_t k, const double* X, int64_t ldx,
                             double* norms);
/* Y[:, i] = X[:, i] / s[i] */
int rcg_scale_columns(rcg_ctx* ctx, int64_t n, int64_t k, const double* X, int64_t ldx,
                      const double* s, double* Y, int64_t ldy);

#ifdef __cplusplus
}
#endif
#endif /* RCG_H */
