/*
 * hessketch_b200.h -- C ABI of the B200-native sketched Hessenberg (sCMRH) /
 * sketched LSLU (sLSLU) iteration loop.
 *
 * The reference (arXiv 2502.02721 `hessketch`, pure Python) has no native
 * boundary; its hot path is reached through Python calls.  Each entry point
 * below replaces one reference interface (paths relative to
 * pkg/src/hessketch/ of the reference):
 *
 *   hs_op_dense_create      LinearOperator.from_matrix(ndarray)      linops.py:142-145
 *   hs_op_csr_create        LinearOperator.from_matrix(scipy CSR)    linops.py:137-141
 *   hs_op_psf_create        make_deblur forward/transpose closures   problems.py:257-267
 *   hs_op_tomo_create       tomography_matrix + from_matrix          problems.py:311-331, 346
 *   hs_op_apply             LinearOperator.apply / apply_transpose   linops.py:107-125
 *   hs_sketch_create        SketchOperator / make_gaussian_sketch    sketch.py:29-53
 *   hs_sketch_apply         sketch_apply                             sketch.py:56-65
 *   hs_sketch_apply_many    entries @ Q (a block of vectors)         sketch.py:108
 *   hs_pivot_select         pivot_select                             hessenberg.py:93-115
 *   hs_projected_ls         dense_qr_ls / stacked_tikhonov_ls        linops.py:168-229
 *   hs_stepper_*            init_square / step_square /              hessenberg.py:160-226,
 *                           init_generalized / step_generalized      275-390
 *   hs_solve                _hessenberg_solve                        solvers.py:410-539
 *                           via scmrh / slslu / *_tikhonov           solvers.py:562-605
 *                           and cmrh / lslu (unsketched)             solvers.py:542-559
 *   hs_solve_krylov         gmres / lsqr (comparison solvers)        solvers.py:256-403
 *   hs_result_*             SolveResult / SolverTrace / state        solvers.py:119-160,
 *                                                                    hessenberg.py:132-158, 229-272
 *
 * Conventions: plain pointers and sizes, host buffers unless a name says
 * otherwise; every function returns an hs_status and, on failure, leaves a
 * message retrievable with hs_last_error() (thread-local).  The library owns
 * all device memory; handles are released with the matching *_destroy.
 */
#ifndef HESSKETCH_B200_H
#define HESSKETCH_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  HS_OK = 0,
  HS_ERR_VALUE = 1,     /* maps to ValueError (shapes, sketch too small, ...)   */
  HS_ERR_RUNTIME = 2,   /* maps to RuntimeError                                 */
  HS_ERR_CUDA = 3,      /* CUDA runtime failure                                 */
  HS_ERR_NOTIMPL = 4,   /* maps to NotImplementedError                          */
  HS_ERR_TYPE = 5,      /* maps to TypeError                                    */
  HS_ERR_COMM = 6       /* NCCL failure                                         */
} hs_status;

typedef enum { HS_F64 = 0, HS_F32 = 1, HS_BF16 = 2 } hs_dtype;

typedef enum {
  HS_SKETCH_DENSE = 0,       /* explicit row-major ell x m matrix (e.g. PCG64 draw) */
  HS_SKETCH_GAUSSIAN = 1,    /* N(0,1/ell) generated on device from Philox, never stored */
  HS_SKETCH_SPARSE_SIGN = 2, /* zeta nonzeros +-1/sqrt(zeta) per column            */
  HS_SKETCH_CSR = 3          /* explicit sparse S (e.g. a scipy CSR via sketch=)    */
} hs_sketch_kind;

typedef enum { HS_TERM_MAXITER = 0, HS_TERM_BREAKDOWN = 1, HS_TERM_TRIVIAL = 2 } hs_termination;

typedef struct hs_ctx hs_ctx;
typedef struct hs_op hs_op;
typedef struct hs_sketch hs_sketch;
typedef struct hs_result hs_result;

/* SolverConfig (solvers.py:88-116) + device knobs */
typedef struct {
  int32_t maxiter;       /* K >= 1                                               */
  int32_t square;        /* 1: scmrh family (square Hessenberg), 0: slslu family */
  int32_t sketch_basis;  /* solvers.py:483-499 variant                           */
  int32_t work_dtype;    /* HS_F64 or HS_F32: Krylov vector arithmetic           */
  int32_t basis_dtype;   /* HS_F64 / HS_F32 / HS_BF16 storage of the bases       */
  int32_t record_x;      /* keep x of every iteration for rel_err (needs x_true) */
  double lam;            /* Tikhonov lambda >= 0                                  */
  int32_t sketched;      /* 1: scmrh / slslu family; 0: unsketched cmrh / lslu
                            (solvers.py:542-559: min |H y - beta e1|, + lam^2 |y|^2;
                            S2 / S1 must then be NULL)                            */
  int32_t pivot_sample;  /* 0: full pivoting; s > 0: PivotStrategy.sampled(s)
                            (hessenberg.py:93-124)                                */
  /* pivot_sample > 0: the positions rng.choice(pop, s, replace=False) drawn by
     the host for each selection, row-major [slot][s]; slot 0 = r0, then
     square: slot k = step k; rectangular: slot 1 = A^T r0, slots 2k / 2k+1 =
     step k data / solution side.  Slots whose population (dim - k) is <= s
     are not read (full scan, no draw), exactly as the reference skips the
     draw.  Positions index the swap-ordered admissible list t[k:] / g[k:]
     (hessenberg.py:127-129), which the device maintains.                   */
  const int64_t* pivot_positions;
  int32_t diagnostics;   /* compute_diagnostics (solvers.py:523-532): exact
                            residual |b - A x_k| (hs_result_resnorm); Hessenberg
                            solvers also kappa_basis, kappa_dbar, eps_embed
                            (hs_result_diagnostics); serialises the loop      */
  int32_t printed_f;     /* slslu_tikhonov(printed_f_columns=True) comparison
                            variant: penalty columns S1 (A^T d_{k+1}) before the
                            elimination (solvers.py:460-461, 488-490)          */
} hs_config;

const char* hs_last_error(void);
/* per-kernel CUDA-event statistics (bench / roofline): launches, ms, algorithmic bytes */
int hs_ctx_set_profiling(hs_ctx* ctx, int on);
int hs_ctx_reset_stats(hs_ctx* ctx);
int hs_ctx_kernel_stats(hs_ctx* ctx, const char* name, int64_t* launches, double* ms, double* bytes);
int hs_ctx_kernel_names(hs_ctx* ctx, char* buf, int64_t cap);
const char* hs_version(void);
/* number of CUDA kernels this library has launched in this process */
unsigned long long hs_launch_count(void);
/* HS_GUARD=1: buffers released with a changed guard band (out-of-bounds writes) */
unsigned long long hs_guard_violations(void);

/* context: one CUDA device, one stream */
int hs_ctx_create(int device, hs_ctx** out);
int hs_ctx_destroy(hs_ctx* ctx);
int hs_ctx_synchronize(hs_ctx* ctx);

/* multi-GPU: NCCL communicator over `nranks` processes (one per GPU) */
int hs_comm_get_unique_id(void* out_128_bytes);
int hs_comm_init(hs_ctx* ctx, int nranks, int rank, const void* unique_id_128_bytes);
/* runs every NCCL call the sharded loops make (all-gather, fp64 all-reduce,
   grouped send/recv) on a throwaway one-rank communicator and checks the
   results: verifies the run-time NCCL bindings on a single GPU */
int hs_nccl_selftest(hs_ctx* ctx);
int hs_comm_info(const hs_ctx* ctx, int32_t* nranks, int32_t* rank);
/* in-process ranks: contexts ctxs[0..nranks) become ranks 0..nranks-1 of one
   communicator whose collectives are stream-ordered device copies between the
   contexts (one host thread per rank drives its solve).  Same partition and
   message sequence as the NCCL path; used to run P-rank solves on one GPU. */
int hs_comm_init_local(hs_ctx** ctxs, int nranks);
/* release every in-process rank blocked in (or entering) a collective: they fail with HS_ERR_COMM */
int hs_comm_abort(hs_ctx* ctx);
/* test hook: build operators / run solves through the sharded path with one rank */
int hs_ctx_force_sharding(hs_ctx* ctx, int on);
/* after hs_comm_init with nranks > 1, hs_op_tomo_create builds only this
   rank's rows of A (rays) and of A^T (image rows); hs_solve then runs the
   row-sharded loop and returns the full x on every rank */
int hs_op_shard_info(const hs_op* op, int64_t* m_off, int64_t* m_loc, int64_t* m_blk, int64_t* n_off,
                     int64_t* n_loc, int64_t* n_blk);

/* operators: m x n, value dtype HS_F64/HS_F32 (values are uploaded once) */
int hs_op_dense_create(hs_ctx* ctx, int64_t m, int64_t n, const void* M_rowmajor, int vdtype, hs_op** out);
int hs_op_csr_create(hs_ctx* ctx, int64_t m, int64_t n, int64_t nnz, const int64_t* indptr,
                     const int32_t* indices, const void* data, int vdtype, hs_op** out);
int hs_op_psf_create(hs_ctx* ctx, int64_t height, int64_t width, int32_t kh, int32_t kw,
                     const double* kernel, int vdtype, hs_op** out);
/* parallel-beam tomography built on device; cos/sin/offsets computed by the
   caller exactly as problems.py:317-322 (math.cos/math.sin of pi*a/n_angles,
   j + 0.5 - n_bins/2) so every chord length is bit-identical to the reference */
int hs_op_tomo_create(hs_ctx* ctx, int32_t grid, int32_t n_angles, int32_t n_bins, const double* cos_t,
                      const double* sin_t, const double* offsets, int vdtype, hs_op** out);
int hs_op_info(const hs_op* op, int64_t* m, int64_t* n, int64_t* nnz, int64_t* nnz_t);
/* storage of the SELL copy one direction runs on (no reference counterpart: the
   reference keeps scipy CSR, linops.py:137-141): slices, entry slots (with
   padding), slices / slots on compact step codes (2-bit for A, 8-bit for A^T),
   and the stored index bytes per nonzero (4 int32, 2 deltas, 1 or 0.25 codes,
   averaged over the slices).  Zeros for operators without a SELL copy. */
int hs_op_storage(const hs_op* op, int transpose, int64_t* slices, int64_t* slots, int64_t* code_slices,
                  int64_t* code_slots, double* index_bytes_per_nnz);
/* y = A x (transpose = 0) or A^T x (transpose = 1); x, y host float64 or float32 (= work dtype) */
int hs_op_apply(hs_op* op, int transpose, int work_dtype, const void* x, void* y);
/* copy the device CSR (transpose selects A^T) to host buffers (data as float64) */
int hs_op_export_csr(hs_op* op, int transpose, int64_t* indptr, int32_t* indices, double* data);
int hs_op_destroy(hs_op* op);

/* sketches: ell x in_rows; `entries` (row-major, float64) only for HS_SKETCH_DENSE */
int hs_sketch_create(hs_ctx* ctx, int kind, int64_t ell, int64_t in_rows, uint64_t seed, int32_t zeta,
                     const double* entries, hs_sketch** out);
int hs_sketch_create_csr(hs_ctx* ctx, int64_t ell, int64_t in_rows, int64_t nnz, const int64_t* indptr,
                         const int32_t* indices, const double* data, hs_sketch** out);
int hs_sketch_apply(hs_sketch* sk, int work_dtype, const void* v, double* out);
/* out[w*ell + i] = (S v_w)_i for nv vectors stored one after another (v[w*in_rows + c]);
 * a Gaussian sketch generates S once per batch of up to 8 vectors.  Each column
 * is bit-identical to hs_sketch_apply of that vector. */
int hs_sketch_apply_many(hs_sketch* sk, int work_dtype, int32_t nv, const void* v, double* out);
/* dense export (row-major ell x in_rows float64) */
int hs_sketch_materialize(hs_sketch* sk, double* out);
/* sparse-sign export as CSR (ell rows): indptr[ell+1], indices[nnz], data[nnz] */
int hs_sketch_nnz(hs_sketch* sk, int64_t* nnz);
int hs_sketch_export_csr(hs_sketch* sk, int64_t* indptr, int32_t* indices, double* data);
int hs_sketch_destroy(hs_sketch* sk);

/* step-level API (hessenberg.py:160-226 init_square / step_square,
 * 275-390 init_generalized / step_generalized): the state stays on the device
 * between calls.  `positions` (sampled pivoting only, else NULL): the host's
 * rng.choice draws for this call's selection slots, [slot][pivot_sample], one
 * slot (square) or two (rectangular: data side, then solution side).  When the
 * starting residual (or A^T r0) is zero, *trivial is set to 1 (or 2) and no
 * stepper is returned (the reference's TrivialSolution). */
/* pivot_select (hessenberg.py:93-115): largest |v| over the candidate rows
 * cand[ncand] (the sampled subset already drawn by the host, or the full
 * admissible set), ties -> smallest row index; all candidates zero ->
 * (min(cand), 0.0).  v host float64 of length n. */
int hs_pivot_select(hs_ctx* ctx, int64_t n, const double* v, int64_t ncand, const int64_t* cand, int64_t* idx,
                    double* val);
/* dense_qr_ls (linops.py:168-207): min |M y - rhs| for an l x k column-major
 * M (l >= k) with the loop's incremental QR; y = the minimum-norm solution
 * when the 1e-14 rank gate fires, *rank = k - dependent columns (the caller
 * raises RankDeficiencyError when *rank < k).  stacked_tikhonov_ls
 * (linops.py:210-229) is this on [M; lam N] with rhs [rhs; 0]. */
int hs_projected_ls(hs_ctx* ctx, int64_t l, int32_t k, const double* M, const double* rhs, double* y, int32_t* rank);
typedef struct hs_stepper hs_stepper;
int hs_stepper_create(hs_ctx* ctx, hs_op* op, int32_t square, int32_t work_dtype, int32_t basis_dtype,
                      int32_t capacity, const double* b, const double* x0, int32_t pivot_sample,
                      const int64_t* positions, int32_t* trivial, hs_stepper** out);
/* one step; HS_ERR_RUNTIME after a breakdown (hessenberg.py:201-202, 338-339) */
int hs_stepper_step(hs_stepper* sp, int32_t keep_products, const int64_t* positions);
int hs_stepper_info(const hs_stepper* sp, int32_t* k, int32_t* breakdown, int32_t* bd_side, int32_t* n_basis_sol,
                    int32_t* n_basis_data, double* beta, double* alpha);
/* H: (k+1) x k column-major; W: n_basis_data^2 column-major (rectangular) */
int hs_stepper_hessenberg(hs_stepper* sp, double* H, double* W);
/* pivot positions in selection order: t[n_basis_data], g[n_basis_sol] */
int hs_stepper_pivots(hs_stepper* sp, int64_t* t, int64_t* g);
/* basis column j (which: 0 = L, 1 = D) as float64 */
int hs_stepper_basis(hs_stepper* sp, int32_t which, int32_t j, double* out);
/* unreduced products of the last keep_products step: 0 = A l_k (m), 1 = A^T d_{k+1} (n) */
int hs_stepper_product(hs_stepper* sp, int32_t which, double* out);
int hs_stepper_r0(hs_stepper* sp, double* out);
int hs_stepper_destroy(hs_stepper* sp);

/* the solve: b[m], x0[n] or NULL, x_true[n] or NULL (host float64).
   Sketched: S2 required, S1 required iff cfg->lam > 0.  Unsketched: both NULL. */
int hs_solve(hs_ctx* ctx, hs_op* op, const hs_config* cfg, hs_sketch* S2, hs_sketch* S1, const double* b,
             const double* x0, const double* x_true, hs_result** out);

/* the reference's comparison solvers (solvers.py:256-403): method 0 = gmres
   (square), 1 = lsqr; cfg: maxiter, work_dtype, record_x, lam (others
   ignored).  The result has no bases / pivots; its "Hessenberg" accessor
   returns the projected matrix (Arnoldi H or bidiagonal B, (k+1) x k). */
int hs_solve_krylov(hs_ctx* ctx, hs_op* op, const hs_config* cfg, int32_t method, const double* b, const double* x0,
                    const double* x_true, hs_result** out);

/* result accessors */
int hs_result_info(const hs_result* r, int32_t* n_records, int32_t* termination, int32_t* k,
                   int32_t* breakdown_side, int32_t* n_basis_data, int32_t* n_basis_sol);
int hs_result_x(const hs_result* r, double* x);                 /* n */
/* per record |b - A x_k| when cfg->diagnostics was set, else NaN */
int hs_result_resnorm(const hs_result* r, double* out);
/* per record kappa_basis, kappa_dbar (lam > 0), eps_embed (sketched, column
   sketching) when cfg->diagnostics was set (Hessenberg solvers), else NaN */
int hs_result_diagnostics(const hs_result* r, double* kappa_basis, double* kappa_dbar, double* eps_embed);
/* per record: sres_norm, proj_obj, rel_err (NaN if no x_true), rank_fallback,
   counters (matvecs, tmatvecs, dots, sketches), wall_ms (device events) */
int hs_result_trace(const hs_result* r, double* sres, double* proj, double* relerr, int32_t* rank_fallback,
                    int64_t* matvecs, int64_t* tmatvecs, int64_t* dots, int64_t* sketches, double* wall_ms);
int hs_result_pivots(const hs_result* r, int64_t* t, int64_t* g);  /* n_basis_data / n_basis_sol */
/* H: (k+1) x k column-major; W: n_basis_data x n_basis_data column-major (rectangular only) */
int hs_result_hessenberg(const hs_result* r, double* H, double* W);
/* basis column j: which = 0 -> L (n), 1 -> D (m); values as float64 */
int hs_result_basis(const hs_result* r, int which, int32_t j, double* out);
/* sketched quantities: Z (ell x k), sr0 (ell), y (k) */
int hs_result_projected(const hs_result* r, double* Z, double* sr0, double* y);
int hs_result_loop_ms(const hs_result* r, double* ms);
int hs_result_destroy(hs_result* r);

#ifdef __cplusplus
}
#endif

#endif /* HESSKETCH_B200_H */
