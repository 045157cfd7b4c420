/*
 * adrom_b200.h — C-ABI of the B200-native adaptive-ROM online loop.
 *
 * The reference (`adrom`, /root/reference/pkg/src/adrom) is a pure-Python
 * package; its "plugin boundary" for this path is the Python API listed in
 * SURVEY.md §8b.  Each entry point below replaces one reference function
 * (cited file:line) and is what a ctypes / cffi binding of the reference
 * would call (INTEGRATION.md shows the binding).
 *
 * Conventions
 *   - Every array argument is a DEVICE pointer (CUDA global memory, fp64,
 *     C / row-major like numpy), unless its name starts with `host_`.
 *   - State vectors use the reference layout q[cell * n_var + var]
 *     (fom.py:4-5).  Bases are N x r row-major (phi[i * r + j]).
 *   - Calls are enqueued on the context's stream.  Functions that return
 *     scalar results through `host_*` pointers synchronise that stream.
 *   - Inputs are never modified unless documented (reference ownership
 *     rule).
 *   - Status codes map to the reference's exceptions in the Python layer:
 *       ADROM_ERR_NONFINITE / ADROM_ERR_SINGULAR / ADROM_ERR_NOCONV /
 *       ADROM_ERR_DENSE            -> adrom.dense.DenseError (dense.py:35)
 *       ADROM_ERR_ROMSTEP          -> adrom.projection.RomStepError (projection.py:37)
 *       ADROM_ERR_ARG              -> ValueError
 *     Non-convergence of Newton / Gauss-Newton is a FLAG in the result,
 *     never an error (dense.py:170-171, projection.py:202-204).
 */
#ifndef ADROM_B200_H
#define ADROM_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ADROM_ABI_VERSION 2

enum adrom_status {
  ADROM_OK = 0,
  ADROM_ERR_NONFINITE = 1, /* dense._require_finite (dense.py:39-43)            */
  ADROM_ERR_SINGULAR = 2,  /* singular Jacobian / rank deficiency (dense.py:163) */
  ADROM_ERR_ROMSTEP = 3,   /* RomStepError (projection.py:193-198)               */
  ADROM_ERR_ARG = 4,       /* ValueError                                         */
  ADROM_ERR_CUDA = 5,      /* CUDA runtime failure                               */
  ADROM_ERR_NOCONV = 6,    /* SVD did not converge (dense.py:66-71)              */
  ADROM_ERR_DENSE = 7      /* other DenseError (e.g. tol <= 0, dense.py:150)     */
};

enum adrom_model_kind {
  ADROM_BURGERS = 1, /* fom.BurgersProblem (fom.py:161-201): periodic, n_var=1 */
  ADROM_SOD = 2,     /* fom.SodProblem (fom.py:249-282): zero-gradient, n_var=3 */
  ADROM_REACTING = 3 /* configuration-4 reacting Euler (no reference code, SPEC.md:8;
                        defined by oracle/reacting.py): periodic, n_var=13.
                        Every entry point below accepts it.                */
};

/* Physics + grid of one full-order model (replaces the FomProblem instance). */
typedef struct adrom_model {
  int32_t kind;   /* adrom_model_kind                              */
  int32_t n_var;  /* 1 (Burgers), 3 (Sod) or 13 (reacting)         */
  int64_t n_elem; /* number of cells                               */
  double dx;      /* length / n_elem (fom.py:74)                   */
  double nu;      /* Burgers viscosity (fom.py:173)                */
  double gamma;   /* Euler specific-heat ratio (fom.py:260)        */
  const double* mech; /* ADROM_REACTING: device array 5 x 12 (a, b, A, Ta, q
                         per reaction); NULL otherwise                 */
} adrom_model;

typedef struct adrom_ctx adrom_ctx;

/* ---- context ----------------------------------------------------------- */
int adrom_abi_version(void);
/* `stream` is a cudaStream_t (NULL = legacy default stream). */
int adrom_ctx_create(adrom_ctx** out, void* stream);
int adrom_ctx_set_stream(adrom_ctx* ctx, void* stream);
void adrom_ctx_destroy(adrom_ctx* ctx);
const char* adrom_ctx_last_error(const adrom_ctx* ctx);
int adrom_ctx_synchronize(adrom_ctx* ctx);
/* number of kernels this context has launched (bench.py's gpu_launches) */
int64_t adrom_ctx_launch_count(const adrom_ctx* ctx);

/* ---- timing probes ----------------------------------------------------- */
/* CUDA-event probes around the library's kernels on the context stream
 * (used by bench.py to time the dominant kernel inside the timed region). */
enum adrom_probe {
  ADROM_PROBE_ISVD_ROTATE = 0, ADROM_PROBE_ISVD_PROJECT = 1, ADROM_PROBE_ISVD_RESID = 2,
  ADROM_PROBE_ISVD_CORE = 3, ADROM_PROBE_FOM_RESIDUAL = 4, ADROM_PROBE_FOM_JACOBIAN = 5,
  ADROM_PROBE_FOM_SOLVE = 6, ADROM_PROBE_QDEIM_ROUND = 7, ADROM_PROBE_ROM_STEP = 8,
  ADROM_PROBE_DECODE = 9, ADROM_PROBE_OPERATOR = 10, ADROM_PROBE_ENCODE = 11,
  ADROM_PROBE_COUNT = 16
};
int adrom_prof_enable(adrom_ctx* ctx, int enable);
/* host_ms[ADROM_PROBE_COUNT], host_count[ADROM_PROBE_COUNT]; resets probes */
int adrom_prof_read(adrom_ctx* ctx, double* host_ms, int32_t* host_count);

/* ---- full-order residual (kernel 1) ------------------------------------ */
/* f = model.rhs(q)  — BurgersProblem.rhs fom.py:180-188, SodProblem.rhs
 * fom.py:265-269.  Bitwise equal to the reference (no FMA contraction). */
int adrom_rhs(adrom_ctx* ctx, const adrom_model* m, const double* q, double* f);

/* out[k, n_var] = model.rhs_at_cells(gathered[k, 3, n_var])
 * — fom.py:190-198 / fom.py:271-277. */
int adrom_rhs_at_cells(adrom_ctx* ctx, const adrom_model* m, const double* gathered,
                       int64_t k, double* out);

/* ---- sampled residual (kernel 2) --------------------------------------- */
/* SamplingPlan.evaluate (fom.py:154-158), batched over n_dir directions:
 *   values_d = closure_values + h[d] * dirs[:, d]   (d < n_dir; dirs is
 *              n_closure x ld_dirs row-major, column d used), or
 *   values   = closure_values                       (n_dir == 0, h/dirs NULL)
 *   out[d * n_s + j] = rhs_at_cells(values_d[gather])[out_cell[j], out_var[j]]
 * gather: n_cells x 3 x n_var closure positions; out_cell/out_var: n_s. */
int adrom_plan_evaluate(adrom_ctx* ctx, const adrom_model* m, const int64_t* gather,
                        int64_t n_cells, const int64_t* out_cell, const int64_t* out_var,
                        int64_t n_s, const double* closure_values, const double* h,
                        const double* dirs, int64_t ld_dirs, int32_t n_dir, double* out);

/* ---- banded FD Jacobian + backward-Euler Newton ------------------------ */
/* blocks[n_elem, 3, n_var, n_var]: d rhs_i / d q_{left(i)}, d q_i,
 * d q_{right(i)} — the nonzero entries of fd_jacobian (fom.py:301-328),
 * bitwise.  f0 may be NULL (recomputed). */
int adrom_fd_jacobian_blocks(adrom_ctx* ctx, const adrom_model* m, const double* q,
                             double* blocks);

typedef struct adrom_newton_info {
  int32_t converged;     /* NewtonResult.converged   (dense.py:134-137) */
  int32_t iterations;    /* NewtonResult.iterations                    */
  double residual_norm;  /* NewtonResult.residual_norm                 */
} adrom_newton_info;

/* x = implicit_step(model, q, dt).x  — fom.py:331-347 with
 * dense.newton_solve (dense.py:140-171): absolute tol on ||r||_2, at most
 * max_iter updates.  The linear solve is a block-tridiagonal (cyclic for
 * periodic) partitioned solver instead of dense LU.  coarse_step (fom.py:350)
 * is this call with dt = z * dt.  Blocking (fills host_info). */
int adrom_implicit_step(adrom_ctx* ctx, const adrom_model* m, const double* q, double dt,
                        double tol, int32_t max_iter, double* x, adrom_newton_info* host_info);

/* ---- tall-skinny projections (kernel 3) -------------------------------- */
/* out[r] = phi^T x                 (phi N x r)  — projection.py:99 core   */
int adrom_project(adrom_ctx* ctx, const double* phi, const double* x, int64_t n,
                  int32_t r, double* out);
/* a = phi^T (d * (q - q_ref))      — encode, projection.py:96-99 with
 * ScalingTransform.preprocess snapshots.py:47-48 (d = row_scale)          */
int adrom_encode(adrom_ctx* ctx, const double* phi, const double* q_ref, const double* d,
                 const double* q, int64_t n, int32_t r, double* a);
/* q = q_ref + (phi a) / d          — decode, projection.py:102-104 with
 * ScalingTransform.lift snapshots.py:50-51                                 */
int adrom_decode(adrom_ctx* ctx, const double* phi, const double* q_ref, const double* d,
                 const double* a, int64_t n, int32_t r, double* q);

/* ---- diagnostics ------------------------------------------------------- */
/* dev_out[v] = relative_error(primitive_fields(pred)[v], primitive_fields(truth)[v])
 * for every variable v of the model — driver.py:168-175 (relative_error) and
 * driver.py:185-199 (_per_variable_errors / _error_history); primitive fields
 * fom.py:200-201 and fom.py:204-210 / 279-282.  pred, truth: device states. */
int adrom_state_errors(adrom_ctx* ctx, const adrom_model* m, const double* pred,
                       const double* truth, double* dev_out);

/* ---- incremental SVD (kernel 4) ---------------------------------------- */
typedef struct adrom_isvd_info {
  double qnorm;          /* ||q|| (tracking.py:163)                          */
  double ynorm;          /* ||y_hat|| (tracking.py:164)                      */
  double proj_resid;     /* ||y - Phi Phi^T y|| (driver.py:366-367 diag)     */
  int32_t degenerate;    /* took the in-span branch (tracking.py:169-170)    */
  int32_t reorthogonalised; /* explicit residual pass was run                */
  int32_t sweeps;        /* Jacobi sweeps of the core SVD (0: secular path)  */
  int32_t core_path;     /* core SVD: 0 secular equation, 1 Jacobi on K,
                            2 Jacobi on K^T (fallbacks)                      */
} adrom_isvd_info;

/* isvd_update (tracking.py:141-178):
 *   p = Phi^+ y (gelsd least squares), q = y - Phi p,
 *   phi_out = [phi, q/||q||] U_core[:, :r],  sigma_out = s_core[:r]
 * phi: n x r_cur, phi_out: n x r (may alias phi when r == r_cur).
 * gram: optional device r_cur x r_cur matrix holding phi^T phi on entry and
 * phi_out^T phi_out on exit (tracked across a stream of updates; NULL =
 * computed afresh, one extra N r^2 pass).  The least-squares coefficients
 * use it exactly like gelsd uses the basis' actual (not assumed) Gram.
 * host_info may be NULL (then the call does not synchronise). */
int adrom_isvd_update(adrom_ctx* ctx, const double* phi, const double* sigma,
                      const double* y_hat, int64_t n, int32_t r_cur, int32_t r, double lam,
                      double* phi_out, double* sigma_out, double* gram,
                      adrom_isvd_info* host_info);
/* Streaming iSVD (B200 extension, r in {32, 64}): the basis is kept factored,
 * Phi = [A | Q] W (csrc/factored.cu), so an update costs two passes over the
 * basis and O(r^3) work instead of the O(N r^2) rotation of adrom_isvd_update;
 * after 16 updates the anchor A = [A | Q] W is rebuilt on the tensor cores.
 * Each update is mathematically tracking.py:141-178; a failed update leaves
 * the stream unchanged.  read() materialises Phi (n x r). */
typedef struct adrom_isvd_stream adrom_isvd_stream;
int adrom_isvd_stream_create(adrom_ctx* ctx, int64_t n, int32_t r, adrom_isvd_stream** out);
void adrom_isvd_stream_destroy(adrom_isvd_stream* s);
int adrom_isvd_stream_load(adrom_isvd_stream* s, const double* phi, const double* sigma);
int adrom_isvd_stream_update(adrom_isvd_stream* s, const double* y_hat, double lam,
                             adrom_isvd_info* host_info);
int adrom_isvd_stream_read(adrom_isvd_stream* s, double* phi_out, double* sigma_out);

/* gram = phi^T phi (device r x r) */
int adrom_gram(adrom_ctx* ctx, const double* phi, int64_t n, int32_t r, double* gram);

/* thin_svd of a small dense matrix (dense.py:59-72), m x n row-major with
 * m, n <= 256, one thread block: u (m x k), s (k), v (n x k), k = min(m,n). */
int adrom_small_svd(adrom_ctx* ctx, const double* a, int32_t m, int32_t n, double* u,
                    double* s, double* v);

/* ---- tall-skinny FP64 tensor-core products (B200 extension) ------------ */
/* No reference counterpart: numpy's `a.T @ b` / `a @ m` inside least_squares,
 * orth, direct_update (dense.py:100-111, :175-179; tracking.py:201-213) and the
 * large-sample DEIM pseudo-inverse (sampling.py:162-175).  DMMA (mma.sync
 * m8n8k4 f64), deterministic split-K.
 * adrom_ts_tn:    C (m x n, COLUMN-major: C[i + m c]) = A^T B, A row-major
 *                 K x m (A[k lda + i]) or, if a_kmajor, A[i lda + k]; B row-major
 *                 K x n.  m <= 128, n <= 136.
 * adrom_ts_apply: out = A M, A row-major K x m, M row-major m x n; out row-major
 *                 K x n (out[k ldo + c]) or, if out_kmajor, out[c ldo + k].
 *                 m <= 128, n <= 136.  All pointers device memory. */
int adrom_ts_tn(adrom_ctx* ctx, int64_t K, int32_t m, int32_t n, const double* A, int64_t lda,
                int32_t a_kmajor, const double* B, int64_t ldb, double* C);
int adrom_ts_apply(adrom_ctx* ctx, int64_t K, int32_t m, int32_t n, const double* A, int64_t lda,
                   const double* M, double* out, int64_t ldo, int32_t out_kmajor);

/* ---- offline stage and dense helpers ---------- */
/* fit_scaling (snapshots.py:54-69): training is m snapshots of n_dof values
 * (row-major m x n_dof, device); q_ref = training[0], phi_norm[n_var] the
 * per-variable mean squared fluctuation with the 1e-30 floor -> 1. */
int adrom_fit_scaling(adrom_ctx* ctx, const double* training, int32_t m, int64_t n_dof,
                      int32_t n_var, double* q_ref, double* phi_norm);
/* pod(preprocess(training), r) (snapshots.py:72-89 with :48-49): Householder
 * QR + one-sided Jacobi SVD on the device, fix_column_signs (dense.py:182).
 * phi: n_dof x r row-major, sigma: r, s_all: min(m, n_dof) singular values
 * (optional), rank: numerical rank (s > 1e-12 s_0).  r > rank ->
 * ADROM_ERR_DENSE (snapshots.py:86-87). */
int adrom_pod_window(adrom_ctx* ctx, const double* training, int32_t m, int64_t n_dof,
                     int32_t n_var, const double* q_ref, const double* phi_norm, int32_t r,
                     double* phi, double* sigma, double* s_all, int32_t* rank);
/* pod(snapshots, r) (snapshots.py:72-89): y is n x m row-major (one snapshot
 * per column). */
int adrom_pod(adrom_ctx* ctx, const double* y, int64_t n, int32_t m, int32_t r, double* phi,
              double* sigma, double* s_all, int32_t* rank);
/* orth (dense.py:175-179): thin-QR Q of a (n x m row-major, n >= m) with the
 * deterministic column signs; q: n x m row-major. */
int adrom_orth(adrom_ctx* ctx, const double* a, int64_t n, int32_t m, double* q);
/* least_squares (dense.py:100-111): minimum-norm x (k x nb row-major) of
 * ||a x - b|| for a (n x k row-major, n >= k) and b (n x nb row-major),
 * singular values below 1e-12 s_max discarded (gelsd semantics). */
int adrom_least_squares(adrom_ctx* ctx, const double* a, int64_t n, int32_t k, const double* b,
                        int32_t nb, double* x);
/* the LU step of newton_solve (dense.py:160-168): A x = b by LU with partial
 * pivoting, A (n x n row-major) and b overwritten (b -> x); an exactly zero
 * pivot -> ADROM_ERR_SINGULAR. */
int adrom_lu_solve(adrom_ctx* ctx, double* a, int64_t n, double* b);
/* rusanov_flux (fom.py:222-236) on n interface pairs of conserved triplets
 * (ul, ur, out: n x 3 row-major). */
int adrom_rusanov_flux(adrom_ctx* ctx, const double* ul, const double* ur, int64_t n,
                       double gamma, double* out);

/* ---- hyper-reduction sampling + reduced operator ----------------------- */
/* qdeim_sample (sampling.py:107-114): first n_s pivots of the restarted
 * column-pivoted QR of phi^T (exact greedy, ties to the lowest row).
 * idx: device int64[n_s]. Blocking. */
int adrom_qdeim(adrom_ctx* ctx, const double* phi, int64_t n, int32_t r, int32_t n_s,
                int64_t* idx);

/* fgs_sample (sampling.py:117-159): QDEIM rows for n_s - n_extra, then the
 * cells with the largest |grad feature(y_corr)| (feature 0 = pressure-,
 * 1 = velocity-gradient), all variables, skipping duplicates. Blocking. */
int adrom_fgs(adrom_ctx* ctx, const adrom_model* m, const double* phi, int32_t r,
              const double* y_corr, int32_t n_s, int32_t n_extra, int32_t feature,
              int64_t* idx);

/* build_deim_operator (sampling.py:162-175): pinv = (phi[idx, :])^+, r x n_s
 * row-major; rank deficiency (s_min <= 1e-12 s_max) -> ADROM_ERR_SINGULAR. */
int adrom_deim_operator(adrom_ctx* ctx, const double* phi, int64_t n, int32_t r, const int64_t* idx,
                        int32_t n_s, double* pinv);

/* Device-resident reduced operator (projection.py:57-87 RomOperator +
 * fom.py:119-158 SamplingPlan).  All pointers are device buffers allocated
 * by the caller with the listed capacities; sizes[] is written by the build:
 * sizes[0] = n_s, sizes[1] = closure length, sizes[2] = sampled cells. */
typedef struct adrom_rom_op {
  int32_t r, n_var;
  int32_t ns_cap;     /* >= n_s                                  */
  int32_t nc_cap;     /* >= 3 * n_s * n_var  (closure rows)       */
  int32_t ncell_cap;  /* >= n_s                                  */
  int32_t pad;
  int64_t* idx;        /* [ns_cap] sampled rows, sampling order      */
  int64_t* closure;    /* [nc_cap] sorted closure rows               */
  int64_t* gather;     /* [ncell_cap * 3 * n_var] closure positions  */
  int64_t* out_cell;   /* [ns_cap]                                  */
  int64_t* out_var;    /* [ns_cap]                                  */
  int64_t* sample_pos; /* [ns_cap]                                  */
  int32_t* sizes;      /* [4]                                       */
  double* pinv;        /* [r * ns_cap] (P^T Phi)^+, row-major r x n_s */
  double* d_s;         /* [ns_cap]                                  */
  double* q_ref_c;     /* [nc_cap]                                  */
  double* dinv_phi_c;  /* [nc_cap * r]                              */
  double* phi_s;       /* [ns_cap * r]                              */
} adrom_rom_op;

/* stencil_closure (sampling.py:178-189) + build_rom_operator
 * (projection.py:61-80, build_deim_operator sampling.py:162-175) for the
 * rows op->idx[0..n_s) (copied from `idx` if non-NULL).  Blocking. */
int adrom_rom_operator_build(adrom_ctx* ctx, const adrom_model* m, const double* phi, int64_t n,
                             const double* q_ref, const double* d, const int64_t* idx,
                             int32_t n_s, adrom_rom_op* op);

typedef struct adrom_rom_step_info {
  int32_t converged;   /* RomStepResult.converged (projection.py:50-54) */
  int32_t iterations;
  double residual_norm;
} adrom_rom_step_info;

/* rom_step (projection.py:217-221): kind 0 = lspg_step (158-204),
 * 1 = galerkin_step (111-147).  a_out may alias a_prev.  Blocking. */
int adrom_rom_step(adrom_ctx* ctx, const adrom_model* m, const adrom_rom_op* op, int32_t kind,
                   const double* a_prev, double dt, double tol, int32_t max_iter, double* a_out,
                   adrom_rom_step_info* host_info);

/* ---- device-resident online loop (driver.py:291-410) ------------------- */
/* The fields of ExperimentConfig (driver.py:63-91) the online loop reads. */
typedef struct adrom_session_config {
  adrom_model model;
  int32_t r, n_s, n_extra, z;
  int32_t projection;       /* 0 = lspg, 1 = galerkin                      */
  int32_t sampling;         /* 0 = qdeim, 1 = fgs                          */
  int32_t feature;          /* 0 = pressure-gradient, 1 = velocity-gradient */
  int32_t adaptive;         /* 1 = run_adaptive_rom (iSVD), 0 = static     */
  int32_t newton_max_iter;  /* also the reduced steps' max_iter            */
  int32_t pad;
  int64_t w_init, n_t;
  double dt, lam, newton_tol;
} adrom_session_config;

/* one adaptation event (driver.py:351-387 event dict) */
typedef struct adrom_event_record {
  int64_t step;              /* event["step"]                                  */
  int32_t coarse_converged;  /* event["coarse_converged"]                      */
  int32_t coarse_iterations; /* event["coarse_iterations"]                     */
  double residual_norm;      /* event["residual_norm"]                         */
  int32_t error;             /* 0, or the adrom_status of event["update_error"] */
  int32_t pad;
} adrom_event_record;

typedef struct adrom_session adrom_session;

int adrom_session_create(adrom_ctx* ctx, const adrom_session_config* cfg, adrom_session** out);
void adrom_session_destroy(adrom_session* s);
/* offline results (device): q_ref, row scale d, POD basis phi0 (N x r),
 * sigma0 (r) and q_last = training[w_init] (driver.py:296-300). */
int adrom_session_load(adrom_session* s, const double* q_ref, const double* d, const double* phi0,
                       const double* sigma0, const double* q_last);
/* driver.py:321-331 (start of the timed region): lookahead, sampling,
 * operator, encode. */
int adrom_session_start(adrom_session* s);
/* driver.py:337-387 for n_steps fine steps; every save_every-th decoded
 * state is copied to dev_out and/or host_out (pinned).  A reduced-step
 * failure returns ADROM_ERR_ROMSTEP like the reference. */
int adrom_session_advance(adrom_session* s, int64_t n_steps, int64_t save_every, double* dev_out,
                          double* host_out, int64_t* n_saved);
int adrom_session_finish(adrom_session* s);
/* logs and current state; host_step_log is n_steps x [converged,
 * iterations, residual_norm]; dev_* may be NULL. */
int adrom_session_read(adrom_session* s, double* host_step_log, int64_t max_steps,
                       adrom_event_record* host_events, int64_t max_events, int64_t* n_steps,
                       int64_t* n_events, double* dev_a, double* dev_phi, double* dev_sigma,
                       double* dev_q_tilde);
/* the coarse lookahead state of the latest adaptation event (the signal
 * y_corr of driver.py:324-327 / 354-357, recorded at step n + 1 + z by
 * driver.py:356) into a device N-vector */
int adrom_session_signal(adrom_session* s, double* dev_y);
/* current sampled rows (device int64[n_s]) */
int adrom_session_sampling(adrom_session* s, int64_t* dev_idx);
/* host_out of adrom_session_advance as a ring of `slots` states (state k of
 * a call goes to slot k % slots; copies into a slot stay ordered); 0 = the
 * default linear layout.  For streaming consumers of the decoded trajectory
 * that do not keep all of it (driver.py:306 keeps it; this bounds the pinned
 * memory a long run needs). */
int adrom_session_set_host_ring(adrom_session* s, int64_t slots);

#ifdef __cplusplus
}
#endif

#endif /* ADROM_B200_H */
