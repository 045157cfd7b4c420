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

#define ADROM_ABI_VERSION 1

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
  ADROM_SOD = 2      /* fom.SodProblem (fom.py:249-282): zero-gradient, n_var=3 */
};

/* Physics + grid of one full-order model (replaces the FomProblem instance). */
typedef struct adrom_model {
  int32_t kind;   /* adrom_model_kind                              */
  int32_t n_var;  /* 1 (Burgers) or 3 (Sod)                        */
  int64_t n_elem; /* number of cells                               */
  double dx;      /* length / n_elem (fom.py:74)                   */
  double nu;      /* Burgers viscosity (fom.py:173)                */
  double gamma;   /* Euler specific-heat ratio (fom.py:260)        */
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

/* ---- incremental SVD (kernel 4) ---------------------------------------- */
typedef struct adrom_isvd_info {
  double qnorm;          /* ||q|| (tracking.py:163)                          */
  double ynorm;          /* ||y_hat|| (tracking.py:164)                      */
  double proj_resid;     /* ||y - Phi Phi^T y|| (driver.py:366-367 diag)     */
  int32_t degenerate;    /* took the in-span branch (tracking.py:169-170)    */
  int32_t reorthogonalised; /* explicit residual pass was run                */
  int32_t sweeps;        /* Jacobi sweeps of the core SVD                    */
  int32_t pad;
} adrom_isvd_info;

/* isvd_update (tracking.py:141-178):
 *   phi_out = [phi, q/||q||] U_core[:, :r],  sigma_out = s_core[:r]
 * phi: n x r_cur, phi_out: n x r (may alias phi when r <= r_cur).
 * host_info may be NULL (then the call does not synchronise). */
int adrom_isvd_update(adrom_ctx* ctx, const double* phi, const double* sigma,
                      const double* y_hat, int64_t n, int32_t r_cur, int32_t r, double lam,
                      double* phi_out, double* sigma_out, adrom_isvd_info* host_info);

/* thin_svd of a small dense matrix (dense.py:59-72), m x n row-major with
 * m, n <= 256, one thread block: u (m x k), s (k), v (n x k), k = min(m,n). */
int adrom_small_svd(adrom_ctx* ctx, const double* a, int32_t m, int32_t n, double* u,
                    double* s, double* v);

#ifdef __cplusplus
}
#endif

#endif /* ADROM_B200_H */
