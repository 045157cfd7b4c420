// Host-side internal API of the tall-skinny / iSVD / small-SVD kernels.
#pragma once

#include "common.cuh"

namespace adrom {

// out[0..r) = phi^T w, out[r] = sum w^2 with w = x (wkind 1) or
// w = d * (x - q_ref) (wkind 2).  partial: >= 3*num_sms*(r+1) doubles.
int ts_project(adrom_ctx* ctx, const double* phi, int64_t n, int r, int wkind, const double* x,
               const double* q_ref, const double* d, double* out, double* partial, int* flag);
// q_out = q_ref + (phi a) / d
int ts_decode(adrom_ctx* ctx, const double* phi, int64_t n, int r, const double* a,
              const double* q_ref, const double* d, double* q_out);
int ts_decode_project(adrom_ctx* ctx, const double* phi, int64_t n, int r, const double* a,
                      const double* q_ref, const double* d, double* q_out, const double* y,
                      double* out, double* partial, int* flag);
int ts_residual(adrom_ctx* ctx, const double* phi, int64_t n, int r, const double* p,
                const double* y, double* out, double* partial, int* flag, const int* skip);
// out = phi M + y b^T  (phi n x r_in, M r_in x r_out)
int ts_rotate(adrom_ctx* ctx, const double* phi, const double* y, const double* M,
              const double* b, int64_t n, int r_in, int r_out, double* out);

size_t isvd_workspace_bytes(adrom_ctx* ctx, int64_t n, int r_cur, int r);
// Asynchronous iSVD update.  stats_out (device, >= 8 doubles, may be null):
// [qnorm, ynorm, proj_resid, degenerate, reorth, sweeps, converged].
// If dec_a != null the first pass also writes dec_out = q_ref + (phi dec_a)/d.
int isvd_update_async(adrom_ctx* ctx, const double* phi, const double* sigma, const double* y,
                      int64_t n, int r_cur, int r, double lam, double* phi_out,
                      double* sigma_out, void* ws, int* flag, double reorth_ratio,
                      double* stats_out, const double* dec_a, const double* q_ref,
                      const double* d, double* dec_out);

int dense_small_svd(adrom_ctx* ctx, const double* a, int m, int n, double* u, double* s,
                    double* v, int* flag);

constexpr double ISVD_REORTH_RATIO = 1e-3;

}  // namespace adrom
