// extern "C" entry points declared in include/adrom_b200.h.
#include "common.cuh"
#include "fom_internal.cuh"
#include "linalg_internal.cuh"

#include <string.h>

using namespace adrom;

namespace {

int read_flags(adrom_ctx* ctx, int* host_flags) {
  ADROM_CK(ctx, cudaMemcpyAsync(ctx->pinned, ctx->dflags, sizeof(int) * 16,
                                cudaMemcpyDeviceToHost, ctx->stream));
  ADROM_CK(ctx, cudaStreamSynchronize(ctx->stream));
  memcpy(host_flags, ctx->pinned, sizeof(int) * 16);
  return ADROM_OK;
}

int reset_flags(adrom_ctx* ctx) {
  ADROM_CK(ctx, cudaMemsetAsync(ctx->dflags, 0, sizeof(int) * 16, ctx->stream));
  return ADROM_OK;
}

}  // namespace

extern "C" {

int adrom_rhs(adrom_ctx* ctx, const adrom_model* m, const double* q, double* f) {
  if (!ctx || !m) return ADROM_ERR_ARG;
  return fom_rhs(ctx, *m, q, f);
}

int adrom_rhs_at_cells(adrom_ctx* ctx, const adrom_model* m, const double* gathered, int64_t k,
                       double* out) {
  if (!ctx || !m) return ADROM_ERR_ARG;
  return fom_rhs_at_cells(ctx, *m, gathered, k, out);
}

int adrom_plan_evaluate(adrom_ctx* ctx, const adrom_model* m, const int64_t* gather,
                        int64_t n_cells, const int64_t* out_cell, const int64_t* out_var,
                        int64_t n_s, const double* closure_values, const double* h,
                        const double* dirs, int64_t ld_dirs, int32_t n_dir, double* out) {
  if (!ctx || !m) return ADROM_ERR_ARG;
  return fom_plan_evaluate(ctx, *m, gather, n_cells, out_cell, out_var, n_s, closure_values, h,
                           dirs, ld_dirs, n_dir, out);
}

int adrom_fd_jacobian_blocks(adrom_ctx* ctx, const adrom_model* m, const double* q,
                             double* blocks) {
  if (!ctx || !m) return ADROM_ERR_ARG;
  return fom_fd_jacobian(ctx, *m, q, blocks, false, 0.0);
}

int adrom_implicit_step(adrom_ctx* ctx, const adrom_model* m, const double* q, double dt,
                        double tol, int32_t max_iter, double* x, adrom_newton_info* host_info) {
  if (!ctx || !m) return ADROM_ERR_ARG;
  if (!(dt > 0)) return set_error(ctx, ADROM_ERR_ARG, "dt must be positive");
  return fom_implicit_step(ctx, *m, q, dt, tol, max_iter, x, host_info);
}

int adrom_project(adrom_ctx* ctx, const double* phi, const double* x, int64_t n, int32_t r,
                  double* out) {
  if (!ctx) return ADROM_ERR_ARG;
  const size_t need = align_up(sizeof(double) * (size_t)adrom::partial_rows(ctx) * (r + 1)) +
                      align_up(sizeof(double) * (r + 1));
  int st = ensure_scratch(ctx, need);
  if (st) return st;
  double* partial = (double*)ctx->scratch;
  double* tmp = (double*)((char*)ctx->scratch +
                          align_up(sizeof(double) * (size_t)adrom::partial_rows(ctx) * (r + 1)));
  st = ts_project(ctx, phi, n, r, 1, x, nullptr, nullptr, tmp, partial, nullptr);
  if (st) return st;
  ADROM_CK(ctx, cudaMemcpyAsync(out, tmp, sizeof(double) * r, cudaMemcpyDeviceToDevice,
                                ctx->stream));
  return ADROM_OK;
}

int adrom_encode(adrom_ctx* ctx, const double* phi, const double* q_ref, const double* d,
                 const double* q, int64_t n, int32_t r, double* a) {
  if (!ctx) return ADROM_ERR_ARG;
  const size_t pb = align_up(sizeof(double) * (size_t)adrom::partial_rows(ctx) * (r + 1));
  int st = ensure_scratch(ctx, pb + align_up(sizeof(double) * (r + 1)));
  if (st) return st;
  double* partial = (double*)ctx->scratch;
  double* tmp = (double*)((char*)ctx->scratch + pb);
  st = ts_project(ctx, phi, n, r, 2, q, q_ref, d, tmp, partial, nullptr);
  if (st) return st;
  ADROM_CK(ctx, cudaMemcpyAsync(a, tmp, sizeof(double) * r, cudaMemcpyDeviceToDevice,
                                ctx->stream));
  return ADROM_OK;
}

int adrom_decode(adrom_ctx* ctx, const double* phi, const double* q_ref, const double* d,
                 const double* a, int64_t n, int32_t r, double* q) {
  if (!ctx) return ADROM_ERR_ARG;
  return ts_decode(ctx, phi, n, r, a, q_ref, d, q);
}

int adrom_gram(adrom_ctx* ctx, const double* phi, int64_t n, int32_t r, double* gram) {
  if (!ctx) return ADROM_ERR_ARG;
  if (r < 1 || r > 128) return set_error(ctx, ADROM_ERR_ARG, "gram: rank %d unsupported", r);
  const size_t cap = gram_partial_doubles(ctx, r);
  int st = ensure_scratch(ctx, sizeof(double) * cap + 4096);
  if (st) return st;
  return ts_gram(ctx, phi, n, r, gram, (double*)ctx->scratch, cap);
}

int adrom_isvd_update(adrom_ctx* ctx, const double* phi, const double* sigma,
                      const double* y_hat, int64_t n, int32_t r_cur, int32_t r, double lam,
                      double* phi_out, double* sigma_out, double* gram,
                      adrom_isvd_info* host_info) {
  if (!ctx) return ADROM_ERR_ARG;
  int st = ensure_scratch(ctx, isvd_workspace_bytes(ctx, n, r_cur, r) + 4096);
  if (st) return st;
  st = reset_flags(ctx);
  if (st) return st;
  double* stats = (double*)((char*)ctx->scratch + isvd_workspace_bytes(ctx, n, r_cur, r));
  st = isvd_update_async(ctx, phi, sigma, y_hat, n, r_cur, r, lam, phi_out, sigma_out, gram,
                         gram, ctx->scratch, ctx->dflags, ISVD_REORTH_RATIO, stats, nullptr,
                         nullptr, nullptr, nullptr);
  if (st) return st;
  int flags[16];
  ADROM_CK(ctx, cudaMemcpyAsync((char*)ctx->pinned + 256, stats, sizeof(double) * 8,
                                cudaMemcpyDeviceToHost, ctx->stream));
  st = read_flags(ctx, flags);
  if (st) return st;
  const double* hs = (const double*)((char*)ctx->pinned + 256);
  if (flags[0] & 1)
    return set_error(ctx, ADROM_ERR_NONFINITE, "least_squares matrix contains non-finite entries");
  if (flags[0] & 8)
    return set_error(ctx, ADROM_ERR_NOCONV, "SVD did not converge for %dx%d input", r_cur + 1,
                     r_cur + 1);
  if (host_info) {
    host_info->qnorm = hs[0];
    host_info->ynorm = hs[1];
    host_info->proj_resid = hs[2];
    host_info->degenerate = (int)hs[3];
    host_info->reorthogonalised = (int)hs[4];
    host_info->sweeps = (int)hs[5];
    host_info->core_path = (int)hs[7];
  }
  return ADROM_OK;
}

int adrom_small_svd(adrom_ctx* ctx, const double* a, int32_t m, int32_t n, double* u, double* s,
                    double* v) {
  if (!ctx) return ADROM_ERR_ARG;
  int st = reset_flags(ctx);
  if (st) return st;
  st = dense_small_svd(ctx, a, m, n, u, s, v, ctx->dflags);
  if (st) return st;
  int flags[16];
  st = read_flags(ctx, flags);
  if (st) return st;
  if (flags[0] & 1) return set_error(ctx, ADROM_ERR_NONFINITE, "thin_svd input contains non-finite entries");
  if (flags[0] & 8) return set_error(ctx, ADROM_ERR_NOCONV, "SVD did not converge for %dx%d input", m, n);
  return ADROM_OK;
}

}  // extern "C"
