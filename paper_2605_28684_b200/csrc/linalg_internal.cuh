// Host-side internal API of the tall-skinny / iSVD / small-SVD kernels.
#pragma once

#include "common.cuh"

namespace adrom {

// out[0..r) = phi^T w, out[r] = sum w^2 with w = x (wkind 1) or
// w = d * (x - q_ref) (wkind 2).  partial: >= partial_rows*(r+1) doubles.
int ts_project(adrom_ctx* ctx, const double* phi, int64_t n, int r, int wkind, const double* x,
               const double* q_ref, const double* d, double* out, double* partial, int* flag);
// q_out = q_ref + (phi a) / d
int ts_decode(adrom_ctx* ctx, const double* phi, int64_t n, int r, const double* a,
              const double* q_ref, const double* d, double* q_out);
int ts_decode_project(adrom_ctx* ctx, const double* phi, int64_t n, int r, const double* a,
                      const double* q_ref, const double* d, double* q_out, const double* y,
                      double* out, double* partial, int* flag);
// q = y - phi p (stored in qbuf if non-null); out = [phi^T q, ||q||^2];
// a no-op when *skip == 0
int ts_residual(adrom_ctx* ctx, const double* phi, int64_t n, int r, const double* p,
                const double* y, double* out, double* partial, int* flag, const int* skip,
                double* qbuf);
// G = phi^T phi (r x r); partial: >= 2*partial_rows*(r+1) doubles
// G = Phi^T Phi; `partial` holds cap_doubles (gram_partial_doubles for full speed)
int ts_gram(adrom_ctx* ctx, const double* phi, int64_t n, int r, double* gram, double* partial,
            size_t cap_doubles);
size_t gram_partial_doubles(const adrom_ctx* ctx, int r);
// partial-sum region at the start of an iSVD workspace (fits ts_gram's)
size_t isvd_partial_doubles(const adrom_ctx* ctx, int r_cur);

// Work fused into the rotation's epilogue (the rotated rows are in registers):
//   encode: enc_partial[block][0..r) = sum_i phi'_i d_i (x_i - q_ref_i)
//           (projection.py:98-99; reduced by rot_encode_finish)
//   seed  : QDEIM bounds res2 = bnd2(1 + 16 eps) = ||phi'_i||^2, ver = 0
struct RotFuse {
  const double* enc_x = nullptr;
  const double* enc_q_ref = nullptr;
  const double* enc_d = nullptr;
  double* enc_partial = nullptr;  // rot_fuse_partial_doubles(ctx, r)
  double* seed_res2 = nullptr;
  double* seed_bnd2 = nullptr;
  unsigned char* seed_ver = nullptr;
};
// true when ts_rotate runs the fused epilogue for this shape
bool rot_fusable(int r_in, int r_out);
size_t rot_fuse_partial_doubles(const adrom_ctx* ctx, int r);
// out[0..r) = sum over the rotation blocks of enc_partial
int rot_encode_finish(adrom_ctx* ctx, const RotFuse& f, int64_t n, int r, double* out);

size_t isvd_workspace_bytes(adrom_ctx* ctx, int64_t n, int r_cur, int r);
// Asynchronous iSVD update (tracking.py:141-178).
//   gram_in  : tracked Phi^T Phi (r_cur x r_cur) or null (then computed here)
//   gram_out : Phi'^T Phi' of the rotated basis (may alias gram_in) or null
//   stats_out (device, >= 8 doubles, may be null):
//   [qnorm, ynorm, proj_resid, degenerate, reorth, sweeps, converged].
// If dec_a != null the first pass also writes dec_out = q_ref + (phi dec_a)/d.
int isvd_update_async(adrom_ctx* ctx, const double* phi, const double* sigma, const double* y,
                      int64_t n, int r_cur, int r, double lam, double* phi_out,
                      double* sigma_out, const double* gram_in, double* gram_out, void* ws,
                      int* flag, double reorth_ratio, double* stats_out, const double* dec_a,
                      const double* q_ref, const double* d, double* dec_out,
                      const RotFuse* fuse = nullptr);

// pieces of the iSVD used by the factored-basis event (factored.cu)
__global__ void reduce_partials_kernel(const double* __restrict__ partial, int nb, int w,
                                       double* __restrict__ out, const int* skip);
__global__ void set_need_kernel(int* need);
int isvd_solve_launch(adrom_ctx* ctx, const double* red1, const double* G, int r, double* p,
                      int* need);
// least-squares refinement after the explicit residual pass (linalg.cu)
int isvd_refine_launch(adrom_ctx* ctx, const double* G, int r, double* red2, double* p,
                       double* p2, double* p2norm, const int* need);
int isvd_core_launch(adrom_ctx* ctx, const double* sigma, const double* red1, const double* pls,
                     const double* red2, const int* need, const double* G, int r, double lam,
                     double* B, double* qinv, double* T, double* Gout, double* sigma_out,
                     double* stats, int* flag, double* udrop = nullptr);

int dense_small_svd(adrom_ctx* ctx, const double* a, int m, int n, double* u, double* s,
                    double* v, int* flag);

constexpr double ISVD_REORTH_RATIO = 1e-3;

}  // namespace adrom
