// Error diagnostics on the device (driver.py:168-199): per-variable relative
// errors of the primitive fields, ||pf_v(pred) - pf_v(truth)|| / ||pf_v(truth)||
// (the absolute norm when the truth vanishes, driver.py:168-175), for the
// error history and the signal errors of a run whose trajectory is never
// stored (configuration 3: 2064 states x 134 MB).
//
// Primitive fields (fom.py:200-201, fom.py:204-210 / 279-282): Burgers u;
// Euler rho = max(rho, floor), v = m / rho, p = max((gamma-1)(E - (0.5 rho) v^2),
// floor); the reacting model adds Y_k = (rho Y_k) / rho.  Sums: fixed-order
// two-stage reduction (per-block partials, then one block).
#include "common.cuh"
#include "physics.cuh"

namespace adrom {

constexpr int DG_NT = 256;
constexpr int DG_MAXV = 13;

__device__ __forceinline__ void prim_fields(const double* q, int64_t c, int nv, double gamma,
                                            double* f) {
  if (nv == 1) {
    f[0] = q[c];
    return;
  }
  const double* u = q + c * nv;
  const double rho = np_max(u[0], PRIM_FLOOR);
  const double vel = u[1] / rho;
  const double p = np_max((gamma - 1.0) * (u[2] - (0.5 * rho) * (vel * vel)), PRIM_FLOOR);
  f[0] = rho;
  f[1] = vel;
  f[2] = p;
  for (int k = 3; k < nv; ++k) f[k] = u[k] / rho;
}

// partial[b][2v] = sum (pf(pred) - pf(truth))^2, partial[b][2v+1] = sum pf(truth)^2
__global__ void __launch_bounds__(DG_NT) err_partial_kernel(const double* __restrict__ pred,
                                                            const double* __restrict__ truth,
                                                            int64_t n_elem, int nv, double gamma,
                                                            double* __restrict__ partial) {
  __shared__ double red[DG_NT / 32];
  double num[DG_MAXV], den[DG_MAXV];
  for (int v = 0; v < nv; ++v) num[v] = den[v] = 0.0;
  for (int64_t c = blockIdx.x * (int64_t)DG_NT + threadIdx.x; c < n_elem;
       c += (int64_t)gridDim.x * DG_NT) {
    double fp[DG_MAXV], ft[DG_MAXV];
    prim_fields(pred, c, nv, gamma, fp);
    prim_fields(truth, c, nv, gamma, ft);
    for (int v = 0; v < nv; ++v) {
      const double e = fp[v] - ft[v];
      num[v] += e * e;
      den[v] += ft[v] * ft[v];
    }
  }
  for (int v = 0; v < nv; ++v) {
    const double a = block_sum<DG_NT>(num[v], red);
    const double b = block_sum<DG_NT>(den[v], red);
    if (threadIdx.x == 0) {
      partial[(size_t)blockIdx.x * 2 * nv + 2 * v] = a;
      partial[(size_t)blockIdx.x * 2 * nv + 2 * v + 1] = b;
    }
  }
}

__global__ void err_final_kernel(double* __restrict__ partial, int nb, int nv,
                                 double* __restrict__ out) {
  __shared__ double red[32];
  for (int j = 0; j < 2 * nv; ++j) {
    double s = 0.0;
    for (int b = threadIdx.x; b < nb; b += blockDim.x) s += partial[(size_t)b * 2 * nv + j];
    s = block_sum<256>(s, red);
    if (threadIdx.x == 0) partial[(size_t)nb * 2 * nv + j] = s;
  }
  __syncthreads();
  if (threadIdx.x < nv) {
    const double num = partial[(size_t)nb * 2 * nv + 2 * threadIdx.x];
    const double den = partial[(size_t)nb * 2 * nv + 2 * threadIdx.x + 1];
    out[threadIdx.x] = (den == 0.0) ? sqrt(num) : sqrt(num) / sqrt(den);
  }
}

}  // namespace adrom

using namespace adrom;

extern "C" int adrom_state_errors(adrom_ctx* ctx, const adrom_model* m, const double* pred,
                                  const double* truth, double* dev_out) {
  if (!ctx || !m || !pred || !truth || !dev_out) return ADROM_ERR_ARG;
  if (m->n_var < 1 || m->n_var > DG_MAXV) return set_error(ctx, ADROM_ERR_ARG, "n_var %d", m->n_var);
  int64_t nb = (m->n_elem + DG_NT - 1) / DG_NT;
  if (nb > (int64_t)ctx->num_sms * 4) nb = (int64_t)ctx->num_sms * 4;
  if (nb < 1) nb = 1;
  const size_t need = sizeof(double) * ((size_t)nb + 1) * 2 * m->n_var;
  const int st = ensure_scratch(ctx, need);
  if (st) return st;
  double* partial = (double*)ctx->scratch;
  err_partial_kernel<<<(int)nb, DG_NT, 0, ctx->stream>>>(pred, truth, m->n_elem, m->n_var, m->gamma,
                                                         partial);
  ADROM_LAUNCH_CK(ctx);
  err_final_kernel<<<1, 256, 0, ctx->stream>>>(partial, (int)nb, m->n_var, dev_out);
  ADROM_LAUNCH_CK(ctx);
  return ADROM_OK;
}
