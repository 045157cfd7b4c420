// Householder QR of tall matrices and the one-sided Jacobi SVD of its
// triangular factor: the offline POD (snapshots.py:72-89) and the dense
// helpers of the basis-update rules (orth / least_squares, dense.py:100-111,
// :175-179; tracking.py:181-246) on the device, unconditionally stable (no
// Gram matrix is ever factorised, so rank-deficient snapshot sets -- e.g. the
// configuration-0 window, numerical rank 69 of 2001 columns -- are fine).
//
// Layout: A is column-major N x m (A[j lda + i]), every column a contiguous
// N-vector, N >= m.  Reflector k: v = A[k:, k] - alpha e_0, alpha =
// -sign(A[k,k]) ||A[k:, k]|| (LAPACK dlarfg's sign), H_k = I - 2 v v^T / v^T v.
//
// One HBM pass per column: hh_update_kernel applies H_k to the trailing
// columns and, from the updated values it holds in registers, accumulates
// the Gram row of the NEXT column (g_j = a_{k+1}^T a_j, rows >= k+1) as
// per-block partials; hh_reflect_kernel (one block) reduces them in a fixed
// order and forms the next reflector's coefficients, because
//   v^T a_j = g_j - alpha A[k, j].
// The explicit Q (or Q^T x) is applied the same way, one pass per reflector.
#include "common.cuh"
#include "hhqr_internal.cuh"

namespace adrom {
namespace {

constexpr int HH_NTHR = 256;

// Apply H_k (coefficients c_j, j in (k, m)) to rows >= k of columns > k and
// accumulate, per block, g_j = sum_{i >= k+1} A'[i, k+1] A'[i, j] for j >= k+1.
// k = -1: no reflector, Gram row of column 0 (rows >= 0).
template <int RPT>
__global__ void __launch_bounds__(HH_NTHR)
    hh_update_kernel(int64_t N, int m, double* __restrict__ A, int64_t lda, int k,
                     const double* __restrict__ coef, double* __restrict__ part) {
  extern __shared__ double red[];  // (HH_NTHR / 32) x m
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t r0 = (k < 0 ? 0 : k) + (int64_t)blockIdx.x * HH_NTHR * RPT;
  const int kn = k + 1;
  double v[RPT], u[RPT];
  int64_t row[RPT];
#pragma unroll
  for (int q = 0; q < RPT; ++q) {
    row[q] = r0 + tid + (int64_t)q * HH_NTHR;
    v[q] = 0.0;
    if (k >= 0 && row[q] < N) v[q] = row[q] == k ? coef[m] : A[(int64_t)k * lda + row[q]];
  }
  for (int j = kn; j < m; ++j) {
    const double cj = k >= 0 ? coef[j] : 0.0;
    double* col = A + (int64_t)j * lda;
    double acc = 0.0;
#pragma unroll
    for (int q = 0; q < RPT; ++q) {
      if (row[q] < N) {
        double a = col[row[q]];
        if (k >= 0) {
          a = fma(-v[q], cj, a);
          col[row[q]] = a;
        }
        if (j == kn) u[q] = row[q] >= kn ? a : 0.0;
        acc = fma(u[q], a, acc);
      } else if (j == kn) {
        u[q] = 0.0;
      }
    }
    acc = warp_sum(acc);
    if (lane == 0) red[warp * m + j] = acc;
  }
  __syncthreads();
  for (int j = kn + tid; j < m; j += HH_NTHR) {
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < HH_NTHR / 32; ++w) s += red[w * m + j];
    part[(int64_t)blockIdx.x * m + j] = s;
  }
}

// Reduce the Gram row of column k (fixed order), form reflector k: vk[k],
// vtv[k], R[k, k] = alpha, coefficients coef[j] = 2 (g_j - alpha A[k, j]) / vtv
// for j > k, coef[m] = v_k (read by the next hh_update_kernel).
__global__ void __launch_bounds__(512)
    hh_reflect_kernel(int m, double* __restrict__ A, int64_t lda, int k,
                      const double* __restrict__ part, int nblk, double* __restrict__ g,
                      double* __restrict__ coef, double* __restrict__ vk, double* __restrict__ vtv) {
  __shared__ double sh[4];
  for (int j = k + threadIdx.x; j < m; j += blockDim.x) {
    double s = 0.0;
    for (int b = 0; b < nblk; ++b) s += part[(int64_t)b * m + j];
    g[j] = s;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const double x0 = A[(int64_t)k * lda + k];
    const double nrm2 = g[k];
    double alpha = 0.0, t = 0.0, v0 = 0.0;
    if (nrm2 > 0.0) {
      alpha = -copysign(sqrt(nrm2), x0);
      v0 = x0 - alpha;
      t = 2.0 * (nrm2 - alpha * x0);  // v^T v
    } else {
      alpha = x0;  // zero column below and at the diagonal: H = I
    }
    sh[0] = alpha;
    sh[1] = t;
    sh[2] = v0;
    vk[k] = v0;
    vtv[k] = t;
  }
  __syncthreads();
  const double alpha = sh[0], t = sh[1];
  for (int j = k + 1 + threadIdx.x; j < m; j += blockDim.x)
    coef[j] = t > 0.0 ? 2.0 * (g[j] - alpha * A[(int64_t)j * lda + k]) / t : 0.0;
  if (threadIdx.x == 0) {
    coef[m] = sh[2];
    A[(int64_t)k * lda + k] = alpha;
  }
}

// X <- H_ka X on rows >= ka for columns [0, nc) (coefficients cx[c]), then per
// block d_c = w^T X'_c with w the vector of reflector kb (rows >= kb); ka or kb
// may be -1 (none).
template <int RPT>
__global__ void __launch_bounds__(HH_NTHR)
    hh_apply_kernel(int64_t N, const double* __restrict__ A, int64_t lda,
                    const double* __restrict__ vk, double* __restrict__ X, int64_t ldx, int nc,
                    int ka, const double* __restrict__ cx, int kb, double* __restrict__ part) {
  extern __shared__ double red[];  // (HH_NTHR / 32) x nc
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int lo = ka < 0 ? kb : (kb < 0 ? ka : (ka < kb ? ka : kb));
  const int64_t r0 = lo + (int64_t)blockIdx.x * HH_NTHR * RPT;
  double va[RPT], wb[RPT];
  int64_t row[RPT];
#pragma unroll
  for (int q = 0; q < RPT; ++q) {
    row[q] = r0 + tid + (int64_t)q * HH_NTHR;
    va[q] = wb[q] = 0.0;
    if (row[q] < N) {
      if (ka >= 0 && row[q] >= ka) va[q] = row[q] == ka ? vk[ka] : A[(int64_t)ka * lda + row[q]];
      if (kb >= 0 && row[q] >= kb) wb[q] = row[q] == kb ? vk[kb] : A[(int64_t)kb * lda + row[q]];
    }
  }
  for (int c = 0; c < nc; ++c) {
    double* col = X + (int64_t)c * ldx;
    const double cc = ka >= 0 ? cx[c] : 0.0;
    double acc = 0.0;
#pragma unroll
    for (int q = 0; q < RPT; ++q) {
      if (row[q] < N) {
        double x = col[row[q]];
        if (ka >= 0 && row[q] >= ka) {
          x = fma(-va[q], cc, x);
          col[row[q]] = x;
        }
        acc = fma(wb[q], x, acc);
      }
    }
    if (kb >= 0) {
      acc = warp_sum(acc);
      if (lane == 0) red[warp * nc + c] = acc;
    }
  }
  if (kb < 0) return;
  __syncthreads();
  for (int c = tid; c < nc; c += HH_NTHR) {
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < HH_NTHR / 32; ++w) s += red[w * nc + c];
    part[(int64_t)blockIdx.x * nc + c] = s;
  }
}

__global__ void __launch_bounds__(512)
    hh_coef_kernel(int nc, int k, const double* __restrict__ part, int nblk,
                   const double* __restrict__ vtv, double* __restrict__ cx) {
  const double t = vtv[k];
  for (int c = threadIdx.x; c < nc; c += blockDim.x) {
    double s = 0.0;
    for (int b = 0; b < nblk; ++b) s += part[(int64_t)b * nc + c];
    cx[c] = t > 0.0 ? 2.0 * s / t : 0.0;
  }
}

int rpt_for(int64_t rows) { return rows >= (1 << 20) ? 16 : 4; }

int64_t blocks_for(int64_t rows, int rpt) {
  const int64_t per = (int64_t)HH_NTHR * rpt;
  return rows <= 0 ? 1 : (rows + per - 1) / per;
}

}  // namespace

size_t hh_work_doubles(int64_t N, int w) {
  const int64_t nb = blocks_for(N, 4);
  return (size_t)nb * (w + 1) + 3 * (size_t)(w + 1) + 64;
}

int hh_qr(adrom_ctx* ctx, int64_t N, int m, double* A, int64_t lda, double* vk, double* vtv,
          double* work) {
  if (m < 1 || N < m) return set_error(ctx, ADROM_ERR_ARG, "hh_qr: %lld x %d is not tall", (long long)N, m);
  double* coef = work;                 // m + 1
  double* g = coef + (m + 1);          // m
  double* part = g + (m + 1);          // nblk x m
  const size_t red = sizeof(double) * (HH_NTHR / 32) * (size_t)m;
  if (red > 200 * 1024) return set_error(ctx, ADROM_ERR_ARG, "hh_qr: %d columns exceed shared memory", m);
  auto upd4 = hh_update_kernel<4>;
  auto upd16 = hh_update_kernel<16>;
  cudaFuncSetAttribute(upd4, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)red);
  cudaFuncSetAttribute(upd16, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)red);
  for (int k = -1; k < m; ++k) {
    const int64_t rows = N - (k < 0 ? 0 : k);
    const int rpt = rpt_for(rows);
    const int64_t nb = blocks_for(rows, rpt);
    if (k + 1 < m) {  // trailing columns to update / next Gram row
      if (rpt == 16) upd16<<<(unsigned)nb, HH_NTHR, red, ctx->stream>>>(N, m, A, lda, k, coef, part);
      else upd4<<<(unsigned)nb, HH_NTHR, red, ctx->stream>>>(N, m, A, lda, k, coef, part);
      ADROM_LAUNCH_CK(ctx);
    }
    if (k + 1 < m) {
      hh_reflect_kernel<<<1, 512, 0, ctx->stream>>>(m, A, lda, k + 1, part, (int)nb, g, coef, vk, vtv);
      ADROM_LAUNCH_CK(ctx);
    }
  }
  return ADROM_OK;
}

int hh_apply(adrom_ctx* ctx, int64_t N, int m, const double* A, int64_t lda, const double* vk,
             const double* vtv, double* X, int64_t ldx, int nc, bool transpose, double* work) {
  if (nc < 1) return ADROM_OK;
  double* cx = work;        // nc
  double* part = cx + nc;   // nblk x nc
  const size_t red = sizeof(double) * (HH_NTHR / 32) * (size_t)nc;
  if (red > 200 * 1024) return set_error(ctx, ADROM_ERR_ARG, "hh_apply: %d columns exceed shared memory", nc);
  auto ap4 = hh_apply_kernel<4>;
  auto ap16 = hh_apply_kernel<16>;
  cudaFuncSetAttribute(ap4, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)red);
  cudaFuncSetAttribute(ap16, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)red);
  // Q X = H_0 H_1 ... H_{m-1} X: reflectors in decreasing order; Q^T X: increasing
  const int first = transpose ? 0 : m - 1, step = transpose ? 1 : -1;
  int ka = -1;
  for (int s = 0; s <= m; ++s) {
    const int kb = s < m ? first + step * s : -1;
    const int lo = ka < 0 ? kb : (kb < 0 ? ka : (ka < kb ? ka : kb));
    const int64_t rows = N - lo;
    const int rpt = rpt_for(rows);
    const int64_t nb = blocks_for(rows, rpt);
    if (rpt == 16)
      ap16<<<(unsigned)nb, HH_NTHR, red, ctx->stream>>>(N, A, lda, vk, X, ldx, nc, ka, cx, kb, part);
    else
      ap4<<<(unsigned)nb, HH_NTHR, red, ctx->stream>>>(N, A, lda, vk, X, ldx, nc, ka, cx, kb, part);
    ADROM_LAUNCH_CK(ctx);
    if (kb >= 0) {
      hh_coef_kernel<<<1, 512, 0, ctx->stream>>>(nc, kb, part, (int)nb, vtv, cx);
      ADROM_LAUNCH_CK(ctx);
    }
    ka = kb;
  }
  return ADROM_OK;
}

}  // namespace adrom
