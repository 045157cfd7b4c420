// Hand-written FP64 tensor-core GEMMs (DMMA: mma.sync.aligned.m8n8k4 f64) for
// the large-sample reduced operator of configuration 4 (FGS: n_s = 408,954
// sampled rows, r = 128; sampling.py:162-175, projection.py:158-204).  Two
// shapes, both tall in K:
//
//   * dmma_tn:    C (m x n, column-major) = sum_k A(k, i) B(k, c) -- the
//                 tall-skinny inner products: Gram matrices of the sampled
//                 basis rows (CholeskyQR2 pseudo-inverse) and the Gauss-Newton
//                 contraction [jac | rho] = pinv [test | res].  Deterministic
//                 split-K: one K chunk per block (one per SM), each block's
//                 m x n partial accumulated on DMMA and stored, then summed in
//                 a fixed order (the result does not depend on timing).
//   * dmma_apply: Out (K x n) = A (K x m) M (m x n) -- the tall-times-small
//                 products Q1 = phi_s R1^{-1} and pinv^T = phi_s M.
//
// Operand tiles are staged in shared memory by cp.async (8-byte copies: the
// sampled matrices have arbitrary leading dimensions), double buffered; the
// smem row strides are = 4 (mod 16) doubles so that the m8n8k4 fragment loads
// (lane -> (lane >> 2, lane & 3)) hit 16 distinct 8-byte banks per half-warp.
#include "common.cuh"
#include "dgemm_internal.cuh"

namespace adrom {
namespace {

__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp8(double* smem, const double* gmem, bool ok) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem),
               "r"(ok ? 8 : 0));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// ---------------------------------------------------------------------------
// split-K C = A^T B
// ---------------------------------------------------------------------------
constexpr int TN_KC = 32;     // K rows per stage
constexpr int TN_NTHR = 256;  // 8 warps, warp w owns output rows 16w .. 16w + 15
constexpr int TN_NT = 17;     // 8-wide output column tiles (n <= 136)
constexpr int TN_SA = 132;    // A stage [k][i] stride (row-major A), >= 128, = 4 mod 16
constexpr int TN_SAK = TN_KC + 4;  // A stage [i][k] stride (K-major A), = 4 mod 16
constexpr int TN_SB = 148;    // B stage [k][c] stride, >= 136, = 4 mod 16
constexpr int TN_ASZ = (TN_KC * TN_SA > DMMA_TN_MAX_M * TN_SAK) ? TN_KC * TN_SA : DMMA_TN_MAX_M * TN_SAK;
constexpr int TN_STAGE = TN_ASZ + TN_KC * TN_SB;
constexpr size_t TN_SMEM = sizeof(double) * 2 * (size_t)TN_STAGE;

// AKM: A is K-major (A[i * lda + k], e.g. the pseudo-inverse r x n_s);
// otherwise row-major K x m (A[k * lda + i], e.g. the sampled basis rows)
// 2 x 17 accumulator tiles = 136 registers per thread: one block per SM
template <bool AKM>
__global__ void __launch_bounds__(TN_NTHR, 1)
    dmma_tn_kernel(int m, int n, int64_t K, int64_t chunk, const double* __restrict__ A, int64_t lda,
                   const double* __restrict__ B, int64_t ldb, double* __restrict__ part) {
  extern __shared__ __align__(16) double sm[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t k_beg = (int64_t)blockIdx.x * chunk;
  int64_t k_end = k_beg + chunk;
  if (k_end > K) k_end = K;
  const int nstage = k_end > k_beg ? (int)((k_end - k_beg + TN_KC - 1) / TN_KC) : 0;
  const int na = TN_KC * m, nb = TN_KC * n;
  auto load = [&](int s, double* st) {
    const int64_t k0 = k_beg + (int64_t)s * TN_KC;
    double* As = st;
    double* Bs = st + TN_ASZ;
    for (int e = tid; e < na; e += TN_NTHR) {
      int kk, i;
      if (AKM) {
        i = e / TN_KC;
        kk = e - i * TN_KC;
      } else {
        kk = e / m;
        i = e - kk * m;
      }
      const int64_t k = k0 + kk;
      const bool ok = k < k_end;
      const double* src = A + (ok ? (AKM ? (int64_t)i * lda + k : k * lda + i) : 0);
      cp8(As + (AKM ? i * TN_SAK + kk : kk * TN_SA + i), src, ok);
    }
    for (int e = tid; e < nb; e += TN_NTHR) {
      const int kk = e / n, c = e - kk * n;
      const int64_t k = k0 + kk;
      const bool ok = k < k_end;
      cp8(Bs + kk * TN_SB + c, B + (ok ? k * ldb + c : 0), ok);
    }
    cp_commit();
  };
  double acc[2][TN_NT][2];
#pragma unroll
  for (int t = 0; t < 2; ++t)
#pragma unroll
    for (int j = 0; j < TN_NT; ++j) acc[t][j][0] = acc[t][j][1] = 0.0;
  const bool active = 16 * warp < m;
  const int ntn = (n + 7) >> 3;
  const int fr = lane >> 2, fk = lane & 3;
  if (nstage > 0) load(0, sm);
  for (int s = 0; s < nstage; ++s) {
    double* st = sm + (s & 1) * TN_STAGE;
    if (s + 1 < nstage) {
      load(s + 1, sm + ((s + 1) & 1) * TN_STAGE);
      cp_wait<1>();
    } else {
      cp_wait<0>();
    }
    __syncthreads();
    if (active) {
      const double* As = st;
      const double* Bs = st + TN_ASZ;
#pragma unroll
      for (int k4 = 0; k4 < TN_KC; k4 += 4) {
        double af[2];
#pragma unroll
        for (int t = 0; t < 2; ++t) {
          const int i = 16 * warp + 8 * t + fr;
          af[t] = AKM ? As[i * TN_SAK + k4 + fk] : As[(k4 + fk) * TN_SA + i];
        }
#pragma unroll
        for (int j = 0; j < TN_NT; ++j) {
          if (j < ntn) {
            const double bf = Bs[(k4 + fk) * TN_SB + 8 * j + fr];
            dmma884(acc[0][j][0], acc[0][j][1], af[0], bf);
            dmma884(acc[1][j][0], acc[1][j][1], af[1], bf);
          }
        }
      }
    }
    __syncthreads();  // this stage is refilled two iterations on
  }
  // partial (column-major m x n) of this block
  if (!active) return;
  double* P = part + (size_t)blockIdx.x * m * n;
#pragma unroll
  for (int t = 0; t < 2; ++t) {
    const int i = 16 * warp + 8 * t + fr;
#pragma unroll
    for (int j = 0; j < TN_NT; ++j) {
      const int c = 8 * j + 2 * fk;
      if (j < ntn && i < m) {
        if (c < n) P[i + (size_t)m * c] = acc[t][j][0];
        if (c + 1 < n) P[i + (size_t)m * (c + 1)] = acc[t][j][1];
      }
    }
  }
}

// C[e] = sum_b part[b][e] in block order (deterministic)
__global__ void dmma_tn_reduce_kernel(const double* __restrict__ part, int nblk, int64_t sz,
                                      double* __restrict__ C) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < sz;
       e += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int b = 0; b < nblk; ++b) s += part[(size_t)b * sz + e];
    C[e] = s;
  }
}

// ---------------------------------------------------------------------------
// Out = A M, A row-major K x m, M m x n (column- or row-major)
// ---------------------------------------------------------------------------
constexpr int AP_TM = 32;    // rows per tile: 4 row tiles of 8
constexpr int AP_NTHR = 256; // 8 warps: 4 (row tiles) x 2 (interleaved column tiles)
constexpr int AP_SA = 132;   // A tile [row][j] stride (>= 128, = 4 mod 16)
constexpr int AP_SM = 148;   // M [j][c] stride (>= 136, = 4 mod 16)
constexpr int AP_NT = 9;     // column tiles per warp (2 x 9 >= 17)
constexpr size_t AP_SMEM =
    sizeof(double) * ((size_t)2 * AP_TM * AP_SA + (size_t)DMMA_TN_MAX_M * AP_SM);

__global__ void __launch_bounds__(AP_NTHR, 1)
    dmma_apply_kernel(int64_t K, int m, int n, const double* __restrict__ A, int64_t lda,
                      const double* __restrict__ M, int m_rowmajor, double* __restrict__ out,
                      int64_t ldo, int out_kmajor) {
  extern __shared__ __align__(16) double sm[];
  double* As0 = sm;                      // 2 stages x TM x SA
  double* Ms = sm + 2 * AP_TM * AP_SA;   // m x SM
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp >> 1, wn = warp & 1;
  for (int e = tid; e < m * n; e += AP_NTHR) {
    if (m_rowmajor) {
      const int j = e / n, c = e - j * n;  // M[j n + c]
      Ms[j * AP_SM + c] = M[e];
    } else {
      const int j = e % m, c = e / m;  // M[j + m c]
      Ms[j * AP_SM + c] = M[e];
    }
  }
  // zero the padding rows / columns the fragments can touch
  const int mp = (m + 3) & ~3;
  for (int e = tid; e < (mp - m) * AP_SM; e += AP_NTHR) Ms[m * AP_SM + e] = 0.0;
  const int64_t ntiles = (K + AP_TM - 1) / AP_TM;
  const int na = AP_TM * m;
  auto load = [&](int64_t t, double* As) {
    const int64_t r0 = t * AP_TM;
    for (int e = tid; e < na; e += AP_NTHR) {
      const int rr = e / m, j = e - rr * m;
      const bool ok = r0 + rr < K;
      cp8(As + rr * AP_SA + j, A + (ok ? (r0 + rr) * lda + j : 0), ok);
    }
    cp_commit();
  };
  // padding columns m .. mp of both stages are zero (never written by load)
  for (int e = tid; e < 2 * AP_TM * (mp - m); e += AP_NTHR) {
    const int q = e / (mp - m), j = m + e % (mp - m);
    As0[q * AP_SA + j] = 0.0;
  }
  const int ntn = (n + 7) >> 3;
  const int fr = lane >> 2, fk = lane & 3;
  int64_t t = blockIdx.x;
  if (t < ntiles) load(t, As0);
  int stage = 0;
  for (; t < ntiles; t += gridDim.x) {
    double* As = As0 + stage * AP_TM * AP_SA;
    const int64_t tn = t + gridDim.x;
    if (tn < ntiles) {
      load(tn, As0 + (stage ^ 1) * AP_TM * AP_SA);
      cp_wait<1>();
    } else {
      cp_wait<0>();
    }
    __syncthreads();
    double acc[AP_NT][2];
#pragma unroll
    for (int jj = 0; jj < AP_NT; ++jj) acc[jj][0] = acc[jj][1] = 0.0;
    const int ar = 8 * wm + fr;
#pragma unroll 4
    for (int k4 = 0; k4 < mp; k4 += 4) {
      const double af = As[ar * AP_SA + k4 + fk];
#pragma unroll
      for (int jj = 0; jj < AP_NT; ++jj) {
        const int j = wn + 2 * jj;
        if (j < ntn) dmma884(acc[jj][0], acc[jj][1], af, Ms[(k4 + fk) * AP_SM + 8 * j + fr]);
      }
    }
    const int64_t row = t * AP_TM + 8 * wm + fr;
    if (row < K) {
#pragma unroll
      for (int jj = 0; jj < AP_NT; ++jj) {
        const int j = wn + 2 * jj;
        const int c = 8 * j + 2 * fk;
        if (j < ntn) {
          if (out_kmajor) {
            if (c < n) out[(int64_t)c * ldo + row] = acc[jj][0];
            if (c + 1 < n) out[(int64_t)(c + 1) * ldo + row] = acc[jj][1];
          } else {
            if (c < n) out[row * ldo + c] = acc[jj][0];
            if (c + 1 < n) out[row * ldo + c + 1] = acc[jj][1];
          }
        }
      }
    }
    __syncthreads();  // this stage is refilled next-next tile
    stage ^= 1;
  }
}

}  // namespace

int dmma_tn_blocks(const adrom_ctx* ctx) { return ctx->num_sms; }

int dmma_tn(adrom_ctx* ctx, int m, int n, int64_t K, const double* A, int64_t lda, bool a_kmajor,
            const double* B, int64_t ldb, double* C, double* part, int max_blocks) {
  if (m < 1 || n < 1 || m > DMMA_TN_MAX_M || n > DMMA_TN_MAX_N)
    return set_error(ctx, ADROM_ERR_ARG, "dmma_tn: %d x %d output unsupported", m, n);
  if (K <= 0) {
    ADROM_CK(ctx, cudaMemsetAsync(C, 0, sizeof(double) * (size_t)m * n, ctx->stream));
    return ADROM_OK;
  }
  int nblk = dmma_tn_blocks(ctx);
  if (max_blocks > 0 && nblk > max_blocks) nblk = max_blocks;
  const int64_t min_chunk = 4 * TN_KC;  // at least 4 stages per block
  if ((int64_t)nblk * min_chunk > K) nblk = (int)((K + min_chunk - 1) / min_chunk);
  if (nblk < 1) nblk = 1;
  int64_t chunk = (K + nblk - 1) / nblk;
  chunk = (chunk + TN_KC - 1) / TN_KC * TN_KC;
  nblk = (int)((K + chunk - 1) / chunk);
  auto kern = a_kmajor ? dmma_tn_kernel<true> : dmma_tn_kernel<false>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)TN_SMEM);
  kern<<<nblk, TN_NTHR, TN_SMEM, ctx->stream>>>(m, n, K, chunk, A, lda, B, ldb, part);
  ADROM_LAUNCH_CK(ctx);
  const int64_t sz = (int64_t)m * n;
  dmma_tn_reduce_kernel<<<(int)((sz + 255) / 256), 256, 0, ctx->stream>>>(part, nblk, sz, C);
  ADROM_LAUNCH_CK(ctx);
  return ADROM_OK;
}

int dmma_apply(adrom_ctx* ctx, int64_t K, int m, int n, const double* A, int64_t lda,
               const double* M, double* out, int64_t ldo, bool out_kmajor, bool m_rowmajor) {
  if (m < 1 || n < 1 || m > DMMA_TN_MAX_M || n > DMMA_TN_MAX_N)
    return set_error(ctx, ADROM_ERR_ARG, "dmma_apply: %d x %d factor unsupported", m, n);
  if (K <= 0) return ADROM_OK;
  const int64_t ntiles = (K + AP_TM - 1) / AP_TM;
  int64_t g = ctx->num_sms;
  if (g > ntiles) g = ntiles;
  cudaFuncSetAttribute(dmma_apply_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)AP_SMEM);
  dmma_apply_kernel<<<(int)g, AP_NTHR, AP_SMEM, ctx->stream>>>(
      K, m, n, A, lda, M, m_rowmajor ? 1 : 0, out, ldo, out_kmajor ? 1 : 0);
  ADROM_LAUNCH_CK(ctx);
  return ADROM_OK;
}

int ts_tn(adrom_ctx* ctx, int64_t K, int m, int n, const double* A, int64_t lda, bool a_kmajor,
          const double* B, int64_t ldb, double* C) {
  const size_t bytes = sizeof(double) * (size_t)dmma_tn_blocks(ctx) * m * n;
  int st = ensure_scratch(ctx, bytes);
  if (st) return st;
  return dmma_tn(ctx, m, n, K, A, lda, a_kmajor, B, ldb, C, (double*)scratch(ctx, bytes));
}

}  // namespace adrom

extern "C" {

int adrom_ts_tn(adrom_ctx* ctx, int64_t K, int32_t m, int32_t n, const double* A, int64_t lda,
                int32_t a_kmajor, const double* B, int64_t ldb, double* C) {
  if (!ctx || K < 0) return ADROM_ERR_ARG;
  return adrom::ts_tn(ctx, K, m, n, A, lda, a_kmajor != 0, B, ldb, C);
}

int adrom_ts_apply(adrom_ctx* ctx, int64_t K, int32_t m, int32_t n, const double* A, int64_t lda,
                   const double* M, double* out, int64_t ldo, int32_t out_kmajor) {
  if (!ctx || K < 0) return ADROM_ERR_ARG;
  return adrom::dmma_apply(ctx, K, m, n, A, lda, M, out, ldo, out_kmajor != 0, true);
}

}  // extern "C"
