// Large sampling sets (configuration 4: FGS on 3 % of 2^20 cells x 13
// variables = 408,954 sampled rows, r = 128).  The one-block kernels of
// sampling.cu / sampled.cu hold the whole sampled system in shared memory
// (n_s <= 4096); here every stage is a grid-wide kernel chain:
//
//   * FGS ranking (sampling.py:117-159): |grad feature| keys, a stable radix
//     sort (CUB) gives np.lexsort's order (descending |grad|, ascending
//     cell), then a prefix sum of the rows each cell adds (its variables not
//     already sampled by QDEIM) places every row without a serial loop;
//   * stencil closure + gather plan (sampling.py:178-189, fom.py:127-152):
//     per-cell marks (sampled / stencil / per-variable bit masks) and two
//     prefix sums, so the closure is sorted by construction; the sampled rows
//     are also grouped by cell (CSR) for the reduced step;
//   * DEIM pseudo-inverse (sampling.py:162-175) by CholeskyQR2 with a
//     certified condition bound (DMMA GEMMs of dgemm.cu for the n_s x r
//     products);
//   * LSPG Gauss-Newton step (projection.py:158-204): closure decode, base
//     residual and the r finite-difference directions evaluated per sampled
//     CELL (one residual evaluation serves all of its sampled rows), then one
//     split-K DMMA GEMM forms [jac | rho] = pinv [test | res]; the r x r update runs in
//     one block (sampled.cu: lspg_update_kernel).
//
// Compiled with --fmad=false: the sampled residuals and the perturbed closure
// values `qc + h_j * Dc[:, j]` reproduce numpy's unfused arithmetic, and the
// FGS feature gradient is bitwise the reference's.
#include "reacting.cuh"
#include "rom_internal.cuh"
#include "sampling_internal.cuh"
#include "dgemm_internal.cuh"

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <stdlib.h>

namespace adrom {

// split-K partial buffers: one r x (r+1) partial per K chunk (dmma_tn runs
// one chunk per SM; more than 296 SMs would be capped here)
constexpr int SPLITK_MAX = 296;

static size_t al(size_t b) { return (b + 255) & ~(size_t)255; }

// ---------------------------------------------------------------------------
// FGS on many cells
// ---------------------------------------------------------------------------
// feature of cell c (sampling.py:64-74 with fom.py:200-201 / 279-282);
// __dmul_rn keeps (0.5 rho)(v v) out of an FMA with the subtraction
__device__ __forceinline__ double fgs_feature(const double* y, int64_t c, int kind, int nv,
                                              double gamma, int feature) {
  if (kind == ADROM_BURGERS) return y[c];
  const double m0 = y[nv * c], m1 = y[nv * c + 1], m2 = y[nv * c + 2];
  const double rho = np_max(m0, PRIM_FLOOR);
  const double vel = m1 / rho;
  if (feature == 1) return vel;
  const double kin = __dmul_rn(0.5 * rho, __dmul_rn(vel, vel));
  return np_max((gamma - 1.0) * (m2 - kin), PRIM_FLOOR);
}

// sort key: ascending key = descending |grad| (NaN last, as np.lexsort)
__global__ void fgs_keys_kernel(const double* __restrict__ y, int64_t n, int kind, int nv,
                                double dx, double gamma, int feature,
                                unsigned long long* __restrict__ keys, int* __restrict__ vals) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < n;
       c += (int64_t)gridDim.x * blockDim.x) {
    double gr;
    if (c == 0)  // sampling.py:135-138
      gr = (fgs_feature(y, 1, kind, nv, gamma, feature) - fgs_feature(y, 0, kind, nv, gamma, feature)) / dx;
    else if (c == n - 1)
      gr = (fgs_feature(y, c, kind, nv, gamma, feature) -
            fgs_feature(y, c - 1, kind, nv, gamma, feature)) / dx;
    else
      gr = (fgs_feature(y, c + 1, kind, nv, gamma, feature) -
            fgs_feature(y, c - 1, kind, nv, gamma, feature)) / (2.0 * dx);
    const double g = fabs(gr);
    unsigned long long k;
    if (g != g) k = 0x7FF0000000000001ull;
    else k = 0x7FF0000000000000ull - (unsigned long long)__double_as_longlong(g);
    keys[c] = k;
    vals[c] = (int)c;
  }
}

__device__ __forceinline__ bool in_sorted(const unsigned long long* a, int n, unsigned long long x) {
  int lo = 0, hi = n - 1;
  while (lo <= hi) {
    const int mid = (lo + hi) >> 1;
    if (a[mid] == x) return true;
    if (a[mid] < x) lo = mid + 1;
    else hi = mid - 1;
  }
  return false;
}

// rows cell order[p] adds: its variables that QDEIM did not already pick
__global__ void fgs_count_kernel(const int* __restrict__ order, int64_t n, int nv,
                                 const unsigned long long* __restrict__ base, int n_base,
                                 int* __restrict__ cnt) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n;
       p += (int64_t)gridDim.x * blockDim.x) {
    const int64_t cell = order[p];
    int k = 0;
    for (int v = 0; v < nv; ++v)
      k += in_sorted(base, n_base, (unsigned long long)(cell * nv + v)) ? 0 : 1;
    cnt[p] = k;
  }
}

__global__ void fgs_emit_kernel(const int* __restrict__ order, int64_t n, int nv,
                                const unsigned long long* __restrict__ base, int n_base,
                                const int* __restrict__ cnt, const int* __restrict__ off,
                                int64_t* __restrict__ idx, int n_extra, int* __restrict__ flag) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n;
       p += (int64_t)gridDim.x * blockDim.x) {
    int o = off[p];
    if (p == n - 1 && o + cnt[p] < n_extra) atomicOr(flag, 16);  // sampling.py:156-157
    if (o >= n_extra) continue;
    const int64_t cell = order[p];
    for (int v = 0; v < nv && o < n_extra; ++v) {
      const int64_t row = cell * nv + v;
      if (in_sorted(base, n_base, (unsigned long long)row)) continue;
      idx[n_base + o] = row;
      ++o;
    }
  }
}

int fgs_extend_big(adrom_ctx* ctx, const adrom_model& m, const double* y_corr, int feature_kind,
                   int64_t* idx, int n_base, int n_extra) {
  const int64_t n = m.n_elem;
  if (n > (int64_t)1 << 30) return set_error(ctx, ADROM_ERR_ARG, "fgs: too many cells");
  size_t t_sort = 0, t_scan = 0, t_base = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, t_sort, (unsigned long long*)nullptr,
                                  (unsigned long long*)nullptr, (int*)nullptr, (int*)nullptr, (int)n);
  cub::DeviceScan::ExclusiveSum(nullptr, t_scan, (int*)nullptr, (int*)nullptr, (int)n);
  cub::DeviceRadixSort::SortKeys(nullptr, t_base, (unsigned long long*)nullptr,
                                 (unsigned long long*)nullptr, n_base > 0 ? n_base : 1);
  size_t tmp = t_sort > t_scan ? t_sort : t_scan;
  tmp = tmp > t_base ? tmp : t_base;
  const size_t bytes = 2 * al(8 * n) + 4 * al(4 * n) + 2 * al(8 * (size_t)(n_base + 1)) + al(tmp);
  int st = ensure_aux(ctx, bytes);
  if (st) return st;
  char* w = (char*)ctx->aux;
  auto take = [&](size_t b) {
    void* p = w;
    w += al(b);
    return p;
  };
  auto* kin = (unsigned long long*)take(8 * n);
  auto* kout = (unsigned long long*)take(8 * n);
  int* vin = (int*)take(4 * n);
  int* vout = (int*)take(4 * n);
  int* cnt = (int*)take(4 * n);
  int* off = (int*)take(4 * n);
  auto* bin = (unsigned long long*)take(8 * (size_t)(n_base + 1));
  auto* bout = (unsigned long long*)take(8 * (size_t)(n_base + 1));
  void* tws = take(tmp);
  const int grid = ctx->num_sms * 8;
  fgs_keys_kernel<<<grid, 256, 0, ctx->stream>>>(y_corr, n, m.kind, m.n_var, m.dx, m.gamma,
                                                 feature_kind, kin, vin);
  ADROM_LAUNCH_CK(ctx);
  size_t t = tmp;
  ADROM_CK(ctx, cub::DeviceRadixSort::SortPairs(tws, t, kin, kout, vin, vout, (int)n, 0, 64,
                                                ctx->stream));
  ++ctx->launches;
  if (n_base > 0) {
    ADROM_CK(ctx, cudaMemcpyAsync(bin, idx, sizeof(int64_t) * n_base, cudaMemcpyDeviceToDevice,
                                  ctx->stream));
    t = tmp;
    ADROM_CK(ctx, cub::DeviceRadixSort::SortKeys(tws, t, bin, bout, n_base, 0, 64, ctx->stream));
    ++ctx->launches;
  }
  fgs_count_kernel<<<grid, 256, 0, ctx->stream>>>(vout, n, m.n_var, bout, n_base, cnt);
  ADROM_LAUNCH_CK(ctx);
  t = tmp;
  ADROM_CK(ctx, cub::DeviceScan::ExclusiveSum(tws, t, cnt, off, (int)n, ctx->stream));
  ++ctx->launches;
  fgs_emit_kernel<<<grid, 256, 0, ctx->stream>>>(vout, n, m.n_var, bout, n_base, cnt, off, idx,
                                                 n_extra, ctx->dflags);
  ADROM_LAUNCH_CK(ctx);
  return ADROM_OK;
}

// ---------------------------------------------------------------------------
// stencil closure + gather plan + rows grouped by cell
// ---------------------------------------------------------------------------
__device__ __forceinline__ int64_t nb_cell(int64_t c, int s, int64_t n, bool periodic) {
  if (s == 1) return c;
  if (s == 0) return periodic ? (c == 0 ? n - 1 : c - 1) : (c == 0 ? 0 : c - 1);
  return periodic ? (c == n - 1 ? 0 : c + 1) : (c == n - 1 ? n - 1 : c + 1);
}

__global__ void plan_mark_kernel(const int64_t* __restrict__ idx, int n_s, int nv, int64_t n,
                                 bool periodic, unsigned* __restrict__ mask,
                                 int* __restrict__ fe, int* __restrict__ flag) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n_s; j += gridDim.x * blockDim.x) {
    const int64_t row = idx[j];
    const int64_t c = row / nv;
    const int v = (int)(row - c * nv);
    if (row < 0 || c >= n) {
      atomicOr(flag, 32);
      continue;
    }
    const unsigned old = atomicOr(mask + c, 1u << v);
    if (old & (1u << v)) atomicOr(flag, 32);  // sampling indices must be distinct
    fe[nb_cell(c, 0, n, periodic)] = 1;
    fe[c] = 1;
    fe[nb_cell(c, 2, n, periodic)] = 1;
  }
}

__global__ void plan_flags_kernel(const unsigned* __restrict__ mask, int64_t n,
                                  int* __restrict__ fs, int* __restrict__ rc) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < n;
       c += (int64_t)gridDim.x * blockDim.x) {
    const unsigned mk = mask[c];
    fs[c] = mk ? 1 : 0;
    rc[c] = __popc(mk);
  }
}

__global__ void plan_fill_kernel(int64_t n, int nv, bool periodic, const unsigned* __restrict__ mask,
                                 const int* __restrict__ fe, const int* __restrict__ pe,
                                 const int* __restrict__ ps, const int* __restrict__ pr,
                                 DevOp op, BigOp big, int n_s) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < n;
       c += (int64_t)gridDim.x * blockDim.x) {
    if (fe[c])
      for (int v = 0; v < nv; ++v) op.closure[(int64_t)pe[c] * nv + v] = c * nv + v;
    const unsigned mk = mask[c];
    if (mk) {
      const int64_t ks = ps[c];
      for (int s = 0; s < 3; ++s) {
        const int64_t e = pe[nb_cell(c, s, n, periodic)];
        for (int v = 0; v < nv; ++v) op.gather[(ks * 3 + s) * nv + v] = e * nv + v;
      }
      big.cell_start[ks] = pr[c];
      big.cell_cnt[ks] = __popc(mk);
    }
    if (c == n - 1) {
      op.sizes[0] = n_s;
      op.sizes[1] = (int)((pe[c] + fe[c]) * (int64_t)nv);
      op.sizes[2] = ps[c] + (mk ? 1 : 0);
    }
  }
}

__global__ void plan_rows_kernel(const int64_t* __restrict__ idx, int n_s, int nv,
                                 const unsigned* __restrict__ mask, const int* __restrict__ pe,
                                 const int* __restrict__ ps, const int* __restrict__ pr, DevOp op,
                                 BigOp big) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n_s; j += gridDim.x * blockDim.x) {
    const int64_t row = idx[j];
    const int64_t c = row / nv;
    const int v = (int)(row - c * nv);
    op.out_cell[j] = ps[c];
    op.out_var[j] = v;
    op.sample_pos[j] = (int64_t)pe[c] * nv + v;
    big.rows[pr[c] + __popc(mask[c] & ((1u << v) - 1u))] = j;  // rows of a cell by variable
  }
}

int plan_build_big(adrom_ctx* ctx, const adrom_model& m, DevOp& op, const BigOp& big, int n_s,
                   int* flag) {
  const int64_t n = m.n_elem;
  const int nv = m.n_var;
  if (nv > 32) return set_error(ctx, ADROM_ERR_ARG, "plan_build: n_var > 32");
  if (n > (int64_t)1 << 30) return set_error(ctx, ADROM_ERR_ARG, "plan_build: too many cells");
  const bool periodic = m.kind != ADROM_SOD;
  size_t tmp = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tmp, (int*)nullptr, (int*)nullptr, (int)n);
  const size_t bytes = 7 * al(4 * n) + al(tmp);
  int st = ensure_aux(ctx, bytes);
  if (st) return st;
  char* w = (char*)ctx->aux;
  auto take = [&](size_t b) {
    void* p = w;
    w += al(b);
    return p;
  };
  auto* mask = (unsigned*)take(4 * n);
  int* fe = (int*)take(4 * n);
  int* fs = (int*)take(4 * n);
  int* rc = (int*)take(4 * n);
  int* pe = (int*)take(4 * n);
  int* ps = (int*)take(4 * n);
  int* pr = (int*)take(4 * n);
  void* tws = take(tmp);
  ADROM_CK(ctx, cudaMemsetAsync(mask, 0, 2 * al(4 * n), ctx->stream));  // mask, fe
  const int grid = ctx->num_sms * 8;
  plan_mark_kernel<<<grid, 256, 0, ctx->stream>>>(op.idx, n_s, nv, n, periodic, mask, fe, flag);
  ADROM_LAUNCH_CK(ctx);
  plan_flags_kernel<<<grid, 256, 0, ctx->stream>>>(mask, n, fs, rc);
  ADROM_LAUNCH_CK(ctx);
  size_t t = tmp;
  ADROM_CK(ctx, cub::DeviceScan::ExclusiveSum(tws, t, fe, pe, (int)n, ctx->stream));
  t = tmp;
  ADROM_CK(ctx, cub::DeviceScan::ExclusiveSum(tws, t, fs, ps, (int)n, ctx->stream));
  t = tmp;
  ADROM_CK(ctx, cub::DeviceScan::ExclusiveSum(tws, t, rc, pr, (int)n, ctx->stream));
  ctx->launches += 3;
  plan_fill_kernel<<<grid, 256, 0, ctx->stream>>>(n, nv, periodic, mask, fe, pe, ps, pr, op, big,
                                                  n_s);
  ADROM_LAUNCH_CK(ctx);
  plan_rows_kernel<<<grid, 256, 0, ctx->stream>>>(op.idx, n_s, nv, mask, pe, ps, pr, op, big);
  ADROM_LAUNCH_CK(ctx);
  return ADROM_OK;
}

// ---------------------------------------------------------------------------
// DEIM pseudo-inverse by CholeskyQR2 (sampling.py:162-175)
// ---------------------------------------------------------------------------
// G (r x r, column-major, symmetric) -> upper R with G = R^T R, R^{-1};
// mode 0: out = R, out2 = R^{-1}.  mode 1 (second pass, R1 = the first
// factor): Rt = R R1, certify ||Rt||_F ||Rt^{-1}||_F <= PINV_BIG_CERT and
// write M = Rt^{-1} Rt^{-T} into out.  Failure -> flag 128.
constexpr double PINV_BIG_CERT = 1e8;

__global__ void __launch_bounds__(512) chol_kernel(const double* __restrict__ G, int r, int mode,
                                                   const double* __restrict__ R1,
                                                   double* __restrict__ out,
                                                   double* __restrict__ out2,
                                                   double* __restrict__ X,
                                                   int* __restrict__ flag) {
  extern __shared__ double sm[];
  const int ld = r + 1;
  double* A = sm;                 // r x ld, column-major; upper triangle -> R
  double* red = A + (size_t)r * ld;
  // X (r x ld, global scratch, L2-resident): R^{-1}
  __shared__ int sh_bad;
  const int tid = threadIdx.x;
  for (int e = tid; e < r * r; e += blockDim.x) {
    const int i = e % r, j = e / r;
    A[j * ld + i] = G[e];
  }
  if (tid == 0) sh_bad = 0;
  __syncthreads();
  // right-looking Cholesky on the upper triangle: R[k][k] = sqrt(A[k][k]),
  // R[k][j] = A[k][j] / R[k][k], A[i][j] -= R[k][i] R[k][j]  (i, j > k)
  for (int k = 0; k < r; ++k) {
    if (tid == 0) {
      const double d = A[k * ld + k];
      if (!(d > 0.0) || !isfinite(d)) sh_bad = 1;
      A[k * ld + k] = sqrt(d > 0.0 ? d : 1.0);
    }
    __syncthreads();
    const double rkk = A[k * ld + k];
    for (int j = k + 1 + tid; j < r; j += blockDim.x) A[j * ld + k] = A[j * ld + k] / rkk;
    __syncthreads();
    const int m = r - k - 1;
    for (int e = tid; e < m * m; e += blockDim.x) {
      const int i = k + 1 + e % m, j = k + 1 + e / m;
      if (i <= j) A[j * ld + i] -= A[i * ld + k] * A[j * ld + k];
    }
    __syncthreads();
  }
  // R^{-1}: column c solves R x = e_c (back substitution, thread per column)
  for (int c = tid; c < r; c += blockDim.x) {
    for (int i = r - 1; i >= 0; --i) {
      double s = (i == c) ? 1.0 : 0.0;
      if (i < c)
        for (int l = i + 1; l <= c; ++l) s -= A[l * ld + i] * X[c * ld + l];
      X[c * ld + i] = (i <= c) ? s / A[i * ld + i] : 0.0;
    }
  }
  __syncthreads();
  if (mode == 0) {
    for (int e = tid; e < r * r; e += blockDim.x) {
      const int i = e % r, j = e / r;
      out[e] = (i <= j) ? A[j * ld + i] : 0.0;
      out2[e] = (i <= j) ? X[j * ld + i] : 0.0;
    }
    if (tid == 0 && sh_bad) atomicOr(flag, 128);
    return;
  }
  // Rt = R2 R1 (upper), Rt^{-1} = R1^{-1} R2^{-1}: R1^{-1} is supplied in out2
  // by the first pass; Rt itself only for the certificate
  double rf = 0.0, xf = 0.0;
  for (int e = tid; e < r * r; e += blockDim.x) {
    const int i = e % r, j = e / r;
    if (i > j) continue;
    double a = 0.0, x = 0.0;
    for (int l = i; l <= j; ++l) {
      a += A[l * ld + i] * R1[j * r + l];     // (R2 R1)[i][j]
      x += out2[l * r + i] * X[j * ld + l];   // (R1^{-1} R2^{-1})[i][j]
    }
    rf += a * a;
    xf += x * x;
  }
  rf = block_sum_dyn(rf, red);
  xf = block_sum_dyn(xf, red);
  __syncthreads();
  // Y = Rt^{-1} = R1^{-1} R2^{-1} into A's storage, then M = Y Y^T
  for (int e = tid; e < r * r; e += blockDim.x) {
    const int i = e % r, j = e / r;
    double x = 0.0;
    for (int l = i; l <= j; ++l) x += out2[l * r + i] * X[j * ld + l];
    A[j * ld + i] = (i <= j) ? x : 0.0;
  }
  __syncthreads();
  for (int e = tid; e < r * r; e += blockDim.x) {
    const int i = e % r, j = e / r;
    double s = 0.0;
    for (int l = (i > j ? i : j); l < r; ++l) s += A[l * ld + i] * A[l * ld + j];
    out[e] = s;
  }
  if (tid == 0 && (sh_bad || !(isfinite(rf) && isfinite(xf)) || !(sqrt(rf) * sqrt(xf) <= PINV_BIG_CERT)))
    atomicOr(flag, 128);
}

static size_t chol_smem(int r) { return sizeof(double) * ((size_t)r * (r + 1) + 40); }

int deim_pinv_big(adrom_ctx* ctx, DevOp& op, int n_s, double* work, int* flag) {
  const int r = op.r;
  if (r > 128) return set_error(ctx, ADROM_ERR_ARG, "deim pinv: rank %d > 128", r);
  double* G = work;                        // r x r
  double* R1 = G + (size_t)r * r;          // r x r
  double* R1i = R1 + (size_t)r * r;        // r x r
  double* M = R1i + (size_t)r * r;         // r x r
  double* X = M + (size_t)r * r;           // r x (r+1) chol scratch
  double* Q1 = X + (size_t)r * (r + 1);    // n_s x r, row-major (like phi_s)
  double* part = Q1 + (size_t)n_s * r;     // split-K partials
  const size_t sm = chol_smem(r);
  cudaFuncSetAttribute(chol_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  // phi_s is row-major n_s x r
  int st = dmma_tn(ctx, r, r, n_s, op.phi_s, r, false, op.phi_s, r, G, part, SPLITK_MAX);  // G = phi_s^T phi_s
  if (st) return st;
  chol_kernel<<<1, 512, sm, ctx->stream>>>(G, r, 0, nullptr, R1, R1i, X, flag);
  ADROM_LAUNCH_CK(ctx);
  st = dmma_apply(ctx, n_s, r, r, op.phi_s, r, R1i, Q1, r, false);  // Q1 = phi_s R1^{-1}
  if (st) return st;
  st = dmma_tn(ctx, r, r, n_s, Q1, r, false, Q1, r, G, part, SPLITK_MAX);        // G2 = Q1^T Q1
  if (st) return st;
  chol_kernel<<<1, 512, sm, ctx->stream>>>(G, r, 1, R1, M, R1i, X, flag);
  ADROM_LAUNCH_CK(ctx);
  // pinv^T = phi_s (Rt^T Rt)^{-1}, stored K-major: pinv row-major r x n_s
  return dmma_apply(ctx, n_s, r, r, op.phi_s, r, M, op.pinv, n_s, true);
}

size_t deim_pinv_big_work_doubles(int n_s, int r) {
  return 5 * (size_t)r * (r + 1) + (size_t)n_s * r + (size_t)SPLITK_MAX * r * r + 64;
}

// ---------------------------------------------------------------------------
// LSPG Gauss-Newton step (projection.py:158-204) on a large sampled set
// ---------------------------------------------------------------------------
// state layout (BigOp::st): [0,r) a, [r,2r) h, [2r,...) scalars:
//   ST_IT iterations, ST_DONE, ST_GN gradient norm, ST_STATUS
// decode_closure (projection.py:86-87): qc = q_ref_c + Dc a, warp per row
__global__ void bl_decode_kernel(const double* __restrict__ Dc, const double* __restrict__ q_ref_c,
                                 const int* __restrict__ sizes, int r,
                                 const double* __restrict__ a, const double* __restrict__ done,
                                 double* __restrict__ qc) {
  if (done && *done != 0.0) return;
  const int n_c = sizes[1];
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  double al[4];
#pragma unroll
  for (int t = 0; t < 4; ++t) al[t] = (lane + 32 * t < r) ? a[lane + 32 * t] : 0.0;
  for (int64_t i = w0; i < n_c; i += nw) {
    const double* row = Dc + i * r;
    double s = 0.0;
#pragma unroll
    for (int t = 0; t < 4; ++t)
      if (lane + 32 * t < r) s = fma(row[lane + 32 * t], al[t], s);
    s = warp_sum(s);
    if (lane == 0) qc[i] = q_ref_c[i] + s;
  }
}

// cell residual of sampled cell slot ks from closure values (+ h dir[:, d])
template <int KIND, int NV>
__device__ __forceinline__ void bl_cell(const DevOp& op, const PlanParams& pp, int64_t ks,
                                        const double* qc, const double* Dc, int r, int d, double h,
                                        double* o) {
  const int64_t* g = op.gather + ks * 3 * NV;
  auto val = [&](int s, int v) {
    const int64_t pos = g[s * NV + v];
    return Dc ? qc[pos] + h * Dc[pos * r + d] : qc[pos];
  };
  if (KIND == ADROM_BURGERS) {
    o[0] = burgers_cell(val(0, 0), val(1, 0), val(2, 0), pp.bp);
  } else if (KIND == ADROM_SOD) {
    const Cons l{val(0, 0), val(0, 1), val(0, 2)}, c{val(1, 0), val(1, 1), val(1, 2)},
        rr{val(2, 0), val(2, 1), val(2, 2)};
    const Cons x = sod_cell(l, c, rr, pp.gamma, pp.bp.dx);
    o[0] = x.m0;
    o[1] = x.m1;
    o[2] = x.m2;
  } else {
    rx_cell_res_get<false>(val, pp.gamma, pp.bp.dx, pp.mech, o);
  }
}

template <int NV>
__device__ __forceinline__ double pick(const double* o, int v) {
  double x = o[0];
#pragma unroll
  for (int k = 1; k < NV; ++k)
    if (k == v) x = o[k];
  return x;
}

// base residual at the sampled rows; res -> column r of test (ld r+1);
// the first iteration also records prev_sampled (projection.py:170)
template <int KIND, int NV>
__global__ void bl_base_kernel(DevOp op, BigOp big, PlanParams pp, const double* __restrict__ qc,
                               double dt, double* __restrict__ fs, double* __restrict__ prev,
                               double* __restrict__ test, const double* __restrict__ st) {
  if (st[2 * op.r + 1] != 0.0) return;
  const bool first = st[2 * op.r] == 0.0;
  const int k = op.sizes[2];
  const int r = op.r;
  for (int64_t ks = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; ks < k;
       ks += (int64_t)gridDim.x * blockDim.x) {
    double o[NV];
    bl_cell<KIND, NV>(op, pp, ks, qc, nullptr, r, 0, 0.0, o);
    const int64_t b = big.cell_start[ks];
    const int cnt = big.cell_cnt[ks];
    for (int q = 0; q < cnt; ++q) {
      const int j = big.rows[b + q];
      const double f = pick<NV>(o, (int)op.out_var[j]);
      const double qs = qc[op.sample_pos[j]];
      if (first) prev[j] = qs;
      const double pv = first ? qs : prev[j];
      fs[j] = f;
      test[(int64_t)j * (r + 1) + r] = op.d_s[j] * ((qs - pv) - dt * f);
    }
  }
}

// finite-difference directions (projection.py:181-186): block = 128
// directions, a grid-stride loop over sampled cells; thread d computes the
// cell residual at qc + h_d Dc[:, d] and writes test[j][d] = phi_s[j][d] -
// dt (d_s[j] dfs[j][d]) for the cell's sampled rows.  The next cell's
// stencil rows of Dc (3 n_var rows, one column per thread) are staged into
// shared memory by cp.async while the current cell is computed.
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n"); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;\n"); }

constexpr int BL_DIR_T = 128;

template <int KIND, int NV, int NBUF>
__global__ void __launch_bounds__(BL_DIR_T, NBUF == 1 ? 4 : 2)
    bl_dir_kernel(DevOp op, BigOp big, PlanParams pp, const double* __restrict__ qc,
                  const double* __restrict__ fs, double dt, double* __restrict__ test,
                  const double* __restrict__ st) {
  constexpr int NS = 3 * NV;
  extern __shared__ double sdc[];  // [NBUF][NS][BL_DIR_T]
  __shared__ int64_t spos[NBUF][NS];
  __shared__ double sqc[NBUF][NS];
  const int r = op.r;
  if (st[2 * r + 1] != 0.0) return;
  const int k = op.sizes[2];
  const int d = threadIdx.x;
  const bool act = d < r;
  const double h = act ? st[r + d] : 1.0;
  const double* __restrict__ Dc = op.dinv_phi_c;
  int64_t ks = blockIdx.x;
  if (ks >= k) return;
  auto stage = [&](int buf, int64_t cell) {
    if (d < NS) {
      const int64_t p = op.gather[cell * NS + d];
      spos[buf][d] = p;
      sqc[buf][d] = qc[p];
    }
    __syncthreads();
    if (act)
#pragma unroll
      for (int s = 0; s < NS; ++s) cp_async8(sdc + (buf * NS + s) * BL_DIR_T + d, Dc + spos[buf][s] * r + d);
    cp_async_commit();
  };
  if (NBUF == 2) stage(0, ks);
  for (int buf = 0; ks < k; buf ^= (NBUF - 1)) {
    const int64_t nx = ks + gridDim.x;
    if (NBUF == 2) {
      if (nx < k) stage(buf ^ 1, nx);
      else cp_async_commit();
      cp_async_wait1();
    } else {
      stage(0, ks);
      asm volatile("cp.async.wait_group 0;\n");
    }
    __syncthreads();
    if (act) {
      const double* sd = sdc + buf * NS * BL_DIR_T + d;
      const double* sq = sqc[buf];
      auto val = [&](int s, int v) { return sq[s * NV + v] + h * sd[(s * NV + v) * BL_DIR_T]; };
      double o[NV];
      if (KIND == ADROM_BURGERS) {
        o[0] = burgers_cell(val(0, 0), val(1, 0), val(2, 0), pp.bp);
      } else if (KIND == ADROM_SOD) {
        const Cons l{val(0, 0), val(0, 1), val(0, 2)}, c{val(1, 0), val(1, 1), val(1, 2)},
            rr{val(2, 0), val(2, 1), val(2, 2)};
        const Cons x = sod_cell(l, c, rr, pp.gamma, pp.bp.dx);
        o[0] = x.m0;
        o[1] = x.m1;
        o[2] = x.m2;
      } else {
        rx_cell_res_once<false>(val, pp.gamma, pp.bp.dx, pp.mech, o);
      }
      const int64_t b = big.cell_start[ks];
      const int cnt = big.cell_cnt[ks];
      for (int q = 0; q < cnt; ++q) {
        const int j = big.rows[b + q];
        const double df = (pick<NV>(o, (int)op.out_var[j]) - fs[j]) / h;
        test[(int64_t)j * (r + 1) + d] = op.phi_s[(int64_t)j * r + d] - dt * (op.d_s[j] * df);
      }
    }
    __syncthreads();
    ks = nx;
  }
}

// [jac | rho] (r x n, column-major) = pinv (r x K, row-major: K-major) times
// [test | res] (K x n, row-major): split-K DMMA GEMM (dgemm.cu), a fixed-order
// sum of one partial per K chunk (one chunk per SM), so the 128 x 129 output
// keeps every SM busy and the result is deterministic.
static int gemm_jac(adrom_ctx* ctx, int r, int n, int64_t K, const double* pinv,
                    const double* test, double* C, double* part) {
  return dmma_tn(ctx, r, n, K, pinv, K, true, test, n, C, part, SPLITK_MAX);
}

__global__ void bl_init_kernel(const double* __restrict__ a_prev, int r, double* __restrict__ st) {
  for (int k = threadIdx.x; k < r; k += blockDim.x) {
    st[k] = a_prev[k];
    st[r + k] = FD_EPS * np_max(1.0, fabs(a_prev[k]));  // _fd_steps (projection.py:107-108)
  }
  if (threadIdx.x == 0) {
    st[2 * r] = 0.0;      // iterations
    st[2 * r + 1] = 0.0;  // done
    st[2 * r + 2] = INFINITY;
    st[2 * r + 3] = 0.0;  // status
    st[2 * r + 4] = 0.0;  // condition number (RomStepError message)
  }
}

size_t big_work_doubles(const DevOp& op) {
  const size_t r = op.r;
  // qc, fs, prev, test, C, state (a, h, scalars) + the update's V scratch
  return (size_t)op.nc_cap + 2 * (size_t)op.ns_cap + (size_t)op.ns_cap * (r + 1) + r * (r + 1) +
         2 * r + 8 + r * (r | 1) + (SPLITK_MAX + 1) * r * (r + 1) + 64;
}

int lspg_step_big(adrom_ctx* ctx, const RomStepArgs& A, const BigOp& big, int n_s) {
  const DevOp& op = A.op;
  const int r = op.r;
  if (r > 128) return set_error(ctx, ADROM_ERR_ARG, "lspg: rank %d > 128", r);
  double* qc = A.work;
  double* fs = qc + op.nc_cap;
  double* prev = fs + op.ns_cap;
  double* test = prev + op.ns_cap;               // n_s x (r+1)
  double* C = test + (size_t)op.ns_cap * (r + 1);  // r x (r+1) column-major: [jac | rho]
  double* st = C + (size_t)r * (r + 1);          // a, h, scalars, update scratch
  double* part = st + 2 * r + 8 + (size_t)r * (r | 1);  // split-K partials
  PlanParams pp{A.bp, A.gamma, A.mech};
  const int pr = prof_begin(ctx, PROBE_ROM_STEP);
  bl_init_kernel<<<1, 128, 0, ctx->stream>>>(A.a_prev, r, st);
  ADROM_LAUNCH_CK(ctx);
  const int grid = ctx->num_sms * 8;
  for (int it = 0; it < A.max_iter; ++it) {
    bl_decode_kernel<<<grid, 256, 0, ctx->stream>>>(op.dinv_phi_c, op.q_ref_c, op.sizes, r, st,
                                                    st + 2 * r + 1, qc);
    ADROM_LAUNCH_CK(ctx);
    // ADROM_BL_DIR_NBUF: 1 = one staged cell per block (4 blocks / SM),
    // 2 = next cell prefetched by cp.async (2 blocks / SM)
    static const int nbuf = getenv("ADROM_BL_DIR_NBUF") ? atoi(getenv("ADROM_BL_DIR_NBUF")) : 1;
    auto dir1 = [&](auto kern, int nv, int nb) {
      const size_t sm = sizeof(double) * nb * 3 * nv * BL_DIR_T;
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      kern<<<ctx->num_sms * (nb == 1 ? 4 : 2), BL_DIR_T, sm, ctx->stream>>>(op, big, pp, qc, fs, A.dt,
                                                                          test, st);
    };
    auto dir = [&](auto k1, auto k2, int nv) {
      if (nbuf == 2) dir1(k2, nv, 2);
      else dir1(k1, nv, 1);
    };
    if (A.kind == ADROM_REACTING) {
      bl_base_kernel<ADROM_REACTING, RX_NV><<<grid, 128, 0, ctx->stream>>>(op, big, pp, qc, A.dt, fs, prev, test, st);
      dir(bl_dir_kernel<ADROM_REACTING, RX_NV, 1>, bl_dir_kernel<ADROM_REACTING, RX_NV, 2>, RX_NV);
    } else if (A.kind == ADROM_SOD) {
      bl_base_kernel<ADROM_SOD, 3><<<grid, 128, 0, ctx->stream>>>(op, big, pp, qc, A.dt, fs, prev, test, st);
      dir(bl_dir_kernel<ADROM_SOD, 3, 1>, bl_dir_kernel<ADROM_SOD, 3, 2>, 3);
    } else {
      bl_base_kernel<ADROM_BURGERS, 1><<<grid, 128, 0, ctx->stream>>>(op, big, pp, qc, A.dt, fs, prev, test, st);
      dir(bl_dir_kernel<ADROM_BURGERS, 1, 1>, bl_dir_kernel<ADROM_BURGERS, 1, 2>, 1);
    }
    ctx->launches += 1;
    ADROM_LAUNCH_CK(ctx);
    // [jac | rho] = pinv [test | res]  (projection.py:176, :187)
    int s2 = gemm_jac(ctx, r, r + 1, n_s, op.pinv, test, C, part);
    if (s2) return s2;
    s2 = lspg_update_launch(ctx, C, r, st, A.tol, A.max_iter);
    if (s2) return s2;
    // stop as soon as the device says so (one small read per iteration)
    ADROM_CK(ctx, cudaMemcpyAsync(ctx->pinned, st + 2 * r + 1, sizeof(double),
                                  cudaMemcpyDeviceToHost, ctx->stream));
    ADROM_CK(ctx, cudaStreamSynchronize(ctx->stream));
    if (*(volatile double*)ctx->pinned != 0.0) break;
  }
  lspg_finish_launch(ctx, st, r, A.tol, A.a_out, A.info);
  prof_end(ctx, pr);
  ADROM_LAUNCH_CK(ctx);
  return ADROM_OK;
}

}  // namespace adrom
