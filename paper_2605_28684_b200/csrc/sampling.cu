// Hyper-reduction sampling on the device: feature-guided sampling
// (sampling.py:117-159), stencil closure + gather plan (sampling.py:178-189,
// fom.py:119-158) and the reduced-operator assembly with the DEIM
// pseudo-inverse (sampling.py:162-175, projection.py:61-80).  The exact
// greedy QDEIM (sampling.py:77-114) is in qdeim.cu.
#include "common.cuh"
#include "jacobi.cuh"
#include "sampling_internal.cuh"
#include <stdlib.h>
#include "rom_internal.cuh"
#include "factored_internal.cuh"

#include <limits.h>

namespace adrom {

// ---------------------------------------------------------------------------
// feature-guided sampling (sampling.py:117-159)
// ---------------------------------------------------------------------------
constexpr int FGS_MAX_CELLS = 8192;

// |gradient| of the feature field; feature: 0 = pressure-gradient,
// 1 = velocity-gradient (sampling.py:64-74, fom.py:200-201 / 279-282)
__device__ __forceinline__ double fgs_theta(const double* y, int64_t c, int kind, int nv,
                                            double gamma, int feature) {
  if (kind == ADROM_BURGERS) return y[c];
  const double m0 = y[nv * c], m1 = y[nv * c + 1], m2 = y[nv * c + 2];
  const double rho = np_max(m0, 1e-10);
  const double vel = m1 / rho;
  if (feature == 1) return vel;
  // __dmul_rn: never contracted into an FMA with the subtraction (numpy order)
  const double kin = __dmul_rn(0.5 * rho, __dmul_rn(vel, vel));
  return np_max((gamma - 1.0) * (m2 - kin), 1e-10);
}

__global__ void __launch_bounds__(1024) fgs_kernel(const double* __restrict__ y, int64_t n_cells,
                                                   int kind, int nv, double dx, double gamma,
                                                   int feature, int64_t* __restrict__ idx,
                                                   int n_base, int n_extra, int* __restrict__ flag) {
  extern __shared__ double sm[];
  int np2 = 1;
  while (np2 < n_cells) np2 <<= 1;
  double* key = sm;               // np2
  int* cid = (int*)(key + np2);   // np2
  int64_t* base = (int64_t*)(cid + np2 + (np2 & 1));  // n_base sorted
  const int tid = threadIdx.x;
  // gradient (sampling.py:135-138)
  for (int c = tid; c < np2; c += blockDim.x) {
    double gk;
    if (c < n_cells) {
      double gr;
      if (c == 0) gr = (fgs_theta(y, 1, kind, nv, gamma, feature) -
                        fgs_theta(y, 0, kind, nv, gamma, feature)) / dx;
      else if (c == n_cells - 1)
        gr = (fgs_theta(y, c, kind, nv, gamma, feature) -
              fgs_theta(y, c - 1, kind, nv, gamma, feature)) / dx;
      else
        gr = (fgs_theta(y, c + 1, kind, nv, gamma, feature) -
              fgs_theta(y, c - 1, kind, nv, gamma, feature)) / (2.0 * dx);
      gk = fabs(gr);
      if (gk != gk) gk = -1.0;  // NaN ranks last (numpy sorts NaN to the end)
    } else {
      gk = -2.0;  // padding
    }
    key[c] = gk;
    cid[c] = c;
  }
  for (int j = tid; j < n_base; j += blockDim.x) {
    const int64_t x = idx[j];
    int rank = 0;
    for (int k = 0; k < n_base; ++k) {
      const int64_t yv = idx[k];
      if (yv < x || (yv == x && k < j)) ++rank;
    }
    base[rank] = x;
  }
  __syncthreads();
  // bitonic sort: |grad| descending, cell index ascending (np.lexsort order)
  for (int size = 2; size <= np2; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = tid; i < np2; i += blockDim.x) {
        const int j = i ^ stride;
        if (j > i) {
          const bool up = ((i & size) == 0);
          const double ki = key[i], kj = key[j];
          const int ci = cid[i], cj = cid[j];
          // "i before j" in the target order
          const bool i_first = (ki > kj) || (ki == kj && ci < cj);
          if (i_first != up) {
            key[i] = kj;
            key[j] = ki;
            cid[i] = cj;
            cid[j] = ci;
          }
        }
      }
      __syncthreads();
    }
  }
  if (tid == 0) {
    int budget = n_extra, out = n_base;
    for (int p = 0; p < n_cells && budget > 0; ++p) {
      const int64_t cell = cid[p];
      for (int v = 0; v < nv && budget > 0; ++v) {
        const int64_t row = cell * nv + v;
        int lo = 0, hi = n_base - 1;
        bool have = false;
        while (lo <= hi) {
          const int mid = (lo + hi) >> 1;
          if (base[mid] == row) {
            have = true;
            break;
          }
          if (base[mid] < row) lo = mid + 1;
          else hi = mid - 1;
        }
        if (have) continue;
        idx[out++] = row;
        --budget;
      }
    }
    if (budget > 0) atomicOr(flag, 16);  // sampling.py:156-157
  }
}

size_t fgs_workspace_bytes(const adrom_model& m) {
  (void)m;
  return 0;
}

int fgs_extend(adrom_ctx* ctx, const adrom_model& m, const double* y_corr, int feature_kind,
               int64_t* idx, int n_base, int n_extra, void* ws) {
  (void)ws;
  const char* ev = getenv("ADROM_FGS_GRID");  // tests: force the grid-wide ranking
  if (m.n_elem > FGS_MAX_CELLS || (ev && atoi(ev) != 0))
    return fgs_extend_big(ctx, m, y_corr, feature_kind, idx, n_base, n_extra);
  int np2 = 1;
  while (np2 < m.n_elem) np2 <<= 1;
  const size_t sm = sizeof(double) * np2 + sizeof(int) * (np2 + 2) + sizeof(int64_t) * (n_base + 1) + 64;
  cudaFuncSetAttribute(fgs_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  fgs_kernel<<<1, 1024, sm, ctx->stream>>>(y_corr, m.n_elem, m.kind, m.n_var, m.dx, m.gamma,
                                           feature_kind, idx, n_base, n_extra, ctx->dflags);
  ADROM_LAUNCH_CK(ctx);
  return ADROM_OK;
}

// ---------------------------------------------------------------------------
// stencil closure + gather plan (one block; n_s <= 4096)
// ---------------------------------------------------------------------------
constexpr int PLAN_MAX_NS = 4096;

__device__ void bitonic_i32(int* a, int np2) {
  for (int size = 2; size <= np2; size <<= 1)
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = threadIdx.x; i < np2; i += blockDim.x) {
        const int j = i ^ stride;
        if (j > i) {
          const bool up = ((i & size) == 0);
          const int x = a[i], y = a[j];
          if ((x > y) == up) {
            a[i] = y;
            a[j] = x;
          }
        }
      }
      __syncthreads();
    }
}

// unique in place (sorted input, first n valid) -> returns count (all threads)
__device__ int unique_sorted(int* a, int n, int* tmp, int* sh_cnt) {
  // flags -> serial compaction by thread 0 (n <= 12288; cheap relative to sorts)
  (void)tmp;
  if (threadIdx.x == 0) {
    int k = 0;
    for (int i = 0; i < n; ++i)
      if (i == 0 || a[i] != a[i - 1]) a[k++] = a[i];
    *sh_cnt = k;
  }
  __syncthreads();
  const int k = *sh_cnt;
  __syncthreads();
  return k;
}

__device__ __forceinline__ int find_sorted(const int* a, int n, int x) {
  int lo = 0, hi = n - 1;
  while (lo <= hi) {
    const int mid = (lo + hi) >> 1;
    if (a[mid] == x) return mid;
    if (a[mid] < x) lo = mid + 1;
    else hi = mid - 1;
  }
  return -1;
}

__global__ void __launch_bounds__(1024) plan_kernel_build(int64_t n_elem, int nv, bool periodic,
                                                          DevOp op, int n_s, int* flag) {
  extern __shared__ int ism[];
  __shared__ int sh_cnt;
  int np2 = 1;
  while (np2 < 3 * n_s) np2 <<= 1;
  int* cells = ism;            // np2 (sorted unique sampled cells)
  int* every = cells + np2;    // np2 (sorted unique stencil cells)
  const int tid = threadIdx.x;
  for (int i = tid; i < np2; i += blockDim.x) cells[i] = (i < n_s) ? (int)(op.idx[i] / nv) : INT_MAX;
  __syncthreads();
  bitonic_i32(cells, np2);
  const int k = unique_sorted(cells, n_s, nullptr, &sh_cnt);
  for (int i = tid; i < np2; i += blockDim.x) {
    int v = INT_MAX;
    if (i < 3 * k) {
      const int c = cells[i / 3], s = i % 3;
      if (s == 1) v = c;
      else if (s == 0) v = periodic ? (c == 0 ? (int)n_elem - 1 : c - 1) : (c == 0 ? 0 : c - 1);
      else v = periodic ? (c == n_elem - 1 ? 0 : c + 1) : (c == n_elem - 1 ? (int)n_elem - 1 : c + 1);
    }
    every[i] = v;
  }
  __syncthreads();
  bitonic_i32(every, np2);
  const int a = unique_sorted(every, 3 * k, nullptr, &sh_cnt);
  // closure rows: every stencil cell, all variables (sampling.py:186-188)
  for (int t = tid; t < a * nv; t += blockDim.x) op.closure[t] = (int64_t)every[t / nv] * nv + t % nv;
  for (int t = tid; t < k * 3 * nv; t += blockDim.x) {
    const int kk = t / (3 * nv), rem = t % (3 * nv), s = rem / nv, v = rem % nv;
    const int c = cells[kk];
    int nb;
    if (s == 1) nb = c;
    else if (s == 0) nb = periodic ? (c == 0 ? (int)n_elem - 1 : c - 1) : (c == 0 ? 0 : c - 1);
    else nb = periodic ? (c == n_elem - 1 ? 0 : c + 1) : (c == n_elem - 1 ? (int)n_elem - 1 : c + 1);
    op.gather[t] = (int64_t)find_sorted(every, a, nb) * nv + v;
  }
  for (int j = tid; j < n_s; j += blockDim.x) {
    const int64_t row = op.idx[j];
    const int c = (int)(row / nv), v = (int)(row % nv);
    op.out_cell[j] = find_sorted(cells, k, c);
    op.out_var[j] = v;
    op.sample_pos[j] = (int64_t)find_sorted(every, a, c) * nv + v;
    // duplicate check
    for (int jj = j + 1; jj < n_s; ++jj)
      if (op.idx[jj] == row) atomicOr(flag, 32);
  }
  if (tid == 0) {
    op.sizes[0] = n_s;
    op.sizes[1] = a * nv;
    op.sizes[2] = k;
  }
}

int plan_build(adrom_ctx* ctx, const adrom_model& m, DevOp& op, int n_s, int* flag) {
  if (n_s > PLAN_MAX_NS || n_s > op.ns_cap)
    return set_error(ctx, ADROM_ERR_ARG, "plan_build: n_s=%d exceeds capacity", n_s);
  int np2 = 1;
  while (np2 < 3 * n_s) np2 <<= 1;
  const size_t sm = sizeof(int) * 2 * np2;
  cudaFuncSetAttribute(plan_kernel_build, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  plan_kernel_build<<<1, 1024, sm, ctx->stream>>>(m.n_elem, m.n_var, m.kind != ADROM_SOD, op,
                                                  n_s, flag);
  ADROM_LAUNCH_CK(ctx);
  return ADROM_OK;
}

// ---------------------------------------------------------------------------
// reduced operator: gathers (projection.py:72-80) + DEIM pinv (sampling.py:162-175)
// ---------------------------------------------------------------------------
// rows_c / rows_s (factored basis): the closure / sampled rows of Phi
// materialised by fact_gather_rows (row j at j * r); otherwise gathered from phi
__global__ void op_gather_kernel(DevOp op, const double* __restrict__ phi,
                                 const double* __restrict__ q_ref, const double* __restrict__ d,
                                 int n_s, const double* __restrict__ rows_c,
                                 const double* __restrict__ rows_s) {
  const int r = op.r;
  const int n_c = op.sizes[1];
  const int64_t total = (int64_t)(n_c + n_s) * (r + 1);
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int row = (int)(t / (r + 1)), col = (int)(t % (r + 1));
    if (row < n_c) {
      const int64_t g = op.closure[row];
      if (col < r)
        op.dinv_phi_c[(int64_t)row * r + col] =
            (rows_c ? rows_c[(int64_t)row * r + col] : phi[g * r + col]) / d[g];
      else op.q_ref_c[row] = q_ref[g];
    } else {
      const int j = row - n_c;
      const int64_t g = op.idx[j];
      if (col < r) op.phi_s[(int64_t)j * r + col] = rows_s ? rows_s[(int64_t)j * r + col] : phi[g * r + col];
      else op.d_s[j] = d[g];
    }
  }
}

// ---------------------------------------------------------------------------
// DEIM pseudo-inverse, fast path: Householder QR of phi_s (n_s x r) with a
// certified condition bound ||R||_F ||R^-1||_F <= 1e10.  Then phi_s has full
// column rank with s_min > 1e-10 s_max, the reference's test
// (s_min <= 1e-12 s_max, sampling.py:171-174) cannot fire, and
// pinv = R^{-1} Q_1^T equals the SVD pseudo-inverse.  Otherwise *need_svd = 1
// and deim_pinv_kernel (Jacobi SVD, the reference's formulation) runs.
// ---------------------------------------------------------------------------
constexpr double PINV_CERT = 1e10;

__global__ void __launch_bounds__(1024) deim_pinv_qr_kernel(DevOp op, int n_s,
                                                           int* __restrict__ need_svd) {
  extern __shared__ double sm[];
  const int r = op.r, m = n_s;
  const int ld = m | 1, ldr = r | 1;
  double* A = sm;                      // r columns of length m (Householder vectors below R)
  double* M = A + (size_t)r * ld;      // r columns of length m: pinv^T accumulator
  double* Ri = M + (size_t)r * ld;     // R^{-1}, column c at Ri[c * ldr]
  double* Rd = Ri + (size_t)r * ldr;   // diag(R)
  double* beta = Rd + r;               // r
  double* red = beta + r;              // 32
  __shared__ int sh_bad;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  for (int e = tid; e < m * r; e += blockDim.x) {
    const int j = e / r, c = e - j * r;
    A[c * ld + j] = op.phi_s[e];
  }
  if (tid == 0) sh_bad = 0;
  __syncthreads();
  for (int k = 0; k < r; ++k) {
    double* col = A + (size_t)k * ld;
    // the column norm by one warp (m is a few hundred at most): one barrier
    // per reflector instead of a block-wide reduction
    if (warp == 0) {
      double a = 0.0;
      for (int i = k + lane; i < m; i += 32) a += col[i] * col[i];
      a = warp_sum(a);
      if (lane == 0) red[0] = a;
    }
    __syncthreads();
    if (tid == 0) {
      const double a = red[0];
      const double x0 = col[k], nrm = sqrt(a);
      const double alpha = (x0 >= 0.0) ? -nrm : nrm;
      const double vtv_half = a - x0 * alpha;
      beta[k] = (vtv_half > 0.0) ? 1.0 / vtv_half : 0.0;
      Rd[k] = alpha;
      col[k] = x0 - alpha;  // v_k (v_i = col[i] below)
    }
    __syncthreads();
    const double bk = beta[k];
    for (int j = k + 1 + warp; j < r; j += nw) {
      double* cj = A + (size_t)j * ld;
      double sdot = 0.0;
      for (int i = k + lane; i < m; i += 32) sdot += col[i] * cj[i];
      sdot = warp_sum(sdot) * bk;
      for (int i = k + lane; i < m; i += 32) cj[i] -= sdot * col[i];
    }
    __syncthreads();
  }
  // R^{-1} (column c: R x = e_c, column-oriented substitution, warp per column)
  double rf = 0.0;
  for (int e = tid; e < r * r; e += blockDim.x) {
    const int l = e / r, k = e - l * r;  // R[k][l], k <= l
    if (k < l) rf += A[(size_t)l * ld + k] * A[(size_t)l * ld + k];
    else if (k == l) rf += Rd[k] * Rd[k];
  }
  rf = block_sum_dyn(rf, red);
  double inv2 = 0.0;
  bool bad = false;
  for (int c = warp; c < r; c += nw) {
    double b[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) b[t] = (lane + 32 * t == c) ? 1.0 : 0.0;
    for (int i = c; i >= 0; --i) {
      const int ti = i >> 5, li = i & 31;
      double bi = 0.0;
#pragma unroll
      for (int t = 0; t < 4; ++t)
        if (t == ti) bi = b[t];
      bi = __shfl_sync(0xffffffffu, bi, li);
      const double d = Rd[i];
      double xi = 0.0;
      if (d == 0.0 || !isfinite(d)) bad = true;
      else xi = bi / d;
      if (lane == 0) {
        Ri[(size_t)c * ldr + i] = xi;
        inv2 += xi * xi;
      }
      const double* coli = A + (size_t)i * ld;
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const int j = lane + 32 * t;
        if (j < i) b[t] -= coli[j] * xi;
      }
    }
    for (int i = c + 1 + lane; i < r; i += 32) Ri[(size_t)c * ldr + i] = 0.0;
  }
  inv2 = block_sum_dyn(inv2, red);
  if (bad) sh_bad = 1;
  __syncthreads();
  const bool cert = !sh_bad && isfinite(rf) && isfinite(inv2) && sqrt(rf) * sqrt(inv2) <= PINV_CERT;
  if (!cert) {
    if (tid == 0) *need_svd = 1;
    return;
  }
  if (tid == 0) *need_svd = 0;
  // M = [R^{-T}; 0]: column c of M is row c of R^{-1}
  for (int e = tid; e < r * m; e += blockDim.x) {
    const int c = e / m, i = e - c * m;
    M[(size_t)c * ld + i] = (i < r) ? Ri[(size_t)i * ldr + c] : 0.0;
  }
  __syncthreads();
  // pinv^T = H_0 ... H_{r-1} M
  for (int k = r - 1; k >= 0; --k) {
    const double* v = A + (size_t)k * ld;
    const double bk = beta[k];
    for (int c = warp; c < r; c += nw) {
      double* mc = M + (size_t)c * ld;
      double sdot = 0.0;
      for (int i = k + lane; i < m; i += 32) sdot += v[i] * mc[i];
      sdot = warp_sum(sdot) * bk;
      for (int i = k + lane; i < m; i += 32) mc[i] -= sdot * v[i];
    }
    __syncthreads();
  }
  for (int e = tid; e < r * m; e += blockDim.x) {
    const int c = e / m, j = e - c * m;
    op.pinv[e] = M[(size_t)c * ld + j];  // pinv[c][j] = (pinv^T)[j][c]
  }
}

static size_t pinv_qr_smem(int n_s, int r) {
  return sizeof(double) * (2 * (size_t)r * (n_s | 1) + (size_t)r * (r | 1) + 2 * r + 32) + 64;
}

__global__ void __launch_bounds__(1024) deim_pinv_kernel(DevOp op, int n_s, int* flag,
                                                         const int* need) {
  extern __shared__ double sm[];
  if (need && *need == 0) return;  // the certified QR path produced pinv
  const int r = op.r;
  const int ld = n_s | 1, ldv = r | 1;
  double* A = sm;                        // r columns of length n_s
  double* V = A + (size_t)r * ld;        // r x r
  double* s = V + (size_t)r * ldv;       // r
  int* order = (int*)(s + r);
  __shared__ int sh_flag;
  for (int e = threadIdx.x; e < n_s * r; e += blockDim.x) {
    const int j = e / r, c = e - j * r;
    A[c * ld + j] = op.phi_s[e];
  }
  __syncthreads();
  const JacobiResult jr = block_jacobi(A, ld, n_s, r, V, ldv, 60, 1e-15, &sh_flag);
  column_norms_sorted(A, ld, n_s, r, s, order);
  const double smax = s[order[0]], smin = s[order[r - 1]];
  if (threadIdx.x == 0) {
    if (!jr.converged) atomicOr(flag, 8);
    if (!(smin > 1e-12 * smax)) atomicOr(flag, 64);  // sampling.py:171-174
  }
  // pinv[k][j] = sum_c V[k][c] W[j][c] / s_c^2
  for (int e = threadIdx.x; e < r * n_s; e += blockDim.x) {
    const int k = e / n_s, j = e - k * n_s;
    double acc = 0.0;
    for (int c = 0; c < r; ++c) {
      const double sc = s[c];
      if (sc > 0.0) acc += V[c * ldv + k] * A[c * ld + j] / (sc * sc);
    }
    op.pinv[e] = acc;
  }
}

// certified QR fast path, Jacobi SVD when it cannot certify (device-side choice)
static int deim_pinv_launch(adrom_ctx* ctx, DevOp& op, int n_s, int* flag) {
  const int r = op.r;
  const size_t sm = sizeof(double) * ((size_t)r * (n_s | 1) + (size_t)r * (r | 1) + r) +
                    sizeof(int) * r + 64;
  if (sm > 220 * 1024)
    return set_error(ctx, ADROM_ERR_ARG, "deim pinv: %d x %d exceeds one block", n_s, r);
  int* need = ctx->dflags + 32;  // 1 = SVD path needed
  const size_t qsm = pinv_qr_smem(n_s, r);
  const bool qr_ok = n_s >= r && r <= 128 && qsm <= 220 * 1024;
  if (qr_ok) {
    cudaFuncSetAttribute(deim_pinv_qr_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)qsm);
    deim_pinv_qr_kernel<<<1, 1024, qsm, ctx->stream>>>(op, n_s, need);
    ADROM_LAUNCH_CK(ctx);
  }
  cudaFuncSetAttribute(deim_pinv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  deim_pinv_kernel<<<1, 1024, sm, ctx->stream>>>(op, n_s, flag, qr_ok ? need : nullptr);
  ADROM_LAUNCH_CK(ctx);
  return ADROM_OK;
}

int operator_fill(adrom_ctx* ctx, DevOp& op, const double* phi, const double* q_ref,
                  const double* d, int n_s, int* flag, const FactBasis* fb, double* fact_rows,
                  double* big_work) {
  const int r = op.r;
  const int64_t total = (int64_t)(op.nc_cap + n_s) * (r + 1);
  int64_t g = (total + 255) / 256;
  if (g > ctx->num_sms * 8) g = ctx->num_sms * 8;
  double* rows_c = nullptr;
  double* rows_s = nullptr;
  if (fb && fb->W) {
    rows_c = fact_rows;
    rows_s = fact_rows + (size_t)op.nc_cap * r;
    int st = fact_gather_rows(ctx, *fb, op.closure, op.nc_cap, rows_c, op.sizes + 1);
    if (st) return st;
    st = fact_gather_rows(ctx, *fb, op.idx, n_s, rows_s);
    if (st) return st;
  }
  op_gather_kernel<<<(int)g, 256, 0, ctx->stream>>>(op, phi, q_ref, d, n_s, rows_c, rows_s);
  ADROM_LAUNCH_CK(ctx);
  if (big_work) return deim_pinv_big(ctx, op, n_s, big_work, flag);
  return deim_pinv_launch(ctx, op, n_s, flag);
}

}  // namespace adrom

namespace adrom {

__global__ void gather_rows_kernel(const double* __restrict__ phi, const int64_t* __restrict__ idx,
                                   int n_s, int r, double* __restrict__ out) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n_s * r; e += gridDim.x * blockDim.x) {
    const int j = e / r, c = e - j * r;
    out[e] = phi[idx[j] * r + c];
  }
}

// build_deim_operator alone (sampling.py:162-175): pinv (r x n_s)
int deim_pinv_only(adrom_ctx* ctx, const double* phi, const int64_t* idx, int n_s, int r,
                   double* phi_s, double* pinv, int* flag) {
  gather_rows_kernel<<<(n_s * r + 255) / 256, 256, 0, ctx->stream>>>(phi, idx, n_s, r, phi_s);
  ADROM_LAUNCH_CK(ctx);
  DevOp op{};
  op.r = r;
  op.phi_s = phi_s;
  op.pinv = pinv;
  return deim_pinv_launch(ctx, op, n_s, flag);
}

}  // namespace adrom
