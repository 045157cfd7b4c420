// The offline stage and the dense helpers of the basis-update rules on the
// device:
//
//   * fit_scaling (snapshots.py:54-69): reference state + per-variable mean
//     squared fluctuation, fixed-order reduction; preprocess into the
//     column-major snapshot matrix Y = D (q - q_ref) (snapshots.py:48-49);
//   * pod (snapshots.py:72-89): Householder QR of the tall factor (Y, or Y^T
//     when the window is wider than the grid), one-sided Jacobi SVD of the
//     triangular factor on many blocks (round-robin pairs, one warp per pair;
//     its columns converge to U S, so no rotation is accumulated), the
//     numerical-rank check s > 1e-12 s_0, U = Q U_R and fix_column_signs
//     (dense.py:182-189: the largest-|.| entry of each column made >= 0,
//     first index on ties as np.argmax);
//   * orth (dense.py:175-179) and least_squares (dense.py:100-111: minimum
//     norm with the 1e-12 relative cutoff, as gelsd) on the same QR.
#include "common.cuh"
#include "hhqr_internal.cuh"

#include <string.h>

namespace adrom {
namespace {

constexpr double SVD_CUT = 1e-12;  // dense.py:32 / snapshots.py:86
constexpr double VAR_FLOOR_D = 1e-30;  // snapshots.py:23

// ---------------------------------------------------------------------------
// one-sided Jacobi on the columns of M (n x nc, column-major, ld n)
// ---------------------------------------------------------------------------
// Round t of the circle schedule over np (even) players: (t, np-1) and
// ((t + i) mod (np-1), (t - i) mod (np-1)), i = 1 .. np/2 - 1.  Player
// indices >= nc are zero padding (skipped).  One warp per pair.
// Rows n_dot .. n-1 (if any) are carried along (rotated, not in the dots):
// appending c^T to M yields (V^T c)^T there without accumulating V.
__global__ void __launch_bounds__(256)
    jac_round_kernel(double* __restrict__ M, int64_t n, int64_t n_dot, int nc, int np, int t,
                     double tol, unsigned long long* __restrict__ off) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  const int npair = np / 2;
  if (warp >= npair) return;
  int p, q;
  if (warp == 0) {
    p = t;
    q = np - 1;
  } else {
    p = (t + warp) % (np - 1);
    q = (t - warp + (np - 1)) % (np - 1);
  }
  if (p > q) {
    const int x = p;
    p = q;
    q = x;
  }
  if (q >= nc) return;
  double* a = M + (int64_t)p * n;
  double* b = M + (int64_t)q * n;
  double al = 0.0, be = 0.0, ga = 0.0;
  for (int64_t i = lane; i < n_dot; i += 32) {
    const double x = a[i], y = b[i];
    al = fma(x, x, al);
    be = fma(y, y, be);
    ga = fma(x, y, ga);
  }
  al = warp_sum(al);
  be = warp_sum(be);
  ga = warp_sum(ga);
  if (al == 0.0 || be == 0.0 || ga == 0.0) return;
  const double rel = fabs(ga) / sqrt(al * be);
  if (lane == 0) atomicMax(off, (unsigned long long)__double_as_longlong(rel));
  if (rel <= tol) return;
  const double zeta = (be - al) / (2.0 * ga);
  const double tt = fabs(zeta) > 1e150 ? 0.5 / zeta
                                      : copysign(1.0, zeta) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
  const double c = 1.0 / sqrt(1.0 + tt * tt), s = c * tt;
  for (int64_t i = lane; i < n; i += 32) {
    const double x = a[i], y = b[i];
    a[i] = c * x - s * y;
    b[i] = s * x + c * y;
  }
}

// column norms (first n rows of columns of stride ld), descending order
// (ties: lower index first), rank
__global__ void __launch_bounds__(1024)
    jac_order_kernel(const double* __restrict__ M, int64_t n, int64_t ld, int nc, double* __restrict__ nrm,
                     int* __restrict__ order, double* __restrict__ s_out, int* __restrict__ rank) {
  for (int c = threadIdx.x >> 5; c < nc; c += blockDim.x >> 5) {
    double s = 0.0;
    for (int64_t i = threadIdx.x & 31; i < n; i += 32) s = fma(M[(int64_t)c * ld + i], M[(int64_t)c * ld + i], s);
    s = warp_sum(s);
    if ((threadIdx.x & 31) == 0) nrm[c] = sqrt(s);
  }
  __syncthreads();
  for (int c = threadIdx.x; c < nc; c += blockDim.x) {
    const double v = nrm[c];
    int pos = 0;
    for (int j = 0; j < nc; ++j) {
      const double w = nrm[j];
      pos += (w > v || (w == v && j < c)) ? 1 : 0;
    }
    order[pos] = c;
  }
  __syncthreads();
  for (int c = threadIdx.x; c < nc; c += blockDim.x) s_out[c] = nrm[order[c]];
  __syncthreads();
  if (threadIdx.x == 0) {
    const double s0 = s_out[0];
    int k = 0;
    if (s0 > 0.0)
      for (int c = 0; c < nc; ++c) k += s_out[c] > SVD_CUT * s0 ? 1 : 0;
    *rank = k;
  }
}

// ---------------------------------------------------------------------------
// layout and sign helpers
// ---------------------------------------------------------------------------
// out (rows x cols, column-major) = in (rows x cols, row-major), 32 x 32 tiles
__global__ void transpose_kernel(const double* __restrict__ in, int64_t rows, int cols,
                                 double* __restrict__ out, int64_t ldo) {
  __shared__ double t[32][33];
  const int64_t r0 = (int64_t)blockIdx.x * 32;
  const int c0 = blockIdx.y * 32;
  for (int y = threadIdx.y; y < 32; y += blockDim.y) {
    const int64_t r = r0 + y;
    const int c = c0 + threadIdx.x;
    t[y][threadIdx.x] = (r < rows && c < cols) ? in[r * cols + c] : 0.0;
  }
  __syncthreads();
  for (int y = threadIdx.y; y < 32; y += blockDim.y) {
    const int c = c0 + y;
    const int64_t r = r0 + threadIdx.x;
    if (r < rows && c < cols) out[(int64_t)c * ldo + r] = t[threadIdx.x][y];
  }
}

// per column of X (column-major, ld n): sign of the first largest-|.| entry
__global__ void __launch_bounds__(1024)
    colsign_kernel(const double* __restrict__ X, int64_t n, double* __restrict__ sign) {
  __shared__ double sv[32];
  __shared__ long long si[32];
  const double* x = X + (int64_t)blockIdx.x * n;
  double best = -1.0, bval = 0.0;
  long long bi = 0x7fffffffffffffffll;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    const double v = fabs(x[i]);
    if (v > best) {  // first occurrence within the thread (increasing i)
      best = v;
      bi = i;
      bval = x[i];
    }
  }
  // warp / block arg-max, ties to the lower index
  for (int o = 16; o > 0; o >>= 1) {
    const double ob = __shfl_xor_sync(0xffffffffu, best, o);
    const long long oi = __shfl_xor_sync(0xffffffffu, bi, o);
    const double ov = __shfl_xor_sync(0xffffffffu, bval, o);
    if (ob > best || (ob == best && oi < bi)) {
      best = ob;
      bi = oi;
      bval = ov;
    }
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  __shared__ double sb[32];
  if (lane == 0) {
    sv[w] = best;
    si[w] = bi;
    sb[w] = bval;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double B = -1.0, V = 0.0;
    long long I = 0x7fffffffffffffffll;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k)
      if (sv[k] > B || (sv[k] == B && si[k] < I)) {
        B = sv[k];
        I = si[k];
        V = sb[k];
      }
    sign[blockIdx.x] = V < 0.0 ? -1.0 : 1.0;  // np.sign, 0 -> +1 (dense.py:187-188)
  }
}

// out[i * r + c] = sign[c] * X[c * ldx + i] (row-major result), 32 x 32 tiles
__global__ void signed_untranspose_kernel(const double* __restrict__ X, int64_t n, int64_t ldx,
                                          int r, const double* __restrict__ sign,
                                          double* __restrict__ out) {
  __shared__ double t[32][33];
  const int64_t i0 = (int64_t)blockIdx.x * 32;
  const int c0 = blockIdx.y * 32;
  for (int y = threadIdx.y; y < 32; y += blockDim.y) {
    const int c = c0 + y;
    const int64_t i = i0 + threadIdx.x;
    t[y][threadIdx.x] = (i < n && c < r) ? sign[c] * X[(int64_t)c * ldx + i] : 0.0;
  }
  __syncthreads();
  for (int y = threadIdx.y; y < 32; y += blockDim.y) {
    const int64_t i = i0 + y;
    const int c = c0 + threadIdx.x;
    if (i < n && c < r) out[i * r + c] = t[threadIdx.x][y];
  }
}

// ---------------------------------------------------------------------------
// scaling
// ---------------------------------------------------------------------------
// per-block partial sums of (q_s - q_ref)^2 per variable over all snapshots
__global__ void __launch_bounds__(256)
    scaling_partial_kernel(const double* __restrict__ tr, int m, int64_t N, int nv,
                           double* __restrict__ part) {
  __shared__ double sh[256 * 16];
  double acc[16];
#pragma unroll
  for (int v = 0; v < 16; ++v) acc[v] = 0.0;
  const int64_t total = (int64_t)m * N;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e % N;
    const double d = tr[e] - tr[i];
    const int v = (int)(i % nv);
#pragma unroll
    for (int w = 0; w < 16; ++w)
      if (w == v) acc[w] = fma(d, d, acc[w]);
  }
  for (int v = 0; v < nv; ++v) sh[v * 256 + threadIdx.x] = acc[v];
  __syncthreads();
  for (int v = 0; v < nv; ++v) {
    for (int s = 128; s > 0; s >>= 1) {
      if ((int)threadIdx.x < s) sh[v * 256 + threadIdx.x] += sh[v * 256 + threadIdx.x + s];
      __syncthreads();
    }
  }
  if ((int)threadIdx.x < nv) part[(int64_t)blockIdx.x * nv + threadIdx.x] = sh[threadIdx.x * 256];
}

__global__ void scaling_final_kernel(const double* __restrict__ part, int nblk, int nv, int m,
                                     int64_t N, double* __restrict__ phi_norm) {
  const int v = threadIdx.x;
  if (v >= nv) return;
  double s = 0.0;
  for (int b = 0; b < nblk; ++b) s += part[(int64_t)b * nv + v];
  double pn = s / ((double)m * (double)(N / nv));
  pn = np_max(pn, VAR_FLOOR_D);
  if (pn <= VAR_FLOOR_D) pn = 1.0;  // snapshots.py:68
  phi_norm[v] = pn;
}

// Y (column-major N x m, == m rows of N) = (1 / phi_norm) * (q_s - q_ref)
__global__ void preprocess_window_kernel(const double* __restrict__ tr, int m, int64_t N, int nv,
                                         const double* __restrict__ q_ref,
                                         const double* __restrict__ phi_norm,
                                         double* __restrict__ Y) {
  const int64_t total = (int64_t)m * N;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e % N;
    Y[e] = (1.0 / phi_norm[i % nv]) * (tr[e] - q_ref[i]);
  }
}

// ---------------------------------------------------------------------------
// small helpers on the triangular factor
// ---------------------------------------------------------------------------
// M (k x k, column-major) = R (tr = 0) or R^T (tr = 1), R = upper triangle of A
__global__ void extract_r_kernel(const double* __restrict__ A, int64_t lda, int k, int tr,
                                 double* __restrict__ M) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < (int64_t)k * k;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(e / k), i = (int)(e % k);  // M[i, c]
    const int rr = tr ? c : i, cc = tr ? i : c;   // R[rr, cc]
    M[e] = rr <= cc ? A[(int64_t)cc * lda + rr] : 0.0;
  }
}

// X (n x r, column-major, ldx) = [M[:, order[c]] / s_c ; 0] for c < r
__global__ void lift_u_kernel(const double* __restrict__ M, int k, const int* __restrict__ order,
                              const double* __restrict__ s, int r, int64_t n,
                              double* __restrict__ X, int64_t ldx) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < (int64_t)r * n;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(e / n);
    const int64_t i = e % n;
    const double sv = s[c];
    X[(int64_t)c * ldx + i] = (i < k && sv > 0.0) ? M[(int64_t)order[c] * k + i] / sv : 0.0;
  }
}

// X (n x m, column-major) = [I; 0]
__global__ void identity_kernel(double* __restrict__ X, int64_t n, int m) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n * m;
       e += (int64_t)gridDim.x * blockDim.x)
    X[e] = (e % n) == (e / n) ? 1.0 : 0.0;
}

// least squares from the Jacobi of [R^T; C^T] (k + nb rows, k columns): the
// columns are W = R^T V (W = U' S, R = V S U'^T) over the first k rows and
// D = C^T V below; x = R^+ C = sum_c W[:, c] D[:, c]^T / s_c^2 over the kept
// singular values (s_c > 1e-12 s_0, as gelsd with rcond 1e-12)
__global__ void lstsq_finish_kernel(const double* __restrict__ M, int k, int nb,
                                    const int* __restrict__ order, const double* __restrict__ s,
                                    double* __restrict__ x) {
  const int ld = k + nb;
  const double s0 = s[0];
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < k * nb; e += gridDim.x * blockDim.x) {
    const int i = e / nb, j = e - i * nb;  // x[i, j] (row-major k x nb)
    double acc = 0.0;
    for (int c = 0; c < k; ++c) {
      const double sc = s[c];
      if (!(sc > SVD_CUT * s0)) break;
      const int col = order[c];
      acc += M[(int64_t)col * ld + i] * M[(int64_t)col * ld + k + j] / (sc * sc);
    }
    x[e] = acc;
  }
}

// M (k + nb rows, k columns, column-major) = [R^T; C^T]: R from A's upper
// triangle, C (k x nb) the top of Q^T B (column-major, ld n)
__global__ void lstsq_stack_kernel(const double* __restrict__ A, int64_t lda, int k,
                                   const double* __restrict__ QtB, int64_t ldb, int nb,
                                   double* __restrict__ M) {
  const int ld = k + nb;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < ld * k; e += gridDim.x * blockDim.x) {
    const int c = e / ld, i = e - c * ld;  // M[i, c]
    double v;
    if (i < k) v = c <= i ? A[(int64_t)i * lda + c] : 0.0;  // R^T[i, c] = R[c, i]
    else v = QtB[(int64_t)(i - k) * ldb + c];               // C^T[j, c] = C[c, j]
    M[e] = v;
  }
}

// Dense LU with partial pivoting (getrf's choice: largest |a|, first index)
// and the solve of A x = b, one block, A row-major n x n (overwritten), b
// overwritten by x.  flag |= 2 on an exactly zero pivot (dense.py:163-166).
__global__ void __launch_bounds__(1024) lu_solve_kernel(double* __restrict__ A, int n,
                                                        double* __restrict__ b, int* flag) {
  __shared__ double sv[32];
  __shared__ int si[32];
  __shared__ int piv_s;
  __shared__ double red[32];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5, nw = blockDim.x >> 5;
  for (int k = 0; k < n; ++k) {
    double best = -1.0;
    int bi = n;
    for (int i = k + tid; i < n; i += blockDim.x) {
      const double v = fabs(A[(int64_t)i * n + k]);
      if (v > best) {
        best = v;
        bi = i;
      }
    }
    for (int o = 16; o > 0; o >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ob > best || (ob == best && oi < bi)) {
        best = ob;
        bi = oi;
      }
    }
    if (lane == 0) {
      sv[w] = best;
      si[w] = bi;
    }
    __syncthreads();
    if (tid == 0) {
      double B = -1.0;
      int I = n;
      for (int q = 0; q < nw; ++q)
        if (sv[q] > B || (sv[q] == B && si[q] < I)) {
          B = sv[q];
          I = si[q];
        }
      piv_s = I;
      if (!(B > 0.0)) atomicOr(flag, 2);
    }
    __syncthreads();
    const int p = piv_s;
    if (p != k) {
      for (int j = tid; j < n; j += blockDim.x) {
        const double t = A[(int64_t)k * n + j];
        A[(int64_t)k * n + j] = A[(int64_t)p * n + j];
        A[(int64_t)p * n + j] = t;
      }
      if (tid == 0) {
        const double t = b[k];
        b[k] = b[p];
        b[p] = t;
      }
    }
    __syncthreads();
    const double akk = A[(int64_t)k * n + k];
    if (akk == 0.0) return;  // singular (flagged)
    for (int i = k + 1 + tid; i < n; i += blockDim.x) A[(int64_t)i * n + k] /= akk;
    __syncthreads();
    const int m = n - k - 1;
    for (int64_t e = tid; e < (int64_t)m * m; e += blockDim.x) {
      const int i = k + 1 + (int)(e / m), j = k + 1 + (int)(e % m);
      A[(int64_t)i * n + j] -= A[(int64_t)i * n + k] * A[(int64_t)k * n + j];
    }
    for (int i = k + 1 + tid; i < n; i += blockDim.x) b[i] -= A[(int64_t)i * n + k] * b[k];
    __syncthreads();
  }
  // back substitution U x = y
  for (int k = n - 1; k >= 0; --k) {
    double s = 0.0;
    for (int j = k + 1 + tid; j < n; j += blockDim.x) s += A[(int64_t)k * n + j] * b[j];
    s = warp_sum(s);
    if (lane == 0) red[w] = s;
    __syncthreads();
    if (tid == 0) {
      double t = 0.0;
      for (int q = 0; q < nw; ++q) t += red[q];
      b[k] = (b[k] - t) / A[(int64_t)k * n + k];
    }
    __syncthreads();
  }
}

int grid_for(adrom_ctx* ctx, int64_t work) {
  int64_t g = (work + 255) / 256;
  const int64_t cap = (int64_t)ctx->num_sms * 8;
  if (g > cap) g = cap;
  return (int)(g < 1 ? 1 : g);
}

struct DevBuf {
  adrom_ctx* ctx;
  void* p = nullptr;
  DevBuf(adrom_ctx* c, size_t bytes) : ctx(c) {
    if (cudaMallocAsync(&p, bytes < 256 ? 256 : bytes, c->stream) != cudaSuccess) p = nullptr;
  }
  ~DevBuf() {
    if (p) cudaFreeAsync(p, ctx->stream);
  }
  double* d(size_t off = 0) const { return (double*)p + off; }
};

}  // namespace

// one-sided Jacobi: M (n x nc, column-major; the dots over the first n_dot
// rows) -> columns U S; s (descending), order, rank (s > 1e-12 s_0).  Host
// loop: one launch per round, one convergence read per sweep.
int jacobi_columns(adrom_ctx* ctx, double* M, int64_t n, int64_t n_dot, int nc, double* s,
                   int* order, int* rank, double* scratch_nrm) {
  const int np = nc + (nc & 1) < 2 ? 2 : nc + (nc & 1);
  DevBuf ob(ctx, sizeof(unsigned long long));
  if (!ob.p) return set_error(ctx, ADROM_ERR_CUDA, "jacobi: out of device memory");
  unsigned long long* off = (unsigned long long*)ob.p;
  int st = ensure_pinned(ctx, 4096);
  if (st) return st;
  const int npair = np / 2;
  const int blocks = (npair * 32 + 255) / 256;
  const double tol = 1e-15;
  bool conv = false;
  for (int sweep = 0; sweep < 60 && !conv; ++sweep) {
    ADROM_CK(ctx, cudaMemsetAsync(off, 0, sizeof(unsigned long long), ctx->stream));
    for (int t = 0; t < np - 1; ++t) {
      jac_round_kernel<<<blocks, 256, 0, ctx->stream>>>(M, n, n_dot, nc, np, t, tol, off);
      ADROM_LAUNCH_CK(ctx);
    }
    ADROM_CK(ctx, cudaMemcpyAsync(ctx->pinned, off, sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                                  ctx->stream));
    ADROM_CK(ctx, cudaStreamSynchronize(ctx->stream));
    unsigned long long bits;
    memcpy(&bits, ctx->pinned, sizeof(bits));
    double rel;
    memcpy(&rel, &bits, sizeof(rel));
    conv = rel <= tol;
  }
  if (!conv) return set_error(ctx, ADROM_ERR_NOCONV, "SVD did not converge for %lld x %d input",
                              (long long)n_dot, nc);
  jac_order_kernel<<<1, 1024, 0, ctx->stream>>>(M, n_dot, n, nc, scratch_nrm, order, s, rank);
  ADROM_LAUNCH_CK(ctx);
  return ADROM_OK;
}

namespace {

int check_finite(adrom_ctx* ctx, const double* x, int64_t n, const char* what);

__global__ void nonfinite_kernel(const double* __restrict__ x, int64_t n, int* flag) {
  bool bad = false;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    bad |= !isfinite(x[i]);
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flag, 1);
}

int read_flag0(adrom_ctx* ctx, int* out) {
  ADROM_CK(ctx, cudaMemcpyAsync(ctx->pinned, ctx->dflags, sizeof(int), cudaMemcpyDeviceToHost,
                                ctx->stream));
  ADROM_CK(ctx, cudaStreamSynchronize(ctx->stream));
  memcpy(out, ctx->pinned, sizeof(int));
  return ADROM_OK;
}

int check_finite(adrom_ctx* ctx, const double* x, int64_t n, const char* what) {
  ADROM_CK(ctx, cudaMemsetAsync(ctx->dflags, 0, sizeof(int), ctx->stream));
  nonfinite_kernel<<<grid_for(ctx, n), 256, 0, ctx->stream>>>(x, n, ctx->dflags);
  ADROM_LAUNCH_CK(ctx);
  int f = 0;
  int st = read_flag0(ctx, &f);
  if (st) return st;
  if (f) return set_error(ctx, ADROM_ERR_NONFINITE, "%s contains non-finite entries", what);
  return ADROM_OK;
}

// Y (column-major N x m, consumed) -> phi (N x r row-major), sigma (r),
// s_all (min(N, m), optional), rank.  Tall: QR of Y, SVD of R, U = Q U_R;
// wide: QR of Y^T, SVD of R^T (its left vectors are Y's).
int pod_core(adrom_ctx* ctx, double* Y, int64_t N, int m, int r, double* phi, double* sigma,
             double* s_all, int* rank_out) {
  const bool tall = N >= m;
  const int64_t rows = tall ? N : m;
  const int k = tall ? m : (int)N;  // columns of the QR'd matrix = order of R
  DevBuf yt(ctx, tall ? 0 : sizeof(double) * (size_t)N * m);
  double* A = Y;
  if (!tall) {  // A = Y^T (column-major m x N) = Y row-major ... transpose
    A = yt.d();
    dim3 g((unsigned)((m + 31) / 32), (unsigned)((N + 31) / 32));  // (rows = m) x (cols = N)
    // Y column-major N x m == row-major m x N; A column-major m x N needs
    // A[j m + i] = Y[i N + j]: the transpose of the row-major m x N array
    transpose_kernel<<<g, dim3(32, 8), 0, ctx->stream>>>(Y, m, (int)N, A, m);
    // (rows = m, cols = N): out[c * m + r] = in[r * N + c]
    ADROM_LAUNCH_CK(ctx);
  }
  const size_t hw = hh_work_doubles(rows, k > r ? k : r);
  DevBuf work(ctx, sizeof(double) * (hw + 2 * (size_t)k + 4 * (size_t)k + (size_t)k * k + 64));
  DevBuf ib(ctx, sizeof(int) * ((size_t)k + 8));
  if (!work.p || !ib.p || (!tall && !yt.p)) return set_error(ctx, ADROM_ERR_CUDA, "pod: out of device memory");
  double* vk = work.d(hw);
  double* vtv = vk + k;
  double* s = vtv + k;
  double* nrm = s + k;
  double* M = nrm + k;               // k x k
  int* order = (int*)ib.p;
  int* rank = order + k;
  int st = hh_qr(ctx, rows, k, A, rows, vk, vtv, work.d());
  if (st) return st;
  extract_r_kernel<<<grid_for(ctx, (int64_t)k * k), 256, 0, ctx->stream>>>(A, rows, k, tall ? 0 : 1, M);
  ADROM_LAUNCH_CK(ctx);
  st = jacobi_columns(ctx, M, k, k, k, s, order, rank, nrm);
  if (st) return st;
  int hrank = 0;
  ADROM_CK(ctx, cudaMemcpyAsync(ctx->pinned, rank, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  ADROM_CK(ctx, cudaStreamSynchronize(ctx->stream));
  memcpy(&hrank, ctx->pinned, sizeof(int));
  if (rank_out) *rank_out = hrank;
  if (s_all) ADROM_CK(ctx, cudaMemcpyAsync(s_all, s, sizeof(double) * k, cudaMemcpyDeviceToDevice, ctx->stream));
  if (r > hrank)
    return set_error(ctx, ADROM_ERR_DENSE, "requested %d modes but snapshot matrix has numerical rank %d", r, hrank);
  // X (N x r, column-major) = U[:, :r]
  DevBuf xb(ctx, sizeof(double) * (size_t)N * r + 64);
  DevBuf sg(ctx, sizeof(double) * (size_t)r + 64);
  if (!xb.p || !sg.p) return set_error(ctx, ADROM_ERR_CUDA, "pod: out of device memory");
  double* X = xb.d();
  lift_u_kernel<<<grid_for(ctx, (int64_t)r * N), 256, 0, ctx->stream>>>(M, k, order, s, r, N, X, N);
  ADROM_LAUNCH_CK(ctx);
  if (tall) {
    st = hh_apply(ctx, N, k, A, N, vk, vtv, X, N, r, false, work.d());
    if (st) return st;
  }
  colsign_kernel<<<r, 1024, 0, ctx->stream>>>(X, N, sg.d());
  ADROM_LAUNCH_CK(ctx);
  dim3 g((unsigned)((N + 31) / 32), (unsigned)((r + 31) / 32));
  signed_untranspose_kernel<<<g, dim3(32, 8), 0, ctx->stream>>>(X, N, N, r, sg.d(), phi);
  ADROM_LAUNCH_CK(ctx);
  ADROM_CK(ctx, cudaMemcpyAsync(sigma, s, sizeof(double) * r, cudaMemcpyDeviceToDevice, ctx->stream));
  return ADROM_OK;
}

}  // namespace
}  // namespace adrom

using namespace adrom;

extern "C" {

int adrom_fit_scaling(adrom_ctx* ctx, const double* training, int32_t m, int64_t n_dof,
                      int32_t n_var, double* q_ref, double* phi_norm) {
  if (!ctx || m < 1 || n_var < 1 || n_var > 16 || n_dof % n_var) return ADROM_ERR_ARG;
  const int nblk = ctx->num_sms * 2;
  DevBuf part(ctx, sizeof(double) * (size_t)nblk * n_var);
  if (!part.p) return set_error(ctx, ADROM_ERR_CUDA, "fit_scaling: out of device memory");
  scaling_partial_kernel<<<nblk, 256, 0, ctx->stream>>>(training, m, n_dof, n_var, part.d());
  ADROM_LAUNCH_CK(ctx);
  scaling_final_kernel<<<1, 32, 0, ctx->stream>>>(part.d(), nblk, n_var, m, n_dof, phi_norm);
  ADROM_LAUNCH_CK(ctx);
  ADROM_CK(ctx, cudaMemcpyAsync(q_ref, training, sizeof(double) * n_dof, cudaMemcpyDeviceToDevice,
                                ctx->stream));
  return ADROM_OK;
}

int adrom_pod_window(adrom_ctx* ctx, const double* training, int32_t m, int64_t n_dof,
                     int32_t n_var, const double* q_ref, const double* phi_norm, int32_t r,
                     double* phi, double* sigma, double* s_all, int32_t* rank) {
  if (!ctx || m < 1 || r < 1 || r > m || r > n_dof || n_var < 1) return ADROM_ERR_ARG;
  DevBuf y(ctx, sizeof(double) * (size_t)m * n_dof);
  if (!y.p) return set_error(ctx, ADROM_ERR_CUDA, "pod: out of device memory");
  preprocess_window_kernel<<<grid_for(ctx, (int64_t)m * n_dof), 256, 0, ctx->stream>>>(
      training, m, n_dof, n_var, q_ref, phi_norm, y.d());
  ADROM_LAUNCH_CK(ctx);
  int st = check_finite(ctx, y.d(), (int64_t)m * n_dof, "thin_svd input");
  if (st) return st;
  int rk = 0;
  st = pod_core(ctx, y.d(), n_dof, m, r, phi, sigma, s_all, &rk);
  if (rank) *rank = rk;
  return st;
}

int adrom_pod(adrom_ctx* ctx, const double* y, int64_t n, int32_t m, int32_t r, double* phi,
              double* sigma, double* s_all, int32_t* rank) {
  if (!ctx || m < 1 || r < 1 || n < 1) return ADROM_ERR_ARG;
  if (r > m || r > n)
    return set_error(ctx, ADROM_ERR_DENSE, "cannot extract %d modes from a %lldx%d matrix", r, (long long)n, m);
  int st = check_finite(ctx, y, n * m, "thin_svd input");
  if (st) return st;
  DevBuf yc(ctx, sizeof(double) * (size_t)n * m);
  if (!yc.p) return set_error(ctx, ADROM_ERR_CUDA, "pod: out of device memory");
  // y row-major n x m -> column-major copy
  dim3 g((unsigned)((n + 31) / 32), (unsigned)((m + 31) / 32));
  transpose_kernel<<<g, dim3(32, 8), 0, ctx->stream>>>(y, n, m, yc.d(), n);
  ADROM_LAUNCH_CK(ctx);
  int rk = 0;
  st = pod_core(ctx, yc.d(), n, m, r, phi, sigma, s_all, &rk);
  if (rank) *rank = rk;
  return st;
}

int adrom_orth(adrom_ctx* ctx, const double* a, int64_t n, int32_t m, double* q) {
  if (!ctx || m < 1 || n < m) return ADROM_ERR_ARG;
  int st = check_finite(ctx, a, n * m, "orth input");
  if (st) return st;
  const size_t hw = hh_work_doubles(n, m);
  DevBuf ac(ctx, sizeof(double) * (size_t)n * m);
  DevBuf xb(ctx, sizeof(double) * (size_t)n * m);
  DevBuf work(ctx, sizeof(double) * (hw + 2 * (size_t)m + (size_t)m + 64));
  if (!ac.p || !xb.p || !work.p) return set_error(ctx, ADROM_ERR_CUDA, "orth: out of device memory");
  dim3 g((unsigned)((n + 31) / 32), (unsigned)((m + 31) / 32));
  transpose_kernel<<<g, dim3(32, 8), 0, ctx->stream>>>(a, n, m, ac.d(), n);
  ADROM_LAUNCH_CK(ctx);
  double* vk = work.d(hw);
  double* vtv = vk + m;
  double* sg = vtv + m;
  st = hh_qr(ctx, n, m, ac.d(), n, vk, vtv, work.d());
  if (st) return st;
  // X = Q [I; 0]
  identity_kernel<<<grid_for(ctx, n * m), 256, 0, ctx->stream>>>(xb.d(), n, m);
  ADROM_LAUNCH_CK(ctx);
  st = hh_apply(ctx, n, m, ac.d(), n, vk, vtv, xb.d(), n, m, false, work.d());
  if (st) return st;
  colsign_kernel<<<m, 1024, 0, ctx->stream>>>(xb.d(), n, sg);
  ADROM_LAUNCH_CK(ctx);
  dim3 g2((unsigned)((n + 31) / 32), (unsigned)((m + 31) / 32));
  signed_untranspose_kernel<<<g2, dim3(32, 8), 0, ctx->stream>>>(xb.d(), n, n, m, sg, q);
  ADROM_LAUNCH_CK(ctx);
  return ADROM_OK;
}

int adrom_least_squares(adrom_ctx* ctx, const double* a, int64_t n, int32_t k, const double* b,
                        int32_t nb, double* x) {
  if (!ctx || k < 1 || nb < 1) return ADROM_ERR_ARG;
  if (n < k) return set_error(ctx, ADROM_ERR_DENSE, "least_squares expects rows >= cols, got shape (%lld, %d)",
                              (long long)n, k);
  int st = check_finite(ctx, a, n * k, "least_squares matrix");
  if (st) return st;
  st = check_finite(ctx, b, n * nb, "least_squares rhs");
  if (st) return st;
  const int w = k > nb ? k : nb;
  const size_t hw = hh_work_doubles(n, w);
  DevBuf ac(ctx, sizeof(double) * (size_t)n * k);
  DevBuf bc(ctx, sizeof(double) * (size_t)n * nb);
  DevBuf work(ctx, sizeof(double) * (hw + 4 * (size_t)k + (size_t)(k + nb) * k + 64));
  DevBuf ib(ctx, sizeof(int) * ((size_t)k + 8));
  if (!ac.p || !bc.p || !work.p || !ib.p) return set_error(ctx, ADROM_ERR_CUDA, "least_squares: out of device memory");
  dim3 g((unsigned)((n + 31) / 32), (unsigned)((k + 31) / 32));
  transpose_kernel<<<g, dim3(32, 8), 0, ctx->stream>>>(a, n, k, ac.d(), n);
  ADROM_LAUNCH_CK(ctx);
  dim3 g2((unsigned)((n + 31) / 32), (unsigned)((nb + 31) / 32));
  transpose_kernel<<<g2, dim3(32, 8), 0, ctx->stream>>>(b, n, nb, bc.d(), n);
  ADROM_LAUNCH_CK(ctx);
  double* vk = work.d(hw);
  double* vtv = vk + k;
  double* s = vtv + k;
  double* nrm = s + k;
  double* M = nrm + k;
  int* order = (int*)ib.p;
  int* rank = order + k;
  st = hh_qr(ctx, n, k, ac.d(), n, vk, vtv, work.d());
  if (st) return st;
  st = hh_apply(ctx, n, k, ac.d(), n, vk, vtv, bc.d(), n, nb, true, work.d());  // Q^T B
  if (st) return st;
  lstsq_stack_kernel<<<grid_for(ctx, (int64_t)(k + nb) * k), 256, 0, ctx->stream>>>(ac.d(), n, k, bc.d(), n, nb, M);
  ADROM_LAUNCH_CK(ctx);
  st = jacobi_columns(ctx, M, k + nb, k, k, s, order, rank, nrm);
  if (st) return st;
  lstsq_finish_kernel<<<grid_for(ctx, (int64_t)k * nb), 256, 0, ctx->stream>>>(M, k, nb, order, s, x);
  ADROM_LAUNCH_CK(ctx);
  return ADROM_OK;
}

int adrom_lu_solve(adrom_ctx* ctx, double* a, int64_t n, double* b) {
  if (!ctx || n < 1 || n > (1 << 20)) return ADROM_ERR_ARG;
  ADROM_CK(ctx, cudaMemsetAsync(ctx->dflags, 0, sizeof(int), ctx->stream));
  lu_solve_kernel<<<1, 1024, 0, ctx->stream>>>(a, (int)n, b, ctx->dflags);
  ADROM_LAUNCH_CK(ctx);
  int f = 0;
  int st = read_flag0(ctx, &f);
  if (st) return st;
  if (f & 2) return set_error(ctx, ADROM_ERR_SINGULAR, "singular Jacobian");
  return ADROM_OK;
}

}  // extern "C"
