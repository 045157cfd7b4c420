// Tall-skinny basis kernels (kernel 3), the iSVD update (kernel 4) and the
// one-block dense SVD.  Compiled WITH FMA contraction: these are reductions
// whose order differs from BLAS anyway; FMA only improves them.
#include "common.cuh"
#include "jacobi.cuh"
#include "linalg_internal.cuh"

#include <math.h>

namespace adrom {

// ---------------------------------------------------------------------------
// tile kernel: one pass over a row-major N x r basis, staged through shared
// memory in tiles of T rows (stride r|1 doubles: conflict-free both for
// thread-per-row and thread-per-column access).
//   ROWDOT: rd_i = phi_i . v                           (v: r-vector)
//   DECODE: out_q_i = q_ref_i + rd_i / d_i            (projection.py:104,
//                                                      snapshots.py:50-51)
//   weight kinds for the column sums acc_j += phi_ij w_i:
//     W_X      w_i = x_i                              (phi^T x)
//     W_ENCODE w_i = d_i (x_i - q_ref_i)              (projection.py:98-99)
//     W_RESID  w_i = x_i - rd_i                       (tracking.py:162)
//   the scalar partial is sum w_i^2.
// ---------------------------------------------------------------------------
enum { W_NONE = 0, W_X = 1, W_ENCODE = 2, W_RESID = 3 };

constexpr int TS_NT = 256;

__host__ __device__ inline int ts_stride(int r) { return (r % 2 == 0) ? r + 1 : r; }
__host__ __device__ inline int ts_tile_rows(int r) { return r <= 64 ? 128 : (r <= 128 ? 64 : 32); }

struct TileArgs {
  const double* phi;
  int64_t n;
  int r;
  const double* v;      // ROWDOT vector (r)
  const double* x;      // weight input / snapshot
  const double* q_ref;  // encode / decode
  const double* d;      // row scale
  double* out_q;        // decode output
  double* partial;      // gridDim.x x (r+1)
  int* flag;            // bit 0: non-finite basis / input
  const int* skip;      // if non-null and *skip == 0 the kernel is a no-op
};

template <bool ROWDOT, bool DECODE, int WKIND>
__global__ void __launch_bounds__(TS_NT) tile_kernel(TileArgs a) {
  extern __shared__ double sm[];
  if (a.skip && *a.skip == 0) return;
  const int r = a.r;
  const int S = ts_stride(r);
  const int T = ts_tile_rows(r);
  double* tile = sm;              // T x S
  double* vv = tile + T * S;      // r
  double* ww = vv + r;            // T (weights)
  double* red = ww + T;           // TS_NT (column reduction)
  const int tid = threadIdx.x;
  const int RS = TS_NT / r;       // row groups for the column sums
  const int col = tid % r, grp = tid / r;
  const bool colthread = grp < RS;
  if (ROWDOT)
    for (int j = tid; j < r; j += TS_NT) vv[j] = a.v[j];
  double acc = 0.0, sacc = 0.0;
  bool bad = false;
  const int64_t ntiles = (a.n + T - 1) / T;
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int64_t row0 = t * T;
    const int rows = (int)((a.n - row0 < T) ? (a.n - row0) : T);
    __syncthreads();
    const double* src = a.phi + row0 * r;
    const int cnt = rows * r;
    for (int e = tid; e < cnt; e += TS_NT) {
      const int rr = e / r, cc = e - rr * r;
      const double vph = src[e];
      bad |= !isfinite(vph);
      tile[rr * S + cc] = vph;
    }
    __syncthreads();
    // phase 1: one thread per row
    if (tid < rows) {
      const int64_t i = row0 + tid;
      double rd = 0.0;
      if (ROWDOT) {
        const double* trow = tile + tid * S;
#pragma unroll 8
        for (int k = 0; k < r; ++k) rd += trow[k] * vv[k];
      }
      if (DECODE) a.out_q[i] = a.q_ref[i] + rd / a.d[i];
      double w = 0.0;
      if (WKIND == W_X) w = a.x[i];
      if (WKIND == W_ENCODE) w = a.d[i] * (a.x[i] - a.q_ref[i]);
      if (WKIND == W_RESID) w = a.x[i] - rd;
      if (WKIND != W_NONE) {
        bad |= !isfinite(w);
        sacc += w * w;
        ww[tid] = w;
      }
    }
    if (WKIND != W_NONE) {
      __syncthreads();
      // phase 2: column sums, thread (grp, col) takes rows grp, grp+RS, ...
      if (colthread) {
        for (int rr = grp; rr < rows; rr += RS) acc += tile[rr * S + col] * ww[rr];
      }
    }
  }
  if (WKIND == W_NONE) {
    if (bad && a.flag) atomicOr(a.flag, 1);
    return;
  }
  __syncthreads();
  red[tid] = colthread ? acc : 0.0;
  __syncthreads();
  double* out = a.partial + (size_t)blockIdx.x * (r + 1);
  for (int j = tid; j < r; j += TS_NT) {
    double s = 0.0;
    for (int g = 0; g < RS; ++g) s += red[g * r + j];
    out[j] = s;
  }
  __syncthreads();
  const double tot = block_sum<TS_NT>(sacc, red);
  if (tid == 0) out[r] = tot;
  if (bad && a.flag) atomicOr(a.flag, 1);
}

// out[j] = sum_b partial[b*(w) + j], one block per j (deterministic tree)
__global__ void reduce_partials_kernel(const double* __restrict__ partial, int nb, int w,
                                       double* __restrict__ out, const int* skip) {
  __shared__ double red[32];
  if (skip && *skip == 0) return;
  const int j = blockIdx.x;
  double s = 0.0;
  for (int b = threadIdx.x; b < nb; b += blockDim.x) s += partial[(size_t)b * w + j];
  s = block_sum<256>(s, red);
  if (threadIdx.x == 0) out[j] = s;
}

static size_t tile_smem(int r) {
  const int T = ts_tile_rows(r);
  return sizeof(double) * ((size_t)T * ts_stride(r) + r + T + TS_NT);
}

static int tile_grid(adrom_ctx* ctx, int64_t n, int r) {
  const int64_t ntiles = (n + ts_tile_rows(r) - 1) / ts_tile_rows(r);
  int64_t g = (int64_t)ctx->num_sms * 3;
  if (g > ntiles) g = ntiles;
  return (int)(g < 1 ? 1 : g);
}

template <bool ROWDOT, bool DECODE, int WKIND>
static int launch_tile(adrom_ctx* ctx, const TileArgs& a, int grid) {
  const size_t sm = tile_smem(a.r);
  static bool attr_done = false;
  if (!attr_done) {
    cudaFuncSetAttribute(tile_kernel<ROWDOT, DECODE, WKIND>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    attr_done = true;
  }
  tile_kernel<ROWDOT, DECODE, WKIND><<<grid, TS_NT, sm, ctx->stream>>>(a);
  ADROM_LAUNCH_CK(ctx);
  return ADROM_OK;
}

static int check_r(adrom_ctx* ctx, int r) {
  if (r < 1 || r > 256) return set_error(ctx, ADROM_ERR_ARG, "basis rank %d outside [1, 256]", r);
  return ADROM_OK;
}

// out[0..r) = phi^T w, out[r] = sum w^2  (w per WKIND); blocking-free
int ts_project(adrom_ctx* ctx, const double* phi, int64_t n, int r, int wkind, const double* x,
               const double* q_ref, const double* d, double* out, double* partial, int* flag) {
  int st = check_r(ctx, r);
  if (st) return st;
  TileArgs a{};
  a.phi = phi;
  a.n = n;
  a.r = r;
  a.x = x;
  a.q_ref = q_ref;
  a.d = d;
  a.partial = partial;
  a.flag = flag;
  const int grid = tile_grid(ctx, n, r);
  if (wkind == W_X)
    st = launch_tile<false, false, W_X>(ctx, a, grid);
  else
    st = launch_tile<false, false, W_ENCODE>(ctx, a, grid);
  if (st) return st;
  reduce_partials_kernel<<<r + 1, 256, 0, ctx->stream>>>(partial, grid, r + 1, out, nullptr);
  ADROM_LAUNCH_CK(ctx);
  return ADROM_OK;
}

int ts_decode(adrom_ctx* ctx, const double* phi, int64_t n, int r, const double* a_vec,
              const double* q_ref, const double* d, double* q_out) {
  int st = check_r(ctx, r);
  if (st) return st;
  TileArgs a{};
  a.phi = phi;
  a.n = n;
  a.r = r;
  a.v = a_vec;
  a.q_ref = q_ref;
  a.d = d;
  a.out_q = q_out;
  return launch_tile<true, true, W_NONE>(ctx, a, tile_grid(ctx, n, r));
}

// fused: q_out = decode(a) and [phi^T y, ||y||^2] partials -> out
int ts_decode_project(adrom_ctx* ctx, const double* phi, int64_t n, int r, const double* a_vec,
                      const double* q_ref, const double* d, double* q_out, const double* y,
                      double* out, double* partial, int* flag) {
  int st = check_r(ctx, r);
  if (st) return st;
  TileArgs a{};
  a.phi = phi;
  a.n = n;
  a.r = r;
  a.v = a_vec;
  a.q_ref = q_ref;
  a.d = d;
  a.out_q = q_out;
  a.x = y;
  a.partial = partial;
  a.flag = flag;
  const int grid = tile_grid(ctx, n, r);
  // ROWDOT with the decode vector, weights = y (W_X); DECODE writes q_out
  st = launch_tile<true, true, W_X>(ctx, a, grid);
  if (st) return st;
  reduce_partials_kernel<<<r + 1, 256, 0, ctx->stream>>>(partial, grid, r + 1, out, nullptr);
  ADROM_LAUNCH_CK(ctx);
  return ADROM_OK;
}

// residual pass: q = y - phi p ; out = [phi^T q, ||q||^2]; no-op if *skip == 0
int ts_residual(adrom_ctx* ctx, const double* phi, int64_t n, int r, const double* p,
                const double* y, double* out, double* partial, int* flag, const int* skip) {
  TileArgs a{};
  a.phi = phi;
  a.n = n;
  a.r = r;
  a.v = p;
  a.x = y;
  a.partial = partial;
  a.flag = flag;
  a.skip = skip;
  const int grid = tile_grid(ctx, n, r);
  int st = launch_tile<true, false, W_RESID>(ctx, a, grid);
  if (st) return st;
  reduce_partials_kernel<<<r + 1, 256, 0, ctx->stream>>>(partial, grid, r + 1, out, skip);
  ADROM_LAUNCH_CK(ctx);
  return ADROM_OK;
}

// ---------------------------------------------------------------------------
// rotation  out = [phi | y] [M ; b^T]   (tracking.py:176-177 with q_hat
// formed on the fly: [phi, q/||q||] U = phi (U_top - p u_bot^T/||q||) +
// y u_bot^T/||q||).  out may alias phi (each block stages its rows first).
// ---------------------------------------------------------------------------
template <int R>
struct RotCfg {
  static constexpr int TM = (R <= 64) ? 128 : 64;  // rows per tile
  static constexpr int RM = TM / 16;               // rows per thread
  static constexpr int RN = R / 16;                // cols per thread
  static constexpr int SA = R + 1;                 // odd smem stride
};

template <int R>
__global__ void __launch_bounds__(256) rot_tiled_kernel(const double* __restrict__ phi,
                                                        const double* __restrict__ y,
                                                        const double* __restrict__ M,
                                                        const double* __restrict__ b, int64_t n,
                                                        double* out) {
  using C = RotCfg<R>;
  extern __shared__ double sm[];
  double* As = sm;                    // TM x SA  (col R = y)
  double* Bs = As + C::TM * C::SA;    // (R+1) x R
  const int tid = threadIdx.x;
  for (int e = tid; e < R * R; e += 256) Bs[e] = M[e];
  for (int e = tid; e < R; e += 256) Bs[R * R + e] = b[e];
  const int rg = tid >> 4, cg = tid & 15;
  const int64_t ntiles = (n + C::TM - 1) / C::TM;
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int64_t row0 = t * C::TM;
    const int rows = (int)((n - row0 < C::TM) ? (n - row0) : C::TM);
    __syncthreads();
    const double2* src = reinterpret_cast<const double2*>(phi + row0 * R);
    const int cnt2 = rows * R / 2;
    for (int e = tid; e < cnt2; e += 256) {
      const double2 v = src[e];
      const int rr = (2 * e) / R, cc = (2 * e) - rr * R;
      As[rr * C::SA + cc] = v.x;
      As[rr * C::SA + cc + 1] = v.y;
    }
    for (int e = tid; e < C::TM; e += 256) As[e * C::SA + R] = (e < rows) ? y[row0 + e] : 0.0;
    __syncthreads();
    double acc[C::RM][C::RN];
#pragma unroll
    for (int m = 0; m < C::RM; ++m)
#pragma unroll
      for (int q = 0; q < C::RN; ++q) acc[m][q] = 0.0;
#pragma unroll 4
    for (int k = 0; k <= R; ++k) {
      double av[C::RM], bv[C::RN];
#pragma unroll
      for (int m = 0; m < C::RM; ++m) av[m] = As[(rg * C::RM + m) * C::SA + k];
#pragma unroll
      for (int q = 0; q < C::RN; ++q) bv[q] = Bs[k * R + cg * C::RN + q];
#pragma unroll
      for (int m = 0; m < C::RM; ++m)
#pragma unroll
        for (int q = 0; q < C::RN; ++q) acc[m][q] = fma(av[m], bv[q], acc[m][q]);
    }
    // the tile is fully consumed before any row of it is overwritten
    __syncthreads();
#pragma unroll
    for (int m = 0; m < C::RM; ++m) {
      const int rr = rg * C::RM + m;
      if (rr < rows) {
        double* dst = out + (row0 + rr) * R + cg * C::RN;
#pragma unroll
        for (int q = 0; q < C::RN; ++q) dst[q] = acc[m][q];
      }
    }
  }
}

// generic sizes: out (n x r_out) = phi (n x r_in) M (r_in x r_out) + y b^T
__global__ void __launch_bounds__(256) rot_generic_kernel(const double* __restrict__ phi,
                                                          const double* __restrict__ y,
                                                          const double* __restrict__ M,
                                                          const double* __restrict__ b,
                                                          int64_t n, int r_in, int r_out,
                                                          double* out) {
  extern __shared__ double sm[];
  const int T = 32;
  const int S = r_in + 1;
  double* As = sm;           // T x S
  double* Bs = As + T * S;   // (r_in+1) x r_out
  const int tid = threadIdx.x;
  for (int e = tid; e < r_in * r_out; e += 256) Bs[e] = M[e];
  for (int e = tid; e < r_out; e += 256) Bs[r_in * r_out + e] = b[e];
  const int64_t ntiles = (n + T - 1) / T;
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int64_t row0 = t * T;
    const int rows = (int)((n - row0 < T) ? (n - row0) : T);
    __syncthreads();
    for (int e = tid; e < rows * r_in; e += 256) {
      const int rr = e / r_in, cc = e - rr * r_in;
      As[rr * S + cc] = phi[row0 * r_in + e];
    }
    for (int e = tid; e < rows; e += 256) As[e * S + r_in] = y[row0 + e];
    __syncthreads();
    double res[32];
    int cntv = 0;
    for (int e = tid; e < rows * r_out; e += 256) {
      const int rr = e / r_out, cc = e - rr * r_out;
      double s = 0.0;
      for (int k = 0; k <= r_in; ++k) s = fma(As[rr * S + k], Bs[k * r_out + cc], s);
      res[cntv++] = s;
    }
    __syncthreads();
    cntv = 0;
    for (int e = tid; e < rows * r_out; e += 256) out[row0 * r_out + e] = res[cntv++];
  }
}

int ts_rotate(adrom_ctx* ctx, const double* phi, const double* y, const double* M,
              const double* b, int64_t n, int r_in, int r_out, double* out) {
  if (r_in == r_out && (r_in == 16 || r_in == 32 || r_in == 64 || r_in == 128)) {
    int64_t g = (int64_t)ctx->num_sms * 2;
    auto launch = [&](auto kern, int TM, int R) -> int {
      const size_t sm = sizeof(double) * ((size_t)TM * (R + 1) + (size_t)(R + 1) * R);
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      const int64_t nt = (n + TM - 1) / TM;
      const int64_t gg = g < nt ? g : nt;
      kern<<<(int)(gg < 1 ? 1 : gg), 256, sm, ctx->stream>>>(phi, y, M, b, n, out);
      ADROM_LAUNCH_CK(ctx);
      return ADROM_OK;
    };
    if (r_in == 16) return launch(rot_tiled_kernel<16>, RotCfg<16>::TM, 16);
    if (r_in == 32) return launch(rot_tiled_kernel<32>, RotCfg<32>::TM, 32);
    if (r_in == 64) return launch(rot_tiled_kernel<64>, RotCfg<64>::TM, 64);
    return launch(rot_tiled_kernel<128>, RotCfg<128>::TM, 128);
  }
  if (r_in > 256 || r_out > 256)
    return set_error(ctx, ADROM_ERR_ARG, "rotation size %d x %d unsupported", r_in, r_out);
  const size_t sm = sizeof(double) * ((size_t)32 * (r_in + 1) + (size_t)(r_in + 1) * r_out);
  cudaFuncSetAttribute(rot_generic_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  int64_t g = (int64_t)ctx->num_sms * 4, nt = (n + 31) / 32;
  if (g > nt) g = nt;
  rot_generic_kernel<<<(int)(g < 1 ? 1 : g), 256, sm, ctx->stream>>>(phi, y, M, b, n, r_in,
                                                                     r_out, out);
  ADROM_LAUNCH_CK(ctx);
  return ADROM_OK;
}

// ---------------------------------------------------------------------------
// iSVD core (one block): K, its SVD, the rotation factors
// ---------------------------------------------------------------------------
// stats layout (doubles): [0] qnorm [1] ynorm [2] proj_resid [3] degenerate
//                         [4] reorth [5] sweeps [6] converged [7] nonfinite
__global__ void isvd_decide_kernel(const double* __restrict__ red1, int r, double ratio,
                                   int* __restrict__ need) {
  // red1 = [p (r), ||y||^2]
  double pp = 0.0;
  for (int j = 0; j < r; ++j) pp += red1[j] * red1[j];
  const double yy = red1[r];
  const double est = yy - pp;
  *need = (est > ratio * yy) ? 0 : 1;
}

__global__ void __launch_bounds__(1024) isvd_core_kernel(
    const double* __restrict__ sigma, const double* __restrict__ red1,
    const double* __restrict__ red2, const int* __restrict__ need, int r_cur, int r, double lam,
    double* __restrict__ Mout, double* __restrict__ bout, double* __restrict__ sigma_out,
    double* __restrict__ stats, int* __restrict__ flag) {
  extern __shared__ double sm[];
  const int n = r_cur + 1;
  const int ld = n + ((n & 1) ? 0 : 1);  // odd leading dimension
  double* A = sm;            // n x ld (column-major: column j = row j of K)
  double* V = A + n * ld;    // n x ld
  double* p = V + n * ld;    // r_cur
  double* s = p + r_cur;     // n
  int* order = (int*)(s + n);
  __shared__ int sh_flag;
  __shared__ double sh_q[4];
  const int tid = threadIdx.x;
  const bool reorth = need[0] != 0;
  if (tid == 0) {
    double yy = red1[r_cur], pp = 0.0;
    double qq, proj;
    if (reorth) {
      double p2 = 0.0;
      for (int j = 0; j < r_cur; ++j) p2 += red2[j] * red2[j];
      proj = red2[r_cur];    // ||y - Phi Phi^T y||^2
      qq = proj - p2;        // ||q||^2 after one re-orthogonalisation
    } else {
      for (int j = 0; j < r_cur; ++j) pp += red1[j] * red1[j];
      proj = yy - pp;
      qq = proj;
    }
    sh_q[0] = sqrt(qq > 0.0 ? qq : 0.0);
    sh_q[1] = sqrt(yy);
    sh_q[2] = sqrt(proj > 0.0 ? proj : 0.0);
  }
  for (int j = tid; j < r_cur; j += blockDim.x) p[j] = red1[j] + (reorth ? red2[j] : 0.0);
  __syncthreads();
  const double qnorm = sh_q[0], ynorm = sh_q[1];
  // tracking.py:169 — degenerate residual keeps the subspace
  const bool degenerate = qnorm <= 1e-12 * fmax(ynorm, 1e-300);
  for (int e = tid; e < n * ld; e += blockDim.x) A[e] = 0.0;
  __syncthreads();
  bool bad = false;
  for (int j = tid; j < r_cur; j += blockDim.x) {
    const double dj = lam * sigma[j];
    A[j * ld + j] = dj;       // K[j][j]   (tracking.py:167)
    A[j * ld + r_cur] = p[j]; // K[j][r]   (tracking.py:168)
    bad |= !isfinite(dj) || !isfinite(p[j]);
  }
  if (tid == 0) {
    A[r_cur * ld + r_cur] = degenerate ? 0.0 : qnorm;  // tracking.py:172
    bad |= !isfinite(qnorm) || !isfinite(ynorm);
  }
  if (bad) atomicOr(flag, 1);
  __syncthreads();
  const JacobiResult jr = block_jacobi(A, ld, n, n, V, ld, 60, 1e-15, &sh_flag);
  column_norms_sorted(A, ld, n, n, s, order);
  // M[k][c] = U_top[k][order[c]] - p_k u_bot[order[c]] / qnorm ; b[c] = u_bot/qnorm
  const double inv = degenerate ? 0.0 : 1.0 / qnorm;
  for (int e = tid; e < r_cur * r; e += blockDim.x) {
    const int k = e / r, c = e - k * r;
    const int jc = order[c];
    const double ub = V[jc * ld + r_cur];
    Mout[e] = V[jc * ld + k] - (degenerate ? 0.0 : p[k] * ub * inv);
  }
  for (int c = tid; c < r; c += blockDim.x) {
    const int jc = order[c];
    bout[c] = degenerate ? 0.0 : V[jc * ld + r_cur] * inv;
  }
  __syncthreads();
  for (int c = tid; c < r; c += blockDim.x) sigma_out[c] = s[order[c]];
  if (tid == 0) {
    stats[0] = qnorm;
    stats[1] = ynorm;
    stats[2] = sh_q[2];
    stats[3] = degenerate ? 1.0 : 0.0;
    stats[4] = reorth ? 1.0 : 0.0;
    stats[5] = jr.sweeps;
    stats[6] = jr.converged;
    if (!jr.converged) atomicOr(flag, 8);
  }
}

static size_t core_smem(int r_cur) {
  const int n = r_cur + 1;
  const int ld = n + ((n & 1) ? 0 : 1);
  return sizeof(double) * (2 * (size_t)n * ld + r_cur + n) + sizeof(int) * n + 64;
}

size_t isvd_workspace_bytes(adrom_ctx* ctx, int64_t n, int r_cur, int r) {
  const int64_t grid = (int64_t)ctx->num_sms * 3;
  size_t b = 0;
  b += align_up(sizeof(double) * grid * (r_cur + 1));  // partials
  b += 2 * align_up(sizeof(double) * (r_cur + 1));     // red1, red2
  b += align_up(sizeof(double) * r_cur * r);           // M
  b += align_up(sizeof(double) * r);                   // b
  b += align_up(sizeof(double) * 16);                  // stats
  b += align_up(sizeof(int) * 4);                      // need
  (void)n;
  return b;
}

int isvd_update_async(adrom_ctx* ctx, const double* phi, const double* sigma, const double* y,
                      int64_t n, int r_cur, int r, double lam, double* phi_out,
                      double* sigma_out, void* ws, int* flag, double reorth_ratio,
                      double* stats_out, const double* dec_a, const double* q_ref,
                      const double* d, double* dec_out) {
  if (r_cur < 1 || r_cur > 110 || r < 1 || r > r_cur + 1)
    return set_error(ctx, ADROM_ERR_ARG, "isvd_update: bad ranks r_cur=%d r=%d", r_cur, r);
  if (phi_out == phi && r != r_cur)
    return set_error(ctx, ADROM_ERR_ARG, "isvd_update: in-place update needs r == r_cur");
  char* w = (char*)ws;
  const int64_t grid = (int64_t)ctx->num_sms * 3;
  double* partial = (double*)w;
  w += align_up(sizeof(double) * grid * (r_cur + 1));
  double* red1 = (double*)w;
  w += align_up(sizeof(double) * (r_cur + 1));
  double* red2 = (double*)w;
  w += align_up(sizeof(double) * (r_cur + 1));
  double* M = (double*)w;
  w += align_up(sizeof(double) * r_cur * r);
  double* bv = (double*)w;
  w += align_up(sizeof(double) * r);
  double* stats = stats_out ? stats_out : (double*)w;
  w += align_up(sizeof(double) * 16);
  int* need = (int*)w;
  int st;
  // pass 1: p = Phi^T y, ||y||^2 (+ fused decode of the ROM state if asked)
  if (dec_a)
    st = ts_decode_project(ctx, phi, n, r_cur, dec_a, q_ref, d, dec_out, y, red1, partial, flag);
  else
    st = ts_project(ctx, phi, n, r_cur, W_X, y, nullptr, nullptr, red1, partial, flag);
  if (st) return st;
  isvd_decide_kernel<<<1, 1, 0, ctx->stream>>>(red1, r_cur, reorth_ratio, need);
  ADROM_LAUNCH_CK(ctx);
  // pass 2 (only if cancellation threatens ||q||): q = y - Phi p, Phi^T q, ||q||^2
  st = ts_residual(ctx, phi, n, r_cur, red1, y, red2, partial, flag, need);
  if (st) return st;
  const size_t csm = core_smem(r_cur);
  cudaFuncSetAttribute(isvd_core_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)csm);
  isvd_core_kernel<<<1, 1024, csm, ctx->stream>>>(sigma, red1, red2, need, r_cur, r, lam, M, bv,
                                                  sigma_out, stats, flag);
  ADROM_LAUNCH_CK(ctx);
  return ts_rotate(ctx, phi, y, M, bv, n, r_cur, r, phi_out);
}

// ---------------------------------------------------------------------------
// thin SVD of a small dense matrix (dense.py:59-72), one block
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(1024) small_svd_kernel(const double* __restrict__ a, int m,
                                                         int n, double* __restrict__ u,
                                                         double* __restrict__ s_out,
                                                         double* __restrict__ v, int* flag) {
  extern __shared__ double sm[];
  // work on B = a (m >= n) or B = a^T (m < n): B is mm x nn with mm >= nn
  const bool tr = m < n;
  const int mm = tr ? n : m, nn = tr ? m : n;
  const int ld = mm | 1, ldv = nn | 1;
  double* B = sm;                 // nn columns of length mm
  double* V = B + (size_t)nn * ld;
  double* s = V + (size_t)nn * ldv;
  int* order = (int*)(s + nn);
  __shared__ int sh_flag;
  bool bad = false;
  for (int e = threadIdx.x; e < m * n; e += blockDim.x) {
    const int i = e / n, j = e - i * n;  // a[i][j]
    const double x = a[e];
    bad |= !isfinite(x);
    if (!tr) B[j * ld + i] = x;
    else B[i * ld + j] = x;
  }
  if (bad) atomicOr(flag, 1);
  __syncthreads();
  const JacobiResult jr = block_jacobi(B, ld, mm, nn, V, ldv, 60, 1e-15, &sh_flag);
  if (!jr.converged && threadIdx.x == 0) atomicOr(flag, 8);
  column_norms_sorted(B, ld, mm, nn, s, order);
  // B = U_B S V_B^T with U_B = W/s.  a = B (tr=0): u = U_B, v = V_B;
  // a = B^T (tr=1): u = V_B, v = U_B.  k = nn.
  for (int e = threadIdx.x; e < mm * nn; e += blockDim.x) {
    const int i = e / nn, c = e - i * nn;
    const int jc = order[c];
    const double sv = s[jc];
    const double wv = (sv > 0.0) ? B[jc * ld + i] / sv : 0.0;
    if (!tr) u[i * nn + c] = wv;
    else v[i * nn + c] = wv;
  }
  for (int e = threadIdx.x; e < nn * nn; e += blockDim.x) {
    const int i = e / nn, c = e - i * nn;
    const double vv = V[order[c] * ldv + i];
    if (!tr) v[i * nn + c] = vv;
    else u[i * nn + c] = vv;
  }
  for (int c = threadIdx.x; c < nn; c += blockDim.x) s_out[c] = s[order[c]];
}

int dense_small_svd(adrom_ctx* ctx, const double* a, int m, int n, double* u, double* s,
                    double* v, int* flag) {
  if (m < 1 || n < 1) return set_error(ctx, ADROM_ERR_DENSE, "thin_svd expects a non-empty 2-d array");
  const int mm = m < n ? n : m, nn = m < n ? m : n;
  const size_t sm = sizeof(double) * ((size_t)nn * (mm | 1) + (size_t)nn * (nn | 1) + nn) +
                    sizeof(int) * nn + 64;
  if (sm > 220 * 1024)
    return set_error(ctx, ADROM_ERR_ARG, "small_svd: %d x %d too large for one block", m, n);
  cudaFuncSetAttribute(small_svd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  small_svd_kernel<<<1, 1024, sm, ctx->stream>>>(a, m, n, u, s, v, flag);
  ADROM_LAUNCH_CK(ctx);
  return ADROM_OK;
}

}  // namespace adrom
