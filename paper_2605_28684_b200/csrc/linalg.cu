// Tall-skinny basis kernels (kernel 3), the iSVD update (kernel 4) and the
// one-block dense SVD.  Compiled WITH FMA contraction: these are reductions
// whose order differs from BLAS anyway; FMA only improves them.
#include "common.cuh"
#include "jacobi.cuh"
#include "secular.cuh"
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
  double* out_w;        // if non-null: out_w[i] = w_i (the iSVD residual q)
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
        if (a.out_w) a.out_w[i] = w;
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


// ---------------------------------------------------------------------------
// streaming variant for r in {16, 32, 64, 128}: one row per LPR lanes,
// 16-byte loads straight from global (no smem staging), U rows in flight per
// lane.  Same semantics as tile_kernel.
// ---------------------------------------------------------------------------
template <int R, bool ROWDOT, bool DECODE, int WKIND>
__global__ void __launch_bounds__(256) stream_kernel(TileArgs a) {
  constexpr int LPR = R / 8;                   // lanes per row (8 columns each)
  constexpr int RPW = 32 / LPR;                // rows per warp per sub-iteration
  constexpr int U = 4;                         // sub-iterations in flight
  __shared__ double red[8 * R];
  __shared__ double sred[32];
  if (a.skip && *a.skip == 0) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int seg = lane / LPR, sl = lane - seg * LPR;
  // lane columns: 2 (sl + LPR h) + {0, 1}, h < 4
  double2 vv[4];
  if (ROWDOT) {
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      vv[h].x = a.v[2 * (sl + LPR * h)];
      vv[h].y = a.v[2 * (sl + LPR * h) + 1];
    }
  }
  double2 acc[4];
#pragma unroll
  for (int h = 0; h < 4; ++h) acc[h] = make_double2(0.0, 0.0);
  double sacc = 0.0;
  bool bad = false;
  const int64_t total_warps = (int64_t)gridDim.x * 8;
  const int64_t rows_per_iter = (int64_t)RPW * U;
  for (int64_t g = (int64_t)blockIdx.x * 8 + warp; g * rows_per_iter < a.n; g += total_warps) {
    const int64_t base = g * rows_per_iter;
    double2 val[U][4];
    double xw[U], qr[U], dd[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = base + u * RPW + seg;
      const bool live = i < a.n;
      if (live) {
        const double2* rowp = reinterpret_cast<const double2*>(a.phi + i * R);
#pragma unroll
        for (int h = 0; h < 4; ++h) val[u][h] = rowp[sl + LPR * h];
      } else {
#pragma unroll
        for (int h = 0; h < 4; ++h) val[u][h] = make_double2(0.0, 0.0);
      }
      xw[u] = (WKIND != W_NONE && live) ? a.x[i] : 0.0;
      qr[u] = ((DECODE || WKIND == W_ENCODE) && live) ? a.q_ref[i] : 0.0;
      dd[u] = ((DECODE || WKIND == W_ENCODE) && live) ? a.d[i] : 1.0;
    }
    double rd[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      double t = 0.0;
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        bad |= !(isfinite(val[u][h].x) && isfinite(val[u][h].y));
        if (ROWDOT) t += val[u][h].x * vv[h].x + val[u][h].y * vv[h].y;
      }
      rd[u] = t;
    }
    if (ROWDOT) {
#pragma unroll
      for (int o = LPR / 2; o > 0; o >>= 1)
#pragma unroll
        for (int u = 0; u < U; ++u) rd[u] += __shfl_xor_sync(0xffffffffu, rd[u], o);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = base + u * RPW + seg;
      const bool live = i < a.n;
      if (DECODE && live && sl == 0) a.out_q[i] = qr[u] + rd[u] / dd[u];
      if (WKIND != W_NONE && live) {
        double w;
        if (WKIND == W_X) w = xw[u];
        else if (WKIND == W_ENCODE) w = dd[u] * (xw[u] - qr[u]);
        else w = xw[u] - rd[u];
        bad |= !isfinite(w);
        if (sl == 0) {
          sacc += w * w;
          if (a.out_w) a.out_w[i] = w;
        }
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          acc[h].x += val[u][h].x * w;
          acc[h].y += val[u][h].y * w;
        }
      }
    }
  }
  if (WKIND == W_NONE) {
    if (bad && a.flag) atomicOr(a.flag, 1);
    return;
  }
  // fold segments sharing columns, then warps
#pragma unroll
  for (int o = LPR; o < 32; o <<= 1)
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      acc[h].x += __shfl_xor_sync(0xffffffffu, acc[h].x, o);
      acc[h].y += __shfl_xor_sync(0xffffffffu, acc[h].y, o);
    }
  if (seg == 0) {
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      red[warp * R + 2 * (sl + LPR * h)] = acc[h].x;
      red[warp * R + 2 * (sl + LPR * h) + 1] = acc[h].y;
    }
  }
  __syncthreads();
  double* out = a.partial + (size_t)blockIdx.x * (R + 1);
  for (int c = threadIdx.x; c < R; c += 256) {
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < 8; ++w) s += red[w * R + c];
    out[c] = s;
  }
  const double tot = block_sum<256>(sacc, sred);
  if (threadIdx.x == 0) out[R] = tot;
  if (bad && a.flag) atomicOr(a.flag, 1);
}

template <int R, bool ROWDOT, bool DECODE, int WKIND>
static int launch_stream_t(adrom_ctx* ctx, const TileArgs& a, int grid) {
  stream_kernel<R, ROWDOT, DECODE, WKIND><<<grid, 256, 0, ctx->stream>>>(a);
  ADROM_LAUNCH_CK(ctx);
  return ADROM_OK;
}

static bool stream_ok(int r) { return r == 16 || r == 32 || r == 64 || r == 128; }

static int stream_grid(adrom_ctx* ctx, int64_t n) {
  int64_t g = (int64_t)ctx->num_sms * 4;
  const int64_t need = (n + 31) / 32;
  if (g > need) g = need;
  return (int)(g < 1 ? 1 : g);
}

template <bool ROWDOT, bool DECODE, int WKIND>
static int launch_stream(adrom_ctx* ctx, const TileArgs& a, int grid) {
  switch (a.r) {
    case 16: return launch_stream_t<16, ROWDOT, DECODE, WKIND>(ctx, a, grid);
    case 32: return launch_stream_t<32, ROWDOT, DECODE, WKIND>(ctx, a, grid);
    case 64: return launch_stream_t<64, ROWDOT, DECODE, WKIND>(ctx, a, grid);
    default: return launch_stream_t<128, ROWDOT, DECODE, WKIND>(ctx, a, grid);
  }
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
  const bool fast = stream_ok(r);
  const int grid = fast ? stream_grid(ctx, n) : tile_grid(ctx, n, r);
  if (fast)
    st = (wkind == W_X) ? launch_stream<false, false, W_X>(ctx, a, grid)
                        : launch_stream<false, false, W_ENCODE>(ctx, a, grid);
  else if (wkind == W_X)
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
  if (stream_ok(r)) return launch_stream<true, true, W_NONE>(ctx, a, stream_grid(ctx, n));
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
  const bool fast = stream_ok(r);
  const int grid = fast ? stream_grid(ctx, n) : tile_grid(ctx, n, r);
  // ROWDOT with the decode vector, weights = y (W_X); DECODE writes q_out
  st = fast ? launch_stream<true, true, W_X>(ctx, a, grid) : launch_tile<true, true, W_X>(ctx, a, grid);
  if (st) return st;
  reduce_partials_kernel<<<r + 1, 256, 0, ctx->stream>>>(partial, grid, r + 1, out, nullptr);
  ADROM_LAUNCH_CK(ctx);
  return ADROM_OK;
}

// residual pass: q = y - phi p (stored to qbuf if non-null);
// out = [phi^T q, ||q||^2]; no-op if *skip == 0
int ts_residual(adrom_ctx* ctx, const double* phi, int64_t n, int r, const double* p,
                const double* y, double* out, double* partial, int* flag, const int* skip,
                double* qbuf) {
  TileArgs a{};
  a.phi = phi;
  a.n = n;
  a.r = r;
  a.v = p;
  a.x = y;
  a.partial = partial;
  a.flag = flag;
  a.skip = skip;
  a.out_w = qbuf;
  const bool fast = stream_ok(r);
  const int grid = fast ? stream_grid(ctx, n) : tile_grid(ctx, n, r);
  int st = fast ? launch_stream<true, false, W_RESID>(ctx, a, grid)
                : launch_tile<true, false, W_RESID>(ctx, a, grid);
  if (st) return st;
  reduce_partials_kernel<<<r + 1, 256, 0, ctx->stream>>>(partial, grid, r + 1, out, skip);
  ADROM_LAUNCH_CK(ctx);
  return ADROM_OK;
}

// ---------------------------------------------------------------------------
// rotation  out = [phi | q_hat] [U_top ; u_bot^T]     (tracking.py:176-177)
// q_hat_i = q_i / ||q|| with q_i read from the residual pass (qbuf) or formed
// here as y_i - phi_i . p from the staged tile; the same q feeds the Gram
// update, so the tracked Phi^T Phi stays consistent with the rotated basis.
// out may alias phi (each block stages its rows before writing them).
// ---------------------------------------------------------------------------
struct RotArgs {
  const double* phi;
  const double* y;
  const double* qbuf;   // may be null
  const int* need;      // q is read from qbuf iff *need (null: iff qbuf)
  const double* p;      // r_in (used when q is formed here)
  const double* qinv;   // device scalar 1/||q|| (0 when degenerate)
  const double* B;      // (r_in + 1) x r_out row-major: [U_top ; u_bot]
  int64_t n;
  int r_in, r_out;
  double* out;
  RotFuse fuse;  // fused epilogue work (rot_tc_kernel only)
  const double* p2 = nullptr;  // least-squares refinement (r_in; null = none):
                               // with q from qbuf, q_hat = (qbuf - phi p2) qinv
};

template <int R>
struct RotCfg {
  static constexpr int TM = (R <= 64) ? 128 : 64;  // rows per tile
  static constexpr int RM = TM / 16;               // rows per thread
  static constexpr int RN = R / 16;                // cols per thread
  static constexpr int SA = R + 1;                 // odd smem stride
};

template <int R>
__global__ void __launch_bounds__(256) rot_tiled_kernel(RotArgs a) {
  using C = RotCfg<R>;
  extern __shared__ double sm[];
  double* As = sm;                    // TM x SA  (col R = q_hat)
  double* Bs = As + C::TM * C::SA;    // (R+1) x R
  double* ps = Bs + (R + 1) * R;      // R
  const int tid = threadIdx.x;
  const bool use_q = a.qbuf && (a.need == nullptr || *a.need != 0);
  for (int e = tid; e < (R + 1) * R; e += 256) Bs[e] = a.B[e];
  for (int e = tid; e < R; e += 256) ps[e] = use_q ? (a.p2 ? a.p2[e] : 0.0) : a.p[e];
  const bool dot = !use_q || a.p2 != nullptr;
  const double qinv = *a.qinv;
  const int rg = tid >> 4, cg = tid & 15;
  const int64_t n = a.n;
  const int64_t ntiles = (n + C::TM - 1) / C::TM;
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int64_t row0 = t * C::TM;
    const int rows = (int)((n - row0 < C::TM) ? (n - row0) : C::TM);
    __syncthreads();
    const double2* src = reinterpret_cast<const double2*>(a.phi + row0 * R);
    const int cnt2 = rows * R / 2;
    for (int e = tid; e < cnt2; e += 256) {
      const double2 v = src[e];
      const int rr = (2 * e) / R, cc = (2 * e) - rr * R;
      As[rr * C::SA + cc] = v.x;
      As[rr * C::SA + cc + 1] = v.y;
    }
    __syncthreads();
    for (int e = tid; e < C::TM; e += 256) {
      double qh = 0.0;
      if (e < rows) {
        double s = 0.0;
        if (dot)
          for (int k = 0; k < R; ++k) s = fma(As[e * C::SA + k], ps[k], s);
        const double qv = (use_q ? a.qbuf[row0 + e] : a.y[row0 + e]) - s;
        qh = qv * qinv;
      }
      As[e * C::SA + R] = qh;
    }
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
      for (int q = 0; q < C::RN; ++q) bv[q] = Bs[k * R + cg + 16 * q];  // conflict-free
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
        double* dst = a.out + (row0 + rr) * R + cg;
#pragma unroll
        for (int q = 0; q < C::RN; ++q) dst[16 * q] = acc[m][q];
      }
    }
  }
}

// ---------------------------------------------------------------------------
// FP64 tensor-core rotation (R in {32, 64, 128}): out = [phi | q_hat] B on DMMA
// (mma.sync m8n8k4 f64).  64-row tiles double-buffered in smem by cp.async
// (row stride R + 4: conflict-free fragment loads; column R holds q_hat);
// 8 warps as 4 (rows) x 2 (cols), each warp 16 rows x R/2 columns; two
// blocks per SM so one block's epilogue overlaps the other's MMAs.  The
// q_hat column is a rank-1 FMA update in the epilogue.
// ---------------------------------------------------------------------------
template <int R>
struct RotTC {
  // R <= 64: 64-row tiles, 2 blocks per SM; R = 128: 32-row tiles (B alone is
  // 132 KB of smem), 1 block per SM with 8 warps as 2 (rows) x 4 (cols)
  static constexpr int TM = R <= 64 ? 64 : 32;  // rows per tile
  static constexpr int WGN = R <= 64 ? 2 : 4;   // column groups of warps
  static constexpr int MT = 2;             // 8-row tiles per warp
  static constexpr int WR = 8 * MT;        // rows per warp
  static constexpr int NTHR = TM / WR * WGN * 32;
  static constexpr int S = R + 4;          // smem row stride (doubles)
  static constexpr int WN = R / WGN;       // columns per warp
  static constexpr int NT = WN / 8;        // 8-wide column tiles per warp
  static constexpr size_t smem_doubles = 2 * (size_t)TM * S + (size_t)(R + 1) * S + R + WGN * TM;
};

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int src_bytes) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem),
               "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

template <int R>
__global__ void __launch_bounds__(RotTC<R>::NTHR, R <= 64 ? 2 : 1) rot_tc_kernel(RotArgs a) {
  using C = RotTC<R>;
  extern __shared__ __align__(16) double sm[];
  double* As0 = sm;                      // 2 stages x TM x S
  double* Bs = sm + 2 * C::TM * C::S;    // (R+1) x S
  double* ps = Bs + (R + 1) * C::S;      // R
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp / C::WGN, wn = warp % C::WGN;  // warp tile: rows WR wm.., cols WN wn..
  const bool use_q = a.qbuf && (a.need == nullptr || *a.need != 0);
  const bool enc = a.fuse.enc_partial != nullptr, seed = a.fuse.seed_res2 != nullptr;
  double* rn = ps + R;  // WGN x TM row-norm parts
  double enc_acc[C::NT][2];
#pragma unroll
  for (int j = 0; j < C::NT; ++j) enc_acc[j][0] = enc_acc[j][1] = 0.0;
  for (int e = tid; e < (R + 1) * R; e += C::NTHR) Bs[(e / R) * C::S + (e % R)] = a.B[e];
  for (int e = tid; e < R; e += C::NTHR) ps[e] = use_q ? (a.p2 ? a.p2[e] : 0.0) : a.p[e];
  const bool dot = !use_q || a.p2 != nullptr;
  const double qinv = *a.qinv;
  const int64_t n = a.n;
  const int64_t ntiles = (n + C::TM - 1) / C::TM;
  constexpr int CHUNKS = C::TM * R / 2;  // 16-byte chunks per tile
  auto load_tile = [&](int64_t t, double* As) {
    const int64_t row0 = t * C::TM;
    for (int c = tid; c < CHUNKS; c += C::NTHR) {
      const int rr = c / (R / 2), cc = 2 * (c % (R / 2));
      const bool ok = row0 + rr < n;
      const double* src = a.phi + (ok ? (row0 + rr) * R + cc : 0);
      cp_async16(As + rr * C::S + cc, src, ok ? 16 : 0);
    }
    cp_async_commit();
  };
  int64_t t = blockIdx.x;
  if (t < ntiles) load_tile(t, As0);
  int stage = 0;
  for (; t < ntiles; t += gridDim.x) {
    double* As = As0 + stage * C::TM * C::S;
    const int64_t tn = t + gridDim.x;
    if (tn < ntiles) {
      load_tile(tn, As0 + (stage ^ 1) * C::TM * C::S);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const int64_t row0 = t * C::TM;
    // q_hat into column R (2 threads per row)
    for (int e = tid; e < 2 * C::TM; e += C::NTHR) {
      const int rr = e >> 1, half = e & 1;
      double qv = 0.0;
      double s = 0.0;
      if (dot) {
#pragma unroll 8
        for (int k = half * (R / 2); k < (half + 1) * (R / 2); ++k) s = fma(As[rr * C::S + k], ps[k], s);
        s += __shfl_xor_sync(0xffffffffu, s, 1);
      }
      if (row0 + rr < n) qv = (use_q ? a.qbuf[row0 + rr] : a.y[row0 + rr]) - s;
      if (half == 0) As[rr * C::S + R] = qv * qinv;
    }
    double acc[C::MT][C::NT][2];
#pragma unroll
    for (int i = 0; i < C::MT; ++i)
#pragma unroll
      for (int j = 0; j < C::NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    const int ar = wm * C::WR + (lane >> 2), ak = lane & 3;
    const int bn = wn * C::WN + (lane >> 2), bk = lane & 3;
#pragma unroll 2
    for (int k0 = 0; k0 < R; k0 += 4) {
      double af[C::MT], bf[C::NT];
#pragma unroll
      for (int i = 0; i < C::MT; ++i) af[i] = As[(ar + 8 * i) * C::S + k0 + ak];
#pragma unroll
      for (int j = 0; j < C::NT; ++j) bf[j] = Bs[(k0 + bk) * C::S + bn + 8 * j];
#pragma unroll
      for (int i = 0; i < C::MT; ++i)
#pragma unroll
        for (int j = 0; j < C::NT; ++j) dmma884(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
    __syncthreads();  // q_hat column visible
    // epilogue: + q_hat (x) B[R, :], store; fused encode / QDEIM seed
    const int er = wm * C::WR + (lane >> 2), ec = wn * C::WN + 2 * (lane & 3);
#pragma unroll
    for (int i = 0; i < C::MT; ++i) {
      const int rr = er + 8 * i;
      const double qh = As[rr * C::S + R];
      const bool ok = row0 + rr < n;
      double w = 0.0;
      if (enc && ok) {
        const int64_t gi = row0 + rr;
        w = a.fuse.enc_d[gi] * (a.fuse.enc_x[gi] - a.fuse.enc_q_ref[gi]);
      }
      double nrm = 0.0;
      double* dst = a.out + (row0 + rr) * R;
#pragma unroll
      for (int j = 0; j < C::NT; ++j) {
        const int cc = ec + 8 * j;
        double2 v;
        v.x = fma(qh, Bs[R * C::S + cc], acc[i][j][0]);
        v.y = fma(qh, Bs[R * C::S + cc + 1], acc[i][j][1]);
        if (ok) *reinterpret_cast<double2*>(dst + cc) = v;
        nrm += v.x * v.x + v.y * v.y;
        enc_acc[j][0] = fma(v.x, w, enc_acc[j][0]);
        enc_acc[j][1] = fma(v.y, w, enc_acc[j][1]);
      }
      if (seed) {
        nrm += __shfl_xor_sync(0xffffffffu, nrm, 1);
        nrm += __shfl_xor_sync(0xffffffffu, nrm, 2);
        if ((lane & 3) == 0) rn[wn * C::TM + rr] = nrm;
      }
    }
    __syncthreads();  // this stage is reloaded next-next iteration; row norms visible
    if (seed) {
      for (int rr = tid; rr < C::TM; rr += C::NTHR) {
        const int64_t gi = row0 + rr;
        if (gi < n) {
          double nv = 0.0;
#pragma unroll
          for (int q = 0; q < C::WGN; ++q) nv += rn[q * C::TM + rr];
          a.fuse.seed_res2[gi] = nv;
          a.fuse.seed_bnd2[gi] = nv + 16.0 * 2.220446049250313e-16 * nv;
          a.fuse.seed_ver[gi] = 0;
        }
      }
    }
    stage ^= 1;
  }
  if (enc) {
    // column sums: lanes with equal (lane & 3) share columns; then the wm warps
#pragma unroll
    for (int j = 0; j < C::NT; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        double v = enc_acc[j][h];
        v += __shfl_xor_sync(0xffffffffu, v, 4);
        v += __shfl_xor_sync(0xffffffffu, v, 8);
        v += __shfl_xor_sync(0xffffffffu, v, 16);
        enc_acc[j][h] = v;
      }
    __syncthreads();
    double* red = As0;  // (TM/WR) x R
    if (lane < 4) {
#pragma unroll
      for (int j = 0; j < C::NT; ++j) {
        const int cc = wn * C::WN + 2 * lane + 8 * j;
        red[wm * R + cc] = enc_acc[j][0];
        red[wm * R + cc + 1] = enc_acc[j][1];
      }
    }
    __syncthreads();
    for (int c = tid; c < R; c += C::NTHR) {
      double sum = 0.0;
      for (int q = 0; q < C::TM / C::WR; ++q) sum += red[q * R + c];
      a.fuse.enc_partial[(size_t)blockIdx.x * R + c] = sum;
    }
  }
}

// generic sizes: out (n x r_out) = [phi | q_hat] B
__global__ void __launch_bounds__(256) rot_generic_kernel(RotArgs a) {
  extern __shared__ double sm[];
  const int T = 32;
  const int r_in = a.r_in, r_out = a.r_out;
  const int S = r_in + 1;
  double* As = sm;                   // T x S
  double* Bs = As + T * S;           // (r_in+1) x r_out
  double* ps = Bs + (r_in + 1) * r_out;
  const int tid = threadIdx.x;
  const bool use_q = a.qbuf && (a.need == nullptr || *a.need != 0);
  for (int e = tid; e < (r_in + 1) * r_out; e += 256) Bs[e] = a.B[e];
  for (int e = tid; e < r_in; e += 256) ps[e] = use_q ? (a.p2 ? a.p2[e] : 0.0) : a.p[e];
  const bool dot = !use_q || a.p2 != nullptr;
  const double qinv = *a.qinv;
  const int64_t ntiles = (a.n + T - 1) / T;
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int64_t row0 = t * T;
    const int rows = (int)((a.n - row0 < T) ? (a.n - row0) : T);
    __syncthreads();
    for (int e = tid; e < rows * r_in; e += 256) {
      const int rr = e / r_in, cc = e - rr * r_in;
      As[rr * S + cc] = a.phi[row0 * r_in + e];
    }
    __syncthreads();
    for (int e = tid; e < rows; e += 256) {
      double s = 0.0;
      if (dot)
        for (int k = 0; k < r_in; ++k) s = fma(As[e * S + k], ps[k], s);
      const double qv = (use_q ? a.qbuf[row0 + e] : a.y[row0 + e]) - s;
      As[e * S + r_in] = qv * qinv;
    }
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
    for (int e = tid; e < rows * r_out; e += 256) a.out[row0 * r_out + e] = res[cntv++];
  }
}

bool rot_fusable(int r_in, int r_out) {
  return r_in == r_out && (r_in == 32 || r_in == 64 || r_in == 128) && !getenv("ADROM_NO_TC_ROT");
}

static int64_t rot_tc_grid(const adrom_ctx* ctx, int64_t n, int r) {
  const int tm = r <= 64 ? RotTC<64>::TM : RotTC<128>::TM;
  const int64_t nt = (n + tm - 1) / tm;
  int64_t gg = (int64_t)ctx->num_sms * (r <= 64 ? 2 : 1);
  if (gg > nt) gg = nt;
  return gg < 1 ? 1 : gg;
}

size_t rot_fuse_partial_doubles(const adrom_ctx* ctx, int r) {
  return (size_t)ctx->num_sms * 2 * (size_t)r;
}

int rot_encode_finish(adrom_ctx* ctx, const RotFuse& f, int64_t n, int r, double* out) {
  reduce_partials_kernel<<<r, 256, 0, ctx->stream>>>(f.enc_partial, (int)rot_tc_grid(ctx, n, r), r,
                                                     out, nullptr);
  ADROM_LAUNCH_CK(ctx);
  return ADROM_OK;
}

int ts_rotate(adrom_ctx* ctx, const RotArgs& a) {
  const int64_t n = a.n;
  const int r_in = a.r_in, r_out = a.r_out;
  if (rot_fusable(r_in, r_out)) {
    auto launch_tc = [&](auto kern, size_t sm_doubles) -> int {
      const size_t sm = sizeof(double) * sm_doubles;
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      kern<<<(int)rot_tc_grid(ctx, n, r_in), 256, sm, ctx->stream>>>(a);
      ADROM_LAUNCH_CK(ctx);
      return ADROM_OK;
    };
    static_assert(RotTC<32>::NTHR == 256 && RotTC<64>::NTHR == 256 && RotTC<128>::NTHR == 256,
                  "rot_tc_kernel launches 256 threads");
    if (r_in == 32) return launch_tc(rot_tc_kernel<32>, RotTC<32>::smem_doubles);
    if (r_in == 64) return launch_tc(rot_tc_kernel<64>, RotTC<64>::smem_doubles);
    return launch_tc(rot_tc_kernel<128>, RotTC<128>::smem_doubles);
  }
  if (r_in == r_out && (r_in == 16 || r_in == 32 || r_in == 64 || r_in == 128)) {
    int64_t g = (int64_t)ctx->num_sms * 2;
    auto launch = [&](auto kern, int TM, int R) -> int {
      const size_t sm = sizeof(double) * ((size_t)TM * (R + 1) + (size_t)(R + 1) * R + R);
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      const int64_t nt = (n + TM - 1) / TM;
      const int64_t gg = g < nt ? g : nt;
      kern<<<(int)(gg < 1 ? 1 : gg), 256, sm, ctx->stream>>>(a);
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
  const size_t sm = sizeof(double) * ((size_t)32 * (r_in + 1) + (size_t)(r_in + 1) * r_out + r_in);
  cudaFuncSetAttribute(rot_generic_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  int64_t g = (int64_t)ctx->num_sms * 4, nt = (n + 31) / 32;
  if (g > nt) g = nt;
  rot_generic_kernel<<<(int)(g < 1 ? 1 : g), 256, sm, ctx->stream>>>(a);
  ADROM_LAUNCH_CK(ctx);
  return ADROM_OK;
}

// ---------------------------------------------------------------------------
// Gram matrix G = Phi^T Phi (tracked across updates; computed afresh once)
// ---------------------------------------------------------------------------
// 16 x 16 thread grid; thread (ti, tj) owns G[ti + 16 a][tj + 16 b],
// a, b < RB = ceil(r / 16): register accumulators, rows staged in smem
template <int RB>
__global__ void __launch_bounds__(256) gram_kernel(const double* __restrict__ phi, int64_t n,
                                                   int r, double* __restrict__ partial) {
  extern __shared__ double sm[];
  constexpr int T = 64;
  const int S = r | 1;
  double* tile = sm;  // T x S, zero-padded to 16 * RB columns
  const int tid = threadIdx.x, ti = tid & 15, tj = tid >> 4;
  double acc[RB][RB];
#pragma unroll
  for (int x = 0; x < RB; ++x)
#pragma unroll
    for (int y = 0; y < RB; ++y) acc[x][y] = 0.0;
  const int64_t ntiles = (n + T - 1) / T;
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int64_t row0 = t * T;
    const int rows = (int)((n - row0 < T) ? (n - row0) : T);
    __syncthreads();
    for (int e = tid; e < rows * r; e += 256) {
      const int a = e / r, c = e - a * r;
      tile[a * S + c] = phi[row0 * r + e];
    }
    __syncthreads();
    for (int a = 0; a < rows; ++a) {
      const double* row = tile + a * S;
      double u[RB], v[RB];
#pragma unroll
      for (int x = 0; x < RB; ++x) {
        const int i = ti + 16 * x, j = tj + 16 * x;
        u[x] = (i < r) ? row[i] : 0.0;
        v[x] = (j < r) ? row[j] : 0.0;
      }
#pragma unroll
      for (int x = 0; x < RB; ++x)
#pragma unroll
        for (int y = 0; y < RB; ++y) acc[x][y] = fma(u[x], v[y], acc[x][y]);
    }
  }
  const int rr2 = r * r;
#pragma unroll
  for (int x = 0; x < RB; ++x)
#pragma unroll
    for (int y = 0; y < RB; ++y) {
      const int i = ti + 16 * x, j = tj + 16 * y;
      if (i < r && j < r) partial[(size_t)blockIdx.x * rr2 + i * r + j] = acc[x][y];
    }
}

size_t gram_partial_doubles(const adrom_ctx* ctx, int r) {
  return (size_t)ctx->num_sms * 2 * (size_t)r * r;
}

size_t isvd_partial_doubles(const adrom_ctx* ctx, int r_cur) {
  const size_t a = (size_t)partial_rows(ctx) * (r_cur + 1), b = gram_partial_doubles(ctx, r_cur);
  return a > b ? a : b;
}

int ts_gram(adrom_ctx* ctx, const double* phi, int64_t n, int r, double* gram, double* partial,
            size_t cap_doubles) {
  if (r > 128) return set_error(ctx, ADROM_ERR_ARG, "gram: rank %d unsupported", r);
  int64_t g = (n + 63) / 64;
  const int64_t cap = (int64_t)(cap_doubles / ((size_t)r * r));
  if (cap < 1)  // every block writes an r x r partial
    return set_error(ctx, ADROM_ERR_ARG, "gram: partials buffer of %zu doubles is smaller than r^2",
                     cap_doubles);
  int64_t lim = (int64_t)ctx->num_sms * 2;
  if (lim > cap) lim = cap;
  if (g > lim) g = lim;
  if (g < 1) g = 1;
  const size_t sm = sizeof(double) * 64 * (r | 1);
  auto kern = (r <= 16)   ? gram_kernel<1>
              : (r <= 32) ? gram_kernel<2>
              : (r <= 64) ? gram_kernel<4>
                          : gram_kernel<8>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  kern<<<(int)g, 256, sm, ctx->stream>>>(phi, n, r, partial);
  ADROM_LAUNCH_CK(ctx);
  reduce_partials_kernel<<<r * r, 256, 0, ctx->stream>>>(partial, (int)g, r * r, gram, nullptr);
  ADROM_LAUNCH_CK(ctx);
  return ADROM_OK;
}

// ---------------------------------------------------------------------------
// iSVD core (one block): K, its SVD, the rotation factors
// ---------------------------------------------------------------------------
// stats layout (doubles): [0] qnorm [1] ynorm [2] proj_resid [3] degenerate
//                         [4] reorth [5] sweeps [6] converged [7] nonfinite
// Least-squares coefficients p = (Phi^T Phi)^{-1} Phi^T y (tracking.py:161,
// gelsd) from the tracked Gram matrix G: Neumann series in E = G - I (the
// tracked basis is orthonormal to << 1), Gaussian elimination otherwise.
// Decides whether the explicit residual pass is needed:
//   ||q||^2 = ||y||^2 - p . p1 cancels when ||q||^2 / ||y||^2 < ratio.
// red1 = [p1 = Phi^T y (r), ||y||^2]; writes p (r) and *need.
__global__ void __launch_bounds__(128) isvd_solve_kernel(const double* __restrict__ red1,
                                                         const double* __restrict__ G, int r,
                                                         double ratio, double* __restrict__ p,
                                                         int* __restrict__ need) {
  __shared__ double sp[128], st[128], sn[128];
  __shared__ int sh_done;
  const int tid = threadIdx.x;
  for (int j = tid; j < r; j += blockDim.x) {
    sp[j] = red1[j];
    st[j] = red1[j];
  }
  __syncthreads();
  bool conv = false;
  for (int it = 0; it < 40 && !conv; ++it) {
    // term <- -(G - I) term
    for (int i = tid; i < r; i += blockDim.x) {
      double s = 0.0;
      for (int k = 0; k < r; ++k) s = fma(G[i * r + k] - (i == k ? 1.0 : 0.0), st[k], s);
      sn[i] = -s;
    }
    __syncthreads();
    if (tid == 0) {
      double tn = 0.0, pn = 0.0;
      for (int j = 0; j < r; ++j) {
        sp[j] += sn[j];
        st[j] = sn[j];
        tn += sn[j] * sn[j];
        pn += sp[j] * sp[j];
      }
      sh_done = (tn <= 1e-34 * pn) ? 1 : (!(tn <= 1e300) ? 2 : 0);
    }
    __syncthreads();
    conv = sh_done != 0;
  }
  // a basis far from orthonormal (the Neumann series did not converge):
  // isvd_solve_direct_kernel solves G p = p1 directly; need[1] tells it to
  if (tid == 0) need[1] = (sh_done != 1) ? 1 : 0;
  if (sh_done != 1) return;
  if (tid == 0) {
    double pdot = 0.0;
    for (int j = 0; j < r; ++j) pdot += sp[j] * red1[j];
    const double yy = red1[r];
    const double est = yy - pdot;
    *need = (est > ratio * yy) ? 0 : 1;
  }
  __syncthreads();
  for (int j = tid; j < r; j += blockDim.x) p[j] = sp[j];
}

// G p = p1 by Gaussian elimination with partial pivoting on the whole block
// (G = Phi^T Phi is SPD; pivoting only guards a drifted tracked Gram), run
// when isvd_solve_kernel flagged need[1]; O(r^3 / 3) in shared memory
// instead of the former one-thread Gauss-Seidel (200 serial sweeps, ~14 ms
// at r = 64 late in a 2000-step configuration-3 run).
__global__ void __launch_bounds__(256) isvd_solve_direct_kernel(const double* __restrict__ red1,
                                                                const double* __restrict__ G, int r,
                                                                double ratio, double* __restrict__ p,
                                                                int* __restrict__ need) {
  if (need[1] == 0) return;
  extern __shared__ double sa[];  // r x (r + 1) augmented, row-major (ld r + 1)
  __shared__ int piv_sh;
  const int tid = threadIdx.x, ld = r + 1;
  for (int e = tid; e < r * r; e += blockDim.x) sa[(e / r) * ld + (e % r)] = G[e];
  for (int i = tid; i < r; i += blockDim.x) sa[i * ld + r] = red1[i];
  __syncthreads();
  for (int k = 0; k < r; ++k) {
    if (tid == 0) {
      int pv = k;
      double best = fabs(sa[k * ld + k]);
      for (int i = k + 1; i < r; ++i) {
        const double v = fabs(sa[i * ld + k]);
        if (v > best) {
          best = v;
          pv = i;
        }
      }
      piv_sh = pv;
    }
    __syncthreads();
    const int pv = piv_sh;
    if (pv != k)
      for (int j = tid; j <= r; j += blockDim.x) {
        const double t = sa[k * ld + j];
        sa[k * ld + j] = sa[pv * ld + j];
        sa[pv * ld + j] = t;
      }
    __syncthreads();
    const double akk = sa[k * ld + k];
    const int m = r - k - 1;
    for (int e = tid; e < m * (m + 1); e += blockDim.x) {
      const int i = k + 1 + e / (m + 1), j = k + 1 + e % (m + 1);
      sa[i * ld + j] -= (sa[i * ld + k] / akk) * sa[k * ld + j];
    }
    __syncthreads();
  }
  if (tid == 0) {
    for (int i = r - 1; i >= 0; --i) {
      double s = sa[i * ld + r];
      for (int j = i + 1; j < r; ++j) s -= sa[i * ld + j] * p[j];
      p[i] = s / sa[i * ld + i];
    }
    double pdot = 0.0;
    for (int j = 0; j < r; ++j) pdot += p[j] * red1[j];
    const double yy = red1[r];
    need[0] = (yy - pdot > ratio * yy) ? 0 : 1;
    need[1] = 0;
  }
}

// iSVD core (tracking.py:163-177) for p = lstsq coefficients (isvd_solve_kernel):
//   ||q||^2: explicit pass (red2[r]) or ||y||^2 - p.p1 when that does not cancel
//   K = [[lam Sigma, p], [0, ||q||]] (last row 0 if degenerate), K = U S V^T
//   B = [U_top ; u_bot][:, :r] sorted by S (rotation factors), qinv = 1/||q||
//   G' = B^T [[G, c_hat], [c_hat^T, 1]] B with c_hat = Phi^T q / ||q||
//   proj_resid = ||y - Phi Phi^T y|| = sqrt(||q||^2 + d^T G d), d = p - p1
//                                                       (driver.py:366-367)
template <bool VG>
__global__ void __launch_bounds__(1024) isvd_core_kernel(
    const double* __restrict__ sigma, const double* __restrict__ red1,
    const double* __restrict__ pls, const double* __restrict__ red2,
    const int* __restrict__ need, const double* __restrict__ G, int r_cur, int r, double lam,
    double* __restrict__ Bout, double* __restrict__ qinv_out, double* __restrict__ Tws,
    double* __restrict__ Gout, double* __restrict__ sigma_out, double* __restrict__ stats,
    int* __restrict__ flag, double* __restrict__ udrop_out, double* __restrict__ vglob,
    int force_jacobi) {
  extern __shared__ double sm[];
  const int n = r_cur + 1;
  const int ld = n + ((n & 1) ? 0 : 1);  // odd leading dimension
  double* A = sm;            // n x ld (column-major: column j = row j of K)
  // V (n x ld) in shared memory, or in global memory (L2-resident) when
  // both matrices do not fit (r_cur > 110); a compile-time choice so the
  // loops below use shared-memory loads, not generic ones
  double* V = VG ? vglob : A + n * ld;
  double* p = VG ? A + n * ld : V + n * ld;       // r_cur
  double* s = p + r_cur;     // n
  double* chat = s + n;      // r_cur
  double* dv = chat + r_cur; // r_cur (p - p1)
  double* red = dv + r_cur;  // 32
  int* order = (int*)(red + 32);
  // T = Ghat B ((r_cur+1) x r): shared memory after `order` when V is, else Tws
  double* Ts = VG ? Tws : (double*)(((uintptr_t)(order + n) + 15) & ~(uintptr_t)15);
  __shared__ int sh_flag;
  __shared__ double sh_q[4];
  const int tid = threadIdx.x;
  const bool reorth = need[0] != 0;
  for (int j = tid; j < r_cur; j += blockDim.x) {
    p[j] = pls[j];
    dv[j] = pls[j] - red1[j];
  }
  __syncthreads();
  // d^T G d for the driver's residual diagnostic
  double dgd = 0.0;
  for (int e = tid; e < r_cur * r_cur; e += blockDim.x) {
    const int i = e / r_cur, k = e - i * r_cur;
    dgd += dv[i] * G[e] * dv[k];
  }
  dgd = block_sum_dyn(dgd, red);
  if (tid == 0) {
    const double yy = red1[r_cur];
    double qq;
    if (reorth) {
      qq = red2[r_cur];
    } else {
      double pdot = 0.0;
      for (int j = 0; j < r_cur; ++j) pdot += p[j] * red1[j];
      qq = yy - pdot;
    }
    sh_q[0] = sqrt(qq > 0.0 ? qq : 0.0);
    sh_q[1] = sqrt(yy);
    const double proj = (qq > 0.0 ? qq : 0.0) + dgd;
    sh_q[2] = sqrt(proj > 0.0 ? proj : 0.0);
  }
  __syncthreads();
  const double qnorm = sh_q[0], ynorm = sh_q[1];
  // tracking.py:169 — degenerate residual keeps the subspace
  const bool degenerate = qnorm <= 1e-12 * fmax(ynorm, 1e-300);
  // Fast path: one-sided Jacobi on K's own columns (A = K column-major):
  // K V = U S, so U (all the rotation needs) is read off the converged
  // columns and V is never formed — half the work of the K^T form.  The
  // result is verified (kept singular values > 0, max |U^T U - I| <= 1e-13);
  // otherwise (rank-deficient K: a column at rounding level never converges
  // in the relative sense) the K^T form with accumulated rotations runs.
  auto fill_k = [&](bool transposed) {
    for (int e = tid; e < n * ld; e += blockDim.x) A[e] = 0.0;
    __syncthreads();
    for (int j = tid; j < r_cur; j += blockDim.x) {
      A[j * ld + j] = lam * sigma[j];                      // K[j][j] (tracking.py:167)
      if (transposed) A[j * ld + r_cur] = p[j];            // A = K^T
      else A[r_cur * ld + j] = p[j];                       // K[j][r] (tracking.py:168)
    }
    if (tid == 0) A[r_cur * ld + r_cur] = degenerate ? 0.0 : qnorm;  // tracking.py:172
    __syncthreads();
  };
  bool bad = false;
  for (int j = tid; j < r_cur; j += blockDim.x)
    bad |= !isfinite(lam * sigma[j]) || !isfinite(p[j]);
  if (tid == 0) bad |= !isfinite(qnorm) || !isfinite(ynorm);
  __shared__ int sh_bad;
  if (tid == 0) sh_bad = 0;
  __syncthreads();
  if (bad) {
    atomicOr(flag, 1);
    sh_bad = 1;
  }
  __syncthreads();
  if (sh_bad) {  // thin_svd rejects non-finite input (dense.py:61): no SVD, no rotation
    for (int e = tid; e < n * r; e += blockDim.x) Bout[e] = 0.0;
    if (tid == 0) *qinv_out = 0.0;
    return;
  }
  // Fast path: the secular equation of K K^T = diag(d^2) + z z^T (secular.cuh),
  // verified by the residual of every kept column and its orthonormality
  __shared__ SecularShared sec;
  __shared__ int sh_path;  // 0 secular, 1 Jacobi on K, 2 Jacobi on K^T
  JacobiResult jr{0, 1};
  {
    const double rho = degenerate ? 0.0 : qnorm;
    const bool conv = secular_core_svd(sigma, lam, p, rho, n, V, ld, s, A, ld, sec);
    for (int j = tid; j < n; j += blockDim.x) {
      int rank = 0;
      const double sj = isnan(s[j]) ? -1.0 : s[j];
      for (int k = 0; k < n; ++k) {
        const double sk = isnan(s[k]) ? -1.0 : s[k];
        if (sk > sj || (sk == sj && k < j)) ++rank;
      }
      order[rank] = j;
    }
    __syncthreads();
    // || K K^T u - s^2 u ||_inf on the kept columns (K K^T = diag(d^2) + z z^T)
    double zz = 0.0, dm = 0.0;
    for (int i = 0; i < n; ++i) {
      const double zi = (i < r_cur) ? p[i] : rho;
      zz += zi * zi;
      if (i < r_cur) dm = fmax(dm, fabs(lam * sigma[i]));
    }
    double worst = 0.0;
    for (int a = tid >> 5; a < r; a += blockDim.x >> 5) {
      const double* u = V + (size_t)order[a] * ld;
      double zu = 0.0;
      for (int i = (tid & 31); i < n; i += 32) zu += ((i < r_cur) ? p[i] : rho) * u[i];
      zu = warp_sum(zu);
      const double s2 = s[order[a]] * s[order[a]];
      for (int i = (tid & 31); i < n; i += 32) {
        const double di = (i < r_cur) ? lam * sigma[i] : 0.0;
        const double zi = (i < r_cur) ? p[i] : rho;
        worst = fmax(worst, fabs(di * di * u[i] + zi * zu - s2 * u[i]));
      }
    }
    worst = block_max_dyn(worst, red);
    if (tid == 0)
      sh_path = (!force_jacobi && conv &&
                 worst <= 256.0 * n * 2.220446049250313e-16 * (dm * dm + zz)) ? 0 : 1;
    __syncthreads();
  }
  if (sh_path) {
    fill_k(false);
    jr = block_jacobi<16>(A, ld, n, n, nullptr, ld, 30, 1e-15, &sh_flag);
    column_norms_sorted(A, ld, n, n, s, order);
    // U column j = A column j / s_j, stored as V[j][k] = U[k][j]
    for (int e = tid; e < n * n; e += blockDim.x) {
      const int j = e / n, k = e - j * n;
      V[j * ld + k] = (s[j] > 0.0) ? A[j * ld + k] / s[j] : 0.0;
    }
    __syncthreads();
  }
  // sorted kept columns B (column c = U[:, order[c]]) into A's buffer
  double* Bs = A;
  auto gather_b = [&]() {
    for (int e = tid; e < r * n; e += blockDim.x) {
      const int c = e / n, k = e - c * n;
      Bs[c * ld + k] = V[order[c] * ld + k];
    }
    __syncthreads();
  };
  gather_b();
  // orthonormality of the kept columns (upper triangle, two chains per dot)
  double defect = 0.0;
  const int npair = r * (r + 1) / 2;
  for (int e = tid; e < npair; e += blockDim.x) {
    int a = (int)((sqrt(8.0 * e + 1.0) - 1.0) * 0.5);  // e -> (a, b), b <= a
    while ((a + 1) * (a + 2) / 2 <= e) ++a;
    while (a * (a + 1) / 2 > e) --a;
    const int b = e - a * (a + 1) / 2;
    const double* ua = Bs + a * ld;
    const double* ub = Bs + b * ld;
    double d0 = 0.0, d1 = 0.0;
    int k = 0;
    for (; k + 1 < n; k += 2) {
      d0 += ua[k] * ub[k];
      d1 += ua[k + 1] * ub[k + 1];
    }
    if (k < n) d0 += ua[k] * ub[k];
    defect = fmax(defect, fabs((d0 + d1) - (a == b ? 1.0 : 0.0)));
  }
  defect = block_max_dyn(defect, red);
  __shared__ int sh_fallback;
  if (tid == 0) {
    sh_fallback = (!jr.converged || !(defect <= 1e-13) || !(s[order[r - 1]] > 0.0)) ? 1 : 0;
    // a rank-deficient K (a zero kept singular value) is legitimate on the
    // secular path: its vectors are exact eigenvectors, not column norms
    if (sh_path == 0 && jr.converged && defect <= 1e-13) sh_fallback = 0;
    if (sh_fallback) sh_path = 2;
  }
  __syncthreads();
  if (sh_fallback) {
    // one-sided Jacobi on K^T with accumulated rotations: U of K = V
    fill_k(true);
    jr = block_jacobi<16>(A, ld, n, n, V, ld, 60, 1e-15, &sh_flag);
    column_norms_sorted(A, ld, n, n, s, order);
    gather_b();
  }
  // rotation factors B[k][c] = U[k][order[c]] (k = r_cur is u_bot)
  const double inv = degenerate ? 0.0 : 1.0 / qnorm;
  for (int e = tid; e < n * r; e += blockDim.x) {
    const int k = e / r, c = e - k * r;
    Bout[e] = Bs[c * ld + k];
  }
  // the left singular vector the truncation drops (factored basis: exact row norms)
  if (udrop_out && r < n)
    for (int k = tid; k < n; k += blockDim.x) udrop_out[k] = V[order[r] * ld + k];
  if (tid == 0) *qinv_out = inv;
  __syncthreads();
  // G staged in V's buffer when both are in shared memory (V is consumed)
  const double* Gm = G;
  if (!VG) {
    double* Gsh = V;
    for (int e = tid; e < r_cur * r_cur; e += blockDim.x) Gsh[e] = G[e];
    Gm = Gsh;
    __syncthreads();
  }
  // c_hat = Phi^T q / ||q||: explicit (pass 2) or p1 - G p (normal equations)
  for (int k = tid; k < r_cur; k += blockDim.x) {
    double c;
    if (reorth) {
      c = red2[k];
    } else {
      double gp = 0.0;
      for (int j = 0; j < r_cur; ++j) gp += Gm[k * r_cur + j] * p[j];
      c = red1[k] - gp;
    }
    chat[k] = c * inv;
  }
  __syncthreads();
  // T = Ghat B ((r_cur+1) x r), 4 rows per thread (one B column load feeds 4
  // FMA chains); Ghat = [[G, c_hat], [c_hat^T, 1 (0 if degenerate)]]
  const int kb = (n + 3) / 4;
  for (int e = tid; e < kb * r; e += blockDim.x) {
    const int k0 = 4 * (e / r), c = e - (e / r) * r;
    const double* bc = Bs + c * ld;
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    for (int l = 0; l < r_cur; ++l) {
      const double bl = bc[l];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int k = k0 + i;
        const double g = (k < r_cur) ? Gm[k * r_cur + l] : (k == r_cur ? chat[l] : 0.0);
        acc[i] += g * bl;
      }
    }
    const double bl = bc[r_cur];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int k = k0 + i;
      if (k < r_cur) Ts[k * r + c] = acc[i] + chat[k] * bl;
      else if (k == r_cur) Ts[k * r + c] = acc[i] + (degenerate ? 0.0 : 1.0) * bl;
    }
  }
  __syncthreads();
  // G' = B^T T (r x r), 4 columns per thread
  const int cb = (r + 3) / 4;
  for (int e = tid; e < r * cb; e += blockDim.x) {
    const int a = e / cb, b0 = 4 * (e - a * cb);
    const double* ba = Bs + a * ld;
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    for (int k = 0; k < n; ++k) {
      const double x = ba[k];
#pragma unroll
      for (int i = 0; i < 4; ++i)
        if (b0 + i < r) acc[i] += x * Ts[k * r + b0 + i];
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
      if (b0 + i < r) Gout[a * r + b0 + i] = acc[i];
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
    stats[7] = sh_path;
    if (!jr.converged) atomicOr(flag, 8);
  }
}

// ADROM_CORE_JACOBI=1: skip the secular path (A/B diagnostics and tests)
static int core_force_jacobi() {
  static const int v = [] {
    const char* e = getenv("ADROM_CORE_JACOBI");
    return (e && atoi(e) != 0) ? 1 : 0;
  }();
  return v;
}

// one column pair per half-warp: ceil((r+2)/2) pairs, rounded up to whole
// warps (no idle warps in the per-round barrier)
static int core_threads(int r_cur) {
  const int pairs = (r_cur + 2) / 2;
  const int t = ((pairs * 16 + 31) / 32) * 32;
  return t < 64 ? 64 : (t > 1024 ? 1024 : t);
}

static size_t core_smem(int r_cur, bool v_global = false) {
  const int n = r_cur + 1;
  const int ld = n + ((n & 1) ? 0 : 1);
  // A, V (unless global), p, s, chat, dv, red, order, T (unless global)
  return sizeof(double) * ((v_global ? 1 : 2) * (size_t)n * ld + 3 * (size_t)r_cur + n + 32) +
         sizeof(int) * n + 64 + (v_global ? 0 : sizeof(double) * (size_t)n * r_cur + 16);
}

// V of the core SVD leaves shared memory above this size
static bool core_v_global(int r_cur) { return core_smem(r_cur) > 220 * 1024; }

static size_t core_vglob_doubles(int r_cur) {
  const int n = r_cur + 1;
  return (size_t)n * (n + ((n & 1) ? 0 : 1));
}

size_t isvd_workspace_bytes(adrom_ctx* ctx, int64_t n, int r_cur, int r) {
  const int64_t grid = (int64_t)partial_rows(ctx);
  size_t b = 0;
  const int w = (r_cur * r_cur > r_cur + 1) ? r_cur * r_cur : r_cur + 1;
  (void)w;
  b += align_up(sizeof(double) * isvd_partial_doubles(ctx, r_cur));  // partials (Gram's too)
  b += 2 * align_up(sizeof(double) * (r_cur + 1));     // red1, red2
  b += align_up(sizeof(double) * r_cur);               // p (least squares)
  b += align_up(sizeof(double) * r_cur);               // p2 (refinement)
  b += align_up(sizeof(double) * (r_cur + 1) * r);     // B
  b += align_up(sizeof(double) * (r_cur + 1) * r);     // T
  b += align_up(sizeof(double) * r_cur * r_cur);       // Gram (when not supplied)
  b += align_up(sizeof(double) * 16);                  // stats + qinv
  b += align_up(sizeof(int) * 4);                      // need
  b += align_up(sizeof(double) * (size_t)n);           // residual q
  b += align_up(sizeof(double) * core_vglob_doubles(r_cur));  // core V (r_cur > 110)
  return b;
}

// One step of least-squares refinement after the explicit residual pass
// (need[0] != 0): red2 = [c = Phi^T q, ||q||^2] for q = y - Phi p.  With the
// tracked Gram G, p2 = G^{-1} c (Neumann series; Gaussian elimination with
// partial pivoting when it diverges), p += p2, and q' = q - Phi p2 is the
// residual used from here on: red2 <- [c - G p2, ||q||^2 - 2 p2.c +
// p2.G p2].  The tracked-Gram solve alone leaves q off Phi's complement by the
// Gram's error times ||y|| / ||q||, which compounds over events (orthonormality
// defect 7e-2 after 600 configuration-3 events at N = 2^16 against the
// reference's 3e-3); one refinement step makes q orthogonal to the actual
// basis (defect 2e-14 in the numpy prototype).  p2norm (optional) <- ||p2||.
__global__ void __launch_bounds__(256) isvd_refine_kernel(const double* __restrict__ G, int r,
                                                          double* __restrict__ red2,
                                                          double* __restrict__ p,
                                                          double* __restrict__ p2,
                                                          double* __restrict__ p2norm,
                                                          const int* __restrict__ need) {
  extern __shared__ double sa[];  // r x (r + 1) augmented system (fallback)
  __shared__ double c[128], x[128], t[128], nx[128];
  __shared__ double red[32];
  __shared__ int sh_done, piv_sh;
  const int tid = threadIdx.x;
  if (need && need[0] == 0) {
    for (int j = tid; j < r; j += blockDim.x) p2[j] = 0.0;
    if (tid == 0 && p2norm) *p2norm = 0.0;
    return;
  }
  for (int j = tid; j < r; j += blockDim.x) {
    c[j] = red2[j];
    x[j] = red2[j];
    t[j] = red2[j];
  }
  __syncthreads();
  // Neumann series x = sum_m (-(G - I))^m c
  bool conv = false;
  for (int it = 0; it < 60 && !conv; ++it) {
    for (int i = tid; i < r; i += blockDim.x) {
      double sacc = 0.0;
      for (int k = 0; k < r; ++k) sacc = fma(G[i * r + k] - (i == k ? 1.0 : 0.0), t[k], sacc);
      nx[i] = -sacc;
    }
    __syncthreads();
    double tn = 0.0, xn = 0.0;
    for (int j = tid; j < r; j += blockDim.x) {
      t[j] = nx[j];
      x[j] += nx[j];
      tn += nx[j] * nx[j];
      xn += x[j] * x[j];
    }
    tn = block_sum_dyn(tn, red);
    xn = block_sum_dyn(xn, red);
    if (tid == 0) sh_done = (tn <= 1e-34 * xn) ? 1 : (!(tn <= 1e300) ? 2 : 0);
    __syncthreads();
    conv = sh_done != 0;
  }
  if (sh_done != 1) {  // Gaussian elimination with partial pivoting
    const int ld = r + 1;
    for (int e = tid; e < r * r; e += blockDim.x) sa[(e / r) * ld + (e % r)] = G[e];
    for (int i = tid; i < r; i += blockDim.x) sa[i * ld + r] = c[i];
    __syncthreads();
    for (int k = 0; k < r; ++k) {
      if (tid == 0) {
        int pv = k;
        double best = fabs(sa[k * ld + k]);
        for (int i = k + 1; i < r; ++i)
          if (fabs(sa[i * ld + k]) > best) {
            best = fabs(sa[i * ld + k]);
            pv = i;
          }
        piv_sh = pv;
      }
      __syncthreads();
      const int pv = piv_sh;
      if (pv != k)
        for (int j = tid; j <= r; j += blockDim.x) {
          const double tt = sa[k * ld + j];
          sa[k * ld + j] = sa[pv * ld + j];
          sa[pv * ld + j] = tt;
        }
      __syncthreads();
      const double akk = sa[k * ld + k];
      const int m = r - k - 1;
      for (int e = tid; e < m * (m + 1); e += blockDim.x) {
        const int i = k + 1 + e / (m + 1), j = k + 1 + e % (m + 1);
        sa[i * ld + j] -= (sa[i * ld + k] / akk) * sa[k * ld + j];
      }
      __syncthreads();
    }
    if (tid == 0)
      for (int i = r - 1; i >= 0; --i) {
        double sacc = sa[i * ld + r];
        for (int j = i + 1; j < r; ++j) sacc -= sa[i * ld + j] * x[j];
        x[i] = sacc / sa[i * ld + i];
      }
    __syncthreads();
  }
  // G x, the new residual's coefficients and norm
  for (int i = tid; i < r; i += blockDim.x) {
    double sacc = 0.0;
    for (int k = 0; k < r; ++k) sacc = fma(G[i * r + k], x[k], sacc);
    nx[i] = sacc;
  }
  __syncthreads();
  double xc = 0.0, xgx = 0.0, xx = 0.0;
  for (int j = tid; j < r; j += blockDim.x) {
    xc += x[j] * c[j];
    xgx += x[j] * nx[j];
    xx += x[j] * x[j];
  }
  xc = block_sum_dyn(xc, red);
  xgx = block_sum_dyn(xgx, red);
  xx = block_sum_dyn(xx, red);
  for (int j = tid; j < r; j += blockDim.x) {
    p[j] += x[j];
    p2[j] = x[j];
    red2[j] = c[j] - nx[j];
  }
  if (tid == 0) {
    const double qq = red2[r] - 2.0 * xc + xgx;
    red2[r] = qq > 0.0 ? qq : 0.0;
    if (p2norm) *p2norm = sqrt(xx);
  }
}

int isvd_refine_launch(adrom_ctx* ctx, const double* G, int r, double* red2, double* p,
                       double* p2, double* p2norm, const int* need) {
  if (r > 128) return set_error(ctx, ADROM_ERR_ARG, "isvd refine: rank %d > 128", r);
  const size_t sm = sizeof(double) * (size_t)r * (r + 1);
  cudaFuncSetAttribute(isvd_refine_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  isvd_refine_kernel<<<1, 256, sm, ctx->stream>>>(G, r, red2, p, p2, p2norm, need);
  ADROM_LAUNCH_CK(ctx);
  return ADROM_OK;
}

__global__ void set_need_kernel(int* need) { need[0] = 1; }

static int isvd_solve_direct_launch(adrom_ctx* ctx, const double* red1, const double* G, int r,
                                    double ratio, double* p, int* need) {
  const size_t sm = sizeof(double) * (size_t)r * (r + 1);
  cudaFuncSetAttribute(isvd_solve_direct_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  isvd_solve_direct_kernel<<<1, 256, sm, ctx->stream>>>(red1, G, r, ratio, p, need);
  ADROM_LAUNCH_CK(ctx);
  return ADROM_OK;
}

int isvd_update_async(adrom_ctx* ctx, const double* phi, const double* sigma, const double* y,
                      int64_t n, int r_cur, int r, double lam, double* phi_out,
                      double* sigma_out, const double* gram_in, double* gram_out, void* ws,
                      int* flag, double reorth_ratio, double* stats_out, const double* dec_a,
                      const double* q_ref, const double* d, double* dec_out,
                      const RotFuse* fuse) {
  if (fuse && !rot_fusable(r_cur, r))
    return set_error(ctx, ADROM_ERR_ARG, "isvd_update: fused epilogue needs r in {32, 64}");
  if (r_cur < 1 || r_cur > 128 || r < 1 || r > r_cur + 1)
    return set_error(ctx, ADROM_ERR_ARG, "isvd_update: bad ranks r_cur=%d r=%d", r_cur, r);
  if (phi_out == phi && r != r_cur)
    return set_error(ctx, ADROM_ERR_ARG, "isvd_update: in-place update needs r == r_cur");
  if (gram_out && r != r_cur)
    return set_error(ctx, ADROM_ERR_ARG, "isvd_update: a tracked Gram needs r == r_cur");
  char* w = (char*)ws;
  auto take = [&](size_t bytes) {
    void* q = w;
    w += align_up(bytes);
    return q;
  };
  double* partial = (double*)take(sizeof(double) * isvd_partial_doubles(ctx, r_cur));
  double* red1 = (double*)take(sizeof(double) * (r_cur + 1));
  double* red2 = (double*)take(sizeof(double) * (r_cur + 1));
  double* pls = (double*)take(sizeof(double) * r_cur);
  double* p2 = (double*)take(sizeof(double) * r_cur);
  double* B = (double*)take(sizeof(double) * (r_cur + 1) * r);
  double* T = (double*)take(sizeof(double) * (r_cur + 1) * r);
  double* Gloc = (double*)take(sizeof(double) * r_cur * r_cur);
  double* sbuf = (double*)take(sizeof(double) * 16);
  int* need = (int*)take(sizeof(int) * 4);
  double* qbuf = (double*)take(sizeof(double) * (size_t)n);
  double* vglob = (double*)take(sizeof(double) * core_vglob_doubles(r_cur));
  double* stats = stats_out ? stats_out : sbuf;
  double* qinv = sbuf + 12;
  int st;
  const double* G = gram_in;
  if (!G) {  // Gram afresh (one extra N r^2 pass; the session tracks it instead)
    st = ts_gram(ctx, phi, n, r_cur, Gloc, partial, isvd_partial_doubles(ctx, r_cur));
    if (st) return st;
    G = Gloc;
  }
  // pass 1: p1 = Phi^T y, ||y||^2 (+ fused decode of the ROM state if asked)
  int pr = prof_begin(ctx, PROBE_ISVD_PROJECT);
  if (dec_a)
    st = ts_decode_project(ctx, phi, n, r_cur, dec_a, q_ref, d, dec_out, y, red1, partial, flag);
  else
    st = ts_project(ctx, phi, n, r_cur, W_X, y, nullptr, nullptr, red1, partial, flag);
  prof_end(ctx, pr);
  if (st) return st;
  // least squares p = G^{-1} p1 (gelsd semantics for a full-rank basis)
  isvd_solve_kernel<<<1, 128, 0, ctx->stream>>>(red1, G, r_cur, reorth_ratio, pls, need);
  ADROM_LAUNCH_CK(ctx);
  st = isvd_solve_direct_launch(ctx, red1, G, r_cur, reorth_ratio, pls, need);
  if (st) return st;
  // pass 2 always: q = y - Phi p, Phi^T q, ||q||^2, then one least-squares
  // refinement step (isvd_refine_kernel: q' = q - Phi p2 orthogonal to the
  // actual basis; the rotation forms q_hat = (q - Phi p2) / ||q'||)
  set_need_kernel<<<1, 1, 0, ctx->stream>>>(need);
  ADROM_LAUNCH_CK(ctx);
  pr = prof_begin(ctx, PROBE_ISVD_RESID);
  st = ts_residual(ctx, phi, n, r_cur, pls, y, red2, partial, flag, need, qbuf);
  prof_end(ctx, pr);
  if (st) return st;
  st = isvd_refine_launch(ctx, G, r_cur, red2, pls, p2, nullptr, need);
  if (st) return st;
  const bool vg = core_v_global(r_cur);
  const size_t csm = core_smem(r_cur, vg);
  pr = prof_begin(ctx, PROBE_ISVD_CORE);
  // Gout may alias G: the kernel reads G completely before its final barrier
  double* Gout = gram_out ? gram_out : Gloc;
  if (vg) {
    cudaFuncSetAttribute(isvd_core_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)csm);
    isvd_core_kernel<true><<<1, core_threads(r_cur), csm, ctx->stream>>>(
        sigma, red1, pls, red2, need, G, r_cur, r, lam, B, qinv, T, Gout, sigma_out, stats, flag,
        nullptr, vglob, core_force_jacobi());
  } else {
    cudaFuncSetAttribute(isvd_core_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)csm);
    isvd_core_kernel<false><<<1, core_threads(r_cur), csm, ctx->stream>>>(
        sigma, red1, pls, red2, need, G, r_cur, r, lam, B, qinv, T, Gout, sigma_out, stats, flag,
        nullptr, nullptr, core_force_jacobi());
  }
  prof_end(ctx, pr);
  ADROM_LAUNCH_CK(ctx);
  // the rotation reads q from pass 2 when it ran, else forms it from y and p
  RotArgs ra{phi, y, qbuf, need, pls, qinv, B, n, r_cur, r, phi_out};
  if (fuse) ra.fuse = *fuse;
  ra.p2 = p2;
  pr = prof_begin(ctx, PROBE_ISVD_ROTATE);
  st = ts_rotate(ctx, ra);
  prof_end(ctx, pr);
  return st;
}

int isvd_solve_launch(adrom_ctx* ctx, const double* red1, const double* G, int r, double* p,
                      int* need) {
  isvd_solve_kernel<<<1, 128, 0, ctx->stream>>>(red1, G, r, ISVD_REORTH_RATIO, p, need);
  ADROM_LAUNCH_CK(ctx);
  int st = isvd_solve_direct_launch(ctx, red1, G, r, ISVD_REORTH_RATIO, p, need);
  if (st) return st;
  return ADROM_OK;
}


int isvd_core_launch(adrom_ctx* ctx, const double* sigma, const double* red1, const double* pls,
                     const double* red2, const int* need, const double* G, int r, double lam,
                     double* B, double* qinv, double* T, double* Gout, double* sigma_out,
                     double* stats, int* flag, double* udrop) {
  const size_t csm = core_smem(r);
  cudaFuncSetAttribute(isvd_core_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)csm);
  isvd_core_kernel<false><<<1, core_threads(r), csm, ctx->stream>>>(sigma, red1, pls, red2, need, G, r, r,
                                                             lam, B, qinv, T, Gout, sigma_out, stats,
                                                             flag, udrop, nullptr, core_force_jacobi());
  ADROM_LAUNCH_CK(ctx);
  return ADROM_OK;
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
