// Exact-greedy QDEIM with a certified candidate pool (sampling.py:77-114).
//
// The pivots of a column-pivoted QR of phi^T are chosen one at a time: the
// row with the largest residual norm after projecting out the directions of
// the rows already chosen (ties -> lowest row, LAPACK idamax).  Each choice
// depends on all earlier ones, so a naive GPU version makes one pass over
// the N x r basis per pivot (r passes).  Here one pass certifies many pivots:
//
//   pass:    res2_i <- res2_i - sum_{new l} (phi_i . d_l)^2 for every row
//            (downdating, as geqp3 does; each value carries an error bound)
//   extract: per chunk of CH rows keep the T rows with the largest res2 (the
//            pool) and record the largest res2 + error bound among the rest
//            (tau: no row outside the pool can exceed it, now or later,
//            because residual norms never increase)
//   vectors: exact residual vectors of the pool rows (CGS2 against the
//            confirmed directions)
//   greedy:  cooperative kernel over the pool: pick the pool argmax, accept
//            it iff its residual^2 > tau, orthogonalise the pool against its
//            direction, repeat.  Every accepted pivot is exactly the global
//            greedy choice.
// Small grids (N <= POOL_ALL) put every row in the pool: one pass.
#include <cooperative_groups.h>

#include "common.cuh"
#include "sampling_internal.cuh"

#include <limits.h>

namespace cg = cooperative_groups;

namespace adrom {

constexpr int QP_CH = 4096;        // rows per extraction chunk
constexpr int QP_T = 32;           // pool rows per chunk
constexpr int64_t POOL_ALL = 1 << 16;
constexpr double QP_EPS = 2.220446049250313e-16;
constexpr int QP_TILE = 128;       // rows per pass tile (one thread per row)

__device__ __forceinline__ bool excluded_row(int64_t i, const int64_t* ex, int n_ex) {
  int a = 0, b = n_ex - 1;
  while (a <= b) {
    const int mid = (a + b) >> 1;
    const int64_t v = ex[mid];
    if (v == i) return true;
    if (v < i) a = mid + 1;
    else b = mid - 1;
  }
  return false;
}

// ---------------------------------------------------------------------------
// pass: res2 / bound update for the directions d_lo..d_hi-1 (D: r x r,
// column l = d_l, row-major D[j*r + l]); the first pass seeds res2 =
// ||phi_i||^2.  Excluded rows (earlier restarts, confirmed pivots) -> -1.
// The tile is staged in smem (coalesced), one thread per row; for r <= 64
// the row lives in registers, the directions are broadcast from smem.
// ---------------------------------------------------------------------------
template <int RMAX>
__global__ void __launch_bounds__(QP_TILE) qp_pass_kernel(const double* __restrict__ phi,
                                                          int64_t n, int r,
                                                          const double* __restrict__ D, int lo,
                                                          int hi, bool first,
                                                          double* __restrict__ res2,
                                                          double* __restrict__ bnd2,
                                                          const int64_t* __restrict__ ex,
                                                          int n_ex) {
  extern __shared__ double sm[];
  const int S = r | 1;
  const int nd = hi - lo;
  double* tile = sm;                   // QP_TILE x S
  double* Ds = tile + QP_TILE * S;     // nd x r  (direction-major: Ds[l*r + j])
  const int tid = threadIdx.x;
  for (int e = tid; e < r * nd; e += blockDim.x) {
    const int l = e / r, j = e - l * r;
    Ds[l * r + j] = D[j * r + lo + l];
  }
  const int64_t ntiles = (n + QP_TILE - 1) / QP_TILE;
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int64_t row0 = t * QP_TILE;
    const int rows = (int)((n - row0 < QP_TILE) ? (n - row0) : QP_TILE);
    __syncthreads();
    for (int e = tid; e < rows * r; e += blockDim.x) {
      const int a = e / r, c = e - a * r;
      tile[a * S + c] = phi[row0 * r + e];
    }
    __syncthreads();
    if (tid < rows) {
      const int64_t i = row0 + tid;
      const double* rowp = tile + tid * S;
      double v[RMAX <= 64 ? RMAX : 1];
      double nrm = 0.0;
      if (RMAX <= 64) {
#pragma unroll
        for (int c = 0; c < (RMAX <= 64 ? RMAX : 1); ++c) {
          v[c] = (c < r) ? rowp[c] : 0.0;
          nrm = fma(v[c], v[c], nrm);
        }
      } else {
        for (int c = 0; c < r; ++c) nrm = fma(rowp[c], rowp[c], nrm);
      }
      const double old = first ? 0.0 : res2[i];
      bool excl = (!first && old < 0.0) || excluded_row(i, ex, n_ex);
      double r2 = first ? nrm : old;
      if (!excl && !first) {
        for (int l = 0; l < nd; ++l) {
          const double* dl = Ds + l * r;
          double s = 0.0;
          if (RMAX <= 64) {
#pragma unroll
            for (int c = 0; c < (RMAX <= 64 ? RMAX : 1); ++c)
              if (c < r) s = fma(v[c], dl[c], s);
          } else {
            for (int c = 0; c < r; ++c) s = fma(rowp[c], dl[c], s);
          }
          r2 -= s * s;
        }
      }
      res2[i] = excl ? -1.0 : r2;
      // downdating error bound (geqp3-style norm updates)
      bnd2[i] = excl ? -1.0 : r2 + 8.0 * (double)(hi + 2) * QP_EPS * nrm;
    }
  }
}

// streaming variant for r in {16, 32, 64, 128}: LPR lanes per row, 16-byte
// loads straight from global, U rows in flight per warp, segmented shuffles
template <int R>
__global__ void __launch_bounds__(256) qp_pass_stream_kernel(const double* __restrict__ phi,
                                                             int64_t n,
                                                             const double* __restrict__ D,
                                                             int lo, int hi, bool first,
                                                             double* __restrict__ res2,
                                                             double* __restrict__ bnd2,
                                                             const int64_t* __restrict__ ex,
                                                             int n_ex) {
  constexpr int LPR = R / 8;  // 8 doubles per lane: 32/LPR rows share a warp
  constexpr int VPL = R / LPR;
  constexpr int RPW = 32 / LPR;
  constexpr int U = 4;
  extern __shared__ __align__(16) double Ds[];  // nd x R (direction-major)
  const int nd = hi - lo;
  for (int e = threadIdx.x; e < R * nd; e += blockDim.x) {
    const int l = e / R, j = e - l * R;
    Ds[l * R + j] = D[j * R + lo + l];
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int seg = lane / LPR, sl = lane - seg * LPR;
  const int64_t total_warps = (int64_t)gridDim.x * 8;
  const int64_t rows_per_iter = (int64_t)RPW * U;
  for (int64_t g = (int64_t)blockIdx.x * 8 + warp; g * rows_per_iter < n; g += total_warps) {
    const int64_t base = g * rows_per_iter;
    double2 val[U][VPL / 2];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = base + u * RPW + seg;
      if (i < n) {
        const double2* rowp = reinterpret_cast<const double2*>(phi + i * R);
#pragma unroll
        for (int h = 0; h < VPL / 2; ++h) val[u][h] = rowp[sl + LPR * h];
      } else {
#pragma unroll
        for (int h = 0; h < VPL / 2; ++h) val[u][h] = make_double2(0.0, 0.0);
      }
    }
    double nrm[U], sub[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      double a = 0.0;
#pragma unroll
      for (int h = 0; h < VPL / 2; ++h) a += val[u][h].x * val[u][h].x + val[u][h].y * val[u][h].y;
#pragma unroll
      for (int o = LPR / 2; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
      nrm[u] = a;
      sub[u] = 0.0;
    }
    for (int l = 0; l < nd; ++l) {
      const double2* dl = reinterpret_cast<const double2*>(Ds + l * R);
      double2 d2[VPL / 2];
#pragma unroll
      for (int h = 0; h < VPL / 2; ++h) d2[h] = dl[sl + LPR * h];
      double s[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        double a = 0.0;
#pragma unroll
        for (int h = 0; h < VPL / 2; ++h) a += val[u][h].x * d2[h].x + val[u][h].y * d2[h].y;
        s[u] = a;
      }
#pragma unroll
      for (int o = LPR / 2; o > 0; o >>= 1)
#pragma unroll
        for (int u = 0; u < U; ++u) s[u] += __shfl_xor_sync(0xffffffffu, s[u], o);
#pragma unroll
      for (int u = 0; u < U; ++u) sub[u] += s[u] * s[u];
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = base + u * RPW + seg;
      if (sl == 0 && i < n) {
        const double old = first ? 0.0 : res2[i];
        const bool excl = (!first && old < 0.0) || excluded_row(i, ex, n_ex);
        const double r2 = first ? nrm[u] : old - sub[u];
        res2[i] = excl ? -1.0 : r2;
        bnd2[i] = excl ? -1.0 : r2 + 8.0 * (double)(hi + 2) * QP_EPS * nrm[u];
      }
    }
  }
}

// mark confirmed pivots as excluded
__global__ void qp_mark_kernel(const int64_t* __restrict__ piv, int lo, int hi,
                               double* __restrict__ res2, double* __restrict__ bnd2) {
  for (int k = lo + threadIdx.x; k < hi; k += blockDim.x) {
    res2[piv[k]] = -1.0;
    bnd2[piv[k]] = -1.0;
  }
}

// ---------------------------------------------------------------------------
// extract: per chunk, the T largest res2 (ties: lower row first) -> pool;
// bound = max bnd2 over the other (non-excluded) rows of the chunk
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned long long qp_key(double v) {
  // non-negative doubles order like their bit patterns; excluded (-1) -> 0
  return v < 0.0 ? 0ull : (unsigned long long)__double_as_longlong(v) + 1ull;
}

constexpr int QP_EX_NT = 256;

// exclusive block scan (blockDim.x multiple of 32, <= 1024); *total = sum
__device__ __forceinline__ int block_excl_scan(int v, int* wsum, int* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  __syncthreads();
  if (lane == 31) wsum[warp] = x;
  __syncthreads();
  int off = 0, tot = 0;
  for (int w = 0; w < nw; ++w) {
    const int s = wsum[w];
    if (w < warp) off += s;
    tot += s;
  }
  *total = tot;
  return off + x - v;
}

__global__ void __launch_bounds__(QP_EX_NT) qp_extract_kernel(const double* __restrict__ res2,
                                                              const double* __restrict__ bnd2,
                                                              int64_t n, int ch, int T,
                                                              int64_t* __restrict__ pool_idx,
                                                              double* __restrict__ chunk_bound) {
  __shared__ unsigned long long keys[QP_CH];
  __shared__ int cnt_sh, dig_sh, above_sh;
  __shared__ int hist[256], wsum[QP_EX_NT / 32];
  __shared__ double bred[QP_EX_NT / 32];
  const int64_t c0 = (int64_t)blockIdx.x * ch;
  const int rows = (int)((n - c0 < ch) ? (n - c0) : ch);
  const int tid = threadIdx.x;
  for (int j = tid; j < rows; j += blockDim.x) keys[j] = qp_key(res2[c0 + j]);
  __syncthreads();
  // threshold = T-th largest key: radix select, 8 digits of 8 bits
  unsigned long long thr = 0ull;
  if (rows >= T) {
    unsigned long long mask = 0ull;
    int need = T;
    for (int shift = 56; shift >= 0; shift -= 8) {
      hist[tid] = 0;
      __syncthreads();
      for (int j = tid; j < rows; j += blockDim.x) {
        const unsigned long long k = keys[j];
        if ((k & mask) == thr) atomicAdd(&hist[(int)((k >> shift) & 255ull)], 1);
      }
      __syncthreads();
      // suffix counts: thread t holds bins >= 255 - t ... via inclusive scan of
      // the reversed histogram
      int v = hist[255 - tid];
      const int lane = tid & 31, warp = tid >> 5;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int x = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += x;
      }
      if (lane == 31) wsum[warp] = v;
      __syncthreads();
      int off = 0;
      for (int w = 0; w < warp; ++w) off += wsum[w];
      const int incl = v + off;                    // keys with digit >= 255 - tid
      const int excl = incl - hist[255 - tid];     // keys with digit >  255 - tid
      if (excl < need && incl >= need) {
        dig_sh = 255 - tid;
        above_sh = excl;
      }
      __syncthreads();
      thr |= (unsigned long long)dig_sh << shift;
      mask |= 255ull << shift;
      need -= above_sh;
      __syncthreads();
    }
  }
  // each thread owns a contiguous run of rows (index order preserved)
  const int per = (rows + QP_EX_NT - 1) / QP_EX_NT;
  const int j0 = tid * per, j1 = (j0 + per < rows) ? j0 + per : rows;
  int gt = 0, eq = 0;
  for (int j = j0; j < j1; ++j) {
    const unsigned long long k = keys[j];
    if (k == 0ull) continue;
    if (k > thr) ++gt;
    else if (k == thr) ++eq;
  }
  int tot_gt, tot_eq;
  const int gpos0 = block_excl_scan(gt, wsum, &tot_gt);
  const int epos0 = block_excl_scan(eq, wsum, &tot_eq);
  if (tid == 0) cnt_sh = tot_gt;  // total above the threshold (< T when ties fill the rest)
  __syncthreads();
  const int total_gt = cnt_sh;
  const int eq_allowed = T - total_gt;
  int64_t* out = pool_idx + (int64_t)blockIdx.x * T;
  int gpos = gpos0, epos = epos0;
  double bmax = -1.0;
  for (int j = j0; j < j1; ++j) {
    const unsigned long long k = keys[j];
    if (k == 0ull) continue;
    bool in = false;
    if (k > thr) {
      in = true;
      out[gpos++] = c0 + j;
    } else if (k == thr && epos < eq_allowed) {
      in = true;
      out[total_gt + epos] = c0 + j;
      ++epos;
    } else if (k == thr) {
      ++epos;
    }
    if (!in) bmax = fmax(bmax, bnd2[c0 + j]);
  }
  // (pool slots beyond the chunk's valid rows keep the -1 of qp_fill_kernel)
  for (int o = 16; o > 0; o >>= 1) bmax = fmax(bmax, __shfl_xor_sync(0xffffffffu, bmax, o));
  if ((tid & 31) == 0) bred[tid >> 5] = bmax;
  __syncthreads();
  if (tid == 0) {
    double b = -1.0;
    for (int q = 0; q < QP_EX_NT / 32; ++q) b = fmax(b, bred[q]);
    chunk_bound[blockIdx.x] = b;
  }
}

// -1 in every pool slot (rows with fewer than T valid candidates keep -1)
__global__ void qp_fill_kernel(int64_t* __restrict__ p, int64_t P) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < P;
       i += (int64_t)gridDim.x * blockDim.x)
    p[i] = -1;
}

// ---------------------------------------------------------------------------
// exact residual vectors of the pool rows (CGS2 against confirmed d_0..d_k-1)
// warp per pool row; R row-major P x r; excluded rows -> pres2 = -1
// ---------------------------------------------------------------------------
template <int RMAX>
__global__ void __launch_bounds__(256) qp_resvec_kernel(const double* __restrict__ phi, int r,
                                                        const int64_t* __restrict__ pool_idx,
                                                        int64_t P, const double* __restrict__ D,
                                                        int k, const double* __restrict__ res2,
                                                        double* __restrict__ Rv,
                                                        double* __restrict__ pres2) {
  constexpr int H = (RMAX + 31) / 32;
  extern __shared__ double Ds[];  // r x 65
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int e = threadIdx.x; e < r * k; e += blockDim.x) {
    const int j = e / k, l = e - j * k;
    Ds[j * 65 + l] = D[j * r + l];
  }
  __syncthreads();
  const int64_t total_warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t p = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp; p < P; p += total_warps) {
    const int64_t i = pool_idx[p];
    const bool live = i >= 0 && res2[i] >= 0.0;
    double v[H];
#pragma unroll
    for (int h = 0; h < H; ++h) {
      const int c = lane + 32 * h;
      v[h] = (live && c < r) ? phi[i * r + c] : 0.0;
    }
    for (int pass = 0; pass < 2; ++pass) {
      for (int l = 0; l < k; ++l) {
        double s = 0.0;
#pragma unroll
        for (int h = 0; h < H; ++h) {
          const int c = lane + 32 * h;
          if (c < r) s += v[h] * Ds[c * 65 + l];
        }
        s = warp_sum(s);
#pragma unroll
        for (int h = 0; h < H; ++h) {
          const int c = lane + 32 * h;
          if (c < r) v[h] -= s * Ds[c * 65 + l];
        }
      }
    }
    double nr = 0.0;
#pragma unroll
    for (int h = 0; h < H; ++h) {
      const int c = lane + 32 * h;
      if (c < r) Rv[p * r + c] = v[h];
      nr += v[h] * v[h];
    }
    nr = warp_sum(nr);
    if (lane == 0) pres2[p] = live ? nr : -1.0;
  }
}

// ---------------------------------------------------------------------------
// cooperative greedy over the pool
// state[0] = k (confirmed count), state[2] = rank-deficient step + 1
// ---------------------------------------------------------------------------
struct GreedyArgs {
  const int64_t* pool_idx;
  int64_t P;
  double* Rv;        // P x r
  double* pres2;     // P
  const double* chunk_bound;
  int nchunks;
  double* D;         // r x r (column l = d_l)
  int64_t* piv;      // pivots (chunk-local list, m entries)
  int m;             // pivots wanted in this restart chunk
  int r;
  int* state;
  double* bv;        // per-block best value [grid]
  int64_t* bi;       // per-block best pool slot [grid]
  int64_t* brow;     // per-block best row [grid]
  double* err_res;   // residual at the failing step
  int all_in_pool;   // no rows outside the pool (tau = -inf)
};

// (value, row) order: larger residual first, ties to the lower row
__device__ __forceinline__ bool cand_better(double v, int64_t row, double bv, int64_t brow) {
  return v > bv || (v == bv && row < brow);
}

struct Cand {
  double v;
  int64_t row, slot;
};

__device__ __forceinline__ void cand_merge(Cand& a, const Cand& b) {
  if (cand_better(b.v, b.row, a.v, a.row)) a = b;
}

__device__ __forceinline__ Cand cand_warp_reduce(Cand c) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    Cand t;
    t.v = __shfl_xor_sync(0xffffffffu, c.v, o);
    t.row = __shfl_xor_sync(0xffffffffu, c.row, o);
    t.slot = __shfl_xor_sync(0xffffffffu, c.slot, o);
    cand_merge(c, t);
  }
  return c;
}

// block-wide reduce; result valid in every thread
__device__ __forceinline__ Cand cand_block_reduce(Cand c, Cand* sc) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  c = cand_warp_reduce(c);
  if (lane == 0) sc[warp] = c;
  __syncthreads();
  if (warp == 0) {
    Cand t = (lane < nw) ? sc[lane] : Cand{-1.0, LLONG_MAX, -1};
    t = cand_warp_reduce(t);
    if (lane == 0) sc[0] = t;
  }
  __syncthreads();
  const Cand out = sc[0];
  __syncthreads();
  return out;
}

// Row update of the pool against the accepted direction d (smem): R > 0 uses
// R/8 lanes per row (8 values per lane, 32/(R/8) rows per warp); R == 0 is
// the generic warp-per-row path.  Tracks the best updated candidate.
template <int R>
__device__ __forceinline__ void qp_pool_update(const GreedyArgs& A, const double* d, int64_t gs,
                                               bool apply, Cand& best) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t total_warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int64_t gw = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp;
  if constexpr (R > 0) {
    constexpr int LPR = R / 8, RPW = 32 / LPR;
    const int seg = lane / LPR, sl = lane - seg * LPR;
    double2 dv[4];
#pragma unroll
    for (int h = 0; h < 4; ++h) dv[h] = reinterpret_cast<const double2*>(d)[sl + LPR * h];
    for (int64_t p0 = gw * RPW; p0 < A.P; p0 += total_warps * RPW) {
      const int64_t p = p0 + seg;
      const bool valid = p < A.P;
      const double old = valid ? A.pres2[p] : -1.0;
      const bool live = old >= 0.0 && p != gs;
      double2* rv = reinterpret_cast<double2*>(A.Rv + p * R);
      double2 x[4];
      double s = 0.0;
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        x[h] = live ? rv[sl + LPR * h] : make_double2(0.0, 0.0);
        s += x[h].x * dv[h].x + x[h].y * dv[h].y;
      }
#pragma unroll
      for (int o = LPR / 2; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (!apply) s = 0.0;
      double nr = 0.0;
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        x[h].x -= s * dv[h].x;
        x[h].y -= s * dv[h].y;
        nr += x[h].x * x[h].x + x[h].y * x[h].y;
      }
#pragma unroll
      for (int o = LPR / 2; o > 0; o >>= 1) nr += __shfl_xor_sync(0xffffffffu, nr, o);
      if (live && apply) {
#pragma unroll
        for (int h = 0; h < 4; ++h) rv[sl + LPR * h] = x[h];
      }
      const double nv = live ? (apply ? nr : old) : -1.0;
      if (sl == 0 && valid && (old >= 0.0) && apply) A.pres2[p] = nv;
      if (nv >= 0.0) {
        const int64_t row = A.pool_idx[p];
        if (cand_better(nv, row, best.v, best.row)) best = Cand{nv, row, p};
      }
    }
  } else {
    const int r = A.r;
    for (int64_t p = gw; p < A.P; p += total_warps) {
      const double old = A.pres2[p];
      if (old < 0.0) continue;
      if (p == gs) {
        if (lane == 0 && apply) A.pres2[p] = -1.0;
        continue;
      }
      double nv = old;
      if (apply) {
        double* rv = A.Rv + p * r;
        double s = 0.0;
        for (int c = lane; c < r; c += 32) s += rv[c] * d[c];
        s = warp_sum(s);
        double nr = 0.0;
        for (int c = lane; c < r; c += 32) {
          const double x = rv[c] - s * d[c];
          rv[c] = x;
          nr += x * x;
        }
        nv = warp_sum(nr);
        if (lane == 0) A.pres2[p] = nv;
      }
      const int64_t row = A.pool_idx[p];
      if (cand_better(nv, row, best.v, best.row)) best = Cand{nv, row, p};
    }
  }
}

// One grid barrier per accepted pivot: the update of step k also produces the
// per-block candidates of step k + 1 (double-buffered per parity).
template <int R>
__global__ void __launch_bounds__(256) qp_greedy_kernel(GreedyArgs A) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(16) double dsm[];
  double* d = dsm;  // r
  __shared__ Cand sc[8];
  __shared__ double tau_sh;
  const int tid = threadIdx.x;
  const int r = A.r;
  {
    double t = -1.0;
    if (!A.all_in_pool)
      for (int c = tid; c < A.nchunks; c += blockDim.x) t = fmax(t, A.chunk_bound[c]);
    Cand c{t, 0, 0};
    c = cand_block_reduce(c, sc);
    if (tid == 0) tau_sh = c.v;
    __syncthreads();
  }
  const double tau = tau_sh;
  const int G = gridDim.x;
  int k = A.state[0];
  // initial candidates (no update)
  {
    Cand c{-1.0, LLONG_MAX, -1};
    qp_pool_update<R>(A, d, -1, false, c);
    c = cand_block_reduce(c, sc);
    if (tid == 0) {
      A.bv[blockIdx.x] = c.v;
      A.brow[blockIdx.x] = c.row;
      A.bi[blockIdx.x] = c.slot;
    }
  }
  grid.sync();
  int par = 0;
  while (k < A.m) {
    Cand gc{-1.0, LLONG_MAX, -1};
    for (int q = tid; q < G; q += blockDim.x) {
      const Cand t{A.bv[par * G + q], A.brow[par * G + q], A.bi[par * G + q]};
      if (t.slot >= 0) cand_merge(gc, t);
    }
    gc = cand_block_reduce(gc, sc);
    const double g = gc.v;
    const int64_t gs = gc.slot;
    // uniform across the grid: every block reduced the same per-block results
    if (!(gs >= 0 && g > tau)) {
      if (blockIdx.x == 0 && tid == 0) *A.err_res = (gs >= 0) ? sqrt(g) : 0.0;
      break;
    }
    if (!(sqrt(g) >= 1e-14)) {  // sampling.py:97-101 rank deficiency
      if (blockIdx.x == 0 && tid == 0) {
        A.state[2] = k + 1;
        *A.err_res = sqrt(g);
      }
      break;
    }
    const double inv = 1.0 / sqrt(g);
    // row gs itself is never rewritten (only its pres2), so no barrier here
    for (int c = tid; c < r; c += blockDim.x) d[c] = A.Rv[gs * r + c] * inv;
    __syncthreads();
    if (blockIdx.x == 0) {
      for (int c = tid; c < r; c += blockDim.x) A.D[c * r + k] = d[c];
      if (tid == 0) A.piv[k] = gc.row;
    }
    if (blockIdx.x == (int)(gs % G) && tid == 0) A.pres2[gs] = -1.0;
    Cand c{-1.0, LLONG_MAX, -1};
    qp_pool_update<R>(A, d, gs, true, c);
    c = cand_block_reduce(c, sc);
    par ^= 1;
    if (tid == 0) {
      A.bv[par * G + blockIdx.x] = c.v;
      A.brow[par * G + blockIdx.x] = c.row;
      A.bi[par * G + blockIdx.x] = c.slot;
    }
    ++k;
    grid.sync();
  }
  if (blockIdx.x == 0 && tid == 0) A.state[0] = k;
}

size_t qdeim_pool_workspace_bytes(int64_t n, int r, int count) {
  const int64_t nchunks = (n + QP_CH - 1) / QP_CH;
  const int64_t P = (n <= POOL_ALL) ? n : nchunks * QP_T;
  size_t b = 0;
  b += 2 * align_up(sizeof(double) * (size_t)n);           // res2, bnd2
  b += align_up(sizeof(int64_t) * (size_t)P);              // pool idx
  b += align_up(sizeof(double) * (size_t)P * r);           // Rv
  b += align_up(sizeof(double) * (size_t)P);               // pres2
  b += align_up(sizeof(double) * (size_t)nchunks);         // chunk bounds
  b += align_up(sizeof(double) * (size_t)r * r);           // D
  b += align_up(sizeof(int64_t) * (size_t)r);              // local pivots
  b += align_up(sizeof(int) * 8) + align_up(sizeof(double) * 2);
  b += 3 * align_up(sizeof(double) * 4096);                // per-block bests
  b += align_up(sizeof(int64_t) * (size_t)(count + 1));    // sorted exclusions
  return b;
}

__global__ void qp_sort_rows_kernel(const int64_t* __restrict__ in, int n, int64_t* __restrict__ out) {
  for (int i = 0; i < n; ++i) {
    const int64_t x = in[i];
    int j = i - 1;
    while (j >= 0 && out[j] > x) {
      out[j + 1] = out[j];
      --j;
    }
    out[j + 1] = x;
  }
}

__global__ void qp_all_rows_kernel(int64_t* __restrict__ pool_idx, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    pool_idx[i] = i;
}

template <int RMAX>
static int qp_pass(adrom_ctx* ctx, const double* phi, int64_t n, int r, const double* D, int lo,
                   int hi, bool first, double* res2, double* bnd2, const int64_t* ex, int n_ex) {
  const int64_t ntiles = (n + QP_TILE - 1) / QP_TILE;
  int64_t g = (int64_t)ctx->num_sms * 8;
  if (g > ntiles) g = ntiles;
  const size_t sm = sizeof(double) * ((size_t)QP_TILE * (r | 1) + (size_t)r * (hi - lo > 0 ? hi - lo : 1));
  cudaFuncSetAttribute(qp_pass_kernel<RMAX>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  qp_pass_kernel<RMAX><<<(int)(g < 1 ? 1 : g), QP_TILE, sm, ctx->stream>>>(
      phi, n, r, D, lo, hi, first, res2, bnd2, ex, n_ex);
  ADROM_LAUNCH_CK(ctx);
  return ADROM_OK;
}

template <int R>
static int qp_pass_stream(adrom_ctx* ctx, const double* phi, int64_t n, const double* D, int lo,
                          int hi, bool first, double* res2, double* bnd2, const int64_t* ex,
                          int n_ex) {
  constexpr int LPR = R / 8;  // 8 doubles per lane: 32/LPR rows share a warp
  const int64_t rows_per_warp_iter = (int64_t)(32 / LPR) * 4;
  const int64_t warps = (n + rows_per_warp_iter - 1) / rows_per_warp_iter;
  int64_t g = (int64_t)ctx->num_sms * 8;
  if (g > (warps + 7) / 8) g = (warps + 7) / 8;
  const size_t sm = sizeof(double) * (size_t)R * (hi - lo > 0 ? hi - lo : 1);
  cudaFuncSetAttribute(qp_pass_stream_kernel<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  qp_pass_stream_kernel<R><<<(int)(g < 1 ? 1 : g), 256, sm, ctx->stream>>>(
      phi, n, D, lo, hi, first, res2, bnd2, ex, n_ex);
  ADROM_LAUNCH_CK(ctx);
  return ADROM_OK;
}

template <int RMAX>
static int qp_resvec(adrom_ctx* ctx, const double* phi, int r, const int64_t* pool_idx, int64_t P,
                     const double* D, int k, const double* res2, double* Rv, double* pres2) {
  int64_t g = (P + 7) / 8;
  if (g > (int64_t)ctx->num_sms * 16) g = (int64_t)ctx->num_sms * 16;
  const size_t sm = sizeof(double) * (size_t)r * 65;
  cudaFuncSetAttribute(qp_resvec_kernel<RMAX>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  qp_resvec_kernel<RMAX><<<(int)(g < 1 ? 1 : g), 256, sm, ctx->stream>>>(phi, r, pool_idx, P, D, k,
                                                                        res2, Rv, pres2);
  ADROM_LAUNCH_CK(ctx);
  return ADROM_OK;
}

int qdeim_pool_select(adrom_ctx* ctx, const double* phi, int64_t n, int r, int count,
                      int64_t* out_idx, void* ws, int* passes_out) {
  if (count > n) return set_error(ctx, ADROM_ERR_DENSE, "cannot select %d pivots from %lld columns",
                                  count, (long long)n);
  if (r < 1 || r > 128) return set_error(ctx, ADROM_ERR_ARG, "qdeim: rank %d unsupported", r);
  const int64_t nchunks = (n + QP_CH - 1) / QP_CH;
  const bool all = n <= POOL_ALL;
  const int64_t P = all ? n : nchunks * QP_T;
  char* w = (char*)ws;
  auto take = [&](size_t bytes) {
    void* p = w;
    w += align_up(bytes);
    return p;
  };
  double* res2 = (double*)take(sizeof(double) * (size_t)n);
  double* bnd2 = (double*)take(sizeof(double) * (size_t)n);
  int64_t* pool_idx = (int64_t*)take(sizeof(int64_t) * (size_t)P);
  double* Rv = (double*)take(sizeof(double) * (size_t)P * r);
  double* pres2 = (double*)take(sizeof(double) * (size_t)P);
  double* cbound = (double*)take(sizeof(double) * (size_t)nchunks);
  double* D = (double*)take(sizeof(double) * (size_t)r * r);
  int64_t* piv = (int64_t*)take(sizeof(int64_t) * (size_t)r);
  int* state = (int*)take(sizeof(int) * 8);
  double* err_res = (double*)take(sizeof(double) * 2);
  double* bv = (double*)take(sizeof(double) * 4096);
  int64_t* bi = (int64_t*)take(sizeof(double) * 4096);
  int64_t* brow = (int64_t*)take(sizeof(double) * 4096);
  int64_t* ex = (int64_t*)take(sizeof(int64_t) * (size_t)(count + 1));
  int* hstate = (int*)ctx->pinned;
  double* hres = (double*)((char*)ctx->pinned + 64);
  int bpm = 0;
  const size_t gsm = sizeof(double) * r;
  void* gkern = (r == 16)    ? (void*)qp_greedy_kernel<16>
                : (r == 32)  ? (void*)qp_greedy_kernel<32>
                : (r == 64)  ? (void*)qp_greedy_kernel<64>
                : (r == 128) ? (void*)qp_greedy_kernel<128>
                             : (void*)qp_greedy_kernel<0>;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bpm, gkern, 256, gsm);
  if (bpm < 1) return set_error(ctx, ADROM_ERR_CUDA, "qdeim: greedy kernel cannot be resident");
  int ggrid = ctx->num_sms * (bpm < 2 ? bpm : 2);
  const int64_t need_blocks = (P + 255) / 256;
  if (ggrid > need_blocks) ggrid = (int)(need_blocks < 1 ? 1 : need_blocks);
  if (ggrid > 2048) ggrid = 2048;  // bests are double-buffered in 4096 slots
  auto pass = [&](int lo, int hi, bool first, int n_ex) -> int {
    if (r == 16) return qp_pass_stream<16>(ctx, phi, n, D, lo, hi, first, res2, bnd2, ex, n_ex);
    if (r == 32) return qp_pass_stream<32>(ctx, phi, n, D, lo, hi, first, res2, bnd2, ex, n_ex);
    if (r == 64) return qp_pass_stream<64>(ctx, phi, n, D, lo, hi, first, res2, bnd2, ex, n_ex);
    if (r == 128) return qp_pass_stream<128>(ctx, phi, n, D, lo, hi, first, res2, bnd2, ex, n_ex);
    if (r <= 32) return qp_pass<32>(ctx, phi, n, r, D, lo, hi, first, res2, bnd2, ex, n_ex);
    if (r <= 64) return qp_pass<64>(ctx, phi, n, r, D, lo, hi, first, res2, bnd2, ex, n_ex);
    return qp_pass<128>(ctx, phi, n, r, D, lo, hi, first, res2, bnd2, ex, n_ex);
  };
  auto resvec = [&](int k) -> int {
    if (r <= 32) return qp_resvec<32>(ctx, phi, r, pool_idx, P, D, k, res2, Rv, pres2);
    if (r <= 64) return qp_resvec<64>(ctx, phi, r, pool_idx, P, D, k, res2, Rv, pres2);
    return qp_resvec<128>(ctx, phi, r, pool_idx, P, D, k, res2, Rv, pres2);
  };
  int chosen = 0, passes = 0;
  while (chosen < count) {
    const int m = (count - chosen < r) ? (count - chosen) : r;
    const int n_ex = chosen;
    if (n_ex > 0) {
      qp_sort_rows_kernel<<<1, 1, 0, ctx->stream>>>(out_idx, n_ex, ex);
      ADROM_LAUNCH_CK(ctx);
    }
    ADROM_CK(ctx, cudaMemsetAsync(state, 0, sizeof(int) * 8, ctx->stream));
    int k = 0, lo = 0;
    bool first = true;
    while (k < m) {
      ++passes;
      const int pr = prof_begin(ctx, PROBE_QDEIM_SCAN);
      int st = pass(first ? 0 : lo, first ? 0 : k, first, n_ex);
      if (st) return st;
      if (!first && k > 0) {
        qp_mark_kernel<<<1, 128, 0, ctx->stream>>>(piv, 0, k, res2, bnd2);
        ADROM_LAUNCH_CK(ctx);
      }
      first = false;
      lo = k;
      int64_t gg = (P + 255) / 256;
      if (gg > ctx->num_sms * 8) gg = ctx->num_sms * 8;
      if (all) {
        qp_all_rows_kernel<<<(int)gg, 256, 0, ctx->stream>>>(pool_idx, n);
        ADROM_LAUNCH_CK(ctx);
      } else {
        qp_fill_kernel<<<(int)gg, 256, 0, ctx->stream>>>(pool_idx, P);
        ADROM_LAUNCH_CK(ctx);
        qp_extract_kernel<<<(int)nchunks, QP_EX_NT, 0, ctx->stream>>>(res2, bnd2, n, QP_CH, QP_T,
                                                                       pool_idx, cbound);
        ADROM_LAUNCH_CK(ctx);
      }
      st = resvec(k);
      if (st) return st;
      GreedyArgs ga{pool_idx, P, Rv, pres2, cbound, (int)nchunks, D, piv, m, r, state, bv, bi, brow,
                    err_res, all ? 1 : 0};
      void* args[] = {&ga};
      ADROM_CK(ctx, cudaLaunchCooperativeKernel(gkern, ggrid, 256, args, gsm,
                                                ctx->stream));
      ++ctx->launches;
      prof_end(ctx, pr);
      ADROM_CK(ctx, cudaMemcpyAsync(hstate, state, sizeof(int) * 4, cudaMemcpyDeviceToHost,
                                    ctx->stream));
      ADROM_CK(ctx, cudaMemcpyAsync(hres, err_res, sizeof(double), cudaMemcpyDeviceToHost,
                                    ctx->stream));
      ADROM_CK(ctx, cudaStreamSynchronize(ctx->stream));
      if (hstate[2])
        return set_error(ctx, ADROM_ERR_SINGULAR,
                         "rank deficiency at pivot step %d (residual column norm %.3e)",
                         chosen + hstate[2] - 1, hres[0]);
      const int knew = hstate[0];
      if (knew == k) {
        // nothing certifiable: only possible when the remaining residuals are
        // ties at (numerically) zero, i.e. the basis is rank deficient
        if (!(hres[0] >= 1e-14))
          return set_error(ctx, ADROM_ERR_SINGULAR,
                           "rank deficiency at pivot step %d (residual column norm %.3e)",
                           chosen + k, hres[0]);
        return set_error(ctx, ADROM_ERR_DENSE, "qdeim: no certified pivot at step %d", chosen + k);
      }
      k = knew;
    }
    ADROM_CK(ctx, cudaMemcpyAsync(out_idx + chosen, piv, sizeof(int64_t) * m,
                                  cudaMemcpyDeviceToDevice, ctx->stream));
    chosen += m;
  }
  if (passes_out) *passes_out = passes;
  return ADROM_OK;
}

}  // namespace adrom
