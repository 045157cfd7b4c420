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
#include <cuda_bf16.h>

#include "common.cuh"
#include "sampling_internal.cuh"
#include "factored_internal.cuh"

#include <limits.h>
#include <stdio.h>
#include <stdlib.h>

#include <vector>

namespace cg = cooperative_groups;

namespace adrom {

// pool target size; ADROM_QDEIM_POOL_M overrides (tuning experiments)
constexpr long long QP_M_DEFAULT = 1 << 15;
// rows refreshed per round = factor x pool size (grows 4x on a stalled
// round); ADROM_QDEIM_REFRESH overrides
static long long qp_refresh_factor() {
  static long long t = [] {
    const char* e = getenv("ADROM_QDEIM_REFRESH");
    const long long v = e ? atoll(e) : 0;
    return (v >= 1 && v <= 4096) ? v : 128ll;
  }();
  return t;
}

// refresh-set capacity over its target, in percent (the selection stops once
// the rows sharing the selected bound prefix fit); ADROM_QDEIM_CAPF overrides
static long long qp_refresh_slack() {
  static long long t = [] {
    const char* e = getenv("ADROM_QDEIM_CAPF");
    const long long v = e ? atoll(e) : -1;
    return (v >= 1 && v <= 1000) ? v : 25ll;
  }();
  return t;
}

// the refresh set may also grow to its capacity (ADROM_QDEIM_EXTEND_REFRESH)
static int qp_extend_refresh() {
  static const int v = getenv("ADROM_QDEIM_EXTEND_REFRESH") ? atoi(getenv("ADROM_QDEIM_EXTEND_REFRESH")) : 0;
  return v;
}

static long long qp_pool_m() {
  static long long t = [] {
    const char* e = getenv("ADROM_QDEIM_POOL_M");
    const long long v = e ? atoll(e) : 0;
    return (v >= 64 && v <= (1ll << 24)) ? v : QP_M_DEFAULT;
  }();
  return t;
}

constexpr int64_t POOL_ALL = 1 << 16;
constexpr double QP_EPS = 2.220446049250313e-16;

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

// mark confirmed pivots as excluded
__global__ void qp_mark_kernel(const int64_t* __restrict__ piv, int lo, int hi,
                               double* __restrict__ res2, double* __restrict__ bnd2) {
  for (int k = lo + threadIdx.x; k < hi; k += blockDim.x) {
    res2[piv[k]] = -1.0;
    bnd2[piv[k]] = -1.0;
  }
}

// lazy refresh: the pool rows' exact residuals (w.r.t. the k confirmed
// directions) tighten their bounds; rows outside the pool keep older, still
// valid bounds (residual norms never increase)
__global__ void qp_writeback_kernel(const int64_t* __restrict__ pool_idx, int64_t P,
                                    const double* __restrict__ pres2,
                                    const double* __restrict__ pn2, int k,
                                    const double* __restrict__ res2, double* __restrict__ bnd2) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < P;
       p += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = pool_idx[p];
    if (i < 0) continue;
    const double v = pres2[p];
    if (v < 0.0 || res2[i] < 0.0) continue;
    const double b = v + 8.0 * (double)(k + 2) * QP_EPS * pn2[p];
    if (b < bnd2[i]) bnd2[i] = b;
  }
}

// ---------------------------------------------------------------------------
// pool selection: the M rows with the largest bounds (global radix select on
// the bound's bit pattern, 8 digits of 8 bits, stopping early once the rows
// sharing the selected prefix fit the pool), then stream compaction.
// tau = an upper bound on every bound left outside the pool.
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned long long qp_key(double v) {
  // non-negative doubles order like their bit patterns; excluded (< 0) -> 0
  return v < 0.0 ? 0ull : (unsigned long long)__double_as_longlong(v) + 1ull;
}

struct SelState {
  unsigned long long prefix, mask;
  unsigned long long theta;  // pool = rows with key >= theta (theta >= 1)
  long long above;           // rows known to have key above the prefix
  long long need;            // rows still to take from the prefix bin
  int done;
  int pad;
  double tau;
  unsigned long long count;  // compaction counter
  // sign + exponent digit of the last selection's threshold, tagged
  // (QS_HINT_TAG | digit): the next selection through this state starts with
  // the mantissa digit inside that bin and falls back if the guess is wrong
  unsigned long long hint;
};
constexpr unsigned long long QS_HINT_TAG = 0xC0FFEE5E1EC70000ull;

// radix select: bits 63..60 (sign + the top three exponent bits) first, then
// 12 bits at a time (passes at shifts 60, 48, 36, 24, 12, 0).  Squared row
// norms of a basis share the top digit, so a selection normally starts from
// the previous one's top digit (SelState::hint) with the pass at shift 48 --
// eight exponent and four mantissa bits, bins 4.4 % wide -- and is done after
// that single pass when the threshold bin fits the capacity's slack.
constexpr int QS_BITS = 12, QS_BINS = 1 << QS_BITS, QS_TOP_SHIFT = 60;
__host__ __device__ inline int qs_bits(int shift) { return shift == QS_TOP_SHIFT ? 4 : QS_BITS; }
__host__ __device__ inline int qs_shift(int pass) { return pass == 0 ? QS_TOP_SHIFT : 60 - QS_BITS * pass; }

__global__ void qs_init_kernel(SelState* st, long long M, unsigned int* hist) {
  if (threadIdx.x == 0) {
    st->prefix = 0ull;
    st->mask = 0ull;
    st->theta = 1ull;
    st->above = 0;
    st->need = M;
    st->done = 0;
    st->tau = -1.0;
    st->count = 0ull;
  }
  for (int j = threadIdx.x; j < QS_BINS + 32; j += blockDim.x) hist[j] = 0u;
}

// ---------------------------------------------------------------------------
// The whole selection in ONE cooperative launch: up to six histogram passes
// (two grid barriers each: histogram -> digit choice by block 0), the stream
// compaction of the selected rows and the -1 fill of the unused output
// slots.  The separate kernels above cost 15 dependent launches per
// selection (7 selections per configuration-3 event), most of them early
// exits; here a finished selection leaves the pass loop at once.
// `hist` must be zero on entry (every digit step leaves it zeroed).
// ---------------------------------------------------------------------------
struct SelArgs {
  const double* vals;   // candidates' bounds (contiguous)
  int64_t n;
  const int64_t* list;  // candidate slot -> row (null: identity)
  SelState* st;
  unsigned int* hist;
  long long M;          // rows wanted
  long long cap;        // output capacity
  int extend;
  int64_t* out;         // cap slots; unused ones -> -1
};

// HINT: `prefix` is a guessed top digit; keys above its bin are counted into
// hist[QS_BINS] (they all belong to the selection)
template <bool HINT>
__device__ __forceinline__ void qs_hist_pass(const double* vals, int64_t n,
                                             unsigned long long prefix, unsigned long long mask,
                                             int shift, unsigned int* hist, unsigned int* sh) {
  constexpr int ITEMS = 8;
  for (int b = threadIdx.x; b < QS_BINS; b += blockDim.x) sh[b] = 0u;
  unsigned int above = 0u;
  __syncthreads();
  const unsigned long long dmask = (1ull << qs_bits(shift)) - 1ull;
  const int lane = threadIdx.x & 31;
  const int64_t tile = (int64_t)blockDim.x * ITEMS;
  for (int64_t t0 = blockIdx.x * tile; t0 < n; t0 += (int64_t)gridDim.x * tile) {
    double v[ITEMS];
#pragma unroll
    for (int q = 0; q < ITEMS; ++q) {
      const int64_t j = t0 + (int64_t)q * blockDim.x + threadIdx.x;
      v[q] = (j < n) ? __ldg(vals + j) : -1.0;
    }
#pragma unroll
    for (int q = 0; q < ITEMS; ++q) {
      const unsigned long long k = qp_key(v[q]);
      const int dig = (k != 0ull && (k & mask) == prefix) ? (int)((k >> shift) & dmask) : -1;
      if (HINT) above += (k & mask) > prefix;
      // bounds crowd into a few bins (or miss the prefix: -1): one vote for the
      // leader's digit, the other lanes add on their own
      const int d0 = __shfl_sync(0xffffffffu, dig, 0);
      const unsigned int same = __ballot_sync(0xffffffffu, dig == d0);
      if (lane == 0) {
        if (d0 >= 0) atomicAdd(&sh[d0], (unsigned int)__popc(same));
      } else if (dig >= 0 && dig != d0) {
        atomicAdd(&sh[dig], 1u);
      }
    }
  }
  if (HINT) {
    above = __reduce_add_sync(0xffffffffu, above);
    if (lane == 0 && above) atomicAdd(&hist[QS_BINS], above);
  }
  __syncthreads();
  for (int b = threadIdx.x; b < QS_BINS; b += blockDim.x) {
    const unsigned int c = sh[b];
    if (c) atomicAdd(&hist[b], c);
  }
}

// digit choice of one pass by ONE block of NT threads (QS_BINS / NT bins per
// thread, from the top): pick the digit holding the need-th largest remaining
// key; the pool may take every bin from the top down to the lowest one whose
// cumulative count still fits the capacity (and holds the need-th key)
template <int NT>
__device__ __forceinline__ void qs_digit_step(volatile SelState* st, int shift, unsigned int* hist,
                                              long long pcap, int extend, long long* wsum,
                                              int* ish, long long* lsh, bool hint_pass = false) {
  constexpr int BPT = QS_BINS / NT;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  long long hb[BPT];
  long long h = 0;
#pragma unroll
  for (int e = 0; e < BPT; ++e) {
    hb[e] = __ldcg(hist + (QS_BINS - 1 - (BPT * tid + e)));
    h += hb[e];
  }
  long long v = h;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const long long x = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += x;
  }
  if (lane == 31) wsum[warp] = v;
  if (tid == 0) {
    ish[0] = -1;        // digit
    ish[1] = QS_BINS;   // lowest bin that still fits
  }
  __syncthreads();
  long long off = 0;
  for (int w = 0; w < warp; ++w) off += wsum[w];
  const long long incl = v + off;
  long long excl = incl - h;
  const long long need = st->need;
  if (extend) {
    const long long limit = pcap - st->above;
    long long c = excl;
#pragma unroll
    for (int e = 0; e < BPT; ++e) {
      c += hb[e];
      if (hb[e] > 0 && c >= need && c <= limit) atomicMin(&ish[1], QS_BINS - 1 - (BPT * tid + e));
    }
  }
  if (excl < need && incl >= need) {
#pragma unroll
    for (int e = 0; e < BPT; ++e) {
      if (excl < need && excl + hb[e] >= need) {
        ish[0] = QS_BINS - 1 - (BPT * tid + e);
        lsh[0] = excl;
        lsh[1] = hb[e];
      }
      excl += hb[e];
    }
  }
  __syncthreads();
#pragma unroll
  for (int e = 0; e < BPT; ++e) hist[BPT * tid + e] = 0u;  // ready for the next pass / selection
  if (tid == 0) {
    const int dig = ish[0], dlow = ish[1];
    if (dig < 0 && hint_pass) {  // the need-th key lies below the guessed bin
      st->done = 2;
    } else if (dig < 0) {  // fewer candidates than M: take every live row
      st->theta = 1ull;
      st->tau = -1.0;
      st->done = 1;
    } else if (dlow < QS_BINS) {  // bins dlow.. of this prefix fit: done
      const unsigned long long th = st->prefix | ((unsigned long long)dlow << shift);
      st->theta = th < 1ull ? 1ull : th;
      st->tau = (th >= 2ull) ? __longlong_as_double((long long)(th - 2ull)) : -1.0;
      st->done = 1;
    } else {
      const unsigned long long pre = st->prefix | ((unsigned long long)dig << shift);
      st->prefix = pre;
      st->mask = st->mask | (((1ull << qs_bits(shift)) - 1ull) << shift);
      const long long above = st->above + lsh[0];
      st->above = above;
      st->need = need - lsh[0];
      const long long with_bin = above + lsh[1];
      if (with_bin <= pcap || shift == 0) {
        const unsigned long long th0 = (with_bin <= pcap) ? pre : pre + 1ull;
        const unsigned long long th = th0 < 1ull ? 1ull : th0;
        st->theta = th;
        st->tau = (th >= 2ull) ? __longlong_as_double((long long)(th - 2ull)) : -1.0;
        st->done = 1;
      }
    }
  }
  __syncthreads();
}

__global__ void __launch_bounds__(256) qs_select_compact_kernel(SelArgs a) {
  cg::grid_group grid = cg::this_grid();
  __shared__ unsigned int sh[QS_BINS];
  __shared__ long long wsum[8];
  __shared__ int ish[2];
  __shared__ long long lsh[2];
  volatile SelState* st = a.st;
  auto init_state = [&]() {  // thread 0 of block 0
    st->prefix = 0ull;
    st->mask = 0ull;
    st->theta = 1ull;
    st->above = 0;
    st->need = a.M;
    st->done = 0;
    st->tau = -1.0;
    st->count = 0ull;
  };
  int pass = 0;
  bool fin = false;  // (the state's own flag is stale until the first digit step)
  // guessed top digit: one pass over the mantissa digit inside its bin
  const unsigned long long hint = st->hint;  // (rewritten only after a grid barrier)
  if ((hint & ~0xFFFFull) == QS_HINT_TAG) {
    const unsigned long long topmask = 0xFull << QS_TOP_SHIFT;
    const unsigned long long hp = (hint & 0xFull) << QS_TOP_SHIFT;
    qs_hist_pass<true>(a.vals, a.n, hp, topmask, qs_shift(1), a.hist, sh);
    grid.sync();
    if (blockIdx.x == 0) {
      __shared__ int hint_ok;
      if (threadIdx.x == 0) {
        const long long above = (long long)__ldcg(a.hist + QS_BINS);
        a.hist[QS_BINS] = 0u;
        init_state();
        hint_ok = above < a.M;  // else the threshold lies above the guessed bin
        if (hint_ok) {
          st->prefix = hp;
          st->mask = topmask;
          st->above = above;
          st->need = a.M - above;
        }
      }
      __syncthreads();
      if (hint_ok) {
        qs_digit_step<256>(st, qs_shift(1), a.hist, a.cap, a.extend, wsum, ish, lsh, true);
      } else {
        for (int b = threadIdx.x; b < QS_BINS; b += blockDim.x) a.hist[b] = 0u;
        if (threadIdx.x == 0) st->done = 2;
      }
      __syncthreads();
      if (threadIdx.x == 0 && st->done == 2) {  // wrong guess: the full selection from the top
        init_state();
        st->hint = 0ull;
      }
      __threadfence();
    }
    grid.sync();
    pass = (st->hint == 0ull) ? 0 : 2;
    fin = st->done != 0;
  }
  for (; pass < 6 && !fin; ++pass) {
    const int shift = qs_shift(pass);
    unsigned long long prefix = 0ull, mask = 0ull;
    if (pass > 0) {
      prefix = st->prefix;
      mask = st->mask;
    }
    qs_hist_pass<false>(a.vals, a.n, prefix, mask, shift, a.hist, sh);
    grid.sync();
    if (blockIdx.x == 0) {
      if (pass == 0) {
        if (threadIdx.x == 0) init_state();
        __syncthreads();
      }
      qs_digit_step<256>(st, shift, a.hist, a.cap, a.extend, wsum, ish, lsh);
      __threadfence();
    }
    grid.sync();
    fin = st->done != 0;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    const unsigned long long th = st->theta;
    st->hint = (th >= 2ull) ? (QS_HINT_TAG | (th >> QS_TOP_SHIFT)) : 0ull;
  }
  // compaction: rows with key >= theta -> out[0..).  One atomic per block and
  // 4096-candidate tile (the counter is a single address: few, large
  // reservations); only the votes are kept between the count and the write.
  {
    constexpr int ITEMS = 16;
    int* wcnt = reinterpret_cast<int*>(sh);
    unsigned long long* base_sh = reinterpret_cast<unsigned long long*>(sh + 16);
    const unsigned long long theta = st->theta;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t tile = (int64_t)blockDim.x * ITEMS;
    for (int64_t t0 = blockIdx.x * tile; t0 < a.n; t0 += (int64_t)gridDim.x * tile) {
      double v[ITEMS];
#pragma unroll
      for (int q = 0; q < ITEMS; ++q) {
        const int64_t j = t0 + (int64_t)q * blockDim.x + threadIdx.x;
        v[q] = (j < a.n) ? __ldg(a.vals + j) : -1.0;
      }
      unsigned int balls[ITEMS];
      int mine = 0;
#pragma unroll
      for (int q = 0; q < ITEMS; ++q) {
        balls[q] = __ballot_sync(0xffffffffu, qp_key(v[q]) >= theta);
        mine += __popc(balls[q]);
      }
      if (lane == 0) wcnt[warp] = mine;
      __syncthreads();
      if (threadIdx.x == 0) {
        int tot = 0;
        for (int w = 0; w < 8; ++w) tot += wcnt[w];
        *base_sh = tot ? atomicAdd((unsigned long long*)&a.st->count, (unsigned long long)tot) : 0ull;
      }
      __syncthreads();
      unsigned long long pos = *base_sh;
      for (int w = 0; w < warp; ++w) pos += wcnt[w];
      if (mine) {
#pragma unroll
        for (int q = 0; q < ITEMS; ++q) {
          if (balls[q] & (1u << lane)) {
            const int64_t j = t0 + (int64_t)q * blockDim.x + threadIdx.x;
            const unsigned long long slot = pos + __popc(balls[q] & ((1u << lane) - 1u));
            if ((long long)slot < a.cap) a.out[slot] = a.list ? a.list[j] : j;
          }
          pos += __popc(balls[q]);
        }
      }
      __syncthreads();
    }
  }
  grid.sync();
  {
    const unsigned long long cnt = st->count;
    const long long from = (long long)cnt < a.cap ? (long long)cnt : a.cap;
    for (int64_t i = from + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < a.cap;
         i += (int64_t)gridDim.x * blockDim.x)
      a.out[i] = -1;
  }
}

// ---------------------------------------------------------------------------
// row pass (D: r x r, column l = d_l, row-major D[j*r + l]):
//   QP_SEED     res2 = bnd2 = ||phi_i||^2 for every row (rows of `ex` -> -1)
//   QP_REFRESH  the rows of `list` (n slots, -1 = empty): res2 -= sum over
//               the directions the row has not seen yet (ver_i <= l < hi) of
//               (phi_i . d_l)^2 (geqp3-style downdating); other rows keep
//               their older (still valid, larger) bounds
// R/8 lanes per row (8 columns each), 32/(R/8) rows per warp, 4 row groups
// in flight; EXACT (r == R) uses 16-byte loads, else scalar loads with the
// columns >= r zero.  Excluded rows (res2 < 0) are never touched.
// ---------------------------------------------------------------------------
enum { QP_SEED = 0, QP_REFRESH = 1 };

template <int R, bool EXACT>
__global__ void __launch_bounds__(256) qp_rows_kernel(const double* __restrict__ phi, int64_t n,
                                                      int r, const double* __restrict__ D, int hi,
                                                      int mode, const int64_t* __restrict__ list,
                                                      double* __restrict__ res2,
                                                      double* __restrict__ bnd2,
                                                      unsigned char* __restrict__ ver,
                                                      const int64_t* __restrict__ ex, int n_ex) {
  constexpr int LPR = R / 8;
  constexpr int RPW = 32 / LPR;
  constexpr int U = 4;
  extern __shared__ __align__(16) double Ds[];  // hi x R (direction-major, zero padded)
  const int nd = (mode == QP_SEED) ? 0 : hi;
  for (int e = threadIdx.x; e < R * nd; e += blockDim.x) {
    const int l = e / R, j = e - l * R;
    Ds[e] = (j < r) ? D[j * r + l] : 0.0;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int seg = lane / LPR, sl = lane - seg * LPR;
  const int64_t total_warps = (int64_t)gridDim.x * 8;
  const int64_t rows_per_iter = (int64_t)RPW * U;
  for (int64_t g = (int64_t)blockIdx.x * 8 + warp; g * rows_per_iter < n; g += total_warps) {
    const int64_t base = g * rows_per_iter;
    double2 val[U][4];
    bool act[U];
    int64_t rowi[U];
    int lv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t pos = base + u * RPW + seg;
      const int64_t i = (pos < n) ? (list ? list[pos] : pos) : -1;
      const bool a = i >= 0;
      rowi[u] = i;
      act[u] = a;
      lv[u] = (a && mode != QP_SEED) ? (int)ver[i] : nd;
      if (a) {
        if (EXACT) {
          const double2* rowp = reinterpret_cast<const double2*>(phi + i * R);
#pragma unroll
          for (int h = 0; h < 4; ++h) val[u][h] = rowp[sl + LPR * h];
        } else {
          const double* rowp = phi + i * r;
#pragma unroll
          for (int h = 0; h < 4; ++h) {
            const int c = 2 * (sl + LPR * h);
            val[u][h].x = (c < r) ? rowp[c] : 0.0;
            val[u][h].y = (c + 1 < r) ? rowp[c + 1] : 0.0;
          }
        }
      } else {
#pragma unroll
        for (int h = 0; h < 4; ++h) val[u][h] = make_double2(0.0, 0.0);
      }
    }
    bool any = false;
#pragma unroll
    for (int u = 0; u < U; ++u) any |= act[u];
    if (!__any_sync(0xffffffffu, any)) continue;
    double nrm[U], sub[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      double a = 0.0;
#pragma unroll
      for (int h = 0; h < 4; ++h) a += val[u][h].x * val[u][h].x + val[u][h].y * val[u][h].y;
#pragma unroll
      for (int o = LPR / 2; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
      nrm[u] = a;
      sub[u] = 0.0;
    }
    // downdate with the directions this row has not seen (ver_i .. hi-1)
    int lmin = nd;
#pragma unroll
    for (int u = 0; u < U; ++u) lmin = min(lmin, lv[u]);
    lmin = __reduce_min_sync(0xffffffffu, lmin);
    for (int l = lmin; l < nd; ++l) {
      const double2* dl = reinterpret_cast<const double2*>(Ds + l * R);
      double2 d2[4];
#pragma unroll
      for (int h = 0; h < 4; ++h) d2[h] = dl[sl + LPR * h];
      double s[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        double a = 0.0;
#pragma unroll
        for (int h = 0; h < 4; ++h) a += val[u][h].x * d2[h].x + val[u][h].y * d2[h].y;
        s[u] = a;
      }
#pragma unroll
      for (int o = LPR / 2; o > 0; o >>= 1)
#pragma unroll
        for (int u = 0; u < U; ++u) s[u] += __shfl_xor_sync(0xffffffffu, s[u], o);
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (l >= lv[u]) sub[u] += s[u] * s[u];
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = rowi[u];
      if (sl == 0 && act[u]) {
        if (mode == QP_SEED && excluded_row(i, ex, n_ex)) {
          res2[i] = -1.0;
          bnd2[i] = -1.0;
        } else if (mode == QP_SEED) {
          res2[i] = nrm[u];
          bnd2[i] = nrm[u] + 16.0 * QP_EPS * nrm[u];
          ver[i] = 0;
        } else {
          const double r2 = res2[i] - sub[u];
          res2[i] = r2;
          ver[i] = (unsigned char)nd;
          // min of two valid bounds (a pool write-back may be tighter)
          bnd2[i] = fmin(bnd2[i], r2 + 8.0 * (double)(nd + 2) * QP_EPS * nrm[u]);
        }
      }
    }
  }
}

// ---------------------------------------------------------------------------
// exact residual vectors of the pool rows (CGS2 against confirmed d_0..d_k-1)
// warp per pool row; R row-major P x r; excluded rows -> pres2 = -1
// ---------------------------------------------------------------------------
template <int R, bool EXACT>
__global__ void __launch_bounds__(256) qp_resvec_kernel(const double* __restrict__ phi, int r,
                                                        const int64_t* __restrict__ pool_idx,
                                                        int64_t P, const double* __restrict__ D,
                                                        int k, const double* __restrict__ res2,
                                                        double* __restrict__ Rv,
                                                        double* __restrict__ pres2,
                                                        double* __restrict__ pn2,
                                                        bool rows_in_rv) {
  constexpr int LPR = R / 8;
  constexpr int RPW = 32 / LPR;
  constexpr int U = 4;
  extern __shared__ __align__(16) double Ds[];  // k x R (direction-major, zero padded)
  for (int e = threadIdx.x; e < R * k; e += blockDim.x) {
    const int l = e / R, j = e - l * R;
    Ds[e] = (j < r) ? D[j * r + l] : 0.0;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int seg = lane / LPR, sl = lane - seg * LPR;
  const int64_t total_warps = (int64_t)gridDim.x * 8;
  const int64_t per_iter = (int64_t)RPW * U;
  for (int64_t g = (int64_t)blockIdx.x * 8 + warp; g * per_iter < P; g += total_warps) {
    double2 v[U][4];
    bool live[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t p = g * per_iter + u * RPW + seg;
      const int64_t i = (p < P) ? pool_idx[p] : -1;
      live[u] = i >= 0 && res2[i] >= 0.0;
      if (live[u]) {
        if (EXACT) {
          // rows_in_rv: the pool rows were materialised into Rv (factored basis)
          const double2* rowp = reinterpret_cast<const double2*>(rows_in_rv ? Rv + p * R : phi + i * R);
#pragma unroll
          for (int h = 0; h < 4; ++h) v[u][h] = rowp[sl + LPR * h];
        } else {
          const double* rowp = phi + i * r;
#pragma unroll
          for (int h = 0; h < 4; ++h) {
            const int c = 2 * (sl + LPR * h);
            v[u][h].x = (c < r) ? rowp[c] : 0.0;
            v[u][h].y = (c + 1 < r) ? rowp[c + 1] : 0.0;
          }
        }
      } else {
#pragma unroll
        for (int h = 0; h < 4; ++h) v[u][h] = make_double2(0.0, 0.0);
      }
    }
    // a warp whose slots are all empty (the pool holds fewer rows than its
    // capacity) or excluded only marks them
    {
      bool any = false;
#pragma unroll
      for (int u = 0; u < U; ++u) any |= live[u];
      if (!__any_sync(0xffffffffu, any)) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int64_t p = g * per_iter + u * RPW + seg;
          if (p < P && sl == 0) {
            pres2[p] = -1.0;
            pn2[p] = 0.0;
          }
        }
        continue;
      }
    }
    double nrm[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      double a = 0.0;
#pragma unroll
      for (int h = 0; h < 4; ++h) a += v[u][h].x * v[u][h].x + v[u][h].y * v[u][h].y;
#pragma unroll
      for (int o = LPR / 2; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
      nrm[u] = a;
    }
    // CGS2 against d_0..d_k-1
    for (int pass = 0; pass < 2; ++pass) {
      for (int l = 0; l < k; ++l) {
        const double2* dl = reinterpret_cast<const double2*>(Ds + l * R);
        double2 d2[4];
#pragma unroll
        for (int h = 0; h < 4; ++h) d2[h] = dl[sl + LPR * h];
        double s[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          double a = 0.0;
#pragma unroll
          for (int h = 0; h < 4; ++h) a += v[u][h].x * d2[h].x + v[u][h].y * d2[h].y;
          s[u] = a;
        }
#pragma unroll
        for (int o = LPR / 2; o > 0; o >>= 1)
#pragma unroll
          for (int u = 0; u < U; ++u) s[u] += __shfl_xor_sync(0xffffffffu, s[u], o);
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
          for (int h = 0; h < 4; ++h) {
            v[u][h].x -= s[u] * d2[h].x;
            v[u][h].y -= s[u] * d2[h].y;
          }
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t p = g * per_iter + u * RPW + seg;
      double a = 0.0;
#pragma unroll
      for (int h = 0; h < 4; ++h) a += v[u][h].x * v[u][h].x + v[u][h].y * v[u][h].y;
#pragma unroll
      for (int o = LPR / 2; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
      if (p < P) {
        if (EXACT) {
          double2* out = reinterpret_cast<double2*>(Rv + p * R);
#pragma unroll
          for (int h = 0; h < 4; ++h) out[sl + LPR * h] = v[u][h];
        } else {
          double* out = Rv + p * r;
#pragma unroll
          for (int h = 0; h < 4; ++h) {
            const int c = 2 * (sl + LPR * h);
            if (c < r) out[c] = v[u][h].x;
            if (c + 1 < r) out[c + 1] = v[u][h].y;
          }
        }
        if (sl == 0) {
          pres2[p] = live[u] ? a : -1.0;
          pn2[p] = nrm[u];
        }
      }
    }
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
  const double* tau_ptr;   // bound on the candidates left out of the pool
  const double* tau_ptr2;  // bound on the rows outside the candidate list
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
// Rows whose residual is already <= tau can never be accepted in this round
// (residuals only decrease): they are left untouched, their stale pres2 stays
// a valid upper bound for the write-back.
template <int R>
__device__ __forceinline__ void qp_pool_update(const GreedyArgs& A, const double* d, int64_t gs,
                                               bool apply, double tau, Cand& best) {
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
      const bool live = old >= 0.0 && old > tau && p != gs;
      if (!__any_sync(0xffffffffu, live)) {
        if (valid && p == gs && apply && sl == 0) A.pres2[p] = -1.0;
        continue;
      }
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
      if (sl == 0 && valid && apply) {
        if (live) A.pres2[p] = nv;
        else if (p == gs) A.pres2[p] = -1.0;
      }
      if (nv >= 0.0) {
        const int64_t row = A.pool_idx[p];
        if (cand_better(nv, row, best.v, best.row)) best = Cand{nv, row, p};
      }
    }
  } else {
    const int r = A.r;
    for (int64_t p = gw; p < A.P; p += total_warps) {
      const double old = A.pres2[p];
      if (p == gs) {
        if (lane == 0 && apply) A.pres2[p] = -1.0;
        continue;
      }
      if (old < 0.0 || !(old > tau)) continue;
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
    if (!A.all_in_pool) t = fmax(*A.tau_ptr, *A.tau_ptr2);
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
    qp_pool_update<R>(A, d, -1, false, tau, c);
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
    qp_pool_update<R>(A, d, gs, true, tau, c);
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

static int64_t qp_pool_capacity(int64_t n) {
  if (n <= POOL_ALL) return n;
  const int64_t cap = 2 * qp_pool_m();
  return cap < n ? cap : n;
}

size_t qdeim_pool_workspace_bytes(int64_t n, int r, int count) {
  const int64_t P = qp_pool_capacity(n);
  size_t b = 0;
  b += 2 * align_up(sizeof(double) * (size_t)n);           // res2, bnd2
  b += align_up(sizeof(int64_t) * (size_t)P);              // pool idx
  b += align_up(sizeof(double) * (size_t)P * r);           // Rv
  b += 2 * align_up(sizeof(double) * (size_t)P);           // pres2, pn2
  b += 2 * align_up(sizeof(SelState)) + align_up(sizeof(unsigned int) * (QS_BINS + 32));  // selection
  b += align_up(sizeof(double) * (size_t)n);               // bounds in refresh-list order
  b += align_up(sizeof(int64_t) * (size_t)n);              // refresh list
  b += align_up(sizeof(double) * (size_t)(r + FACT_KQ) * r);  // W D (factored rows)
  b += align_up((size_t)n);                                // per-row downdate version
  b += 2 * align_up(sizeof(double) * (size_t)r * r);       // D, complement basis E
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

// ---------------------------------------------------------------------------
// QP_REFRESH on the FP64 tensor cores (r in {32, 64, 128}): a warp takes 8
// list rows, S = X_rows D[:, lo:k] by DMMA m8n8k4 (A fragments straight from
// the rows in global memory, B fragments from smem), then
// res2 -= sum_{ver_i <= l < k} S_il^2 as in qp_rows_kernel.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void qp_dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// FACT: rows are X_i = [A_i | Q_i] of a factored basis Phi = X W (factored.cu)
// and Mm = W D ((R + FACT_KQ) x R, rows >= R + kf zero); the bound's norm term
// comes from nrmb (bounds of ||Phi_i||^2).  Otherwise rows are phi_i and Mm = D.
template <int R, bool FACT>
__global__ void __launch_bounds__(256) qp_refresh_tc_kernel(const double* __restrict__ phi,
                                                            const double* __restrict__ Qx, int kf, int64_t qn,
                                                            const double* __restrict__ nrmb,
                                                            const int64_t* __restrict__ list,
                                                            int64_t cap,
                                                            const double* __restrict__ Mm, int k,
                                                            double* __restrict__ res2,
                                                            double* __restrict__ bnd2,
                                                            unsigned char* __restrict__ ver) {
  constexpr int S = R + 4;                          // smem row stride
  constexpr int KX = FACT ? R + FACT_KQ : R;        // inner dimension
  constexpr int KS = KX / 4;                        // k-steps
  constexpr int DT = R / 8;                         // direction tiles
  extern __shared__ __align__(16) double Ds[];      // KX x S: Ds[j*S + l] = Mm[j][l] (l < k)
  for (int e = threadIdx.x; e < KX * R; e += blockDim.x) {
    const int j = e / R, l = e - j * R;
    Ds[j * S + l] = (l < k) ? Mm[j * R + l] : 0.0;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int rq = lane >> 2, cq = lane & 3;  // fragment row / column quad
  const int64_t tiles = (cap + 7) / 8;
  for (int64_t t = (int64_t)blockIdx.x * 8 + warp; t < tiles; t += (int64_t)gridDim.x * 8) {
    const int64_t pos = t * 8 + rq;
    const int64_t i = (pos < cap) ? list[pos] : -1;
    const int v = (i >= 0) ? (int)ver[i] : k;
    const int vmin = __reduce_min_sync(0xffffffffu, v);
    if (vmin >= k) continue;  // nothing new for any of the 8 rows
    double af[KS];
    double nrm = 0.0;
    const double* row = phi + (i >= 0 ? i : 0) * R;
#pragma unroll
    for (int j = 0; j < KS; ++j) {
      const int c = 4 * j + cq;
      double x = 0.0;
      if (i >= 0) {
        if (c < R) x = row[c];
        else if (c - R < kf) x = Qx[qpanel(i, c - R, qn)];
      }
      af[j] = x;
      if (!FACT) nrm = fma(x, x, nrm);
    }
    if (FACT) {
      nrm = (i >= 0) ? nrmb[i] : 0.0;
    } else {
      nrm += __shfl_xor_sync(0xffffffffu, nrm, 1);
      nrm += __shfl_xor_sync(0xffffffffu, nrm, 2);
    }
    double sub = 0.0;
    const int t0 = vmin >> 3, t1 = (k + 7) >> 3;
#pragma unroll
    for (int dt = 0; dt < DT; ++dt) {
      if (dt < t0 || dt >= t1) continue;
      double c0 = 0.0, c1 = 0.0;
#pragma unroll
      for (int j = 0; j < KS; ++j) qp_dmma(c0, c1, af[j], Ds[(4 * j + cq) * S + 8 * dt + rq]);
      // c0, c1 = S[row rq][dir 8 dt + 2 cq + {0, 1}]
      const int l0 = 8 * dt + 2 * cq;
      // rows of the C fragment are lane >> 2 as well: same row as this lane's A
      if (l0 >= v && l0 < k) sub = fma(c0, c0, sub);
      if (l0 + 1 >= v && l0 + 1 < k) sub = fma(c1, c1, sub);
    }
    sub += __shfl_xor_sync(0xffffffffu, sub, 1);
    sub += __shfl_xor_sync(0xffffffffu, sub, 2);
    if (cq == 0 && i >= 0 && v < k) {
      const double r2 = res2[i] - sub;
      res2[i] = r2;
      ver[i] = (unsigned char)k;
      bnd2[i] = fmin(bnd2[i], r2 + 8.0 * (double)(k + 2) * QP_EPS * nrm);
    }
  }
}

template <int R, bool FACT>
static int qp_refresh_tc(adrom_ctx* ctx, const double* phi, const double* Qx, int kf, int64_t qn,
                         const double* nrmb, const int64_t* list, int64_t cap, const double* Mm,
                         int k, double* res2, double* bnd2, unsigned char* ver) {
  constexpr int KX = FACT ? R + FACT_KQ : R;
  const size_t sm = sizeof(double) * (size_t)KX * (R + 4);
  const int64_t tiles = (cap + 7) / 8;
  int64_t g = (tiles + 7) / 8;
  if (g > (int64_t)ctx->num_sms * 8) g = (int64_t)ctx->num_sms * 8;
  cudaFuncSetAttribute(qp_refresh_tc_kernel<R, FACT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)sm);
  qp_refresh_tc_kernel<R, FACT><<<(int)(g < 1 ? 1 : g), 256, sm, ctx->stream>>>(
      phi, Qx, kf, qn, nrmb, list, cap, Mm, k, res2, bnd2, ver);
  ADROM_LAUNCH_CK(ctx);
  return ADROM_OK;
}

// ---------------------------------------------------------------------------
// Split-bf16 refresh (the default).  A refresh only has to produce valid UPPER
// bounds of the residuals -- the pool rows' exact residuals come from
// qp_resvec in fp64 and decide every pivot -- so S = X_rows Mm[:, v:k] runs on
// the bf16 tensor cores (mma.sync m16n8k16, 15x the FP64 DMMA rate here):
// x = x0 + x1 and m = m0 + m1 (bf16 each), x0 m0 + x0 m1 + x1 m0 accumulated
// in fp32.  Rows of Mm are scaled by exact powers of two to max |m| in
// [1/2, 1) and the matching columns of X by the inverse, so
//   |S^_il - S_il| <= delta_l = QP_BF_GAMMA ||x~_i|| ||m~_l|| + tiny
// (Cauchy-Schwarz; the dropped terms are ~3.1 u_bf16^2 |x||m| plus fp32
// accumulation; QP_BF_GAMMA = 8 u_bf16^2 leaves a factor > 2), and the bound
// subtracts only (|S^_il| - delta_l)_+^2 <= S_il^2.  res2 stays an upper
// bound of the residual; bnd2 adds the fp64 slack as before.
// ---------------------------------------------------------------------------
constexpr double QP_BF_GAMMA = 8.0 / 65536.0;
constexpr double QP_BF_TINY = 1e-33;

__device__ __forceinline__ void qp_bmma(float (&c)[4], const uint32_t (&a)[4], uint32_t b0,
                                        uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};\n"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// fast split for the row fragments: x -> f = fp32(x) (error 2^-24 |x|, inside
// the dropped terms), hi = bf16(f), lo = bf16(f - hi) (f - hi exact in fp32)
__device__ __forceinline__ void qp_split2f(double x, double y, uint32_t& hi, uint32_t& lo) {
  const float2 f = make_float2((float)x, (float)y);
  const __nv_bfloat162 h = __float22bfloat162_rn(f);
  const float2 hf = __bfloat1622float2(h);
  const __nv_bfloat162 l = __float22bfloat162_rn(make_float2(f.x - hf.x, f.y - hf.y));
  hi = *reinterpret_cast<const uint32_t*>(&h);
  lo = *reinterpret_cast<const uint32_t*>(&l);
}

// (x, y) -> packed bf16 pairs hi = (x0, y0), lo = (x1, y1); lower half = x
__device__ __forceinline__ void qp_split2(double x, double y, uint32_t& hi, uint32_t& lo) {
  const __nv_bfloat16 xh = __float2bfloat16_rn((float)x), yh = __float2bfloat16_rn((float)y);
  const __nv_bfloat16 xl = __float2bfloat16_rn((float)(x - (double)__bfloat162float(xh)));
  const __nv_bfloat16 yl = __float2bfloat16_rn((float)(y - (double)__bfloat162float(yh)));
  hi = (uint32_t)__bfloat16_as_ushort(xh) | ((uint32_t)__bfloat16_as_ushort(yh) << 16);
  lo = (uint32_t)__bfloat16_as_ushort(xl) | ((uint32_t)__bfloat16_as_ushort(yl) << 16);
}

// T: element type of the staged anchor rows -- the fp64 basis itself, or
// (factored session) its fp32 shadow, half the gather bytes; the fragments
// are fp32 splits either way, so the results are identical.  The residual
// columns Q (factored rows) are gathered in fp64.
template <int R, bool FACT, typename T>
struct QpBf {
  static constexpr int KX = FACT ? R + FACT_KQ : R;  // inner dimension (multiple of 16)
  static constexpr int KS = KX / 16;                 // k-steps
  static constexpr int NT = R / 8;                   // direction tiles
  static constexpr int EPC = 16 / (int)sizeof(T);    // elements per 16-byte chunk
  static constexpr int LC = (sizeof(T) == 8) ? 8 : 4;  // lanes per anchor row in the gather
  static constexpr int RPI = 32 / LC;                // anchor rows per gather instruction
  static constexpr int RS = R + 8;                   // staged anchor row stride (elements):
                                                     // fragment loads are conflict-free
  static constexpr int RSQ = FACT_KQ + 8;            // staged Q row stride (doubles)
  static constexpr int WPB = (R >= 128) ? 4 : (sizeof(T) == 4 ? 12 : 8);  // warps per block
  static constexpr int STAGE = 16 * RS;              // one 16-row anchor tile (elements)
  static constexpr int STAGEQ = FACT ? 16 * RSQ : 0;  // one 16-row Q tile (doubles)
  static constexpr size_t STAGE_BYTES = sizeof(T) * STAGE + sizeof(double) * STAGEQ;
  // smem: B fragments (KS x NT x 32 lanes x uint4), x scales (KX), ||m~_l|| (R),
  // two staged tiles per warp, ||m~_l|| in fp32 (R), x scales in fp32 (KX)
  static constexpr size_t smem_bytes = sizeof(uint4) * KS * NT * 32 +
                                       sizeof(double) * (KX + R) +
                                       (size_t)WPB * 2 * STAGE_BYTES + sizeof(float) * (R + KX);
  static_assert((R / EPC) % LC == 0 && STAGE_BYTES % 16 == 0, "gather split");
};

__device__ __forceinline__ void qp_cp16(void* smem, const void* gmem, int src_bytes) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem),
               "r"(src_bytes));
}

// Each warp owns 16-row tiles of the refresh list and stages the next tile's
// rows (gathered, 16-byte cp.async) while the current one is on the tensor
// cores: the gather is latency bound otherwise.
template <int R, bool FACT, typename T>
__global__ void __launch_bounds__(QpBf<R, FACT, T>::WPB * 32, 1)
    qp_refresh_bf_kernel(const T* __restrict__ phi, const double* __restrict__ Qx, int kf, int64_t qn,
                         const double* __restrict__ nrmb, const int64_t* __restrict__ list,
                         int64_t cap, const double* __restrict__ Mm, int k,
                         double* __restrict__ res2, double* __restrict__ bnd2,
                         unsigned char* __restrict__ ver, double* __restrict__ blist,
                         int kver, const int* __restrict__ cflag) {
  using C = QpBf<R, FACT, T>;
  // complement mode (kver >= 0): the k columns of Mm span the orthogonal
  // complement of the confirmed directions, so a row's residual is the SUM of
  // its squared components, res2 = sum (|S^| + delta)^2 -- no subtraction from
  // the seed, whose slack and the accumulated under-subtractions otherwise
  // swamp the last pivots' small residuals.  Every listed row is recomputed
  // and stamped with version kver.  *cflag != k: the complement basis is
  // incomplete -> bounds are left as they are.
  const bool cmode = kver >= 0;
  const bool cskip = cmode && cflag && *cflag != k;
  constexpr int KX = C::KX, KS = C::KS, NT = C::NT, RS = C::RS, WPB = C::WPB;
  constexpr int EPC = C::EPC, LC = C::LC, RPI = C::RPI;
  extern __shared__ __align__(16) unsigned char qbf_sm[];
  uint4* Bs = reinterpret_cast<uint4*>(qbf_sm);
  double* xsc = reinterpret_cast<double*>(Bs + KS * NT * 32);  // 2^e_j (x side)
  double* mn = xsc + KX;                                       // ||m~_l|| (rounded up)
  unsigned char* stg_all = reinterpret_cast<unsigned char*>(mn + R);
  float* mnf = reinterpret_cast<float*>(stg_all + (size_t)WPB * 2 * C::STAGE_BYTES);
  float* xscf = mnf + R;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int64_t tiles = (cap + 15) / 16;
  const int64_t tstride = (int64_t)gridDim.x * WPB;
  int64_t tl = (int64_t)blockIdx.x * WPB + warp;
  unsigned char* stg = stg_all + (size_t)warp * 2 * C::STAGE_BYTES;
  auto tileA = [&](int b) { return reinterpret_cast<T*>(stg + b * C::STAGE_BYTES); };
  auto tileQ = [&](int b) {
    return reinterpret_cast<double*>(stg + b * C::STAGE_BYTES + sizeof(T) * C::STAGE);
  };
  auto load_list = [&](int64_t tt) -> int64_t {
    const int64_t pos = tt * 16 + (lane & 15);
    return (tt < tiles && pos < cap) ? list[pos] : -1;
  };
  // anchor rows: LC lanes per row (whole 128-byte lines per instruction); Q
  // rows (fp64, 128 bytes): 8 lanes per row
  auto issue = [&](int64_t li, int b) {
    T* dA = tileA(b);
    const int sub = lane % LC;
#pragma unroll
    for (int rr = 0; rr < 16 / RPI; ++rr) {
      const int p = lane / LC + RPI * rr;
      const int64_t i = __shfl_sync(0xffffffffu, li, p);
      const int nb = i >= 0 ? 16 : 0;
      const T* srcA = phi + (i >= 0 ? i : 0) * R + EPC * sub;
      T* d = dA + p * RS + EPC * sub;
#pragma unroll
      for (int j = 0; j < R / EPC / LC; ++j) qp_cp16(d + EPC * LC * j, srcA + EPC * LC * j, nb);
    }
    if (FACT) {
      double* dQ = tileQ(b);
      const int sq = lane & 7;
#pragma unroll
      for (int rr = 0; rr < 4; ++rr) {
        const int p = (lane >> 3) + 4 * rr;
        const int64_t i = __shfl_sync(0xffffffffu, li, p);
        // only the live columns' sectors (zero fill beyond kf)
        const bool live = i >= 0 && 2 * sq < kf;
        qp_cp16(dQ + p * C::RSQ + 2 * sq, Qx + (live ? qpanel(i, 2 * sq, qn) : 0), live ? 16 : 0);
      }
    }
    asm volatile("cp.async.commit_group;\n");
  };
  // first tile's gather overlaps the prologue
  int64_t li_cur = load_list(tl);
  issue(li_cur, 0);
  auto row_ver = [&](int64_t li) -> int {
    if (!(lane < 16 && li >= 0) || cskip) return k;
    return cmode ? 0 : (int)ver[li];
  };
  int v_cur = row_ver(li_cur);
  int64_t li_next = load_list(tl + tstride);
  // row scales of Mm (directions l < k only)
  for (int j = threadIdx.x; j < KX; j += blockDim.x) {
    double mx = 0.0;
    for (int l = 0; l < k; ++l) mx = fmax(mx, fabs(Mm[j * R + l]));
    int e = 0;
    if (mx > 0.0 && isfinite(mx)) frexp(mx, &e);
    xsc[j] = ldexp(1.0, e);
    xscf[j] = (float)xsc[j];
  }
  __syncthreads();
  for (int l = threadIdx.x; l < R; l += blockDim.x) {
    double sm = 0.0;
    if (l < k)
      for (int j = 0; j < KX; ++j) {
        const double m = Mm[j * R + l] / xsc[j];
        sm = fma(m, m, sm);
      }
    mn[l] = sqrt(sm) * (1.0 + 1e-14);
    mnf[l] = __double2float_ru(mn[l]);
  }
  for (int e = threadIdx.x; e < KS * NT * 32; e += blockDim.x) {
    const int ln = e & 31, nt = (e >> 5) % NT, ks = (e >> 5) / NT;
    const int gg = ln >> 2, tt = ln & 3, l = 8 * nt + gg;
    const int j0 = 16 * ks + 2 * tt, j1 = j0 + 8;
    auto m = [&](int j) { return (l < k) ? Mm[j * R + l] / xsc[j] : 0.0; };
    uint4 b;
    qp_split2(m(j0), m(j0 + 1), b.x, b.z);
    qp_split2(m(j1), m(j1 + 1), b.y, b.w);
    Bs[e] = b;
  }
  __syncthreads();
  int s = 0;
  for (; tl < tiles; tl += tstride) {
    const int64_t tn = tl + tstride;
    issue(li_next, s ^ 1);  // empty rows when tn >= tiles
    const int v_next = row_ver(li_next);
    const int64_t li_nn = load_list(tn + tstride);
    const int vmin = __reduce_min_sync(0xffffffffu, v_cur);
    asm volatile("cp.async.wait_group 1;\n" ::: "memory");
    __syncwarp();
    if (vmin >= k) {  // nothing new: the list-order bounds only
      const int64_t pos = tl * 16 + lane;
      if (lane < 16 && pos < cap) blist[pos] = (li_cur >= 0) ? bnd2[li_cur] : -1.0;
    } else {
      int64_t ir[2];
      int vr[2];
      double r2o[2] = {0.0, 0.0}, b2o[2] = {0.0, 0.0}, nrm[2] = {0.0, 0.0};
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        ir[h] = __shfl_sync(0xffffffffu, li_cur, g + 8 * h);
        vr[h] = __shfl_sync(0xffffffffu, v_cur, g + 8 * h);
        if (t == 0 && ir[h] >= 0) {  // consumed after the MMAs
          b2o[h] = bnd2[ir[h]];
          if (vr[h] < k) {
            r2o[h] = res2[ir[h]];
            if (FACT) nrm[h] = nrmb[ir[h]];
          }
        }
      }
      const T* stA = tileA(s);
      const double* stQ = tileQ(s);
      uint32_t ah[KS][4], al[KS][4];
      double ss[2] = {0.0, 0.0}, nn[2] = {0.0, 0.0};
      float ssf[2] = {0.f, 0.f};
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {  // fragment register q: row g + 8 (q & 1), cols + 8 (q >> 1)
          const int h = q & 1;
          const int c = 16 * ks + 8 * (q >> 1) + 2 * t;
          if (sizeof(T) == 8 || c >= R) {
            double2 x;
            if (c < R) {
              x = *reinterpret_cast<const double2*>(stA + (g + 8 * h) * RS + c);
            } else {  // Q columns >= kf may hold a rejected event's data
              x = *reinterpret_cast<const double2*>(stQ + (g + 8 * h) * C::RSQ + c - R);
              if (c - R >= kf) x.x = 0.0;
              if (c + 1 - R >= kf) x.y = 0.0;
            }
            if (!FACT) nn[h] = fma(x.x, x.x, fma(x.y, x.y, nn[h]));
            x.x *= xsc[c];
            x.y *= xsc[c + 1];
            if (sizeof(T) == 8) {
              ss[h] = fma(x.x, x.x, fma(x.y, x.y, ss[h]));
              qp_split2f(x.x, x.y, ah[ks][q], al[ks][q]);
            } else {
              const float2 f = make_float2((float)x.x, (float)x.y);
              ssf[h] = fmaf(f.x, f.x, fmaf(f.y, f.y, ssf[h]));
              qp_split2f(x.x, x.y, ah[ks][q], al[ks][q]);
            }
          } else {
            // fp32 shadow: the same fp32 values qp_split2f would form
            float2 x = *reinterpret_cast<const float2*>(stA + (g + 8 * h) * RS + c);
            x.x *= xscf[c];
            x.y *= xscf[c + 1];
            ssf[h] = fmaf(x.x, x.x, fmaf(x.y, x.y, ssf[h]));
            const __nv_bfloat162 hb = __float22bfloat162_rn(x);
            const float2 hf = __bfloat1622float2(hb);
            const __nv_bfloat162 lb = __float22bfloat162_rn(make_float2(x.x - hf.x, x.y - hf.y));
            ah[ks][q] = *reinterpret_cast<const uint32_t*>(&hb);
            al[ks][q] = *reinterpret_cast<const uint32_t*>(&lb);
          }
        }
      }
      if constexpr (sizeof(T) == 4) {
        // fp32 sum of KX squares: relative error < KX 2^-24, covered by 1e-5
#pragma unroll
        for (int h = 0; h < 2; ++h) ss[h] = (double)ssf[h] * (1.0 + 1e-5);
      }
      // per-row error scale in fp32, rounded up (covers the fp32 rounding of
      // delta = dx * mn_l + tiny)
      float dx[2], dt0[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        ss[h] += __shfl_xor_sync(0xffffffffu, ss[h], 1);
        ss[h] += __shfl_xor_sync(0xffffffffu, ss[h], 2);
        const double xn = sqrt(ss[h]) * (1.0 + 1e-14);
        dx[h] = __double2float_ru(QP_BF_GAMMA * xn * (1.0 + 1e-6));
        dt0[h] = __double2float_ru(QP_BF_TINY * (1.0 + xn) * (1.0 + 1e-6));
        if (!FACT) {
          nn[h] += __shfl_xor_sync(0xffffffffu, nn[h], 1);
          nn[h] += __shfl_xor_sync(0xffffffffu, nn[h], 2);
          nrm[h] = nn[h];
        }
      }
      // sum of (|S^| - delta)_+^2 in fp32; every rounding can only inflate it
      // by (1 + 2^-24) per operation (<= KX + 8 operations per term and sum),
      // removed by the (1 - 2^-14) factor below
      float sub[2] = {0.f, 0.f};
      const int t0 = vmin >> 3, t1 = (k + 7) >> 3;
      // two direction tiles per iteration, the three products in separate
      // accumulators: six independent MMA chains
      for (int d0 = t0; d0 < t1; d0 += 2) {
        const bool two = d0 + 1 < t1;
        float c[2][3][4];
#pragma unroll
        for (int u = 0; u < 2; ++u)
#pragma unroll
          for (int p = 0; p < 3; ++p)
#pragma unroll
            for (int e = 0; e < 4; ++e) c[u][p][e] = 0.f;
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) {
          const uint4 b0 = Bs[(ks * NT + d0) * 32 + lane];
          qp_bmma(c[0][0], ah[ks], b0.x, b0.y);
          qp_bmma(c[0][1], ah[ks], b0.z, b0.w);
          qp_bmma(c[0][2], al[ks], b0.x, b0.y);
          if (two) {
            const uint4 b1 = Bs[(ks * NT + d0 + 1) * 32 + lane];
            qp_bmma(c[1][0], ah[ks], b1.x, b1.y);
            qp_bmma(c[1][1], ah[ks], b1.z, b1.w);
            qp_bmma(c[1][2], al[ks], b1.x, b1.y);
          }
        }
        // c[u][.][2h + e] = S^[row g + 8h][direction 8 (d0 + u) + 2t + e]
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          if (u == 1 && !two) break;
          const float2 m2 = *reinterpret_cast<const float2*>(mnf + 8 * (d0 + u) + 2 * t);
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int h = q >> 1, l = 8 * (d0 + u) + 2 * t + (q & 1);
            const float sv = (c[u][0][q] + c[u][1][q]) + c[u][2][q];
            const float dl = fmaf(dx[h], (q & 1) ? m2.y : m2.x, dt0[h]);
            float a = cmode ? fabsf(sv) + dl : fabsf(sv) - dl;
            a = (l >= vr[h] && l < k && a > 0.f) ? a : 0.f;
            sub[h] = fmaf(a, a, sub[h]);
          }
        }
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        sub[h] += __shfl_xor_sync(0xffffffffu, sub[h], 1);
        sub[h] += __shfl_xor_sync(0xffffffffu, sub[h], 2);
        const int64_t i = ir[h];
        const int64_t pos = tl * 16 + g + 8 * h;
        if (t == 0 && pos < cap) {
          double b = (i >= 0) ? b2o[h] : -1.0;
          if (i >= 0 && vr[h] < k && isfinite(sub[h])) {
            // fp32 rounding of the sum: deflated when subtracted, inflated when it IS the bound
            const double r2 = cmode ? fmin(r2o[h], (double)sub[h] * (1.0 + 1.0 / 16384.0))
                                    : fmax(r2o[h] - (double)sub[h] * (1.0 - 1.0 / 16384.0), 0.0);
            res2[i] = r2;
            ver[i] = (unsigned char)(cmode ? kver : k);
            b = fmin(b, r2 + 8.0 * (double)((cmode ? kver : k) + 2) * QP_EPS * nrm[h]);
            bnd2[i] = b;
          }
          blist[pos] = b;
        }
      }
    }
    __syncwarp();  // stage s is re-filled by the next iteration's issue
    li_cur = li_next;
    v_cur = v_next;
    li_next = li_nn;
    s ^= 1;
  }
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
}

static bool qp_refresh_fp64() {
  static const bool v = getenv("ADROM_QDEIM_REFRESH_FP64") && atoi(getenv("ADROM_QDEIM_REFRESH_FP64"));
  return v;
}

// blist[p] = bound of list[p] (-1 for empty slots): the pool selection reads
// the refreshed bounds contiguously
__global__ void qp_list_bounds_kernel(const int64_t* __restrict__ list, int64_t cap,
                                      const double* __restrict__ bnd2, double* __restrict__ blist) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < cap;
       p += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = list[p];
    blist[p] = (i >= 0) ? bnd2[i] : -1.0;
  }
}

static int qp_list_bounds(adrom_ctx* ctx, const int64_t* list, int64_t cap, const double* bnd2,
                          double* blist) {
  int64_t g = (cap + 255) / 256;
  if (g > (int64_t)ctx->num_sms * 8) g = (int64_t)ctx->num_sms * 8;
  qp_list_bounds_kernel<<<(int)(g < 1 ? 1 : g), 256, 0, ctx->stream>>>(list, cap, bnd2, blist);
  ADROM_LAUNCH_CK(ctx);
  return ADROM_OK;
}

template <int R, bool FACT, typename T>
static int qp_refresh_bf_launch(adrom_ctx* ctx, const T* phi, const double* Qx, int kf, int64_t qn,
                                const double* nrmb, const int64_t* list, int64_t cap,
                                const double* Mm, int k, double* res2, double* bnd2,
                                unsigned char* ver, double* blist, int kver, const int* cflag) {
  using C = QpBf<R, FACT, T>;
  const size_t sm = C::smem_bytes;
  const int64_t tiles = (cap + 15) / 16;
  int64_t g = (tiles + C::WPB - 1) / C::WPB;
  if (g > (int64_t)ctx->num_sms) g = (int64_t)ctx->num_sms;
  cudaFuncSetAttribute(qp_refresh_bf_kernel<R, FACT, T>,
                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  qp_refresh_bf_kernel<R, FACT, T><<<(int)(g < 1 ? 1 : g), C::WPB * 32, sm, ctx->stream>>>(
      phi, Qx, kf, qn, nrmb, list, cap, Mm, k, res2, bnd2, ver, blist, kver, cflag);
  ADROM_LAUNCH_CK(ctx);
  return ADROM_OK;
}

// refresh on the bf16 tensor cores; factored rows come from the fp32 shadows
// when the session keeps them (phi32, Qx32), else from the fp64 basis
template <int R, bool FACT>
static int qp_refresh_bf(adrom_ctx* ctx, const double* phi, const double* Qx, int kf, int64_t qn,
                         const double* nrmb, const int64_t* list, int64_t cap, const double* Mm,
                         int k, double* res2, double* bnd2, unsigned char* ver, double* blist,
                         const float* phi32 = nullptr, int kver = -1, const int* cflag = nullptr) {
  if (qp_refresh_fp64()) {
    const int st = qp_refresh_tc<R, FACT>(ctx, phi, Qx, kf, qn, nrmb, list, cap, Mm, k, res2, bnd2, ver);
    return st ? st : qp_list_bounds(ctx, list, cap, bnd2, blist);
  }
  if (FACT && phi32)
    return qp_refresh_bf_launch<R, FACT, float>(ctx, phi32, Qx, kf, qn, nrmb, list, cap, Mm, k, res2,
                                                bnd2, ver, blist, kver, cflag);
  return qp_refresh_bf_launch<R, FACT, double>(ctx, phi, Qx, kf, qn, nrmb, list, cap, Mm, k, res2, bnd2,
                                               ver, blist, kver, cflag);
}

// ---------------------------------------------------------------------------
// E (r x r row-major, columns 0 .. r-k-1): an orthonormal basis of the
// orthogonal complement of the k confirmed directions D[:, :k] in R^r: the
// pivoted Cholesky factor of the projector P = I - D D^T (P = L L^T with
// rank r - k makes L^T L = I), one block, r <= 64.  A step costs one argmax
// over the running diagonal and one column of L; the diagonal of the
// deflated projector has trace r - k - t, so its largest entry is at least
// 1 / r until the factor is complete.  One Gram-Schmidt pass against D
// removes the rounding of P.  *found = columns produced (r - k unless D has
// lost orthonormality; the refresh then leaves the bounds alone).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) qp_complement_kernel(const double* __restrict__ D, int r, int k,
                                                            double* __restrict__ E,
                                                            int* __restrict__ found) {
  constexpr int RM = 64, S = RM + 1;
  extern __shared__ __align__(16) double csm[];  // QP_COMPLEMENT_SMEM bytes
  double* Ds = csm;           // D[a * S + l], l < k
  double* L = Ds + RM * S;    // L[a * S + t]
  double* cf = L + RM * S;    // D^T L: k x 33 (r - k <= 32 columns)
  double* dg = cf + RM * S;   // running diagonal (RM)
  __shared__ int jsel;
  __shared__ double dsel;
  const int tid = threadIdx.x, lane = tid & 31;
  const int nE = r - k;
  for (int x = tid; x < r * r; x += blockDim.x) {
    const int a = x / r, l = x - a * r;
    Ds[a * S + l] = (l < k) ? D[(size_t)a * r + l] : 0.0;
  }
  __syncthreads();
  // diag(P) = 1 - |row a of D|^2; the columns of P are formed when chosen
  // (four threads per row share the sum over the directions)
  const int row = tid >> 2, part = tid & 3;
  {
    double s0 = 0.0;
    if (row < r)
      for (int l = part; l < k; l += 4) s0 = fma(Ds[row * S + l], Ds[row * S + l], s0);
    s0 += __shfl_xor_sync(0xffffffffu, s0, 1);
    s0 += __shfl_xor_sync(0xffffffffu, s0, 2);
    if (row < r && part == 0) dg[row] = 1.0 - s0;
  }
  __syncthreads();
  int t = 0;
  for (; t < nE; ++t) {
    if (tid < 32) {  // argmax of the running diagonal (ties to the lowest index)
      double v = (lane < r) ? dg[lane] : -1.0;
      int j = lane;
      if (lane + 32 < r && dg[lane + 32] > v) {
        v = dg[lane + 32];
        j = lane + 32;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double v2 = __shfl_xor_sync(0xffffffffu, v, o);
        const int j2 = __shfl_xor_sync(0xffffffffu, j, o);
        if (v2 > v || (v2 == v && j2 < j)) {
          v = v2;
          j = j2;
        }
      }
      if (lane == 0) {
        jsel = j;
        dsel = v;
      }
    }
    __syncthreads();
    if (!(dsel > 1e-6)) break;
    const int j = jsel;
    const double inv = 1.0 / sqrt(dsel);
    // L[:, t] = (P[:, j] - L[:, :t] L[j, :t]^T) / sqrt(d_j),  P[a][j] = delta_aj - D_a . D_j
    double v = 0.0;
    if (row < r) {
      for (int l = part; l < k; l += 4) v = fma(-Ds[row * S + l], Ds[j * S + l], v);
      for (int q = part; q < t; q += 4) v = fma(-L[row * S + q], L[j * S + q], v);
    }
    v += __shfl_xor_sync(0xffffffffu, v, 1);
    v += __shfl_xor_sync(0xffffffffu, v, 2);
    __syncthreads();  // every read of L[:, :t] done before column t is written
    if (row < r && part == 0) {
      v = (v + (row == j ? 1.0 : 0.0)) * inv;
      L[row * S + t] = v;
      dg[row] = (row == j) ? -1.0 : dg[row] - v * v;  // a used pivot never returns
    }
    __syncthreads();
  }
  // one Gram-Schmidt pass against D: L -= D (D^T L)
  for (int x = tid; x < k * t; x += blockDim.x) {
    const int l = x / t, c = x - l * t;
    double s0 = 0.0;
    for (int a = 0; a < r; ++a) s0 = fma(Ds[a * S + l], L[a * S + c], s0);
    cf[l * 33 + c] = s0;
  }
  __syncthreads();
  for (int x = tid; x < r * r; x += blockDim.x) {
    const int a = x / r, c = x - a * r;
    double v = 0.0;
    if (c < t) {
      v = L[a * S + c];
      for (int l = 0; l < k; ++l) v = fma(-Ds[a * S + l], cf[l * 33 + c], v);
    }
    E[(size_t)a * r + c] = v;
  }
  if (tid == 0) *found = t;
}

constexpr size_t QP_COMPLEMENT_SMEM = sizeof(double) * (3 * 64 * 65 + 5 * 64);

// complement-mode refresh (ADROM_QDEIM_COMPLEMENT=0 turns it off)
static bool qp_complement_on() {
  static const bool v = !(getenv("ADROM_QDEIM_COMPLEMENT") && atoi(getenv("ADROM_QDEIM_COMPLEMENT")) == 0);
  return v;
}

// Mm ((r + FACT_KQ) x r) = W D for the directions l < k (rows >= r + kf zero).
// With the dropped direction of the iSVD event (vdrop, X coordinates) column 0
// is vdrop and the directions follow in columns 1..k: the refresh then removes
// the seed's slack (X_i . vdrop)^2 together with the first downdate, and a
// row's version counts columns of this extended list.
__global__ void qp_wd_kernel(const double* __restrict__ W, int rkf, int r,
                             const double* __restrict__ D, int k,
                             const double* __restrict__ vdrop, double* __restrict__ Mm) {
  const int sh = vdrop ? 1 : 0;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < (r + FACT_KQ) * r;
       e += gridDim.x * blockDim.x) {
    const int j = e / r, c = e - j * r, l = c - sh;
    double s = 0.0;
    if (j < rkf) {
      if (l < 0) s = vdrop[j];
      else if (l < k)
        for (int q = 0; q < r; ++q) s += W[(size_t)j * r + q] * D[(size_t)q * r + l];
    }
    Mm[e] = s;
  }
}

template <int R, bool EXACT>
static int qp_rows_launch(adrom_ctx* ctx, const double* phi, int64_t n, int r, const double* D,
                          int hi, int mode, const int64_t* list, double* res2, double* bnd2,
                          unsigned char* ver, const int64_t* ex, int n_ex) {
  constexpr int LPR = R / 8;
  const int64_t rows_per_warp_iter = (int64_t)(32 / LPR) * 4;
  const int64_t warps = (n + rows_per_warp_iter - 1) / rows_per_warp_iter;
  int64_t g = (int64_t)ctx->num_sms * 8;
  if (g > (warps + 7) / 8) g = (warps + 7) / 8;
  const int nd = (mode == QP_SEED) ? 0 : hi;
  const size_t sm = sizeof(double) * (size_t)R * (nd > 0 ? nd : 1);
  cudaFuncSetAttribute(qp_rows_kernel<R, EXACT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  qp_rows_kernel<R, EXACT><<<(int)(g < 1 ? 1 : g), 256, sm, ctx->stream>>>(
      phi, n, r, D, hi, mode, list, res2, bnd2, ver, ex, n_ex);
  ADROM_LAUNCH_CK(ctx);
  return ADROM_OK;
}

template <int R, bool EXACT>
static int qp_resvec(adrom_ctx* ctx, const double* phi, int r, const int64_t* pool_idx, int64_t P,
                     const double* D, int k, const double* res2, double* Rv, double* pres2,
                     double* pn2, bool rows_in_rv = false) {
  const int64_t per_block = (int64_t)(32 / (R / 8)) * 4 * 8;
  int64_t g = (P + per_block - 1) / per_block;
  if (g > (int64_t)ctx->num_sms * 8) g = (int64_t)ctx->num_sms * 8;
  const size_t sm = sizeof(double) * (size_t)R * (k > 0 ? k : 1);
  cudaFuncSetAttribute(qp_resvec_kernel<R, EXACT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  qp_resvec_kernel<R, EXACT><<<(int)(g < 1 ? 1 : g), 256, sm, ctx->stream>>>(
      phi, r, pool_idx, P, D, k, res2, Rv, pres2, pn2, rows_in_rv);
  ADROM_LAUNCH_CK(ctx);
  return ADROM_OK;
}

// diagnostics (ADROM_QDEIM_TRACE >= 2): rows whose bound exceeds g / 4^j
__global__ void qp_count_above_kernel(const double* __restrict__ bnd2, int64_t n, double g,
                                      unsigned long long* __restrict__ cnt) {
  unsigned long long c[4] = {0, 0, 0, 0};
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double b = bnd2[i];
    double t = g;
    for (int j = 0; j < 4; ++j, t *= 0.25) c[j] += b > t;
  }
  for (int j = 0; j < 4; ++j)
    if (c[j]) atomicAdd(&cnt[j], c[j]);
}

void qdeim_seed_buffers(void* ws, int64_t n, double** res2, double** bnd2, unsigned char** ver) {
  char* w = (char*)ws;
  *res2 = (double*)w;
  w += align_up(sizeof(double) * (size_t)n);
  *bnd2 = (double*)w;
  w += align_up(sizeof(double) * (size_t)n);
  *ver = (unsigned char*)w;
}

int qdeim_pool_select(adrom_ctx* ctx, const double* phi, int64_t n, int r, int count,
                      int64_t* out_idx, void* ws, int* passes_out, bool seeded,
                      const FactBasis* fb, const double* nrmb) {
  if (count > n) return set_error(ctx, ADROM_ERR_DENSE, "cannot select %d pivots from %lld columns",
                                  count, (long long)n);
  if (r < 1 || r > 128) return set_error(ctx, ADROM_ERR_ARG, "qdeim: rank %d unsupported", r);
  // factored basis rows (Phi = X W): the k = 0 bounds must come seeded, one
  // restart chunk only (count <= r); the caller materialises Phi otherwise
  const bool fact = fb && fb->W;
  if (fact && (!seeded || count > r || !(r == 32 || r == 64) || !nrmb))
    return set_error(ctx, ADROM_ERR_ARG, "qdeim: factored rows need a seeded single chunk");
  const bool all = n <= POOL_ALL;
  const int64_t P = qp_pool_capacity(n);
  char* w = (char*)ws;
  auto take = [&](size_t bytes) {
    void* p = w;
    w += align_up(bytes);
    return p;
  };
  double* res2 = (double*)take(sizeof(double) * (size_t)n);
  double* bnd2 = (double*)take(sizeof(double) * (size_t)n);
  unsigned char* ver = (unsigned char*)take((size_t)n);  // (qdeim_seed_buffers)
  int64_t* pool_idx = (int64_t*)take(sizeof(int64_t) * (size_t)P);
  double* Rv = (double*)take(sizeof(double) * (size_t)P * r);
  double* pres2 = (double*)take(sizeof(double) * (size_t)P);
  double* pn2 = (double*)take(sizeof(double) * (size_t)P);
  SelState* sel = (SelState*)take(sizeof(SelState));
  SelState* selR = (SelState*)take(sizeof(SelState));
  int64_t* rlist = (int64_t*)take(sizeof(int64_t) * (size_t)n);
  unsigned int* hist = (unsigned int*)take(sizeof(unsigned int) * (QS_BINS + 32));  // [QS_BINS]: rows above a hinted bin
  double* blist = (double*)take(sizeof(double) * (size_t)n);  // bounds in refresh-list order
  double* Mw = (double*)take(sizeof(double) * (size_t)(r + FACT_KQ) * r);
  double* D = (double*)take(sizeof(double) * (size_t)r * r);
  double* Ec = (double*)take(sizeof(double) * (size_t)r * r);
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
  auto rows_pass = [&](int64_t nn, int hi, int mode, const int64_t* sl, int n_ex) -> int {
    if (r == 16) return qp_rows_launch<16, true>(ctx, phi, nn, r, D, hi, mode, sl, res2, bnd2, ver, ex, n_ex);
    if (r == 32) return qp_rows_launch<32, true>(ctx, phi, nn, r, D, hi, mode, sl, res2, bnd2, ver, ex, n_ex);
    if (r == 64) return qp_rows_launch<64, true>(ctx, phi, nn, r, D, hi, mode, sl, res2, bnd2, ver, ex, n_ex);
    if (r == 128) return qp_rows_launch<128, true>(ctx, phi, nn, r, D, hi, mode, sl, res2, bnd2, ver, ex, n_ex);
    if (r < 16) return qp_rows_launch<16, false>(ctx, phi, nn, r, D, hi, mode, sl, res2, bnd2, ver, ex, n_ex);
    if (r < 32) return qp_rows_launch<32, false>(ctx, phi, nn, r, D, hi, mode, sl, res2, bnd2, ver, ex, n_ex);
    if (r < 64) return qp_rows_launch<64, false>(ctx, phi, nn, r, D, hi, mode, sl, res2, bnd2, ver, ex, n_ex);
    return qp_rows_launch<128, false>(ctx, phi, nn, r, D, hi, mode, sl, res2, bnd2, ver, ex, n_ex);
  };
  auto resvec = [&](int k) -> int {
    if (fact) {  // pool rows of Phi = X W materialised into Rv, CGS2 in place
      int st2 = fact_gather_rows(ctx, *fb, pool_idx, P, Rv);
      if (st2) return st2;
      return (r == 32) ? qp_resvec<32, true>(ctx, fb->A, r, pool_idx, P, D, k, res2, Rv, pres2, pn2, true)
                       : qp_resvec<64, true>(ctx, fb->A, r, pool_idx, P, D, k, res2, Rv, pres2, pn2, true);
    }
#define QP_RV(RR, EX) return qp_resvec<RR, EX>(ctx, phi, r, pool_idx, P, D, k, res2, Rv, pres2, pn2)
    if (r == 16) QP_RV(16, true);
    if (r == 32) QP_RV(32, true);
    if (r == 64) QP_RV(64, true);
    if (r == 128) QP_RV(128, true);
    if (r < 16) QP_RV(16, false);
    if (r < 32) QP_RV(32, false);
    if (r < 64) QP_RV(64, false);
    QP_RV(128, false);
#undef QP_RV
  };
  // theta/tau of the rows holding the M largest bounds (<= cap rows taken),
  // compacted into out[0..cap) (unused slots -1): one cooperative launch
  int sbpm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&sbpm, qs_select_compact_kernel, 256, 0);
  if (sbpm < 1) return set_error(ctx, ADROM_ERR_CUDA, "qdeim: selection kernel cannot be resident");
  const int sgrid_max = ctx->num_sms * (sbpm < 4 ? sbpm : 4);
  ADROM_CK(ctx, cudaMemsetAsync(hist, 0, sizeof(unsigned int) * (QS_BINS + 32), ctx->stream));
  auto select_compact = [&](SelState* st, const double* vals, int64_t nn, const int64_t* list,
                            long long M, long long cap, int extend, int64_t* out) -> int {
    int64_t hg = (nn + 2047) / 2048;
    if (hg > sgrid_max) hg = sgrid_max;
    if (hg < 1) hg = 1;
    SelArgs sa{vals, nn, list, st, hist, M, cap, extend, out};
    void* args[] = {&sa};
    ADROM_CK(ctx, cudaLaunchCooperativeKernel((void*)qs_select_compact_kernel, (int)hg, 256, args, 0,
                                              ctx->stream));
    ++ctx->launches;
    return ADROM_OK;
  };
  const long long M = qp_pool_m();
  int chosen = 0, rounds = 0, refreshed = 0;
  while (chosen < count) {
    const int m = (count - chosen < r) ? (count - chosen) : r;
    const int n_ex = chosen;
    if (n_ex > 0) {
      qp_sort_rows_kernel<<<1, 1, 0, ctx->stream>>>(out_idx, n_ex, ex);
      ADROM_LAUNCH_CK(ctx);
    }
    ADROM_CK(ctx, cudaMemsetAsync(state, 0, sizeof(int) * 8, ctx->stream));
    // seed: every bound = ||phi_i||^2 (fresh for k = 0); the first chunk's
    // seed may come from the rotation epilogue
    if (!(seeded && chosen == 0)) {
      int st0 = rows_pass(n, 0, QP_SEED, nullptr, n_ex);
      if (st0) return st0;
    }
    int st = ADROM_OK;
    int k = 0;
    bool fresh = true;                       // bounds of the top rows are current
    int64_t rl_n = 0;                        // refresh-list slots (0: none this round)
    long long mref = qp_refresh_factor() * M;  // rows refreshed per round
    while (k < m) {
      ++rounds;
      const int pr = prof_begin(ctx, PROBE_QDEIM_ROUND);
      int64_t gg = (P + 255) / 256;
      if (gg > ctx->num_sms * 8) gg = ctx->num_sms * 8;
      if (!fresh && !all) {
        // refresh the mref rows with the largest (possibly stale) bounds
        const long long capm = mref + (mref * qp_refresh_slack()) / 100;
        const long long cap = (capm < n) ? capm : n;
        st = select_compact(selR, bnd2, n, nullptr, mref, cap, qp_extend_refresh(), rlist);
        if (st) return st;
        if (getenv("ADROM_QDEIM_TRACE") && atoi(getenv("ADROM_QDEIM_TRACE")) >= 2) {
          // refresh work: direction tiles of 8 computed per 8-row tile vs per row
          std::vector<int64_t> hl(cap);
          std::vector<unsigned char> hv(n);
          cudaMemcpyAsync(hl.data(), rlist, sizeof(int64_t) * cap, cudaMemcpyDeviceToHost, ctx->stream);
          cudaMemcpyAsync(hv.data(), ver, n, cudaMemcpyDeviceToHost, ctx->stream);
          cudaStreamSynchronize(ctx->stream);
          long long rows = 0, v0 = 0, tile_work = 0, row_work = 0;
          for (int64_t t = 0; t < cap; t += 8) {
            int vmin = k;
            for (int64_t p = t; p < t + 8 && p < cap; ++p) {
              if (hl[p] < 0) continue;
              const int v = hv[hl[p]];
              ++rows;
              v0 += v == 0;
              if (v < vmin) vmin = v;
              if (v < k) row_work += (k + 7) / 8 - v / 8;
            }
            if (vmin < k) tile_work += 8LL * ((k + 7) / 8 - vmin / 8);
          }
          fprintf(stderr, "qdeim refresh: k=%d rows=%lld ver0=%lld tile_work=%lld row_work=%lld\n", k,
                  rows, v0, tile_work, row_work);
        }
        // Late rounds (at most as many directions left as confirmed): bounds
        // from the complement basis, see qp_refresh_bf_kernel
        const bool cmode = qp_complement_on() && !qp_refresh_fp64() && (r == 32 || r == 64) &&
                           k >= 1 && (r - k) <= k;
        int* cfound = state + 5;
        if (cmode) {
          cudaFuncSetAttribute(qp_complement_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)QP_COMPLEMENT_SMEM);
          qp_complement_kernel<<<1, 256, QP_COMPLEMENT_SMEM, ctx->stream>>>(D, r, k, Ec, cfound);
          ADROM_LAUNCH_CK(ctx);
        }
        if (fact && cmode) {
          const int kver = k + (fb->vdrop ? 1 : 0);
          qp_wd_kernel<<<(r + FACT_KQ) * r / 256 + 1, 256, 0, ctx->stream>>>(fb->W, r + fb->k, r, Ec,
                                                                            r - k, nullptr, Mw);
          ADROM_LAUNCH_CK(ctx);
          st = (r == 32) ? qp_refresh_bf<32, true>(ctx, fb->A, fb->Q, fb->k, fb->n, nrmb, rlist, cap, Mw,
                                                   r - k, res2, bnd2, ver, blist, fb->A32, kver, cfound)
                         : qp_refresh_bf<64, true>(ctx, fb->A, fb->Q, fb->k, fb->n, nrmb, rlist, cap, Mw,
                                                   r - k, res2, bnd2, ver, blist, fb->A32, kver, cfound);
        } else if (cmode) {
          st = (r == 32) ? qp_refresh_bf<32, false>(ctx, phi, nullptr, 0, (int64_t)0, nullptr, rlist, cap,
                                                    Ec, r - k, res2, bnd2, ver, blist, nullptr, k, cfound)
                         : qp_refresh_bf<64, false>(ctx, phi, nullptr, 0, (int64_t)0, nullptr, rlist, cap,
                                                    Ec, r - k, res2, bnd2, ver, blist, nullptr, k, cfound);
        } else if (fact) {
          // (k < m <= r, so the extended list of k + 1 columns fits the r of Mw)
          const int kx = k + (fb->vdrop ? 1 : 0);
          qp_wd_kernel<<<(r + FACT_KQ) * r / 256 + 1, 256, 0, ctx->stream>>>(fb->W, r + fb->k, r, D,
                                                                            k, fb->vdrop, Mw);
          ADROM_LAUNCH_CK(ctx);
          st = (r == 32) ? qp_refresh_bf<32, true>(ctx, fb->A, fb->Q, fb->k, fb->n, nrmb, rlist, cap, Mw,
                                                   kx, res2, bnd2, ver, blist, fb->A32)
                         : qp_refresh_bf<64, true>(ctx, fb->A, fb->Q, fb->k, fb->n, nrmb, rlist, cap, Mw,
                                                   kx, res2, bnd2, ver, blist, fb->A32);
        } else if (r == 32 || r == 64 || r == 128) {
          st = (r == 32)
                   ? qp_refresh_bf<32, false>(ctx, phi, nullptr, 0, (int64_t)0, nullptr, rlist, cap, D, k, res2, bnd2, ver, blist)
               : (r == 64)
                   ? qp_refresh_bf<64, false>(ctx, phi, nullptr, 0, (int64_t)0, nullptr, rlist, cap, D, k, res2, bnd2, ver, blist)
                   : qp_refresh_bf<128, false>(ctx, phi, nullptr, 0, (int64_t)0, nullptr, rlist, cap, D, k, res2, bnd2, ver, blist);
        } else {
          st = rows_pass(cap, k, QP_REFRESH, rlist, n_ex);
          if (!st) st = qp_list_bounds(ctx, rlist, cap, bnd2, blist);
        }
        if (st) return st;
        ++refreshed;
        rl_n = cap;
      } else {
        rl_n = 0;  // pool straight from every row's bound; nothing else outside
        if (!all) {
          qs_init_kernel<<<1, 256, 0, ctx->stream>>>(selR, 0, hist);
          ADROM_LAUNCH_CK(ctx);
        }
      }
      if (all) {
        qp_all_rows_kernel<<<(int)gg, 256, 0, ctx->stream>>>(pool_idx, n);
        ADROM_LAUNCH_CK(ctx);
      } else {
        // pool = the M largest bounds among the refreshed rows (rows outside the
        // refresh list are bounded by selR->tau), or among all rows
        const int64_t* cl = rl_n ? rlist : nullptr;
        const double* cv = rl_n ? blist : bnd2;
        const int64_t cn = rl_n ? rl_n : n;
        st = select_compact(sel, cv, cn, cl, M, (long long)P, 1, pool_idx);
        if (st) return st;
      }
      st = resvec(k);
      if (st) return st;
      GreedyArgs ga{pool_idx, P, Rv, pres2, &sel->tau, &selR->tau, D, piv, m, r, state, bv, bi, brow,
                    err_res, all ? 1 : 0};
      void* args[] = {&ga};
      ADROM_CK(ctx, cudaLaunchCooperativeKernel(gkern, ggrid, 256, args, gsm, ctx->stream));
      ++ctx->launches;
      prof_end(ctx, pr);
      ADROM_CK(ctx, cudaMemcpyAsync(hstate, state, sizeof(int) * 4, cudaMemcpyDeviceToHost,
                                    ctx->stream));
      ADROM_CK(ctx, cudaMemcpyAsync(hres, err_res, sizeof(double), cudaMemcpyDeviceToHost,
                                    ctx->stream));
      ride_flush(ctx);  // the caller's pending status words share this round trip
      ADROM_CK(ctx, cudaStreamSynchronize(ctx->stream));
      if (hstate[2])
        return set_error(ctx, ADROM_ERR_SINGULAR,
                         "rank deficiency at pivot step %d (residual column norm %.3e)",
                         chosen + hstate[2] - 1, hres[0]);
      const int knew = hstate[0];
      if (getenv("ADROM_QDEIM_TRACE") && atoi(getenv("ADROM_QDEIM_TRACE")) >= 1)
        fprintf(stderr, "qdeim round %d: k %d -> %d (refresh %lld rows)\n", rounds, k, knew,
                (long long)rl_n);
      if (getenv("ADROM_QDEIM_TRACE") && atoi(getenv("ADROM_QDEIM_TRACE")) >= 2 && !all) {
        unsigned long long* dc = nullptr;
        unsigned long long hc[4];
        double taus[2];
        cudaMalloc(&dc, sizeof(hc));
        cudaMemsetAsync(dc, 0, sizeof(hc), ctx->stream);
        const double g2 = hres[0] * hres[0];
        qp_count_above_kernel<<<ctx->num_sms * 4, 256, 0, ctx->stream>>>(bnd2, n, g2, dc);
        cudaMemcpyAsync(hc, dc, sizeof(hc), cudaMemcpyDeviceToHost, ctx->stream);
        cudaMemcpyAsync(&taus[0], &sel->tau, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream);
        cudaMemcpyAsync(&taus[1], &selR->tau, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream);
        cudaStreamSynchronize(ctx->stream);
        cudaFree(dc);
        fprintf(stderr,
                "  stop residual^2 g=%.3e tau_pool=%.3e tau_outside=%.3e rows with bound > g, g/4, "
                "g/16, g/64: %llu %llu %llu %llu\n",
                g2, taus[0], taus[1], hc[0], hc[1], hc[2], hc[3]);
      }
      if (knew == k) {
        if (!all && mref < n) {  // stale bounds block progress: refresh more rows
          mref = (mref * 4 < n) ? mref * 4 : n;
          fresh = false;
          continue;
        }
        // factored rows: the bounds keep the seed's slack, so a stall does not
        // prove rank deficiency -> the caller reruns on the materialised basis
        if (fact) return QDEIM_NEEDS_EXPLICIT;
        // nothing certifiable with every bound fresh: only possible when the
        // remaining residuals tie at (numerically) zero -> rank deficient
        if (!(hres[0] >= 1e-14))
          return set_error(ctx, ADROM_ERR_SINGULAR,
                           "rank deficiency at pivot step %d (residual column norm %.3e)",
                           chosen + k, hres[0]);
        return set_error(ctx, ADROM_ERR_DENSE, "qdeim: no certified pivot at step %d", chosen + k);
      }
      k = knew;
      fresh = false;
      if (k < m && !all) {
        // exclude the new pivots; the pool rows' exact residuals tighten their bounds
        qp_mark_kernel<<<1, 128, 0, ctx->stream>>>(piv, 0, k, res2, bnd2);
        ADROM_LAUNCH_CK(ctx);
        qp_writeback_kernel<<<(int)gg, 256, 0, ctx->stream>>>(pool_idx, P, pres2, pn2, k, res2,
                                                             bnd2);
        ADROM_LAUNCH_CK(ctx);
      }
    }
    ADROM_CK(ctx, cudaMemcpyAsync(out_idx + chosen, piv, sizeof(int64_t) * m,
                                  cudaMemcpyDeviceToDevice, ctx->stream));
    chosen += m;
  }
  if (getenv("ADROM_QDEIM_TRACE"))
    fprintf(stderr, "qdeim: n=%lld r=%d count=%d rounds=%d refreshes=%d\n", (long long)n, r, count,
            rounds, refreshed);
  if (passes_out) *passes_out = rounds;
  return ADROM_OK;
}

}  // namespace adrom
