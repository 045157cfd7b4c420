// Factored basis for the session's iSVD (r in {32, 64}).
//
// The explicit update rotates the whole basis every event, Phi' = [Phi | q^] B
// (tracking.py:176-177): 2 N r (r+1) flop, FP64-tensor bound at N = 2^24.
// Here the basis is kept as
//
//     Phi = X W,   X = [A | Q_0 .. Q_{k-1}]   (A: N x r anchor, Q: raw residuals)
//
// with W ((r+k) x r) on the device.  An event appends its residual q as
// column k of Q and maps W' = [[W, 0], [0, 1/||q||]] B — O(r^3) instead of
// O(N r^2).  Every pass over the basis reads X (r + k columns) and applies W
// to r-vectors; after KQ appended columns the anchor is rebuilt, A = X W, on
// the FP64 tensor cores (reanchor_kernel).  Mathematically the basis is the
// reference's Phi' = [Phi, q^] U[:, :r] at every event; only the rounding
// differs (tests/test_gpu_rom.py compares both representations).
//
//   pass 1 (xpass MODE 1): X^T y, ||y||^2 and the fused decode
//                          q~ = q_ref + (X (W a)) / d        (projection.py:104)
//   pass 2 (xpass MODE 2): q = y - X (W p) stored as Q[:, k];  X^T q, ||q||^2;
//                          X^T w, q.w with w = d (q~ - q_ref) (state transfer,
//                          projection.py:98-99, for the new basis)
#include "common.cuh"
#include "factored_internal.cuh"
#include "linalg_internal.cuh"
#include "tma.cuh"

#include <stdlib.h>

#include <vector>

namespace adrom {

struct XPassArgs {
  const double* A;
  const double* Q;
  int64_t n;
  int k, kq;
  const double* v;      // r + k: decode vector W a (MODE 1) or W p (MODE 2)
  const double* y;      // snapshot y_hat
  const double* q_ref;
  const double* d;
  double* qt;           // MODE 1: decoded q~ (out); MODE 2: q~ (in)
  double* Qw;           // MODE 2: Q (column k written)
  double* qv;           // MODE 2: the residual q also as a contiguous vector
  double* partial;      // per block: see xpass_partial_width
  int* flag;
  const double* vdrop;  // MODE 1 (optional): the previous event's dropped direction in X
  double* nrm2;         //   coordinates; nrm2[i] -= (X_i . vdrop)^2 (bound -> exact norm)
  const double* va;     // MODE 2 (optional): decode vector W a -> q~ written here (qt)
};

__host__ __device__ inline int xpass_width(int r, int kq, int mode) {
  (void)mode;
  return r + kq + 1;
}

constexpr int XP_ROWS = 4096;  // rows per xpass block

template <int R, int MODE>
__global__ void __launch_bounds__(256, 2) xpass_kernel(XPassArgs a) {
  constexpr int LPR = R / 8;        // lanes per row: 8 A columns each
  constexpr int RPW = 32 / LPR;     // rows per warp per sub-iteration
  constexpr int QPL = FACT_KQ / LPR;  // Q columns per lane
  constexpr int U = 2;
  constexpr int NW = 1;  // weight vectors (y in MODE 1, q in MODE 2)
  const int kq = a.kq, k = a.k;
  __shared__ double red[8 * (R + FACT_KQ) * NW];
  __shared__ double sred[3][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int seg = lane / LPR, sl = lane - seg * LPR;
  // the row-dot vectors live in shared memory (registers hold the rows)
  __shared__ __align__(16) double sv[R + FACT_KQ];
  __shared__ __align__(16) double sg[R + FACT_KQ];
  // second row-dot vector: MODE 1 the dropped direction, MODE 2 the decode vector
  const double* v2p = (MODE == 1) ? a.vdrop : a.va;
  const bool drop = v2p != nullptr;
  for (int j = threadIdx.x; j < R + FACT_KQ; j += blockDim.x) {
    const bool ok = j < R + k;
    sv[j] = (ok && a.v) ? a.v[j] : 0.0;
    sg[j] = (drop && ok) ? v2p[j] : 0.0;
  }
  __syncthreads();
  const double2* vA = reinterpret_cast<const double2*>(sv);
  const double2* gA = reinterpret_cast<const double2*>(sg);
  const double* vQ = sv + R;
  const double* gQ = sg + R;
  double2 accA[NW][4];
  double accQ[NW][QPL];
#pragma unroll
  for (int w = 0; w < NW; ++w) {
#pragma unroll
    for (int h = 0; h < 4; ++h) accA[w][h] = make_double2(0.0, 0.0);
#pragma unroll
    for (int t = 0; t < QPL; ++t) accQ[w][t] = 0.0;
  }
  double s0 = 0.0, s1 = 0.0;
  bool bad = false;
  // block b owns rows [b * XP_ROWS, (b+1) * XP_ROWS): many small blocks
  // balance themselves across SMs (pass 1 shares the GPU with the one-block
  // reduced step on the other stream)
  const int64_t rows_per_iter = (int64_t)RPW * U;
  const int64_t blk0 = (int64_t)blockIdx.x * XP_ROWS;
  const int64_t blk1 = (blk0 + XP_ROWS < a.n) ? blk0 + XP_ROWS : a.n;
  for (int64_t base = blk0 + (int64_t)warp * rows_per_iter; base < blk1; base += 8 * rows_per_iter) {
    double2 xa[U][4];
    double xq[U][QPL];
    double yv[U], qr[U], dd[U], qt[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = base + u * RPW + seg;
      const bool live = i < blk1;
      if (live) {
        const double2* rowp = reinterpret_cast<const double2*>(a.A + i * R);
#pragma unroll
        for (int h = 0; h < 4; ++h) xa[u][h] = rowp[sl + LPR * h];
#pragma unroll
        for (int t = 0; t < QPL; ++t) {
          const int j = sl + LPR * t;
          xq[u][t] = (j < k) ? a.Q[qpanel(i, j, a.n)] : 0.0;
        }
      } else {
#pragma unroll
        for (int h = 0; h < 4; ++h) xa[u][h] = make_double2(0.0, 0.0);
#pragma unroll
        for (int t = 0; t < QPL; ++t) xq[u][t] = 0.0;
      }
      yv[u] = (live && a.y) ? a.y[i] : 0.0;
      qr[u] = (live && a.q_ref) ? a.q_ref[i] : 0.0;
      dd[u] = (live && a.d) ? a.d[i] : 1.0;
      qt[u] = 0.0;
    }
    double rd[U], dd2[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      double t0 = 0.0, t2 = 0.0;
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        bad |= !(isfinite(xa[u][h].x) && isfinite(xa[u][h].y));
        const double2 vv = vA[sl + LPR * h];
        t0 += xa[u][h].x * vv.x + xa[u][h].y * vv.y;
        if (drop) {
          const double2 gg = gA[sl + LPR * h];
          t2 += xa[u][h].x * gg.x + xa[u][h].y * gg.y;
        }
      }
#pragma unroll
      for (int t = 0; t < QPL; ++t) {
        t0 += xq[u][t] * vQ[sl + LPR * t];
        if (drop) t2 += xq[u][t] * gQ[sl + LPR * t];
      }
      rd[u] = t0;
      dd2[u] = t2;
    }
#pragma unroll
    for (int o = LPR / 2; o > 0; o >>= 1)
#pragma unroll
      for (int u = 0; u < U; ++u) {
        rd[u] += __shfl_xor_sync(0xffffffffu, rd[u], o);
        if (drop) dd2[u] += __shfl_xor_sync(0xffffffffu, dd2[u], o);
      }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = base + u * RPW + seg;
      if (i >= blk1) continue;
      double w0, w1 = 0.0;
      if (MODE == 1) {
        if (a.qt && sl == 0) a.qt[i] = qr[u] + rd[u] / dd[u];  // decode (projection.py:104)
        if (drop && sl == 0) a.nrm2[i] = fmax(a.nrm2[i] - dd2[u] * dd2[u], 0.0);
        w0 = yv[u];
        bad |= !isfinite(w0);
        if (sl == 0) s0 += w0 * w0;
      } else {
        w0 = yv[u] - rd[u];                    // q = y - Phi p (tracking.py:162)
        if (drop && sl == 0) a.qt[i] = qr[u] + dd2[u] / dd[u];  // fused decode (projection.py:104)
        bad |= !isfinite(w0);
        if (sl == 0) {
          if (a.qv) a.qv[i] = w0;
          s0 += w0 * w0;
        }
        // column k joins its 4-column panel: the 4 lanes owning that panel
        // write the whole 32-byte sector (live columns rewritten unchanged,
        // later ones zeroed), so no partial-sector write reaches L2
#pragma unroll
        for (int t = 0; t < QPL; ++t) {
          const int j = sl + LPR * t;
          if ((j >> 2) == (k >> 2)) a.Qw[qpanel(i, j, a.n)] = (j < k) ? xq[u][t] : (j == k ? w0 : 0.0);
        }
      }
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        accA[0][h].x += xa[u][h].x * w0;
        accA[0][h].y += xa[u][h].y * w0;
        if (NW == 2) {
          accA[NW - 1][h].x += xa[u][h].x * w1;
          accA[NW - 1][h].y += xa[u][h].y * w1;
        }
      }
#pragma unroll
      for (int t = 0; t < QPL; ++t) {
        accQ[0][t] += xq[u][t] * w0;
        if (NW == 2) accQ[NW - 1][t] += xq[u][t] * w1;
      }
    }
  }
  // fold the row segments sharing columns, then the warps (fixed order)
#pragma unroll
  for (int o = LPR; o < 32; o <<= 1)
#pragma unroll
    for (int w = 0; w < NW; ++w) {
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        accA[w][h].x += __shfl_xor_sync(0xffffffffu, accA[w][h].x, o);
        accA[w][h].y += __shfl_xor_sync(0xffffffffu, accA[w][h].y, o);
      }
#pragma unroll
      for (int t = 0; t < QPL; ++t) accQ[w][t] += __shfl_xor_sync(0xffffffffu, accQ[w][t], o);
    }
  constexpr int WD = R + FACT_KQ;
  if (seg == 0) {
#pragma unroll
    for (int w = 0; w < NW; ++w) {
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        red[(w * 8 + warp) * WD + 2 * (sl + LPR * h)] = accA[w][h].x;
        red[(w * 8 + warp) * WD + 2 * (sl + LPR * h) + 1] = accA[w][h].y;
      }
#pragma unroll
      for (int t = 0; t < QPL; ++t) red[(w * 8 + warp) * WD + R + sl + LPR * t] = accQ[w][t];
    }
  }
  __syncthreads();
  const int width = xpass_width(R, kq, MODE);
  double* out = a.partial + (size_t)blockIdx.x * width;
  for (int c = threadIdx.x; c < R + kq; c += 256) {
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      double s = 0.0;
#pragma unroll
      for (int q = 0; q < 8; ++q) s += red[(w * 8 + q) * WD + c];
      out[w * (R + kq + 1) + c] = s;
    }
  }
  const double t0 = block_sum<256>(s0, sred[0]);
  (void)s1;
  if (threadIdx.x == 0) out[R + kq] = t0;
  if (bad && a.flag) atomicOr(a.flag, 1);
}

// ---------------------------------------------------------------------------
// The same two passes with the row tiles staged by the copy engine
// (cp.async.bulk into a STAGES-deep shared-memory ring, one mbarrier per
// stage; tma.cuh).  One elected thread issues a tile's copies — the A rows
// (TR x R doubles, contiguous), the ceil(k/4) live 32-byte Q panels and only
// the per-row vectors the pass reads — so the bytes requested are exactly
// the algorithmic ones and several tiles stay in flight per block whatever
// the consumers' register pressure.  Each warp consumes one RPW-row group of
// every tile with the register-streamed kernel's arithmetic (same fixed
// reduction order).  A block owns the same XP_ROWS rows as xpass_kernel, so
// the partial-sum layout and the host side are shared.
// ---------------------------------------------------------------------------
template <int R>
struct XpT {
  static constexpr int LPR = R / 8, RPW = 32 / LPR;
  static constexpr int TR = 8 * RPW;                 // rows per tile: one group per warp
  static constexpr int STAGES = 4;
  static constexpr int A_BYTES = TR * R * 8;
  static constexpr int Q_BYTES = (FACT_KQ / 4) * TR * 32;
  static constexpr int V_BYTES = TR * 8;
  static constexpr int STAGE = A_BYTES + Q_BYTES + 4 * V_BYTES;  // A | Q | y | q_ref | d | nrm2
  static constexpr size_t SMEM = 128 + (size_t)STAGES * STAGE;
  static_assert(XP_ROWS % TR == 0, "block rows are whole tiles");
};

template <int R, int MODE>
__global__ void __launch_bounds__(256, 2) xpass_tma_kernel(XPassArgs a) {
  using T = XpT<R>;
  constexpr int LPR = T::LPR, RPW = T::RPW, TR = T::TR, STAGES = T::STAGES;
  constexpr int QPL = FACT_KQ / LPR;
  const int kq = a.kq, k = a.k;
  extern __shared__ __align__(128) unsigned char xsm[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(xsm);
  unsigned char* stage0 = xsm + 128;
  __shared__ double red[8 * (R + FACT_KQ)];
  __shared__ double sred[32];
  __shared__ __align__(16) double sv[R + FACT_KQ];
  __shared__ __align__(16) double sg[R + FACT_KQ];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int seg = lane / LPR, sl = lane - seg * LPR;
  const double* v2p = (MODE == 1) ? a.vdrop : a.va;
  const bool drop = v2p != nullptr;
  // which per-row vectors this pass reads
  const bool ld_y = a.y != nullptr;
  const bool ld_qd = (MODE == 1) ? (a.qt != nullptr) : drop;  // q_ref, d (decode)
  const bool ld_n2 = (MODE == 1) && drop;                     // row norms (RMW)
  const int npan = (k + 3) >> 2;
  for (int j = tid; j < R + FACT_KQ; j += blockDim.x) {
    const bool ok = j < R + k;
    sv[j] = (ok && a.v) ? a.v[j] : 0.0;
    sg[j] = (drop && ok) ? v2p[j] : 0.0;
  }
  const int64_t blk0 = (int64_t)blockIdx.x * XP_ROWS;
  const int64_t blk1 = (blk0 + XP_ROWS < a.n) ? blk0 + XP_ROWS : a.n;
  const int ntiles = (int)((blk1 - blk0 + TR - 1) / TR);
  const int nfull = (int)((blk1 - blk0) / TR);
  if (tid == 0) {
    for (int st = 0; st < STAGES; ++st) mbar_init(&bars[st], 1);
    mbar_fence_init();
  }
  __syncthreads();
  auto stage_ptr = [&](int st) { return stage0 + (size_t)st * T::STAGE; };
  auto issue = [&](int t) {  // thread 0; full tiles only
    const int st = t % STAGES;
    unsigned char* b = stage_ptr(st);
    const int64_t row = blk0 + (int64_t)t * TR;
    const uint32_t bytes = T::A_BYTES + npan * TR * 32 + (ld_y ? T::V_BYTES : 0) +
                           (ld_qd ? 2 * T::V_BYTES : 0) + (ld_n2 ? T::V_BYTES : 0);
    mbar_arrive_expect_tx(&bars[st], bytes);
    bulk_g2s(b, a.A + row * R, T::A_BYTES, &bars[st]);
    for (int P = 0; P < npan; ++P)
      bulk_g2s(b + T::A_BYTES + P * TR * 32, a.Q + ((int64_t)P * a.n + row) * 4, TR * 32, &bars[st]);
    unsigned char* vb = b + T::A_BYTES + T::Q_BYTES;
    if (ld_y) bulk_g2s(vb, a.y + row, T::V_BYTES, &bars[st]);
    if (ld_qd) {
      bulk_g2s(vb + T::V_BYTES, a.q_ref + row, T::V_BYTES, &bars[st]);
      bulk_g2s(vb + 2 * T::V_BYTES, a.d + row, T::V_BYTES, &bars[st]);
    }
    if (ld_n2) bulk_g2s(vb + 3 * T::V_BYTES, a.nrm2 + row, T::V_BYTES, &bars[st]);
  };
  if (tid == 0)
    for (int t = 0; t < STAGES && t < nfull; ++t) issue(t);
  __syncthreads();  // sv / sg
  const double2* vA = reinterpret_cast<const double2*>(sv);
  const double2* gA = reinterpret_cast<const double2*>(sg);
  const double* vQ = sv + R;
  const double* gQ = sg + R;
  // this lane's slices of the row-dot vectors, held in registers
  double2 rv[4], rg[4];
  double rvq[QPL], rgq[QPL];
#pragma unroll
  for (int h = 0; h < 4; ++h) {
    rv[h] = vA[sl + LPR * h];
    rg[h] = gA[sl + LPR * h];
  }
#pragma unroll
  for (int q = 0; q < QPL; ++q) {
    rvq[q] = vQ[sl + LPR * q];
    rgq[q] = gQ[sl + LPR * q];
  }
  double2 accA[4];
  double accQ[QPL];
#pragma unroll
  for (int h = 0; h < 4; ++h) accA[h] = make_double2(0.0, 0.0);
#pragma unroll
  for (int t = 0; t < QPL; ++t) accQ[t] = 0.0;
  double s0 = 0.0;
  bool bad = false;
  for (int t = 0; t < ntiles; ++t) {
    const int st = t % STAGES;
    unsigned char* b = stage_ptr(st);
    const double* As = reinterpret_cast<const double*>(b);
    const double* Qs = reinterpret_cast<const double*>(b + T::A_BYTES);
    const double* Vs = reinterpret_cast<const double*>(b + T::A_BYTES + T::Q_BYTES);
    const int64_t row0 = blk0 + (int64_t)t * TR;
    const int cnt = (int)((blk1 - row0 < TR) ? (blk1 - row0) : TR);
    if (t < nfull) {
      mbar_wait(&bars[st], (uint32_t)((t / STAGES) & 1));
    } else {  // the block's ragged last tile: plain loads, zero fill
      double* Aw = reinterpret_cast<double*>(b);
      for (int e = tid; e < TR * R; e += blockDim.x)
        Aw[e] = (e / R < cnt) ? a.A[row0 * R + e] : 0.0;
      double* Qw = reinterpret_cast<double*>(b + T::A_BYTES);
      for (int e = tid; e < (FACT_KQ / 4) * TR * 4; e += blockDim.x) {
        const int P = e / (TR * 4), rr = (e / 4) % TR, c = e & 3;
        Qw[e] = (rr < cnt && P < npan) ? a.Q[((int64_t)P * a.n + row0 + rr) * 4 + c] : 0.0;
      }
      double* Vw = reinterpret_cast<double*>(b + T::A_BYTES + T::Q_BYTES);
      for (int rr = tid; rr < TR; rr += blockDim.x) {
        const bool ok = rr < cnt;
        Vw[rr] = (ok && ld_y) ? a.y[row0 + rr] : 0.0;
        Vw[TR + rr] = (ok && ld_qd) ? a.q_ref[row0 + rr] : 0.0;
        Vw[2 * TR + rr] = (ok && ld_qd) ? a.d[row0 + rr] : 1.0;
        Vw[3 * TR + rr] = (ok && ld_n2) ? a.nrm2[row0 + rr] : 0.0;
      }
      __syncthreads();
    }
    const int rl = warp * RPW + seg;  // this lane group's row in the tile
    const bool live = rl < cnt;
    const int64_t i = row0 + rl;
    double2 xa[4];
    double xq[QPL];
    const double2* rowp = reinterpret_cast<const double2*>(As + rl * R);
#pragma unroll
    for (int h = 0; h < 4; ++h) xa[h] = rowp[sl + LPR * h];
#pragma unroll
    for (int q = 0; q < QPL; ++q) {
      const int j = sl + LPR * q;
      xq[q] = (j < k) ? Qs[(j >> 2) * TR * 4 + rl * 4 + (j & 3)] : 0.0;
    }
    const double yv = ld_y ? Vs[rl] : 0.0;
    const double qr = ld_qd ? Vs[TR + rl] : 0.0;
    const double dd = ld_qd ? Vs[2 * TR + rl] : 1.0;
    double t0 = 0.0, t2 = 0.0;
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      bad |= !(isfinite(xa[h].x) && isfinite(xa[h].y));
      t0 += xa[h].x * rv[h].x + xa[h].y * rv[h].y;
      if (drop) t2 += xa[h].x * rg[h].x + xa[h].y * rg[h].y;
    }
#pragma unroll
    for (int q = 0; q < QPL; ++q) {
      t0 += xq[q] * rvq[q];
      if (drop) t2 += xq[q] * rgq[q];
    }
#pragma unroll
    for (int o = LPR / 2; o > 0; o >>= 1) {
      t0 += __shfl_xor_sync(0xffffffffu, t0, o);
      if (drop) t2 += __shfl_xor_sync(0xffffffffu, t2, o);
    }
    if (live) {
      double w0;
      if (MODE == 1) {
        if (a.qt && sl == 0) a.qt[i] = qr + t0 / dd;  // decode (projection.py:104)
        if (drop && sl == 0) a.nrm2[i] = fmax(Vs[3 * TR + rl] - t2 * t2, 0.0);
        w0 = yv;
        bad |= !isfinite(w0);
        if (sl == 0) s0 += w0 * w0;
      } else {
        w0 = yv - t0;                                  // q = y - Phi p (tracking.py:162)
        if (drop && sl == 0) a.qt[i] = qr + t2 / dd;   // fused decode (projection.py:104)
        bad |= !isfinite(w0);
        if (sl == 0) {
          if (a.qv) a.qv[i] = w0;
          s0 += w0 * w0;
        }
        // column k joins its 4-column panel as one full 32-byte sector
#pragma unroll
        for (int q = 0; q < QPL; ++q) {
          const int j = sl + LPR * q;
          if ((j >> 2) == (k >> 2)) a.Qw[qpanel(i, j, a.n)] = (j < k) ? xq[q] : (j == k ? w0 : 0.0);
        }
      }
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        accA[h].x += xa[h].x * w0;
        accA[h].y += xa[h].y * w0;
      }
#pragma unroll
      for (int q = 0; q < QPL; ++q) accQ[q] += xq[q] * w0;
    }
    __syncthreads();  // stage st fully consumed
    if (tid == 0 && t + STAGES < nfull) issue(t + STAGES);
  }
  // fold the row segments sharing columns, then the warps (fixed order)
#pragma unroll
  for (int o = LPR; o < 32; o <<= 1) {
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      accA[h].x += __shfl_xor_sync(0xffffffffu, accA[h].x, o);
      accA[h].y += __shfl_xor_sync(0xffffffffu, accA[h].y, o);
    }
#pragma unroll
    for (int q = 0; q < QPL; ++q) accQ[q] += __shfl_xor_sync(0xffffffffu, accQ[q], o);
  }
  constexpr int WD = R + FACT_KQ;
  if (seg == 0) {
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      red[warp * WD + 2 * (sl + LPR * h)] = accA[h].x;
      red[warp * WD + 2 * (sl + LPR * h) + 1] = accA[h].y;
    }
#pragma unroll
    for (int q = 0; q < QPL; ++q) red[warp * WD + R + sl + LPR * q] = accQ[q];
  }
  __syncthreads();
  const int width = xpass_width(R, kq, MODE);
  double* out = a.partial + (size_t)blockIdx.x * width;
  for (int c = tid; c < R + kq; c += 256) {
    double sacc = 0.0;
#pragma unroll
    for (int w = 0; w < 8; ++w) sacc += red[w * WD + c];
    out[c] = sacc;
  }
  const double tsum = block_sum<256>(s0, sred);
  if (tid == 0) out[R + kq] = tsum;
  if (bad && a.flag) atomicOr(a.flag, 1);
}

// ADROM_XPASS_TMA=0 selects the register-streamed passes (A/B comparisons)
static bool xpass_use_tma() {
  static const bool v = [] {
    const char* e = getenv("ADROM_XPASS_TMA");
    return !(e && atoi(e) == 0);
  }();
  return v;
}

template <int R, int MODE>
static void xpass_launch(adrom_ctx* ctx, int grid, const XPassArgs& a) {
  if (xpass_use_tma()) {
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(xpass_tma_kernel<R, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)XpT<R>::SMEM);
      attr = true;
    }
    xpass_tma_kernel<R, MODE><<<grid, 256, XpT<R>::SMEM, ctx->stream>>>(a);
  } else {
    xpass_kernel<R, MODE><<<grid, 256, 0, ctx->stream>>>(a);
  }
}

// ---------------------------------------------------------------------------
// small dense helpers (one block)
// ---------------------------------------------------------------------------
// out[c] = sum_j M[j][c] x[j]  (M rows x cols, row-major), i.e. M^T x
__global__ void matT_vec_kernel(const double* __restrict__ M, int rows, int cols,
                                const double* __restrict__ x, double* __restrict__ out) {
  for (int c = threadIdx.x; c < cols; c += blockDim.x) {
    double s = 0.0;
    for (int j = 0; j < rows; ++j) s += M[(size_t)j * cols + c] * x[j];
    out[c] = s;
  }
}

// out[j] = sum_c M[j][c] x[c]  (M x)
__global__ void mat_vec_kernel(const double* __restrict__ M, int rows, int cols,
                               const double* __restrict__ x, double* __restrict__ out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int j = warp; j < rows; j += nw) {
    double s = 0.0;
    for (int c = lane; c < cols; c += 32) s += M[(size_t)j * cols + c] * x[c];
    s = warp_sum(s);
    if (lane == 0) out[j] = s;
  }
}

// W' ((r+k+1) x r) = [[W, 0], [0, qinv]] B  with B ((r+1) x r) from the core
__global__ void wnext_kernel(const double* __restrict__ W, int rk, int r,
                             const double* __restrict__ B, const double* __restrict__ qinv,
                             double* __restrict__ Wn) {
  const double qi = *qinv;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < (rk + 1) * r; e += gridDim.x * blockDim.x) {
    const int i = e / r, c = e - i * r;
    double s = 0.0;
    if (i < rk) {
      if (W) {
        for (int j = 0; j < r; ++j) s += W[(size_t)i * r + j] * B[(size_t)j * r + c];
      } else {
        s = B[(size_t)i * r + c];  // W = I (k = 0, i < r)
      }
    } else {
      s = qi * B[(size_t)r * r + c];
    }
    Wn[e] = s;
  }
}

// state transfer a' = Phi'^T D (q~ - q_ref) = Phi'^T Phi a with
// Phi' = [Phi, q^] B:  a' = B^T [G a ; qinv (Phi^T q) . a]  (no basis pass;
// the reference's rounding of q~ (driver.py:376) is not reproduced — this is
// the exact-arithmetic value, rounding-level close)
__global__ void encode_factored_kernel(const double* __restrict__ G, int r,
                                       const double* __restrict__ a,
                                       const double* __restrict__ phitq,
                                       const double* __restrict__ qinv,
                                       const double* __restrict__ B, double* __restrict__ a_out) {
  __shared__ double z[129];
  __shared__ double red[32];
  for (int c = threadIdx.x; c < r; c += blockDim.x) {
    double s = 0.0;
    for (int j = 0; j < r; ++j) s += G[(size_t)c * r + j] * a[j];
    z[c] = s;
  }
  double t = 0.0;
  for (int j = threadIdx.x; j < r; j += blockDim.x) t += phitq[j] * a[j];
  t = block_sum_dyn(t, red);
  if (threadIdx.x == 0) z[r] = (*qinv) * t;
  __syncthreads();
  for (int c = threadIdx.x; c < r; c += blockDim.x) {
    double s = 0.0;
    for (int j = 0; j <= r; ++j) s += B[(size_t)j * r + c] * z[j];
    a_out[c] = s;
  }
}

// v_drop ((rk + 1)) = [W u_top ; qinv u_bot]  (u = dropped left singular vector of K)
__global__ void vdrop_kernel(const double* __restrict__ W, int rk, int r,
                             const double* __restrict__ u, const double* __restrict__ qinv,
                             double* __restrict__ out) {
  for (int i = threadIdx.x; i <= rk; i += blockDim.x) {
    double s = 0.0;
    if (i < rk) {
      if (W) {
        for (int j = 0; j < r; ++j) s += W[(size_t)i * r + j] * u[j];
      } else {
        s = u[i];
      }
    } else {
      s = (*qinv) * u[r];
    }
    out[i] = s;
  }
}

// QDEIM k = 0 bounds of the new basis: ||Phi'_i||^2 <= ||Phi_i||^2 + (q_i / ||q||)^2
// (B has orthonormal columns); nrm2_next keeps the bound for the next event
// sb = [qinv, ||p2||]: with the refined direction q_hat_i = (q_i - Phi_i p2)
// qinv, |q_hat_i| <= (|q_i| + ||Phi_i|| ||p2||) qinv
__global__ void seed_bounds_kernel(const double* __restrict__ nrm2, const double* __restrict__ qv,
                                   const double* __restrict__ sb, int64_t n,
                                   double* __restrict__ res2, double* __restrict__ bnd2,
                                   unsigned char* __restrict__ ver, double* __restrict__ nrm2_next) {
  const double qi = sb[0], p2n = sb[1];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double qh = (fabs(qv[i]) + (p2n > 0.0 ? sqrt(nrm2[i]) * p2n : 0.0)) * qi;
    const double b = (nrm2[i] + qh * qh) * (1.0 + 64.0 * 2.220446049250313e-16);
    nrm2_next[i] = b;
    res2[i] = b;
    bnd2[i] = b;
    ver[i] = 0;
  }
}

// ---------------------------------------------------------------------------
// re-anchor: A_out = X W on the FP64 tensor cores (DMMA m8n8k4), exact row
// norms into nrm2.  X = [A (R cols) | Q (k of FACT_KQ cols)], W ((R+k) x R).
// 64-row tiles staged by cp.async (stride R + FACT_KQ + 4), 8 warps as
// 4 (rows) x 2 (cols); B fragments (W) from smem.
// ---------------------------------------------------------------------------
template <int R>
struct ReTC {
  static constexpr int TM = 64;
  static constexpr int KX = R + FACT_KQ;      // padded inner dimension
  static constexpr int S = KX + 4;            // row stride (doubles)
  static constexpr int SW = R + 4;            // W row stride
  static constexpr int WN = R / 2, NT = WN / 8, MT = 2, WR = 16;
  static constexpr size_t smem_doubles = 2 * (size_t)TM * S + (size_t)KX * SW + 2 * TM;
};

__device__ __forceinline__ void re_cp16(void* smem, const void* gmem, int src_bytes) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem),
               "r"(src_bytes));
}
__device__ __forceinline__ void re_dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

template <int R>
__global__ void __launch_bounds__(256, 1) reanchor_kernel(const double* __restrict__ A,
                                                          const double* __restrict__ Q, int k,
                                                          const double* __restrict__ W, int64_t n,
                                                          double* __restrict__ out,
                                                          double* __restrict__ nrm2,
                                                          float* __restrict__ out32) {
  using C = ReTC<R>;
  extern __shared__ __align__(16) double sm[];
  double* X0 = sm;                          // 2 stages x TM x S
  double* Ws = sm + 2 * C::TM * C::S;       // KX x SW (rows >= R + k zero)
  double* rn = Ws + C::KX * C::SW;          // 2 x TM
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp >> 1, wn = warp & 1;
  for (int e = tid; e < C::KX * R; e += 256) {
    const int j = e / R, c = e - j * R;
    Ws[j * C::SW + c] = (j < R + k) ? W[(size_t)j * R + c] : 0.0;
  }
  const int64_t ntiles = (n + C::TM - 1) / C::TM;
  auto load_tile = [&](int64_t t, double* Xs) {
    const int64_t row0 = t * C::TM;
    for (int c = tid; c < C::TM * (R / 2); c += 256) {
      const int rr = c / (R / 2), cc = 2 * (c % (R / 2));
      const bool ok = row0 + rr < n;
      re_cp16(Xs + rr * C::S + cc, A + (ok ? (row0 + rr) * R + cc : 0), ok ? 16 : 0);
    }
    for (int c = tid; c < C::TM * (FACT_KQ / 2); c += 256) {
      const int rr = c / (FACT_KQ / 2), cc = 2 * (c % (FACT_KQ / 2));
      const bool ok = row0 + rr < n && cc < k;
      re_cp16(Xs + rr * C::S + R + cc, Q + (ok ? qpanel(row0 + rr, cc, n) : 0), ok ? 16 : 0);
    }
    asm volatile("cp.async.commit_group;\n");
  };
  int64_t t = blockIdx.x;
  if (t < ntiles) load_tile(t, X0);
  int stage = 0;
  const int ksteps = (R + k + 3) / 4;
  for (; t < ntiles; t += gridDim.x) {
    double* Xs = X0 + stage * C::TM * C::S;
    const int64_t tn = t + gridDim.x;
    if (tn < ntiles) {
      load_tile(tn, X0 + (stage ^ 1) * C::TM * C::S);
      asm volatile("cp.async.wait_group 1;\n");
    } else {
      asm volatile("cp.async.wait_group 0;\n");
    }
    __syncthreads();
    // zero the Q columns >= k of this tile (cp.async zero-filled them only
    // for 16-byte chunks with cc >= k; an odd k leaves column k in a live chunk)
    if (k & 1)
      for (int rr = tid; rr < C::TM; rr += 256) Xs[rr * C::S + R + k] = 0.0;
    __syncthreads();
    const int64_t row0 = t * C::TM;
    double acc[C::MT][C::NT][2];
#pragma unroll
    for (int i = 0; i < C::MT; ++i)
#pragma unroll
      for (int j = 0; j < C::NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    const int ar = wm * C::WR + (lane >> 2), ak = lane & 3;
    const int bn = wn * C::WN + (lane >> 2), bk = lane & 3;
    for (int ks = 0; ks < ksteps; ++ks) {
      const int k0 = 4 * ks;
      double af[C::MT], bf[C::NT];
#pragma unroll
      for (int i = 0; i < C::MT; ++i) af[i] = Xs[(ar + 8 * i) * C::S + k0 + ak];
#pragma unroll
      for (int j = 0; j < C::NT; ++j) bf[j] = Ws[(k0 + bk) * C::SW + bn + 8 * j];
#pragma unroll
      for (int i = 0; i < C::MT; ++i)
#pragma unroll
        for (int j = 0; j < C::NT; ++j) re_dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
    const int er = wm * C::WR + (lane >> 2), ec = wn * C::WN + 2 * (lane & 3);
#pragma unroll
    for (int i = 0; i < C::MT; ++i) {
      const int rr = er + 8 * i;
      double nr = 0.0;
      if (row0 + rr < n) {
        double* dst = out + (row0 + rr) * R;
#pragma unroll
        for (int j = 0; j < C::NT; ++j) {
          const double2 v = make_double2(acc[i][j][0], acc[i][j][1]);
          *reinterpret_cast<double2*>(dst + ec + 8 * j) = v;
          if (out32)
            *reinterpret_cast<float2*>(out32 + (row0 + rr) * R + ec + 8 * j) =
                make_float2((float)v.x, (float)v.y);
          nr += v.x * v.x + v.y * v.y;
        }
      }
      nr += __shfl_xor_sync(0xffffffffu, nr, 1);
      nr += __shfl_xor_sync(0xffffffffu, nr, 2);
      if ((lane & 3) == 0) rn[wn * C::TM + rr] = nr;
    }
    __syncthreads();
    if (nrm2)
      for (int rr = tid; rr < C::TM; rr += 256)
        if (row0 + rr < n) nrm2[row0 + rr] = rn[rr] + rn[C::TM + rr];
    stage ^= 1;
  }
}

// rows_out[p][c] = sum_j X_{rows[p]}[j] W[j][c]; warp per row, W in smem
__global__ void __launch_bounds__(256) gather_rows_kernel(FactBasis b, const int64_t* __restrict__ rows,
                                                          int64_t count, const int* dcount,
                                                          double* __restrict__ out) {
  if (dcount && *dcount < count) count = *dcount;
  extern __shared__ double wsm[];  // (r + k) x r, then 8 warps x (r + k)
  const int r = b.r, rk = b.r + b.k;
  double* Ws = wsm;
  double* xs = wsm + (size_t)rk * r;
  for (int e = threadIdx.x; e < rk * r; e += blockDim.x) Ws[e] = b.W ? b.W[e] : ((e / r == e % r) ? 1.0 : 0.0);
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double* x = xs + (size_t)warp * rk;
  for (int64_t p = (int64_t)blockIdx.x * 8 + warp; p < count; p += (int64_t)gridDim.x * 8) {
    const int64_t i = rows[p];
    for (int j = lane; j < rk; j += 32)
      x[j] = (i < 0) ? 0.0 : (j < r ? b.A[i * r + j] : b.Q[qpanel(i, j - r, b.n)]);
    __syncwarp();
    for (int c = lane; c < r; c += 32) {
      double s = 0.0;
      for (int j = 0; j < rk; ++j) s += x[j] * Ws[(size_t)j * r + c];
      out[p * r + c] = s;
    }
    __syncwarp();
  }
}

// DMMA variant (r in {32, 64}): a warp takes 8 rows, Phi_rows = X_rows W with
// A fragments from the rows in global memory and W fragments from smem
template <int R>
__global__ void __launch_bounds__(256) gather_rows_tc_kernel(FactBasis b, const int64_t* __restrict__ rows,
                                                             int64_t count, const int* dcount,
                                                             double* __restrict__ out) {
  constexpr int KX = R + FACT_KQ, KS = KX / 4, S = R + 4, NT = R / 8;
  extern __shared__ __align__(16) double Ws[];  // KX x S
  if (dcount && *dcount < count) count = *dcount;
  const int k = b.k;
  for (int e = threadIdx.x; e < KX * R; e += blockDim.x) {
    const int j = e / R, c = e - j * R;
    Ws[j * S + c] = (j < R + k) ? (b.W ? b.W[(size_t)j * R + c] : (j == c ? 1.0 : 0.0)) : 0.0;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int rq = lane >> 2, cq = lane & 3;
  const int64_t tiles = (count + 7) / 8;
  for (int64_t t = (int64_t)blockIdx.x * 8 + warp; t < tiles; t += (int64_t)gridDim.x * 8) {
    const int64_t p = t * 8 + rq;
    const int64_t i = (p < count) ? rows[p] : -1;
    if (!__any_sync(0xffffffffu, i >= 0)) continue;  // a tile of empty slots (row -1)
    double af[KS];
#pragma unroll
    for (int j = 0; j < KS; ++j) {
      const int c = 4 * j + cq;
      double x = 0.0;
      if (i >= 0) {
        if (c < R) x = b.A[i * R + c];
        else if (c - R < k) x = b.Q[qpanel(i, c - R, b.n)];
      }
      af[j] = x;
    }
    double acc[NT][2];
#pragma unroll
    for (int ct = 0; ct < NT; ++ct) {
      acc[ct][0] = acc[ct][1] = 0.0;
#pragma unroll
      for (int j = 0; j < KS; ++j) re_dmma(acc[ct][0], acc[ct][1], af[j], Ws[(4 * j + cq) * S + 8 * ct + rq]);
    }
    if (p < count) {
#pragma unroll
      for (int ct = 0; ct < NT; ++ct)
        *reinterpret_cast<double2*>(out + p * R + 8 * ct + 2 * cq) = make_double2(acc[ct][0], acc[ct][1]);
    }
  }
}

int fact_gather_rows(adrom_ctx* ctx, const FactBasis& b, const int64_t* rows, int64_t count,
                     double* rows_out, const int* dcount) {
  if (count <= 0) return ADROM_OK;
  if (b.r == 32 || b.r == 64) {
    auto launch = [&](auto kern, int R) -> int {
      const size_t sm = sizeof(double) * (size_t)(R + FACT_KQ) * (R + 4);
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      int64_t g = ((count + 7) / 8 + 7) / 8;
      if (g > (int64_t)ctx->num_sms * 4) g = (int64_t)ctx->num_sms * 4;
      kern<<<(int)(g < 1 ? 1 : g), 256, sm, ctx->stream>>>(b, rows, count, dcount, rows_out);
      ADROM_LAUNCH_CK(ctx);
      return ADROM_OK;
    };
    return b.r == 32 ? launch(gather_rows_tc_kernel<32>, 32) : launch(gather_rows_tc_kernel<64>, 64);
  }
  const int rk = b.r + b.k;
  const size_t sm = sizeof(double) * ((size_t)rk * b.r + 8 * (size_t)rk);
  cudaFuncSetAttribute(gather_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  int64_t g = (count + 7) / 8;
  if (g > (int64_t)ctx->num_sms * 4) g = (int64_t)ctx->num_sms * 4;
  gather_rows_kernel<<<(int)g, 256, sm, ctx->stream>>>(b, rows, count, dcount, rows_out);
  ADROM_LAUNCH_CK(ctx);
  return ADROM_OK;
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
static int xpass_grid(adrom_ctx* ctx, int64_t n) {
  (void)ctx;
  const int64_t g = (n + XP_ROWS - 1) / XP_ROWS;
  return (int)(g < 1 ? 1 : g);
}

int fact_decode(adrom_ctx* ctx, const FactBasis& b, const double* a, const double* q_ref,
                const double* d, double* q_tilde, double* small, double* partial) {
  const int r = b.r, rk = r + b.k;
  double* v = small;
  if (b.W) {
    mat_vec_kernel<<<1, 256, 0, ctx->stream>>>(b.W, rk, r, a, v);
    ADROM_LAUNCH_CK(ctx);
  } else {
    ADROM_CK(ctx, cudaMemcpyAsync(v, a, sizeof(double) * r, cudaMemcpyDeviceToDevice, ctx->stream));
  }
  const int grid = xpass_grid(ctx, b.n);
  XPassArgs a1{b.A, b.Q, b.n, b.k, FACT_KQ, v, nullptr, q_ref, d, q_tilde, nullptr, nullptr, partial,
               nullptr};
  if (r == 64) xpass_launch<64, 1>(ctx, grid, a1);
  else if (r == 32) xpass_launch<32, 1>(ctx, grid, a1);
  else return set_error(ctx, ADROM_ERR_ARG, "factored decode: rank %d", r);
  ADROM_LAUNCH_CK(ctx);
  return ADROM_OK;
}

size_t fact_partial_doubles(adrom_ctx* ctx, int64_t n, int r) {
  (void)ctx;
  return (size_t)((n + XP_ROWS - 1) / XP_ROWS) * xpass_width(r, FACT_KQ, 2);
}

int fact_reanchor(adrom_ctx* ctx, const FactBasis& b, double* out, double* nrm2, float* out32) {
  auto launch = [&](auto kern, size_t smd) -> int {
    const size_t sm = sizeof(double) * smd;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    const int64_t nt = (b.n + 63) / 64;
    int64_t g = (int64_t)ctx->num_sms;
    if (g > nt) g = nt;
    const int pr = prof_begin(ctx, PROBE_ISVD_REANCHOR);
    kern<<<(int)(g < 1 ? 1 : g), 256, sm, ctx->stream>>>(b.A, b.Q, b.k, b.W, b.n, out, nrm2,
                                                         out32);
    prof_end(ctx, pr);
    ADROM_LAUNCH_CK(ctx);
    return ADROM_OK;
  };
  if (!b.W) return set_error(ctx, ADROM_ERR_ARG, "reanchor: identity transform");
  if (b.r == 32) return launch(reanchor_kernel<32>, ReTC<32>::smem_doubles);
  if (b.r == 64) return launch(reanchor_kernel<64>, ReTC<64>::smem_doubles);
  return set_error(ctx, ADROM_ERR_ARG, "reanchor: rank %d unsupported", b.r);
}

struct FactSmall {
  double *vdec, *vp, *red1, *red2, *pls, *t1, *t2, *Bm, *Tm, *sb, *p2;
  int* need;
};

static FactSmall fact_small_layout(double* w, int r) {
  FactSmall f;
  f.vdec = w;                         // r + KQ
  f.vp = f.vdec + r + FACT_KQ;        // r + KQ
  f.red1 = f.vp + r + FACT_KQ;        // r + 1: [p1, ||y||^2]
  f.red2 = f.red1 + r + 1;            // r + 1: [Phi^T q, ||q||^2]
  f.pls = f.red2 + r + 1;             // r
  f.t1 = f.pls + r;                   // r + KQ + 1   (reduced pass-1 sums)
  f.t2 = f.t1 + r + FACT_KQ + 1;      // r + KQ + 1 (reduced pass-2 sums)
  f.Bm = f.t2 + 2 * (r + FACT_KQ) + 2;  // (r + 1) x r
  f.Tm = f.Bm + (r + 1) * r;            // (r + 1) x r
  f.sb = f.Tm + (r + 1) * r;            // [0] qinv, [1] ||p2||, [2 .. r+3) dropped vector
  f.need = (int*)(f.sb + r + 8);        // 4 ints
  f.p2 = f.sb + r + 12;                 // r: least-squares refinement
  return f;
}

// pass 1 (only the snapshot's projection): X^T y, ||y||^2, exact row norms.
// Needs y only, so the session runs it on the coarse-step stream while the
// reduced step (one block) runs on the main stream.
int fact_event_pass_a(adrom_ctx* ctx, const FactBasis& b, const FactEventArgs& e) {
  const int r = b.r, k = b.k, rk = r + k;
  if (!(r == 32 || r == 64) || k < 0 || k >= FACT_KQ)
    return set_error(ctx, ADROM_ERR_ARG, "factored iSVD: r=%d k=%d", r, k);
  const FactSmall f = fact_small_layout(e.small, r);
  const int grid = xpass_grid(ctx, b.n);
  int pr = prof_begin(ctx, PROBE_ISVD_PROJECT);
  XPassArgs a1{b.A, b.Q, b.n, k, FACT_KQ, nullptr, e.y, e.q_ref, e.d, nullptr, nullptr, nullptr,
               e.partial_a, e.flag_a, e.vdrop_in, e.vdrop_in ? e.nrm2_inout : nullptr, nullptr};
  if (r == 64) xpass_launch<64, 1>(ctx, grid, a1);
  else xpass_launch<32, 1>(ctx, grid, a1);
  ADROM_LAUNCH_CK(ctx);
  const int w1 = xpass_width(r, FACT_KQ, 1);
  reduce_partials_kernel<<<w1, 256, 0, ctx->stream>>>(e.partial_a, grid, w1, f.t1, nullptr);
  ADROM_LAUNCH_CK(ctx);
  prof_end(ctx, pr);
  // p1 = W^T (X^T y), ||y||^2
  if (b.W) {
    matT_vec_kernel<<<1, 128, 0, ctx->stream>>>(b.W, rk, r, f.t1, f.red1);
    ADROM_LAUNCH_CK(ctx);
  } else {
    ADROM_CK(ctx, cudaMemcpyAsync(f.red1, f.t1, sizeof(double) * r, cudaMemcpyDeviceToDevice, ctx->stream));
  }
  ADROM_CK(ctx, cudaMemcpyAsync(f.red1 + r, f.t1 + r + FACT_KQ, sizeof(double), cudaMemcpyDeviceToDevice,
                                ctx->stream));
  return ADROM_OK;
}

// the rest of the event on the main stream: least squares, pass 2 with the
// the refined direction q_hat = (q - Phi p2) qinv in factored form: with
// Phi' = Phi B_top + q_hat b_bot = X W (B_top - qinv p2 b_bot) + q qinv b_bot,
// B_top (and the dropped vector's top) absorb the rank-one correction
__global__ void refine_b_kernel(double* __restrict__ B, double* __restrict__ udrop,
                                const double* __restrict__ p2, const double* __restrict__ sb,
                                int r, int r_out) {
  const double qi = sb[0];
  for (int e = threadIdx.x; e < r * r_out; e += blockDim.x) {
    const int k = e / r_out, c = e - k * r_out;
    B[e] -= qi * p2[k] * B[(size_t)r * r_out + c];
  }
  if (udrop)
    for (int k = threadIdx.x; k < r; k += blockDim.x) udrop[k] -= qi * p2[k] * udrop[r];
}

// fused decode of the reduced state, core SVD, W', state transfer, seeds
int fact_event_pass_b(adrom_ctx* ctx, const FactBasis& b, const FactEventArgs& e) {
  const int r = b.r, k = b.k, rk = r + k;
  const FactSmall f = fact_small_layout(e.small, r);
  const int grid = xpass_grid(ctx, b.n);
  // decode vector W a (identity when k == 0 and W == null); no decode without a
  if (e.a && b.W) {
    mat_vec_kernel<<<1, 256, 0, ctx->stream>>>(b.W, rk, r, e.a, f.vdec);
    ADROM_LAUNCH_CK(ctx);
  } else if (e.a) {
    ADROM_CK(ctx, cudaMemcpyAsync(f.vdec, e.a, sizeof(double) * r, cudaMemcpyDeviceToDevice, ctx->stream));
  }
  // least squares p = G^{-1} p1; the explicit residual pass always runs here
  int prs = prof_begin(ctx, PROBE_ISVD_SMALL);
  int st = isvd_solve_launch(ctx, f.red1, e.G, r, f.pls, f.need);
  prof_end(ctx, prs);
  if (st) return st;
  set_need_kernel<<<1, 1, 0, ctx->stream>>>(f.need);
  ADROM_LAUNCH_CK(ctx);
  if (b.W) {
    mat_vec_kernel<<<1, 256, 0, ctx->stream>>>(b.W, rk, r, f.pls, f.vp);
    ADROM_LAUNCH_CK(ctx);
  } else {
    ADROM_CK(ctx, cudaMemcpyAsync(f.vp, f.pls, sizeof(double) * r, cudaMemcpyDeviceToDevice, ctx->stream));
  }
  // pass 2 (+ decode of the reduced state, projection.py:104)
  int pr = prof_begin(ctx, PROBE_ISVD_RESID);
  XPassArgs a2{b.A, b.Q, b.n, k, FACT_KQ, f.vp, e.y, e.q_ref, e.d, e.q_tilde, e.Qw, e.qv, e.partial,
               e.flag, nullptr, nullptr, e.a ? f.vdec : nullptr};
  if (r == 64) xpass_launch<64, 2>(ctx, grid, a2);
  else xpass_launch<32, 2>(ctx, grid, a2);
  ADROM_LAUNCH_CK(ctx);
  const int w2 = xpass_width(r, FACT_KQ, 2);
  reduce_partials_kernel<<<w2, 256, 0, ctx->stream>>>(e.partial, grid, w2, f.t2, nullptr);
  ADROM_LAUNCH_CK(ctx);
  prof_end(ctx, pr);
  // Phi^T q = W^T (X^T q), ||q||^2
  if (b.W) {
    matT_vec_kernel<<<1, 128, 0, ctx->stream>>>(b.W, rk, r, f.t2, f.red2);
    ADROM_LAUNCH_CK(ctx);
  } else {
    ADROM_CK(ctx, cudaMemcpyAsync(f.red2, f.t2, sizeof(double) * r, cudaMemcpyDeviceToDevice, ctx->stream));
  }
  ADROM_CK(ctx, cudaMemcpyAsync(f.red2 + r, f.t2 + r + FACT_KQ, sizeof(double), cudaMemcpyDeviceToDevice,
                                ctx->stream));
  // one least-squares refinement step: q' = q - Phi p2 (isvd_refine_kernel)
  prs = prof_begin(ctx, PROBE_ISVD_SMALL);
  st = isvd_refine_launch(ctx, e.G, r, f.red2, f.pls, f.p2, f.sb + 1, f.need);
  prof_end(ctx, prs);
  if (st) return st;
  // core: K, its SVD, B, qinv, the tracked Gram of the new basis, sigma'
  pr = prof_begin(ctx, PROBE_ISVD_CORE);
  double* udrop = f.sb + 2;
  st = isvd_core_launch(ctx, e.sigma, f.red1, f.pls, f.red2, f.need, e.G, r, e.lam, f.Bm, f.sb, f.Tm,
                        e.G_out, e.sigma_out, e.stats, e.flag, udrop);
  prof_end(ctx, pr);
  if (st) return st;
  // state transfer for the new basis: a' = B_top^T G a + b_bot^T qinv c'.a,
  // from the refined c' = Phi^T q' (red2) and the unmodified B
  if (e.a_out) {
    encode_factored_kernel<<<1, 128, 0, ctx->stream>>>(e.G, r, e.a, f.red2, f.sb, f.Bm, e.a_out);
    ADROM_LAUNCH_CK(ctx);
  }
  refine_b_kernel<<<1, 256, 0, ctx->stream>>>(f.Bm, e.vdrop_out ? udrop : nullptr, f.p2, f.sb, r, r);
  ADROM_LAUNCH_CK(ctx);
  // W' for the new basis
  wnext_kernel<<<(rk + 1) * r / 256 + 1, 256, 0, ctx->stream>>>(b.W, rk, r, f.Bm, f.sb, e.W_out);
  ADROM_LAUNCH_CK(ctx);
  if (e.vdrop_out) {
    vdrop_kernel<<<1, 128, 0, ctx->stream>>>(b.W, rk, r, udrop, f.sb, e.vdrop_out);
    ADROM_LAUNCH_CK(ctx);
  }
  if (e.seed_res2) {
    int64_t g = (b.n + 255) / 256;
    if (g > (int64_t)ctx->num_sms * 8) g = (int64_t)ctx->num_sms * 8;
    seed_bounds_kernel<<<(int)g, 256, 0, ctx->stream>>>(e.nrm2_inout, e.qv, f.sb, b.n,
                                                        e.seed_res2, e.seed_bnd2, e.seed_ver,
                                                        e.nrm2_out);
    ADROM_LAUNCH_CK(ctx);
  }
  return ADROM_OK;
}

int fact_isvd_event(adrom_ctx* ctx, const FactBasis& b, const FactEventArgs& e) {
  int st = fact_event_pass_a(ctx, b, e);
  if (st) return st;
  return fact_event_pass_b(ctx, b, e);
}



}  // namespace adrom

using namespace adrom;

// ---------------------------------------------------------------------------
// C-ABI: a streaming iSVD on the factored basis (include/adrom_b200.h)
// ---------------------------------------------------------------------------
struct adrom_isvd_stream {
  adrom_ctx* ctx = nullptr;
  int64_t n = 0;
  int r = 0;
  int kf = 0, acur = 0, cur = 0;
  bool w_id = true;
  double *A[2] = {nullptr, nullptr}, *Q = nullptr, *W[2] = {nullptr, nullptr};
  double *sigma[2] = {nullptr, nullptr}, *G[2] = {nullptr, nullptr};
  double *partial = nullptr, *partial_a = nullptr, *small = nullptr, *stats = nullptr;
  size_t partial_doubles = 0;  // capacity of `partial`
  std::vector<void*> allocs;
  double* alloc(size_t count) {
    void* p = nullptr;
    if (cudaMalloc(&p, sizeof(double) * (count ? count : 1)) != cudaSuccess) return nullptr;
    allocs.push_back(p);
    return (double*)p;
  }
};

extern "C" {

int adrom_isvd_stream_create(adrom_ctx* ctx, int64_t n, int32_t r, adrom_isvd_stream** out) {
  if (!ctx || !out) return ADROM_ERR_ARG;
  if (!(r == 32 || r == 64) || n < r)
    return set_error(ctx, ADROM_ERR_ARG, "isvd stream: r must be 32 or 64 and n >= r");
  adrom_isvd_stream* s = new adrom_isvd_stream();
  s->ctx = ctx;
  s->n = n;
  s->r = r;
  bool ok = true;
  for (int b = 0; b < 2; ++b) {
    ok &= (s->A[b] = s->alloc((size_t)n * r)) != nullptr;
    ok &= (s->W[b] = s->alloc((size_t)(r + FACT_KQ + 1) * r)) != nullptr;
    ok &= (s->sigma[b] = s->alloc(r)) != nullptr;
    ok &= (s->G[b] = s->alloc((size_t)r * r)) != nullptr;
  }
  ok &= (s->Q = s->alloc((size_t)n * FACT_KQ)) != nullptr;
  // (the load's Gram pass needs r x r doubles per block: a short stream's
  // xpass partials alone are smaller than one of them)
  s->partial_doubles = fact_partial_doubles(ctx, n, r);
  if (s->partial_doubles < gram_partial_doubles(ctx, r)) s->partial_doubles = gram_partial_doubles(ctx, r);
  ok &= (s->partial = s->alloc(s->partial_doubles)) != nullptr;
  ok &= (s->partial_a = s->alloc(fact_partial_doubles(ctx, n, r))) != nullptr;
  ok &= (s->small = s->alloc(fact_small_doubles(r))) != nullptr;
  ok &= (s->stats = s->alloc(16)) != nullptr;
  if (!ok) {
    for (void* p : s->allocs) cudaFree(p);
    delete s;
    return set_error(ctx, ADROM_ERR_CUDA, "isvd stream: device allocation failed");
  }
  cudaMemsetAsync(s->Q, 0, sizeof(double) * (size_t)n * FACT_KQ, ctx->stream);
  *out = s;
  return ADROM_OK;
}

void adrom_isvd_stream_destroy(adrom_isvd_stream* s) {
  if (!s) return;
  cudaStreamSynchronize(s->ctx->stream);
  for (void* p : s->allocs) cudaFree(p);
  delete s;
}

int adrom_isvd_stream_load(adrom_isvd_stream* s, const double* phi, const double* sigma) {
  if (!s) return ADROM_ERR_ARG;
  adrom_ctx* ctx = s->ctx;
  ADROM_CK(ctx, cudaMemcpyAsync(s->A[0], phi, sizeof(double) * (size_t)s->n * s->r,
                                cudaMemcpyDeviceToDevice, ctx->stream));
  ADROM_CK(ctx, cudaMemcpyAsync(s->sigma[0], sigma, sizeof(double) * s->r, cudaMemcpyDeviceToDevice,
                                ctx->stream));
  s->kf = 0;
  s->acur = 0;
  s->cur = 0;
  s->w_id = true;
  return ts_gram(ctx, s->A[0], s->n, s->r, s->G[0], s->partial, s->partial_doubles);
}

int adrom_isvd_stream_update(adrom_isvd_stream* s, const double* y_hat, double lam,
                             adrom_isvd_info* host_info) {
  if (!s) return ADROM_ERR_ARG;
  adrom_ctx* ctx = s->ctx;
  int st;
  auto view = [&]() {
    return FactBasis{s->A[s->acur], s->Q, s->r, s->w_id ? 0 : s->kf, s->w_id ? nullptr : s->W[s->cur], s->n};
  };
  if (s->kf == FACT_KQ) {  // re-anchor (same basis)
    st = fact_reanchor(ctx, view(), s->A[1 - s->acur], nullptr);
    if (st) return st;
    s->acur = 1 - s->acur;
    s->kf = 0;
    s->w_id = true;
  }
  const int nxt = 1 - s->cur;
  const FactBasis b = view();
  FactEventArgs e{};
  e.y = y_hat;
  e.Qw = s->Q;
  e.sigma = s->sigma[s->cur];
  e.G = s->G[s->cur];
  e.lam = lam;
  e.partial = s->partial;
  e.partial_a = s->partial_a;
  e.small = s->small;
  e.W_out = s->W[nxt];
  e.sigma_out = s->sigma[nxt];
  e.G_out = s->G[nxt];
  e.stats = s->stats;
  e.flag = ctx->dflags;
  e.flag_a = ctx->dflags;
  ADROM_CK(ctx, cudaMemsetAsync(ctx->dflags, 0, sizeof(int) * 16, ctx->stream));
  st = fact_isvd_event(ctx, b, e);
  if (st) return st;
  int* hf = (int*)ctx->pinned;
  double* hs = (double*)((char*)ctx->pinned + 256);
  ADROM_CK(ctx, cudaMemcpyAsync(hf, ctx->dflags, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  ADROM_CK(ctx, cudaMemcpyAsync(hs, s->stats, sizeof(double) * 8, cudaMemcpyDeviceToHost, ctx->stream));
  ADROM_CK(ctx, cudaStreamSynchronize(ctx->stream));
  if (hf[0] & 1)  // dense.py:110 / tracking.py: non-finite input, basis unchanged
    return set_error(ctx, ADROM_ERR_NONFINITE, "least_squares matrix contains non-finite entries");
  if (hf[0] & 8)
    return set_error(ctx, ADROM_ERR_NOCONV, "SVD did not converge for %dx%d input", s->r + 1, s->r + 1);
  if (host_info) {
    host_info->qnorm = hs[0];
    host_info->ynorm = hs[1];
    host_info->proj_resid = hs[2];
    host_info->degenerate = (int)hs[3];
    host_info->reorthogonalised = (int)hs[4];
    host_info->sweeps = (int)hs[5];
    host_info->core_path = (int)hs[7];
  }
  s->kf = b.k + 1;
  s->w_id = false;
  s->cur = nxt;
  return ADROM_OK;
}

int adrom_isvd_stream_read(adrom_isvd_stream* s, double* phi_out, double* sigma_out) {
  if (!s) return ADROM_ERR_ARG;
  adrom_ctx* ctx = s->ctx;
  if (sigma_out)
    ADROM_CK(ctx, cudaMemcpyAsync(sigma_out, s->sigma[s->cur], sizeof(double) * s->r,
                                  cudaMemcpyDeviceToDevice, ctx->stream));
  if (phi_out) {
    if (s->w_id) {
      ADROM_CK(ctx, cudaMemcpyAsync(phi_out, s->A[s->acur], sizeof(double) * (size_t)s->n * s->r,
                                    cudaMemcpyDeviceToDevice, ctx->stream));
    } else {
      const FactBasis b{s->A[s->acur], s->Q, s->r, s->kf, s->W[s->cur], s->n};
      const int st = fact_reanchor(ctx, b, phi_out, nullptr);
      if (st) return st;
    }
  }
  return ADROM_OK;
}

}  // extern "C"
