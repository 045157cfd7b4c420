// Hyper-reduction sampling on the device: exact-greedy QDEIM (sampling.py:77-114),
// feature-guided sampling (sampling.py:117-159), stencil closure + gather plan
// (sampling.py:178-189, fom.py:119-158) and the reduced-operator assembly
// with the DEIM pseudo-inverse (sampling.py:162-175, projection.py:61-80).
//
// QDEIM = the pivots of a column-pivoted QR of phi^T, i.e. greedy selection of
// the row with the largest residual norm after projecting out the directions
// of the rows already chosen (ties -> lowest row, LAPACK idamax).  Done
// naively that is r passes over the N x r basis.  Here it is a
// guess-and-verify loop:
//   * directions D = MGS of the guessed pivot rows, completed to an
//     orthonormal basis of R^r (one block);
//   * one pass over the basis computes C_i = D^T phi_i for every row; the
//     residual of row i after k steps is sum_{l>=k} C_il^2, so the exact
//     argmax of every step k is found in the same pass (tiled FP64 GEMM with
//     an argmax epilogue);
//   * the argmax at step k is exact as soon as guesses 0..k-1 are confirmed,
//     so every pass confirms at least one more pivot; with the previous
//     event's pivots as guesses a pass usually confirms all of them.
#include "common.cuh"
#include "jacobi.cuh"
#include "sampling_internal.cuh"

#include <limits.h>

namespace adrom {

// ---------------------------------------------------------------------------
// directions: D (r x r, row-major, padded stride r+1) from guessed rows
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) qd_dirs_kernel(const double* __restrict__ phi, int r,
                                                      const int64_t* __restrict__ L, int g,
                                                      double* __restrict__ Dout,
                                                      double* __restrict__ tau) {
  extern __shared__ double sm[];
  const int S = r + 1;
  double* Ds = sm;          // r x S: Ds[j*S + k] component j of direction k
  double* v = Ds + r * S;   // r
  double* c = v + r;        // r
  double* red = c + r;      // 32
  __shared__ int sh_j;
  const int tid = threadIdx.x;
  for (int k = 0; k < r; ++k) {
    if (k < g) {
      for (int j = tid; j < r; j += blockDim.x) v[j] = phi[L[k] * r + j];
    } else {
      // completion: the unit vector with the largest residual
      double best = -1.0;
      int bj = 0;
      for (int j = tid; j < r; j += blockDim.x) {
        double s = 1.0;
        for (int l = 0; l < k; ++l) s -= Ds[j * S + l] * Ds[j * S + l];
        if (s > best) {
          best = s;
          bj = j;
        }
      }
      // block argmax (lowest j on ties)
      for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int oj = __shfl_xor_sync(0xffffffffu, bj, o);
        if (ob > best || (ob == best && oj < bj)) {
          best = ob;
          bj = oj;
        }
      }
      __shared__ double wb[32];
      __shared__ int wj[32];
      if ((tid & 31) == 0) {
        wb[tid >> 5] = best;
        wj[tid >> 5] = bj;
      }
      __syncthreads();
      if (tid == 0) {
        double b = wb[0];
        int jj = wj[0];
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w)
          if (wb[w] > b || (wb[w] == b && wj[w] < jj)) {
            b = wb[w];
            jj = wj[w];
          }
        sh_j = jj;
      }
      __syncthreads();
      for (int j = tid; j < r; j += blockDim.x) v[j] = (j == sh_j) ? 1.0 : 0.0;
    }
    __syncthreads();
    // CGS2 against directions 0..k-1
    for (int pass = 0; pass < 2; ++pass) {
      for (int l = tid; l < k; l += blockDim.x) {
        double s = 0.0;
        for (int j = 0; j < r; ++j) s += v[j] * Ds[j * S + l];
        c[l] = s;
      }
      __syncthreads();
      for (int j = tid; j < r; j += blockDim.x) {
        double s = 0.0;
        for (int l = 0; l < k; ++l) s += c[l] * Ds[j * S + l];
        v[j] -= s;
      }
      __syncthreads();
    }
    double a = 0.0;
    for (int j = tid; j < r; j += blockDim.x) a += v[j] * v[j];
    a = block_sum_dyn(a, red);
    const double nrm = sqrt(a);
    if (tid == 0 && k < g) tau[k] = nrm;
    for (int j = tid; j < r; j += blockDim.x) Ds[j * S + k] = nrm > 0.0 ? v[j] / nrm : 0.0;
    __syncthreads();
  }
  for (int e = tid; e < r * r; e += blockDim.x) {
    const int j = e / r, k = e - j * r;
    Dout[j * r + k] = Ds[j * S + k];
  }
}

// per-row exclusion: a row that is guess L[pos] leaves the candidate set after
// step pos; rows of earlier restarts (ex) are excluded from every step.
struct Excl {
  const int64_t* lrow;  // sorted guessed rows (smem)
  const int* lpos;      // their positions
  int g;
  const int64_t* ex;    // sorted excluded rows (global)
  int n_ex;
  __device__ __forceinline__ int first_excluded_step(int64_t i) const {
    // rows of earlier restarts first: a stale guess may name one of them
    int lo = 0, hi = n_ex - 1;
    while (lo <= hi) {
      const int mid = (lo + hi) >> 1;
      const int64_t v = ex[mid];
      if (v == i) return 0;
      if (v < i) lo = mid + 1;
      else hi = mid - 1;
    }
    lo = 0;
    hi = g - 1;
    while (lo <= hi) {
      const int mid = (lo + hi) >> 1;
      const int64_t v = lrow[mid];
      if (v == i) return lpos[mid] + 1;
      if (v < i) lo = mid + 1;
      else hi = mid - 1;
    }
    return INT_MAX;
  }
};

__device__ __forceinline__ bool better(double v, int64_t i, double bv, int64_t bi) {
  return v > bv || (v == bv && i < bi && i >= 0) || (bi < 0 && i >= 0);
}

__device__ void load_guess_sorted(const int64_t* L, int g, int64_t* lrow, int* lpos) {
  // insertion rank (g <= 256): lrow sorted ascending with original positions
  for (int k = threadIdx.x; k < g; k += blockDim.x) {
    const int64_t x = L[k];
    int rank = 0;
    for (int j = 0; j < g; ++j) {
      const int64_t y = L[j];
      if (y < x || (y == x && j < k)) ++rank;
    }
    lrow[rank] = x;
    lpos[rank] = k;
  }
}

// ---------------------------------------------------------------------------
// scan, tiled FP64 GEMM C = Phi_tile * D with an argmax epilogue (R in
// {16, 32, 64, 128}); thread (rg, cg) owns rows rg*RM.. and columns cg+16q
// ---------------------------------------------------------------------------
template <int R>
struct ScanCfg {
  static constexpr int TM = (R <= 64) ? 128 : 64;
  static constexpr int RM = TM / 16;
  static constexpr int RN = R / 16;
  static constexpr int SA = R + 1;
};

template <int R>
__global__ void __launch_bounds__(256) qd_scan_kernel(const double* __restrict__ phi, int64_t n,
                                                      const double* __restrict__ D, int m_eval,
                                                      const int64_t* __restrict__ L, int g,
                                                      const int64_t* __restrict__ ex, int n_ex,
                                                      double* __restrict__ pv,
                                                      int64_t* __restrict__ pi) {
  using C = ScanCfg<R>;
  extern __shared__ double sm[];
  double* As = sm;                            // TM x SA
  double* Bs = As + C::TM * C::SA;            // R x R
  int64_t* lrow = (int64_t*)(Bs + R * R);     // R
  int* lpos = (int*)(lrow + R);               // R
  const int tid = threadIdx.x;
  for (int e = tid; e < R * R; e += 256) Bs[e] = D[e];
  load_guess_sorted(L, g, lrow, lpos);
  const Excl exc{lrow, lpos, g, ex, n_ex};
  const int rg = tid >> 4, cg = tid & 15;
  double bv[C::RN];
  int64_t bi[C::RN];
#pragma unroll
  for (int q = 0; q < C::RN; ++q) {
    bv[q] = -1.0;
    bi[q] = -1;
  }
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
    for (int e = rows * R + tid; e < C::TM * R; e += 256) {
      const int rr = e / R, cc = e - rr * R;
      As[rr * C::SA + cc] = 0.0;
    }
    __syncthreads();
    double acc[C::RM][C::RN];
#pragma unroll
    for (int m = 0; m < C::RM; ++m)
#pragma unroll
      for (int q = 0; q < C::RN; ++q) acc[m][q] = 0.0;
#pragma unroll 4
    for (int k = 0; k < R; ++k) {
      double av[C::RM], bw[C::RN];
#pragma unroll
      for (int m = 0; m < C::RM; ++m) av[m] = As[(rg * C::RM + m) * C::SA + k];
#pragma unroll
      for (int q = 0; q < C::RN; ++q) bw[q] = Bs[k * R + cg + 16 * q];
#pragma unroll
      for (int m = 0; m < C::RM; ++m)
#pragma unroll
        for (int q = 0; q < C::RN; ++q) acc[m][q] = fma(av[m], bw[q], acc[m][q]);
    }
    // epilogue: residual after step l = sum_{c >= l} C_c^2, column c = cg + 16 q
#pragma unroll
    for (int m = 0; m < C::RM; ++m) {
      const int64_t i = row0 + rg * C::RM + m;
      double incl[C::RN], tot[C::RN];
#pragma unroll
      for (int q = 0; q < C::RN; ++q) {
        double x = acc[m][q] * acc[m][q];
        // inclusive suffix over cg' >= cg within the 16-lane row group
#pragma unroll
        for (int o = 1; o < 16; o <<= 1) {
          const double y = __shfl_down_sync(0xffffffffu, x, o, 16);
          if (cg + o < 16) x += y;
        }
        incl[q] = x;
        tot[q] = __shfl_sync(0xffffffffu, x, 0, 16);
      }
      if (i < n) {
        const int fx = exc.first_excluded_step(i);
        double later = 0.0;
#pragma unroll
        for (int q = C::RN - 1; q >= 0; --q) {
          const int l = cg + 16 * q;
          const double s = incl[q] + later;
          if (l < m_eval && l < fx && better(s, i, bv[q], bi[q])) {
            bv[q] = s;
            bi[q] = i;
          }
          later += tot[q];
        }
      }
    }
  }
  // block reduction over the 16 row groups: reuse As as scratch
  __syncthreads();
  double* rv = As;                       // 16 x R
  int64_t* ri = (int64_t*)(As + 16 * R); // 16 x R
#pragma unroll
  for (int q = 0; q < C::RN; ++q) {
    rv[rg * R + cg + 16 * q] = bv[q];
    ri[rg * R + cg + 16 * q] = bi[q];
  }
  __syncthreads();
  for (int l = tid; l < m_eval; l += 256) {
    double b = -1.0;
    int64_t bidx = -1;
    for (int w = 0; w < 16; ++w)
      if (better(rv[w * R + l], ri[w * R + l], b, bidx)) {
        b = rv[w * R + l];
        bidx = ri[w * R + l];
      }
    pv[(size_t)blockIdx.x * R + l] = b;
    pi[(size_t)blockIdx.x * R + l] = bidx;
  }
}

// generic r (<= 64): thread per row, local arrays
__global__ void __launch_bounds__(128) qd_scan_generic_kernel(
    const double* __restrict__ phi, int64_t n, int r, const double* __restrict__ D, int m_eval,
    const int64_t* __restrict__ L, int g, const int64_t* __restrict__ ex, int n_ex,
    double* __restrict__ pv, int64_t* __restrict__ pi) {
  extern __shared__ double sm[];
  double* Ds = sm;                           // r x r
  int64_t* lrow = (int64_t*)(Ds + r * r);    // r
  int* lpos = (int*)(lrow + r);              // r
  const int tid = threadIdx.x;
  for (int e = tid; e < r * r; e += blockDim.x) Ds[e] = D[e];
  load_guess_sorted(L, g, lrow, lpos);
  __syncthreads();
  const Excl exc{lrow, lpos, g, ex, n_ex};
  double bv[64];
  int64_t bi[64];
  for (int l = 0; l < m_eval; ++l) {
    bv[l] = -1.0;
    bi[l] = -1;
  }
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + tid; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double row[64], cc[64];
    for (int j = 0; j < r; ++j) row[j] = phi[i * r + j];
    for (int l = 0; l < r; ++l) {
      double s = 0.0;
      for (int j = 0; j < r; ++j) s = fma(row[j], Ds[j * r + l], s);
      cc[l] = s;
    }
    const int fx = exc.first_excluded_step(i);
    double suf = 0.0;
    for (int l = r - 1; l >= 0; --l) {
      suf += cc[l] * cc[l];
      if (l < m_eval && l < fx && better(suf, i, bv[l], bi[l])) {
        bv[l] = suf;
        bi[l] = i;
      }
    }
  }
  // block reduce per step through shared memory (128 threads, one step at a time)
  __shared__ double wv[128];
  __shared__ int64_t wi[128];
  for (int l = 0; l < m_eval; ++l) {
    __syncthreads();
    wv[tid] = bv[l];
    wi[tid] = bi[l];
    __syncthreads();
    if (tid == 0) {
      double b = -1.0;
      int64_t bidx = -1;
      for (int w = 0; w < (int)blockDim.x; ++w)
        if (better(wv[w], wi[w], b, bidx)) {
          b = wv[w];
          bidx = wi[w];
        }
      pv[(size_t)blockIdx.x * r + l] = b;
      pi[(size_t)blockIdx.x * r + l] = bidx;
    }
  }
}

// best per step across blocks (one block per step)
__global__ void qd_reduce_kernel(const double* __restrict__ pv, const int64_t* __restrict__ pi,
                                 int nb, int ld, double* __restrict__ bestv,
                                 int64_t* __restrict__ besti) {
  const int l = blockIdx.x;
  double b = -1.0;
  int64_t bidx = -1;
  for (int k = threadIdx.x; k < nb; k += blockDim.x) {
    const double v = pv[(size_t)k * ld + l];
    const int64_t i = pi[(size_t)k * ld + l];
    if (better(v, i, b, bidx)) {
      b = v;
      bidx = i;
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, b, o);
    const int64_t oi = __shfl_xor_sync(0xffffffffu, bidx, o);
    if (better(ov, oi, b, bidx)) {
      b = ov;
      bidx = oi;
    }
  }
  __shared__ double wv[32];
  __shared__ int64_t wi[32];
  if ((threadIdx.x & 31) == 0) {
    wv[threadIdx.x >> 5] = b;
    wi[threadIdx.x >> 5] = bidx;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w)
      if (better(wv[w], wi[w], b, bidx)) {
        b = wv[w];
        bidx = wi[w];
      }
    bestv[l] = b;
    besti[l] = bidx;
  }
}

// status[0] = done, [1] = new g, [2] = error (1 + pivot step) or 0,
// [3] = step of the error, [4..5] = error residual (double bits)
__global__ void qd_check_kernel(int64_t* __restrict__ L, int g, int m, int m_eval,
                                const double* __restrict__ bestv,
                                const int64_t* __restrict__ besti, int* __restrict__ status,
                                double* __restrict__ err_resid) {
  int kstar = -1;
  const int lim = g < m_eval ? g : m_eval;
  for (int k = 0; k < lim; ++k)
    if (besti[k] != L[k]) {
      kstar = k;
      break;
    }
  int newg, done = 0, confirmed;
  if (kstar >= 0) {
    // keep the remaining old guesses (the pivot SET usually survives a basis
    // update, only its order changes): L[0..k*) + [exact pivot] + old
    // guesses after k* without the exact pivot
    const int64_t piv = besti[kstar];
    int w = kstar + 1;
    int64_t carry = L[kstar];
    for (int j = kstar + 1; j <= g && w < m; ++j) {
      const int64_t nxt = (j < g) ? L[j] : -1;
      if (carry != piv && carry >= 0) L[w++] = carry;
      carry = nxt;
    }
    L[kstar] = piv;
    newg = w;
    confirmed = kstar + 1;
  } else if (g < m) {
    L[g] = besti[g];
    newg = g + 1;
    confirmed = newg;
    done = (newg == m);
  } else {
    newg = g;
    confirmed = g;
    done = 1;
  }
  int err = 0;
  for (int k = 0; k < confirmed && k < m_eval; ++k) {
    if (besti[k] < 0 || !(sqrt(bestv[k]) >= 1e-14)) {  // sampling.py:97-101
      err = k + 1;
      *err_resid = besti[k] < 0 ? 0.0 : sqrt(bestv[k]);
      break;
    }
  }
  status[0] = done;
  status[1] = newg;
  status[2] = err;
}

// sort rows[0..n) ascending (single thread; n <= a few thousand)
__global__ void sort_rows_kernel(const int64_t* __restrict__ in, int n, int64_t* __restrict__ out) {
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

size_t qdeim_workspace_bytes(adrom_ctx* ctx, int r, int count) {
  const int nb = partial_rows(ctx);
  size_t b = 0;
  b += align_up(sizeof(double) * r * r);             // D
  b += align_up(sizeof(double) * r);                 // tau
  b += align_up(sizeof(double) * (size_t)nb * r);    // pv
  b += align_up(sizeof(int64_t) * (size_t)nb * r);   // pi
  b += align_up(sizeof(double) * r);                 // bestv
  b += align_up(sizeof(int64_t) * r);                // besti
  b += align_up(sizeof(int) * 8) + align_up(sizeof(double) * 2);
  b += align_up(sizeof(int64_t) * (size_t)(count + 1));  // sorted exclusions
  b += align_up(sizeof(int64_t) * (size_t)r);            // local guess list
  return b;
}

int qdeim_select(adrom_ctx* ctx, const double* phi, int64_t n, int r, int count, int64_t* out_idx,
                 QdeimGuess* guess, void* ws, int* iterations_out) {
  if (count > n) return set_error(ctx, ADROM_ERR_DENSE, "cannot select %d pivots from %lld columns",
                                  count, (long long)n);
  if (r < 1 || r > 128) return set_error(ctx, ADROM_ERR_ARG, "qdeim: rank %d unsupported", r);
  const int nb = partial_rows(ctx);
  char* w = (char*)ws;
  auto take = [&](size_t bytes) {
    void* p = w;
    w += align_up(bytes);
    return p;
  };
  double* D = (double*)take(sizeof(double) * r * r);
  double* tau = (double*)take(sizeof(double) * r);
  double* pv = (double*)take(sizeof(double) * (size_t)nb * r);
  int64_t* pi = (int64_t*)take(sizeof(int64_t) * (size_t)nb * r);
  double* bestv = (double*)take(sizeof(double) * r);
  int64_t* besti = (int64_t*)take(sizeof(int64_t) * r);
  int* status = (int*)take(sizeof(int) * 8);
  double* err_resid = (double*)take(sizeof(double) * 2);
  int64_t* ex = (int64_t*)take(sizeof(int64_t) * (size_t)(count + 1));
  int64_t* Lloc = (int64_t*)take(sizeof(int64_t) * (size_t)r);
  const bool fast = (r == 16 || r == 32 || r == 64 || r == 128);
  if (!fast && r > 64) return set_error(ctx, ADROM_ERR_ARG, "qdeim: rank %d unsupported", r);
  int* hstat = (int*)ctx->pinned;
  double* hres = (double*)((char*)ctx->pinned + 64);
  int chosen = 0, chunk = 0, iters = 0;
  const size_t dsm = sizeof(double) * ((size_t)r * (r + 1) + 2 * r + 32);
  cudaFuncSetAttribute(qd_dirs_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dsm);
  while (chosen < count) {
    const int m = (count - chosen < r) ? (count - chosen) : r;
    int64_t* L = (guess && chunk < guess->max_chunks) ? guess->rows + (size_t)chunk * guess->r : Lloc;
    int g = (guess && chunk < guess->max_chunks) ? guess->g[chunk] : 0;
    if (g > m) g = m;
    const int n_ex = chosen;
    if (n_ex > 0) {
      sort_rows_kernel<<<1, 1, 0, ctx->stream>>>(out_idx, n_ex, ex);
      ADROM_LAUNCH_CK(ctx);
    }
    bool done = false;
    for (int pass = 0; pass < m + 8 && !done; ++pass) {
      ++iters;
      qd_dirs_kernel<<<1, 256, dsm, ctx->stream>>>(phi, r, L, g, D, tau);
      ADROM_LAUNCH_CK(ctx);
      const int m_eval = (g + 1 < m) ? g + 1 : m;
      const int pr = prof_begin(ctx, PROBE_QDEIM_SCAN);
      int grid;
      if (fast) {
        auto launch = [&](auto kern, int TM, int R) -> int {
          const size_t sm = sizeof(double) * ((size_t)TM * (R + 1) + (size_t)R * R) +
                            (sizeof(int64_t) + sizeof(int)) * R + 64;
          cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
          int64_t gg = (int64_t)ctx->num_sms * 2;
          const int64_t nt = (n + TM - 1) / TM;
          if (gg > nt) gg = nt;
          if (gg > nb) gg = nb;
          grid = (int)(gg < 1 ? 1 : gg);
          kern<<<grid, 256, sm, ctx->stream>>>(phi, n, D, m_eval, L, g, ex, n_ex, pv, pi);
          ADROM_LAUNCH_CK(ctx);
          return ADROM_OK;
        };
        int st2;
        if (r == 16) st2 = launch(qd_scan_kernel<16>, ScanCfg<16>::TM, 16);
        else if (r == 32) st2 = launch(qd_scan_kernel<32>, ScanCfg<32>::TM, 32);
        else if (r == 64) st2 = launch(qd_scan_kernel<64>, ScanCfg<64>::TM, 64);
        else st2 = launch(qd_scan_kernel<128>, ScanCfg<128>::TM, 128);
        if (st2) return st2;
      } else {
        int64_t gg = (n + 127) / 128;
        if (gg > nb) gg = nb;
        grid = (int)(gg < 1 ? 1 : gg);
        const size_t sm = sizeof(double) * r * r + (sizeof(int64_t) + sizeof(int)) * r + 64;
        qd_scan_generic_kernel<<<grid, 128, sm, ctx->stream>>>(phi, n, r, D, m_eval, L, g, ex, n_ex,
                                                               pv, pi);
        ADROM_LAUNCH_CK(ctx);
      }
      prof_end(ctx, pr);
      qd_reduce_kernel<<<m_eval, 256, 0, ctx->stream>>>(pv, pi, grid, r, bestv, besti);
      ADROM_LAUNCH_CK(ctx);
      qd_check_kernel<<<1, 1, 0, ctx->stream>>>(L, g, m, m_eval, bestv, besti, status, err_resid);
      ADROM_LAUNCH_CK(ctx);
      ADROM_CK(ctx, cudaMemcpyAsync(hstat, status, sizeof(int) * 4, cudaMemcpyDeviceToHost,
                                    ctx->stream));
      ADROM_CK(ctx, cudaMemcpyAsync(hres, err_resid, sizeof(double), cudaMemcpyDeviceToHost,
                                    ctx->stream));
      ADROM_CK(ctx, cudaStreamSynchronize(ctx->stream));
      if (hstat[2])
        return set_error(ctx, ADROM_ERR_SINGULAR,
                         "rank deficiency at pivot step %d (residual column norm %.3e)",
                         chosen + hstat[2] - 1, hres[0]);
      g = hstat[1];
      done = hstat[0] != 0;
    }
    if (!done) return set_error(ctx, ADROM_ERR_DENSE, "qdeim: verification did not settle");
    ADROM_CK(ctx, cudaMemcpyAsync(out_idx + chosen, L, sizeof(int64_t) * m,
                                  cudaMemcpyDeviceToDevice, ctx->stream));
    if (guess && chunk < guess->max_chunks) guess->g[chunk] = m;
    chosen += m;
    ++chunk;
  }
  if (iterations_out) *iterations_out = iters;
  return ADROM_OK;
}

// ---------------------------------------------------------------------------
// feature-guided sampling (sampling.py:117-159)
// ---------------------------------------------------------------------------
constexpr int FGS_MAX_CELLS = 8192;

// |gradient| of the feature field; feature: 0 = pressure-gradient,
// 1 = velocity-gradient (sampling.py:64-74, fom.py:200-201 / 279-282)
__device__ __forceinline__ double fgs_theta(const double* y, int64_t c, int kind, int nv,
                                            double gamma, int feature) {
  if (kind == ADROM_BURGERS) return y[c];
  const double m0 = y[3 * c], m1 = y[3 * c + 1], m2 = y[3 * c + 2];
  const double rho = np_max(m0, 1e-10);
  const double vel = m1 / rho;
  if (feature == 1) return vel;
  const double kin = (0.5 * rho) * (vel * vel);
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
  if (m.n_elem > FGS_MAX_CELLS)
    return set_error(ctx, ADROM_ERR_ARG, "fgs: %lld cells exceeds the one-block ranking limit %d",
                     (long long)m.n_elem, FGS_MAX_CELLS);
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
  plan_kernel_build<<<1, 1024, sm, ctx->stream>>>(m.n_elem, m.n_var, m.kind == ADROM_BURGERS, op,
                                                  n_s, flag);
  ADROM_LAUNCH_CK(ctx);
  return ADROM_OK;
}

// ---------------------------------------------------------------------------
// reduced operator: gathers (projection.py:72-80) + DEIM pinv (sampling.py:162-175)
// ---------------------------------------------------------------------------
__global__ void op_gather_kernel(DevOp op, const double* __restrict__ phi,
                                 const double* __restrict__ q_ref, const double* __restrict__ d,
                                 int n_s) {
  const int r = op.r;
  const int n_c = op.sizes[1];
  const int64_t total = (int64_t)(n_c + n_s) * (r + 1);
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int row = (int)(t / (r + 1)), col = (int)(t % (r + 1));
    if (row < n_c) {
      const int64_t g = op.closure[row];
      if (col < r) op.dinv_phi_c[(int64_t)row * r + col] = phi[g * r + col] / d[g];
      else op.q_ref_c[row] = q_ref[g];
    } else {
      const int j = row - n_c;
      const int64_t g = op.idx[j];
      if (col < r) op.phi_s[(int64_t)j * r + col] = phi[g * r + col];
      else op.d_s[j] = d[g];
    }
  }
}

__global__ void __launch_bounds__(1024) deim_pinv_kernel(DevOp op, int n_s, int* flag) {
  extern __shared__ double sm[];
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

int operator_fill(adrom_ctx* ctx, DevOp& op, const double* phi, const double* q_ref,
                  const double* d, int n_s, int* flag) {
  const int r = op.r;
  const int64_t total = (int64_t)(op.nc_cap + n_s) * (r + 1);
  int64_t g = (total + 255) / 256;
  if (g > ctx->num_sms * 8) g = ctx->num_sms * 8;
  op_gather_kernel<<<(int)g, 256, 0, ctx->stream>>>(op, phi, q_ref, d, n_s);
  ADROM_LAUNCH_CK(ctx);
  const size_t sm = sizeof(double) * ((size_t)r * (n_s | 1) + (size_t)r * (r | 1) + r) +
                    sizeof(int) * r + 64;
  if (sm > 220 * 1024)
    return set_error(ctx, ADROM_ERR_ARG, "deim pinv: %d x %d exceeds one block", n_s, r);
  cudaFuncSetAttribute(deim_pinv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  deim_pinv_kernel<<<1, 1024, sm, ctx->stream>>>(op, n_s, flag);
  ADROM_LAUNCH_CK(ctx);
  return ADROM_OK;
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
  const size_t sm = sizeof(double) * ((size_t)r * (n_s | 1) + (size_t)r * (r | 1) + r) +
                    sizeof(int) * r + 64;
  if (sm > 220 * 1024)
    return set_error(ctx, ADROM_ERR_ARG, "deim pinv: %d x %d exceeds one block", n_s, r);
  cudaFuncSetAttribute(deim_pinv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  deim_pinv_kernel<<<1, 1024, sm, ctx->stream>>>(op, n_s, flag);
  ADROM_LAUNCH_CK(ctx);
  return ADROM_OK;
}

}  // namespace adrom
