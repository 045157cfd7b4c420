// One-block one-sided (Hestenes) Jacobi SVD on data resident in shared (or
// global) memory.  Used for the iSVD core matrix K ((r+1) x (r+1),
// tracking.py:175), the LSPG reduced Jacobian (projection.py:193-199) and
// the DEIM pseudo-inverse (sampling.py:168-175).
//
// Columns of A (m x n, column j at A + j*lda) are rotated pairwise in
// round-robin order until mutually orthogonal; the same rotations
// accumulate into V (n x n, column j at V + j*ldv, initialised to I here).
// On exit A = W = A_in V with orthogonal columns, so A_in = U S V^T with
// S_j = ||W_j||, U_j = W_j / S_j.  One-sided Jacobi attains high relative
// accuracy, at least the ||A|| eps accuracy of LAPACK gesdd.
#pragma once

#include "common.cuh"

namespace adrom {

struct JacobiResult {
  int sweeps;
  int converged;
};

// All threads of the block must call.  blockDim.x must be a multiple of 32.
// Each column pair of a round is handled by one half-warp (16 lanes), so up
// to blockDim/16 pairs rotate concurrently and a round costs one barrier.
__device__ __forceinline__ double hw_sum(double v) {
#pragma unroll
  for (int o = 8; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o, 16);
  return v;
}

template <int LP>
__device__ __forceinline__ double lp_sum(double v) {
#pragma unroll
  for (int o = LP / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o, LP);
  return v;
}

// LP lanes per column pair (a power of two <= 32): fewer lanes -> fewer
// warps per round and a cheaper barrier (the iSVD core uses 8).
template <int LP = 16>
__device__ inline JacobiResult block_jacobi(double* A, int lda, int m, int n, double* V, int ldv,
                                            int max_sweeps, double tol, int* sh_flag) {
  constexpr int LSH = (LP == 32) ? 5 : (LP == 16) ? 4 : (LP == 8) ? 3 : (LP == 4) ? 2 : 1;
  const int tid = threadIdx.x, hl = tid & (LP - 1), hw = tid >> LSH, nhw = blockDim.x >> LSH;
  if (V)  // V == nullptr: right rotations not accumulated
    for (int e = tid; e < n * n; e += blockDim.x) {
      const int c = e / n, rr = e - c * n;
      V[c * ldv + rr] = (c == rr) ? 1.0 : 0.0;
    }
  __syncthreads();
  const int ne = n + (n & 1);  // pad to even: index n (if odd) is a virtual zero column
  JacobiResult res{0, 0};
  if (n < 2) {
    res.converged = 1;
    return res;
  }
  for (int sweep = 0; sweep < max_sweeps; ++sweep) {
    if (tid == 0) *sh_flag = 0;
    __syncthreads();
    for (int round = 0; round < ne - 1; ++round) {
      // pb is warp-uniform so both half-warps run the same iterations (the
      // 16-wide shuffles below are issued with the full warp mask)
      constexpr int GPW = 32 / LP;  // pair groups per warp (loop stays warp-uniform)
      for (int pb = (hw & ~(GPW - 1)); pb < ne / 2; pb += nhw) {
        const int pr = pb + (hw & (GPW - 1));
        int a = 0, b = 0;
        if (pr == 0) {
          a = round;
          b = ne - 1;
        } else {
          a = (round + pr) % (ne - 1);
          b = (round - pr + ne - 1) % (ne - 1);
        }
        const bool live = (pr < ne / 2) && (a < n && b < n);
        if (a > b) {
          const int t = a;
          a = b;
          b = t;
        }
        double al = 0.0, be = 0.0, ga = 0.0;
        double* ca = A + (size_t)a * lda;
        double* cb = A + (size_t)b * lda;
        if (live) {
          for (int i = hl; i < m; i += LP) {
            const double x = ca[i], y = cb[i];
            al += x * x;
            be += y * y;
            ga += x * y;
          }
        }
        al = lp_sum<LP>(al);
        be = lp_sum<LP>(be);
        ga = lp_sum<LP>(ga);
        if (!live || al == 0.0 || be == 0.0) continue;
        if (!(fabs(ga) > tol * sqrt(al * be))) continue;
        const double zeta = (be - al) / (2.0 * ga);
        const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
        const double c = 1.0 / sqrt(1.0 + t * t);
        const double s = c * t;
        for (int i = hl; i < m; i += LP) {
          const double x = ca[i], y = cb[i];
          ca[i] = c * x - s * y;
          cb[i] = s * x + c * y;
        }
        if (V) {
          double* va = V + (size_t)a * ldv;
          double* vb = V + (size_t)b * ldv;
          for (int i = hl; i < n; i += LP) {
            const double x = va[i], y = vb[i];
            va[i] = c * x - s * y;
            vb[i] = s * x + c * y;
          }
        }
        if (hl == 0) *sh_flag = 1;
      }
      __syncthreads();
    }
    res.sweeps = sweep + 1;
    const int rotated = *sh_flag;
    __syncthreads();
    if (!rotated) {
      res.converged = 1;
      break;
    }
  }
  return res;
}

// Column norms of A -> s[n]; order[k] = index of the k-th largest
// (descending, ties to the lower index).  All threads call.
__device__ inline void column_norms_sorted(const double* A, int lda, int m, int n, double* s,
                                           int* order) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int j = warp; j < n; j += nw) {
    double a = 0.0;
    for (int i = lane; i < m; i += 32) a += A[(size_t)j * lda + i] * A[(size_t)j * lda + i];
    a = warp_sum(a);
    if (lane == 0) s[j] = sqrt(a);
  }
  __syncthreads();
  // total order (NaN sorts last) so `order` is always a permutation
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    int rank = 0;
    const double sj = isnan(s[j]) ? -1.0 : s[j];
    for (int k = 0; k < n; ++k) {
      const double sk = isnan(s[k]) ? -1.0 : s[k];
      if (sk > sj || (sk == sj && k < j)) ++rank;
    }
    order[rank] = j;
  }
  __syncthreads();
}

}  // namespace adrom
