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
__device__ inline JacobiResult block_jacobi(double* A, int lda, int m, int n, double* V, int ldv,
                                            int max_sweeps, double tol, int* sh_flag) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
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
      for (int pr = warp; pr < ne / 2; pr += nw) {
        int a, b;
        if (pr == 0) {
          a = round;
          b = ne - 1;
        } else {
          a = (round + pr) % (ne - 1);
          b = (round - pr + ne - 1) % (ne - 1);
        }
        if (a >= n || b >= n) continue;
        if (a > b) {
          const int t = a;
          a = b;
          b = t;
        }
        double* ca = A + (size_t)a * lda;
        double* cb = A + (size_t)b * lda;
        double al = 0.0, be = 0.0, ga = 0.0;
        for (int i = lane; i < m; i += 32) {
          const double x = ca[i], y = cb[i];
          al += x * x;
          be += y * y;
          ga += x * y;
        }
        al = warp_sum(al);
        be = warp_sum(be);
        ga = warp_sum(ga);
        if (al == 0.0 || be == 0.0) continue;
        if (!(fabs(ga) > tol * sqrt(al) * sqrt(be))) continue;
        const double zeta = (be - al) / (2.0 * ga);
        const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
        const double c = 1.0 / sqrt(1.0 + t * t);
        const double s = c * t;
        for (int i = lane; i < m; i += 32) {
          const double x = ca[i], y = cb[i];
          ca[i] = c * x - s * y;
          cb[i] = s * x + c * y;
        }
        double* va = V + (size_t)a * ldv;
        double* vb = V + (size_t)b * ldv;
        for (int i = lane; i < n; i += 32) {
          const double x = va[i], y = vb[i];
          va[i] = c * x - s * y;
          vb[i] = s * x + c * y;
        }
        if (lane == 0) *sh_flag = 1;
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
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    int rank = 0;
    const double sj = s[j];
    for (int k = 0; k < n; ++k) {
      const double sk = s[k];
      if (sk > sj || (sk == sj && k < j)) ++rank;
    }
    order[rank] = j;
  }
  __syncthreads();
}

}  // namespace adrom
