// Partitioned block-tridiagonal solver for the backward-Euler Newton systems.
//
// The reference factors the dense N x N matrix I - dt J with LAPACK getrf
// (dense.py:162).  That matrix is block tridiagonal (cyclic for the
// periodic Burgers grid, open chain for Sod's clamped ghosts), so here it is
// solved in O(N) with a recursive partition method:
//
//   level l: rows are cut into partitions of M rows.  Inside partition p
//   the M-1 interior rows are eliminated (block Thomas, partial pivoting
//   inside the nv x nv diagonal blocks) as affine functions of the two
//   "interface" unknowns that bound them — X_{p-1} (last row of the left
//   partition) and X_p (own last row):  x_i = y_i + V_i X_{p-1} + W_i X_p.
//   Substituting into the interface rows gives a block-tridiagonal system
//   of P = ceil(n/M) rows with the same cyclic structure; recurse until a
//   single partition remains, then back-substitute level by level.
//
// Rounding differs from LU with row pivoting at the 1e-16 level; the Newton
// iterate and iteration count are compared with the reference in
// tests/test_gpu_fom.py.
#include "btsolve.cuh"

#include <stdlib.h>

namespace adrom {

constexpr int BT_M = 16;  // rows per partition

template <int NV>
struct Blk {
  double a[NV][NV];
};

template <int NV>
__device__ __forceinline__ void load_blk(const double* p, Blk<NV>& b) {
#pragma unroll
  for (int i = 0; i < NV; ++i)
#pragma unroll
    for (int j = 0; j < NV; ++j) b.a[i][j] = p[i * NV + j];
}
template <int NV>
__device__ __forceinline__ void store_blk(double* p, const Blk<NV>& b) {
#pragma unroll
  for (int i = 0; i < NV; ++i)
#pragma unroll
    for (int j = 0; j < NV; ++j) p[i * NV + j] = b.a[i][j];
}
template <int NV>
__device__ __forceinline__ void zero_blk(Blk<NV>& b) {
#pragma unroll
  for (int i = 0; i < NV; ++i)
#pragma unroll
    for (int j = 0; j < NV; ++j) b.a[i][j] = 0.0;
}
// c = a * b
template <int NV>
__device__ __forceinline__ void mm(const Blk<NV>& a, const Blk<NV>& b, Blk<NV>& c) {
#pragma unroll
  for (int i = 0; i < NV; ++i)
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      double s = 0.0;
#pragma unroll
      for (int k = 0; k < NV; ++k) s += a.a[i][k] * b.a[k][j];
      c.a[i][j] = s;
    }
}
// y = a * x
template <int NV>
__device__ __forceinline__ void mv(const Blk<NV>& a, const double* x, double* y) {
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < NV; ++k) s += a.a[i][k] * x[k];
    y[i] = s;
  }
}

// in-place LU with partial pivoting of a small block; false on zero pivot
template <int NV>
__device__ __forceinline__ bool lu(Blk<NV>& A, int* piv) {
  bool ok = true;
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    int p = k;
    double best = fabs(A.a[k][k]);
#pragma unroll
    for (int i = k + 1; i < NV; ++i)
      if (fabs(A.a[i][k]) > best) {
        best = fabs(A.a[i][k]);
        p = i;
      }
    piv[k] = p;
    if (p != k) {
#pragma unroll
      for (int j = 0; j < NV; ++j) {
        const double t = A.a[k][j];
        A.a[k][j] = A.a[p][j];
        A.a[p][j] = t;
      }
    }
    const double d = A.a[k][k];
    if (d == 0.0 || !isfinite(d)) ok = false;
    const double inv = 1.0 / d;
#pragma unroll
    for (int i = k + 1; i < NV; ++i) {
      A.a[i][k] *= inv;
#pragma unroll
      for (int j = k + 1; j < NV; ++j) A.a[i][j] -= A.a[i][k] * A.a[k][j];
    }
  }
  return ok;
}
template <int NV>
__device__ __forceinline__ void lu_solve(const Blk<NV>& A, const int* piv, double* x) {
#pragma unroll
  for (int k = 0; k < NV; ++k)
    if (piv[k] != k) {
      const double t = x[k];
      x[k] = x[piv[k]];
      x[piv[k]] = t;
    }
#pragma unroll
  for (int i = 1; i < NV; ++i)
#pragma unroll
    for (int k = 0; k < i; ++k) x[i] -= A.a[i][k] * x[k];
#pragma unroll
  for (int i = NV - 1; i >= 0; --i) {
#pragma unroll
    for (int k = i + 1; k < NV; ++k) x[i] -= A.a[i][k] * x[k];
    x[i] /= A.a[i][i];
  }
}
// B <- A^{-1} B  (column by column)
template <int NV>
__device__ __forceinline__ void lu_solve_blk(const Blk<NV>& A, const int* piv, Blk<NV>& B) {
#pragma unroll
  for (int j = 0; j < NV; ++j) {
    double c[NV];
#pragma unroll
    for (int i = 0; i < NV; ++i) c[i] = B.a[i][j];
    lu_solve<NV>(A, piv, c);
#pragma unroll
    for (int i = 0; i < NV; ++i) B.a[i][j] = c[i];
  }
}

// ---------------------------------------------------------------------------
// per-partition elimination of the interior rows
// ---------------------------------------------------------------------------
template <int NV>
__global__ void part_solve_kernel(const double* __restrict__ sys, const double* __restrict__ rhs,
                                  double sign, int64_t n, double* __restrict__ Y,
                                  double* __restrict__ V, double* __restrict__ W,
                                  double* __restrict__ G, int* __restrict__ flag) {
  constexpr int NV2 = NV * NV;
  const int64_t P = (n + BT_M - 1) / BT_M;
  const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= P) return;
  const int64_t s = p * BT_M;
  const int64_t e = ((s + BT_M < n) ? s + BT_M : n) - 1;
  if (e == s) return;
  double cb[NV];
  Blk<NV> cV, Gp, cW;
  bool ok = true;
  zero_blk<NV>(Gp);
  zero_blk<NV>(cW);
  for (int64_t i = s; i < e; ++i) {
    Blk<NV> L, D, U;
    load_blk<NV>(sys + (i * 3 + 0) * NV2, L);
    load_blk<NV>(sys + (i * 3 + 1) * NV2, D);
    load_blk<NV>(sys + (i * 3 + 2) * NV2, U);
    double b[NV];
#pragma unroll
    for (int a = 0; a < NV; ++a) b[a] = sign * rhs[i * NV + a];
    Blk<NV> fV;
    if (i > s) {
      Blk<NV> LG;
      mm<NV>(L, Gp, LG);
#pragma unroll
      for (int a = 0; a < NV; ++a)
#pragma unroll
        for (int c = 0; c < NV; ++c) D.a[a][c] -= LG.a[a][c];
      double Lc[NV];
      mv<NV>(L, cb, Lc);
#pragma unroll
      for (int a = 0; a < NV; ++a) b[a] -= Lc[a];
      Blk<NV> LV;
      mm<NV>(L, cV, LV);
#pragma unroll
      for (int a = 0; a < NV; ++a)
#pragma unroll
        for (int c = 0; c < NV; ++c) fV.a[a][c] = -LV.a[a][c];
    } else {
#pragma unroll
      for (int a = 0; a < NV; ++a)
#pragma unroll
        for (int c = 0; c < NV; ++c) fV.a[a][c] = -L.a[a][c];
    }
    int piv[NV];
    ok &= lu<NV>(D, piv);
    lu_solve<NV>(D, piv, b);
    lu_solve_blk<NV>(D, piv, fV);
#pragma unroll
    for (int a = 0; a < NV; ++a) cb[a] = b[a];
    cV = fV;
    if (i < e - 1) {
      lu_solve_blk<NV>(D, piv, U);
      Gp = U;
    } else {
#pragma unroll
      for (int a = 0; a < NV; ++a)
#pragma unroll
        for (int c = 0; c < NV; ++c) cW.a[a][c] = -U.a[a][c];
      lu_solve_blk<NV>(D, piv, cW);
      zero_blk<NV>(Gp);
    }
#pragma unroll
    for (int a = 0; a < NV; ++a) Y[i * NV + a] = cb[a];
    store_blk<NV>(V + i * NV2, cV);
    store_blk<NV>(G + i * NV2, Gp);
  }
  // backward sweep: z_i = c_i - G_i z_{i+1};  W has no forward part
  double yn[NV];
  Blk<NV> Vn, Wn;
#pragma unroll
  for (int a = 0; a < NV; ++a) yn[a] = cb[a];
  Vn = cV;
  Wn = cW;
  store_blk<NV>(W + (e - 1) * NV2, Wn);
  for (int64_t i = e - 2; i >= s; --i) {
    Blk<NV> Gi, Vi;
    load_blk<NV>(G + i * NV2, Gi);
    load_blk<NV>(V + i * NV2, Vi);
    double yi[NV], t[NV];
#pragma unroll
    for (int a = 0; a < NV; ++a) yi[a] = Y[i * NV + a];
    mv<NV>(Gi, yn, t);
#pragma unroll
    for (int a = 0; a < NV; ++a) yn[a] = yi[a] - t[a];
    Blk<NV> GV, GW;
    mm<NV>(Gi, Vn, GV);
    mm<NV>(Gi, Wn, GW);
#pragma unroll
    for (int a = 0; a < NV; ++a)
#pragma unroll
      for (int c = 0; c < NV; ++c) {
        Vn.a[a][c] = Vi.a[a][c] - GV.a[a][c];
        Wn.a[a][c] = -GW.a[a][c];
      }
#pragma unroll
    for (int a = 0; a < NV; ++a) Y[i * NV + a] = yn[a];
    store_blk<NV>(V + i * NV2, Vn);
    store_blk<NV>(W + i * NV2, Wn);
  }
  if (!ok) atomicOr(flag, 2);
}


// ---------------------------------------------------------------------------
// wide blocks (n_var = 13, configuration 4): one half-warp per partition,
// lane a owns row a of every nv x nv block (registers), rows are broadcast
// by shuffles.  The same elimination as part_solve_kernel (block Thomas with
// partial pivoting inside the diagonal blocks); the triangular solves are
// column-oriented, so rounding differs from the thread-per-partition form at
// the 1e-16 level (the Newton tests compare against the oracle's sparse LU).
// ---------------------------------------------------------------------------
template <int NV>
struct HW {
  unsigned mask;
  int lane;  // 0..15 within the half-warp
  __device__ __forceinline__ double bc(double v, int src) const {
    return __shfl_sync(mask, v, src, 16);
  }
};

// c_row = a_row * B (B row-distributed)
template <int NV>
__device__ __forceinline__ void hw_mm(const HW<NV>& h, const double* a, const double* b, double* c) {
#pragma unroll
  for (int j = 0; j < NV; ++j) c[j] = 0.0;
#pragma unroll
  for (int k = 0; k < NV; ++k) {
#pragma unroll
    for (int j = 0; j < NV; ++j) c[j] += a[k] * h.bc(b[j], k);
  }
}
// y_row = a_row . x (x distributed: x[k] in lane k)
template <int NV>
__device__ __forceinline__ double hw_mv(const HW<NV>& h, const double* a, double x) {
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < NV; ++k) s += a[k] * h.bc(x, k);
  return s;
}
// in-place LU with partial pivoting (rows physically swapped between lanes);
// perm[k] = pivot row of step k (all lanes)
template <int NV>
__device__ __forceinline__ bool hw_lu(const HW<NV>& h, double* A, int* perm) {
  bool ok = true;
  const int a = h.lane;
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    // argmax_{i >= k} |A[i][k]|, lowest row on ties (strict >, as lu())
    double best = (a >= k && a < NV) ? fabs(A[k]) : -1.0;
    int p = a;
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) {
      const double ob = __shfl_xor_sync(h.mask, best, o, 16);
      const int op = __shfl_xor_sync(h.mask, p, o, 16);
      if (ob > best || (ob == best && op < p)) {
        best = ob;
        p = op;
      }
    }
    perm[k] = p;
    if (p != k) {
#pragma unroll
      for (int j = 0; j < NV; ++j) {
        const double vk = h.bc(A[j], k), vp = h.bc(A[j], p);
        if (a == k) A[j] = vp;
        if (a == p) A[j] = vk;
      }
    }
    const double d = h.bc(A[k], k);
    if (d == 0.0 || !isfinite(d)) ok = false;
    const double inv = 1.0 / d;
    if (a > k) A[k] *= inv;
    const double lik = A[k];
#pragma unroll
    for (int j = k + 1; j < NV; ++j) {
      const double akj = h.bc(A[j], k);
      if (a > k) A[j] -= lik * akj;
    }
  }
  return ok;
}
// x <- A^{-1} x for x distributed (x[a] in lane a)
template <int NV>
__device__ __forceinline__ double hw_solve(const HW<NV>& h, const double* A, const int* perm, double x) {
  const int a = h.lane;
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    const int p = perm[k];
    if (p != k) {
      const double xk = h.bc(x, k), xp = h.bc(x, p);
      if (a == k) x = xp;
      if (a == p) x = xk;
    }
  }
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    const double xk = h.bc(x, k);
    if (a > k) x -= A[k] * xk;
  }
#pragma unroll
  for (int i = NV - 1; i >= 0; --i) {
    if (a == i) x /= A[i];
    const double xi = h.bc(x, i);
    if (a < i) x -= A[i] * xi;
  }
  return x;
}
// B <- A^{-1} B, B row-distributed
template <int NV>
__device__ __forceinline__ void hw_solve_blk(const HW<NV>& h, const double* A, const int* perm, double* B) {
  const int a = h.lane;
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    const int p = perm[k];
    if (p != k) {
#pragma unroll
      for (int j = 0; j < NV; ++j) {
        const double vk = h.bc(B[j], k), vp = h.bc(B[j], p);
        if (a == k) B[j] = vp;
        if (a == p) B[j] = vk;
      }
    }
  }
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    const double lak = A[k];
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      const double bkj = h.bc(B[j], k);
      if (a > k) B[j] -= lak * bkj;
    }
  }
#pragma unroll
  for (int i = NV - 1; i >= 0; --i) {
    if (a == i) {
      const double dii = A[i];
#pragma unroll
      for (int j = 0; j < NV; ++j) B[j] /= dii;
    }
    const double ai = A[i];
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      const double bij = h.bc(B[j], i);
      if (a < i) B[j] -= ai * bij;
    }
  }
}

template <int NV>
__global__ void __launch_bounds__(128) part_solve_hw_kernel(
    const double* __restrict__ sys, const double* __restrict__ rhs, double sign, int64_t n,
    double* __restrict__ Y, double* __restrict__ V, double* __restrict__ W,
    double* __restrict__ G, int* __restrict__ flag) {
  constexpr int NV2 = NV * NV;
  const int64_t P = (n + BT_M - 1) / BT_M;
  const int64_t gt = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t p = gt >> 4;
  HW<NV> h;
  h.lane = threadIdx.x & 15;
  h.mask = 0xFFFFu << (threadIdx.x & 16);
  if (p >= P) return;  // uniform per half-warp
  const int64_t s = p * BT_M;
  const int64_t e = ((s + BT_M < n) ? s + BT_M : n) - 1;
  if (e == s) return;
  const int a = h.lane;
  const bool row = a < NV;
  const int ar = row ? a : 0;
  double cb = 0.0;
  double cV[NV], Gp[NV], cW[NV];
#pragma unroll
  for (int j = 0; j < NV; ++j) {
    Gp[j] = 0.0;
    cW[j] = 0.0;
    cV[j] = 0.0;
  }
  bool ok = true;
  for (int64_t i = s; i < e; ++i) {
    double L[NV], D[NV], U[NV];
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      L[j] = row ? sys[(i * 3 + 0) * NV2 + ar * NV + j] : 0.0;
      D[j] = row ? sys[(i * 3 + 1) * NV2 + ar * NV + j] : 0.0;
      U[j] = row ? sys[(i * 3 + 2) * NV2 + ar * NV + j] : 0.0;
    }
    double b = row ? sign * rhs[i * NV + ar] : 0.0;
    double fV[NV];
    if (i > s) {
      double LG[NV];
      hw_mm<NV>(h, L, Gp, LG);
#pragma unroll
      for (int c = 0; c < NV; ++c) D[c] -= LG[c];
      b -= hw_mv<NV>(h, L, cb);
      double LV[NV];
      hw_mm<NV>(h, L, cV, LV);
#pragma unroll
      for (int c = 0; c < NV; ++c) fV[c] = -LV[c];
    } else {
#pragma unroll
      for (int c = 0; c < NV; ++c) fV[c] = -L[c];
    }
    if (!row) {
#pragma unroll
      for (int c = 0; c < NV; ++c) D[c] = 0.0;
    }
    int perm[NV];
    ok &= hw_lu<NV>(h, D, perm);
    b = hw_solve<NV>(h, D, perm, b);
    hw_solve_blk<NV>(h, D, perm, fV);
    cb = b;
#pragma unroll
    for (int c = 0; c < NV; ++c) cV[c] = fV[c];
    if (i < e - 1) {
      hw_solve_blk<NV>(h, D, perm, U);
#pragma unroll
      for (int c = 0; c < NV; ++c) Gp[c] = U[c];
    } else {
#pragma unroll
      for (int c = 0; c < NV; ++c) cW[c] = -U[c];
      hw_solve_blk<NV>(h, D, perm, cW);
#pragma unroll
      for (int c = 0; c < NV; ++c) Gp[c] = 0.0;
    }
    if (row) {
      Y[i * NV + a] = cb;
#pragma unroll
      for (int c = 0; c < NV; ++c) {
        V[i * NV2 + a * NV + c] = cV[c];
        G[i * NV2 + a * NV + c] = Gp[c];
      }
    }
  }
  // backward sweep: z_i = c_i - G_i z_{i+1}
  double yn = cb;
  double Vn[NV], Wn[NV];
#pragma unroll
  for (int c = 0; c < NV; ++c) {
    Vn[c] = cV[c];
    Wn[c] = cW[c];
  }
  if (row)
#pragma unroll
    for (int c = 0; c < NV; ++c) W[(e - 1) * NV2 + a * NV + c] = Wn[c];
  for (int64_t i = e - 2; i >= s; --i) {
    double Gi[NV], Vi[NV];
#pragma unroll
    for (int c = 0; c < NV; ++c) {
      Gi[c] = row ? G[i * NV2 + a * NV + c] : 0.0;
      Vi[c] = row ? V[i * NV2 + a * NV + c] : 0.0;
    }
    const double yi = row ? Y[i * NV + a] : 0.0;
    yn = yi - hw_mv<NV>(h, Gi, yn);
    double GV[NV], GW[NV];
    hw_mm<NV>(h, Gi, Vn, GV);
    hw_mm<NV>(h, Gi, Wn, GW);
#pragma unroll
    for (int c = 0; c < NV; ++c) {
      Vn[c] = Vi[c] - GV[c];
      Wn[c] = -GW[c];
    }
    if (row) {
      Y[i * NV + a] = yn;
#pragma unroll
      for (int c = 0; c < NV; ++c) {
        V[i * NV2 + a * NV + c] = Vn[c];
        W[i * NV2 + a * NV + c] = Wn[c];
      }
    }
  }
  if (!ok && a == 0) atomicOr(flag, 2);
}


// ---------------------------------------------------------------------------
// wide blocks (n_var = 13, configuration 4), tensor-core form: one warp per
// partition, every nv x nv block padded to a 16 x 16 shared-memory tile.
// The block products (L G, L V for the forward sweep, G V and G W for the
// backward one) run on the FP64 tensor cores (DMMA m8n8k4, 16 per product);
// the diagonal block is eliminated by Gauss-Jordan with partial pivoting on
// the augmented [D' | b | -L V | U] with one column per lane (row swaps stay
// in registers, one pivot column broadcast per step).  Rounding differs from
// the thread-per-partition LU at the 1e-16 level.
// ---------------------------------------------------------------------------
constexpr int TC_LD = 20;   // tile leading dimension: conflict-free DMMA fragments
constexpr int TC_TILE = 16 * TC_LD;
constexpr int TC_WARPS = 4;
constexpr int TC_TILES = 7;  // L, D, U, F, V, G, W
__device__ __forceinline__ void dmma884_bt(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}
// C = Cin + alpha A B (16 x 16 tiles, zero padding beyond nv); Cin may alias C
__device__ __forceinline__ void tc_mm(const double* A, const double* B, double* C,
                                      const double* Cin, double alpha, int lane) {
  const int r = lane >> 2, k = lane & 3;
#pragma unroll
  for (int ti = 0; ti < 2; ++ti)
#pragma unroll
    for (int tj = 0; tj < 2; ++tj) {
      double d0 = 0.0, d1 = 0.0;
#pragma unroll
      for (int kk = 0; kk < 4; ++kk)
        dmma884_bt(d0, d1, A[(ti * 8 + r) * TC_LD + kk * 4 + k], B[(kk * 4 + k) * TC_LD + tj * 8 + r]);
      const int row = ti * 8 + r, col = tj * 8 + 2 * k;
      const double c0 = Cin ? Cin[row * TC_LD + col] : 0.0;
      const double c1 = Cin ? Cin[row * TC_LD + col + 1] : 0.0;
      C[row * TC_LD + col] = c0 + alpha * d0;
      C[row * TC_LD + col + 1] = c1 + alpha * d1;
    }
}

// one Gauss-Jordan step on lane-held columns (column K's owner is lane K);
// recursive template so every register index is a compile-time constant
template <int NV, int K>
__device__ __forceinline__ void gj_step(double (&x1)[NV], double (&x2)[NV], bool& ok) {
  int pr = K;
  {
    double best = fabs(x1[K]);
#pragma unroll
    for (int r = K + 1; r < NV; ++r)
      if (fabs(x1[r]) > best) {
        best = fabs(x1[r]);
        pr = r;
      }
  }
  pr = __shfl_sync(0xffffffffu, pr, K);
  if (pr != K) {
    double b1 = 0.0, b2 = 0.0;
#pragma unroll
    for (int r = K + 1; r < NV; ++r)
      if (r == pr) {
        b1 = x1[r];
        b2 = x2[r];
      }
#pragma unroll
    for (int r = K + 1; r < NV; ++r)
      if (r == pr) {
        x1[r] = x1[K];
        x2[r] = x2[K];
      }
    x1[K] = b1;
    x2[K] = b2;
  }
  const double d = __shfl_sync(0xffffffffu, x1[K], K);
  if (d == 0.0 || !isfinite(d)) ok = false;
  const double inv = 1.0 / d;
  const double p1 = x1[K] * inv, p2 = x2[K] * inv;
  x1[K] = p1;
  x2[K] = p2;
#pragma unroll
  for (int r = 0; r < NV; ++r) {
    if (r == K) continue;
    const double m = __shfl_sync(0xffffffffu, x1[r], K);
    x1[r] -= m * p1;
    x2[r] -= m * p2;
  }
  if constexpr (K + 1 < NV) gj_step<NV, K + 1>(x1, x2, ok);
}

template <int NV>
__global__ void __launch_bounds__(32 * TC_WARPS, 3) part_solve_tc_kernel(
    const double* __restrict__ sys, const double* __restrict__ rhs, double sign, int64_t n,
    double* __restrict__ Y, double* __restrict__ V, double* __restrict__ W,
    double* __restrict__ G, int* __restrict__ flag) {
  static_assert(NV <= 16 && 3 * NV <= 64, "tile size");
  constexpr int NV2 = NV * NV;
  extern __shared__ __align__(16) double tsm[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double* base = tsm + (size_t)wid * (TC_TILES * TC_TILE + 64);
  double* tL = base;
  double* tD = tL + TC_TILE;
  double* tU = tD + TC_TILE;
  double* tF = tU + TC_TILE;
  double* tV = tF + TC_TILE;
  double* tG = tV + TC_TILE;
  double* tW = tG + TC_TILE;
  double* vb = tW + TC_TILE;  // 32: b / y
  double* vc = vb + 32;       // 32: c_b / y_n
  const int64_t P = (n + BT_M - 1) / BT_M;
  const int64_t p = blockIdx.x * (int64_t)TC_WARPS + wid;
  if (p >= P) return;
  const int64_t s = p * BT_M;
  const int64_t e = ((s + BT_M < n) ? s + BT_M : n) - 1;
  if (e == s) return;
  for (int i = lane; i < TC_TILES * TC_TILE + 64; i += 32) base[i] = 0.0;
  __syncwarp();
  bool ok = true;
  // augmented column j of lane: j = lane (0..31) and j2 = 32 + lane (lanes < 8)
  // columns: [0, NV) D', NV b, [NV+1, 2NV+1) F = -L V, [2NV+1, 3NV+1) U
  constexpr int NA = 3 * NV + 1;
  auto colval = [&](int j, int i) -> double {
    if (j < NV) return tD[i * TC_LD + j];
    if (j == NV) return vb[i];
    if (j < 2 * NV + 1) return tF[i * TC_LD + (j - NV - 1)];
    if (j < NA) return tU[i * TC_LD + (j - 2 * NV - 1)];
    return 0.0;
  };
  // row i's L, D, U and b are prefetched into registers while row i-1 is
  // eliminated (PF values per lane), then scattered into the tiles
  constexpr int PF = (3 * NV2 + 31) / 32;
  double pre[PF];
  double preb = 0.0;
  auto fetch = [&](int64_t i) {
    const double* src = sys + i * 3 * NV2;
#pragma unroll
    for (int m = 0; m < PF; ++m) {
      const int t = lane + 32 * m;
      pre[m] = (t < 3 * NV2) ? src[t] : 0.0;
    }
    preb = (lane < NV) ? sign * rhs[i * NV + lane] : 0.0;
  };
  fetch(s);
  for (int64_t i = s; i < e; ++i) {
    // stage L, D, U (rows of NV, contiguous in sys) and b
#pragma unroll
    for (int m = 0; m < PF; ++m) {
      const int t = lane + 32 * m;
      if (t < 3 * NV2) {
        const int blk = t / NV2, rem = t - blk * NV2, rr = rem / NV, cc = rem - rr * NV;
        (blk == 0 ? tL : blk == 1 ? tD : tU)[rr * TC_LD + cc] = pre[m];
      }
    }
    if (lane < NV) vb[lane] = preb;
    if (i + 1 < e) fetch(i + 1);
    __syncwarp();
    if (i > s) {
      tc_mm(tL, tG, tD, tD, -1.0, lane);   // D' = D - L G
      tc_mm(tL, tV, tF, nullptr, -1.0, lane);  // F = -L V
      if (lane < NV) {
        double acc = 0.0;
#pragma unroll
        for (int k = 0; k < NV; ++k) acc += tL[lane * TC_LD + k] * vc[k];
        vb[lane] -= acc;  // b' = b - L c_b
      }
    } else {
      for (int t = lane; t < NV2; t += 32) {
        const int rr = t / NV, cc = t - rr * NV;
        tF[rr * TC_LD + cc] = -tL[rr * TC_LD + cc];
      }
    }
    __syncwarp();
    // Gauss-Jordan on the augmented columns (one or two per lane)
    double x1[NV], x2[NV];
#pragma unroll
    for (int r = 0; r < NV; ++r) {
      x1[r] = colval(lane, r);
      x2[r] = (lane + 32 < NA) ? colval(lane + 32, r) : 0.0;
    }
    gj_step<NV, 0>(x1, x2, ok);
    // lanes' solved columns -> c_b, V (= D'^-1 F), G (= D'^-1 U) or W (last row)
    __syncwarp();
    const bool last = (i == e - 1);
#define ADROM_BT_PUT(j, x)                                                                  \
  do {                                                                                      \
    if ((j) == NV) {                                                                        \
      _Pragma("unroll") for (int r = 0; r < NV; ++r) vc[r] = x[r];                          \
    } else if ((j) > NV && (j) < 2 * NV + 1) {                                              \
      _Pragma("unroll") for (int r = 0; r < NV; ++r) tV[r * TC_LD + ((j) - NV - 1)] = x[r]; \
    } else if ((j) >= 2 * NV + 1 && (j) < NA) {                                             \
      double* t_ = last ? tW : tG;                                                          \
      const double sg_ = last ? -1.0 : 1.0;                                                 \
      _Pragma("unroll") for (int r = 0; r < NV; ++r) t_[r * TC_LD + ((j) - 2 * NV - 1)] =   \
          sg_ * x[r];                                                                       \
    }                                                                                       \
  } while (0)
    ADROM_BT_PUT(lane, x1);
    if (lane + 32 < NA) ADROM_BT_PUT(lane + 32, x2);
#undef ADROM_BT_PUT
    __syncwarp();
    if (last)
      for (int t = lane; t < NV2; t += 32) tG[(t / NV) * TC_LD + (t % NV)] = 0.0;
    __syncwarp();
    if (lane < NV) Y[i * NV + lane] = vc[lane];
    for (int t = lane; t < NV2; t += 32) {
      const int rr = t / NV, cc = t - rr * NV;
      V[i * NV2 + t] = tV[rr * TC_LD + cc];
      G[i * NV2 + t] = tG[rr * TC_LD + cc];
    }
    __syncwarp();
  }
  // backward sweep: y_i = c_i - G_i y_{i+1}, V_i -= G_i V_{i+1}, W_i = -G_i W_{i+1}
  for (int t = lane; t < NV2; t += 32) W[(e - 1) * NV2 + t] = tW[(t / NV) * TC_LD + (t % NV)];
  double* cV = tV;
  double* cW = tW;
  double* nV = tF;
  double* nW = tU;
  constexpr int PB = (NV2 + 31) / 32;
  double pg[PB], pv[PB], py = 0.0;
  auto fetch_b = [&](int64_t i) {
#pragma unroll
    for (int m = 0; m < PB; ++m) {
      const int t = lane + 32 * m;
      pg[m] = (t < NV2) ? G[i * NV2 + t] : 0.0;
      pv[m] = (t < NV2) ? V[i * NV2 + t] : 0.0;
    }
    py = (lane < NV) ? Y[i * NV + lane] : 0.0;
  };
  if (e - 2 >= s) fetch_b(e - 2);
  for (int64_t i = e - 2; i >= s; --i) {
#pragma unroll
    for (int m = 0; m < PB; ++m) {
      const int t = lane + 32 * m;
      if (t < NV2) {
        const int rr = t / NV, cc = t - rr * NV;
        tL[rr * TC_LD + cc] = pg[m];  // G_i
        tD[rr * TC_LD + cc] = pv[m];  // V_i
      }
    }
    if (lane < NV) vb[lane] = py;
    if (i - 1 >= s) fetch_b(i - 1);
    __syncwarp();
    double yv = 0.0;
    if (lane < NV) {
      double acc = 0.0;
#pragma unroll
      for (int k = 0; k < NV; ++k) acc += tL[lane * TC_LD + k] * vc[k];
      yv = vb[lane] - acc;
    }
    tc_mm(tL, cV, nV, tD, -1.0, lane);
    tc_mm(tL, cW, nW, nullptr, -1.0, lane);
    __syncwarp();
    if (lane < NV) vc[lane] = yv;
    double* t1 = cV;
    cV = nV;
    nV = t1;
    t1 = cW;
    cW = nW;
    nW = t1;
    __syncwarp();
    if (lane < NV) Y[i * NV + lane] = vc[lane];
    for (int t = lane; t < NV2; t += 32) {
      const int rr = t / NV, cc = t - rr * NV;
      V[i * NV2 + t] = cV[rr * TC_LD + cc];
      W[i * NV2 + t] = cW[rr * TC_LD + cc];
    }
    __syncwarp();
  }
  if (!ok && lane == 0) atomicOr(flag, 2);
}

// ---------------------------------------------------------------------------
// scalar (n_var = 1) partitions: the same elimination, staged through smem so
// that global traffic is coalesced.  A warp owns 32 consecutive partitions
// (1024 rows); lane p walks partition p in smem (stride 33: conflict-free).
// G lives in D's slot, the outputs Y / V / W overwrite rhs / L / U.
// ---------------------------------------------------------------------------
constexpr int PS_WARPS = 4;
constexpr int PS_LD = BT_M + 1;

__global__ void __launch_bounds__(32 * PS_WARPS) part_solve_scalar_kernel(
    const double* __restrict__ sys, const double* __restrict__ rhs, double sign, int64_t n,
    double* __restrict__ Y, double* __restrict__ V, double* __restrict__ W, int* __restrict__ flag) {
  extern __shared__ double sm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double* sL = sm + (size_t)warp * 4 * 32 * PS_LD;
  double* sD = sL + 32 * PS_LD;
  double* sU = sD + 32 * PS_LD;
  double* sB = sU + 32 * PS_LD;
  const int64_t P = (n + BT_M - 1) / BT_M;
  const int64_t groups = (P + 31) / 32;
  bool ok = true;
  for (int64_t gidx = (int64_t)blockIdx.x * PS_WARPS + warp; gidx < groups;
       gidx += (int64_t)gridDim.x * PS_WARPS) {
    const int64_t row0 = gidx * 32 * BT_M;
    const int rows = (int)((n - row0 < 32 * BT_M) ? (n - row0) : 32 * BT_M);
    __syncwarp();
    for (int j = lane; j < rows; j += 32) {
      const int pp = j / BT_M, ii = j - pp * BT_M, o = pp * PS_LD + ii;
      const int64_t gi = row0 + j;
      sL[o] = sys[gi * 3 + 0];
      sD[o] = sys[gi * 3 + 1];
      sU[o] = sys[gi * 3 + 2];
      sB[o] = sign * rhs[gi];
    }
    __syncwarp();
    // lane = partition within the group
    const int64_t s = row0 + (int64_t)lane * BT_M;
    const int m = (s < n) ? (int)(((s + BT_M < n) ? s + BT_M : n) - s) : 0;  // rows in it
    const int base = lane * PS_LD;
    if (m > 1) {
      const int last = m - 1;  // local index of the interface row e
      double cb = 0.0, cV = 0.0, Gp = 0.0, cW = 0.0;
      for (int i = 0; i < last; ++i) {
        const double L = sL[base + i];
        double D = sD[base + i];
        const double U = sU[base + i];
        double b = sB[base + i];
        double fV;
        if (i > 0) {
          D -= L * Gp;
          b -= L * cb;
          fV = -(L * cV);
        } else {
          fV = -L;
        }
        if (D == 0.0 || !isfinite(D)) ok = false;
        // lu<1> / lu_solve<1>: multiply by the reciprocal pivot, then divide
        b /= D;
        fV /= D;
        cb = b;
        cV = fV;
        if (i < last - 1) {
          Gp = U / D;
        } else {
          cW = (-U) / D;
          Gp = 0.0;
        }
        sB[base + i] = cb;
        sL[base + i] = cV;
        sD[base + i] = Gp;
      }
      // backward sweep (as part_solve_kernel)
      double yn = cb, Vn = cV, Wn = cW;
      sU[base + last - 1] = Wn;
      for (int i = last - 2; i >= 0; --i) {
        const double Gi = sD[base + i];
        yn = sB[base + i] - Gi * yn;
        Vn = sL[base + i] - Gi * Vn;
        Wn = -(Gi * Wn);
        sB[base + i] = yn;
        sL[base + i] = Vn;
        sU[base + i] = Wn;
      }
    }
    __syncwarp();
    for (int j = lane; j < rows; j += 32) {
      const int pp = j / BT_M, ii = j - pp * BT_M, o = pp * PS_LD + ii;
      const int64_t ps = row0 + (int64_t)pp * BT_M;
      const int64_t pe = ((ps + BT_M < n) ? ps + BT_M : n) - 1;
      const int64_t gi = row0 + j;
      if (gi < pe) {  // interior rows only (the interface row keeps no Y/V/W)
        Y[gi] = sB[o];
        V[gi] = sL[o];
        W[gi] = sU[o];
      }
    }
  }
  if (!ok) atomicOr(flag, 2);
}

// ---------------------------------------------------------------------------
// interface rows -> reduced system (or, with one partition, its solution)
// ---------------------------------------------------------------------------
template <int NV>
__global__ void assemble_kernel(const double* __restrict__ sys, const double* __restrict__ rhs,
                                double sign, int64_t n, bool cyclic,
                                const double* __restrict__ Y, const double* __restrict__ V,
                                const double* __restrict__ W, double* __restrict__ nsys,
                                double* __restrict__ nrhs, double* __restrict__ xsol,
                                int* __restrict__ flag) {
  constexpr int NV2 = NV * NV;
  const int64_t P = (n + BT_M - 1) / BT_M;
  const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= P) return;
  const int64_t s = p * BT_M;
  const int64_t e = ((s + BT_M < n) ? s + BT_M : n) - 1;
  Blk<NV> L, D, U;
  load_blk<NV>(sys + (e * 3 + 0) * NV2, L);
  load_blk<NV>(sys + (e * 3 + 1) * NV2, D);
  load_blk<NV>(sys + (e * 3 + 2) * NV2, U);
  double bt[NV];
#pragma unroll
  for (int a = 0; a < NV; ++a) bt[a] = sign * rhs[e * NV + a];
  Blk<NV> Lt, Ut, T;
  zero_blk<NV>(Lt);
  zero_blk<NV>(Ut);
  const bool has_left = (p > 0) || cyclic;
  const bool has_right = (p < P - 1) || cyclic;
  // left side: x_{e-1}
  if (e > s) {
    Blk<NV> Vb, Wb;
    load_blk<NV>(V + (e - 1) * NV2, Vb);
    load_blk<NV>(W + (e - 1) * NV2, Wb);
    mm<NV>(L, Vb, Lt);
    mm<NV>(L, Wb, T);
#pragma unroll
    for (int a = 0; a < NV; ++a)
#pragma unroll
      for (int c = 0; c < NV; ++c) D.a[a][c] += T.a[a][c];
    double t[NV];
    mv<NV>(L, Y + (e - 1) * NV, t);
#pragma unroll
    for (int a = 0; a < NV; ++a) bt[a] -= t[a];
  } else if (has_left) {
    Lt = L;
  }
  // right side: x_{e+1} = first row of the next partition
  if (has_right) {
    const int64_t pr = (p + 1 < P) ? p + 1 : 0;
    const int64_t s2 = pr * BT_M;
    const int64_t e2 = ((s2 + BT_M < n) ? s2 + BT_M : n) - 1;
    if (e2 > s2) {
      Blk<NV> Vb, Wb;
      load_blk<NV>(V + s2 * NV2, Vb);
      load_blk<NV>(W + s2 * NV2, Wb);
      mm<NV>(U, Vb, T);
#pragma unroll
      for (int a = 0; a < NV; ++a)
#pragma unroll
        for (int c = 0; c < NV; ++c) D.a[a][c] += T.a[a][c];
      mm<NV>(U, Wb, Ut);
      double t[NV];
      mv<NV>(U, Y + s2 * NV, t);
#pragma unroll
      for (int a = 0; a < NV; ++a) bt[a] -= t[a];
    } else {
      Ut = U;
    }
  }
  if (P == 1) {
    // every neighbour is this partition's own interface unknown
#pragma unroll
    for (int a = 0; a < NV; ++a)
#pragma unroll
      for (int c = 0; c < NV; ++c) D.a[a][c] += Lt.a[a][c] + Ut.a[a][c];
    int piv[NV];
    if (!lu<NV>(D, piv)) atomicOr(flag, 2);
    lu_solve<NV>(D, piv, bt);
#pragma unroll
    for (int a = 0; a < NV; ++a) xsol[a] = bt[a];
    return;
  }
  store_blk<NV>(nsys + (p * 3 + 0) * NV2, Lt);
  store_blk<NV>(nsys + (p * 3 + 1) * NV2, D);
  store_blk<NV>(nsys + (p * 3 + 2) * NV2, Ut);
#pragma unroll
  for (int a = 0; a < NV; ++a) nrhs[p * NV + a] = bt[a];
}

// ---------------------------------------------------------------------------
// back-substitution, one thread per row (coalesced)
// ---------------------------------------------------------------------------
template <int NV>
__global__ void backsub_kernel(int64_t n, bool cyclic, const double* __restrict__ Y,
                               const double* __restrict__ V, const double* __restrict__ W,
                               const double* __restrict__ X, double* out, const double* add_to) {
  constexpr int NV2 = NV * NV;
  const int64_t P = (n + BT_M - 1) / BT_M;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = i / BT_M;
    const int64_t s = p * BT_M;
    const int64_t e = ((s + BT_M < n) ? s + BT_M : n) - 1;
    double xo[NV];
    if (i == e) {
#pragma unroll
      for (int a = 0; a < NV; ++a) xo[a] = X[p * NV + a];
    } else {
      Blk<NV> Vb, Wb;
      load_blk<NV>(V + i * NV2, Vb);
      load_blk<NV>(W + i * NV2, Wb);
      double t[NV];
#pragma unroll
      for (int a = 0; a < NV; ++a) xo[a] = Y[i * NV + a];
      mv<NV>(Wb, X + p * NV, t);
#pragma unroll
      for (int a = 0; a < NV; ++a) xo[a] += t[a];
      if (p > 0 || cyclic) {
        const int64_t pl = (p > 0) ? p - 1 : P - 1;
        mv<NV>(Vb, X + pl * NV, t);
#pragma unroll
        for (int a = 0; a < NV; ++a) xo[a] += t[a];
      }
    }
    if (add_to) {  // out = add_to + solution (the Newton update x += delta, in place)
#pragma unroll
      for (int a = 0; a < NV; ++a) out[i * NV + a] = add_to[i * NV + a] + xo[a];
    } else {
#pragma unroll
      for (int a = 0; a < NV; ++a) out[i * NV + a] = xo[a];
    }
  }
}

// ---------------------------------------------------------------------------
// host driver
// ---------------------------------------------------------------------------
struct LevelBufs {
  int64_t n;
  const double* sys;
  const double* rhs;
  double sign;
  double *Y, *V, *W, *G;
  double* sol;  // solution of this level (n rows)
};

static size_t level_bytes(int64_t n, int nv) {
  return 4 * align_up(sizeof(double) * n * nv * nv) + align_up(sizeof(double) * n * nv);
}

size_t bt_workspace_bytes(int64_t n, int nv) {
  size_t b = 0;
  int64_t cur = n;
  while (true) {
    b += level_bytes(cur, nv);  // Y, V, W, G
    const int64_t P = (cur + BT_M - 1) / BT_M;
    // next level: sys + rhs + sol
    b += align_up(sizeof(double) * P * 3 * nv * nv) + 2 * align_up(sizeof(double) * P * nv);
    if (P == 1) break;
    cur = P;
  }
  return b;
}

template <int NV>
static int bt_solve_t(adrom_ctx* ctx, const double* sys, const double* rhs, double sign,
                      int64_t n, bool cyclic, double* out, void* ws, int* flag,
                      const double* add_to) {
  constexpr int NV2 = NV * NV;
  LevelBufs lv[16];
  int nl = 0;
  char* w = (char*)ws;
  auto take = [&](size_t bytes) {
    double* p = (double*)w;
    w += align_up(bytes);
    return p;
  };
  lv[0].n = n;
  lv[0].sys = sys;
  lv[0].rhs = rhs;
  lv[0].sign = sign;
  lv[0].sol = out;
  // forward: eliminate interiors level by level
  while (true) {
    LevelBufs& L = lv[nl];
    L.Y = take(sizeof(double) * L.n * NV);
    L.V = take(sizeof(double) * L.n * NV2);
    L.W = take(sizeof(double) * L.n * NV2);
    L.G = take(sizeof(double) * L.n * NV2);
    take(0);
    const int64_t P = (L.n + BT_M - 1) / BT_M;
    double* nsys = take(sizeof(double) * P * 3 * NV2);
    double* nrhs = take(sizeof(double) * P * NV);
    double* nsol = take(sizeof(double) * P * NV);
    const int nt = 128;
    const int gb = (int)((P + nt - 1) / nt);
    if (NV == 1) {
      const size_t sm = sizeof(double) * PS_WARPS * 4 * 32 * PS_LD;
      const int64_t groups = (P + 31) / 32;
      int64_t g = (groups + PS_WARPS - 1) / PS_WARPS;
      if (g > (int64_t)ctx->num_sms * 16) g = (int64_t)ctx->num_sms * 16;
      cudaFuncSetAttribute(part_solve_scalar_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)sm);
      part_solve_scalar_kernel<<<(int)(g < 1 ? 1 : g), 32 * PS_WARPS, sm, ctx->stream>>>(
          L.sys, L.rhs, L.sign, L.n, L.Y, L.V, L.W, flag);
    } else if (NV > 8) {  // warp per partition, DMMA block products (13 x 13 blocks)
      static const bool hw = getenv("ADROM_BT_HALFWARP") && atoi(getenv("ADROM_BT_HALFWARP"));
      if (hw) {
        const int64_t g2 = (P * 16 + 127) / 128;
        part_solve_hw_kernel<NV><<<(int)g2, 128, 0, ctx->stream>>>(L.sys, L.rhs, L.sign, L.n,
                                                                   L.Y, L.V, L.W, L.G, flag);
      } else {
        const size_t sm = sizeof(double) * TC_WARPS * (TC_TILES * TC_TILE + 64);
        cudaFuncSetAttribute(part_solve_tc_kernel<NV>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)sm);
        const int64_t g2 = (P + TC_WARPS - 1) / TC_WARPS;
        part_solve_tc_kernel<NV><<<(int)g2, 32 * TC_WARPS, sm, ctx->stream>>>(
            L.sys, L.rhs, L.sign, L.n, L.Y, L.V, L.W, L.G, flag);
      }
    } else {
      part_solve_kernel<NV><<<gb, nt, 0, ctx->stream>>>(L.sys, L.rhs, L.sign, L.n, L.Y, L.V, L.W,
                                                        L.G, flag);
    }
    ADROM_LAUNCH_CK(ctx);
    assemble_kernel<NV><<<gb, nt, 0, ctx->stream>>>(L.sys, L.rhs, L.sign, L.n, cyclic, L.Y, L.V,
                                                    L.W, nsys, nrhs, nsol, flag);
    ADROM_LAUNCH_CK(ctx);
    if (nl + 1 >= 16) return set_error(ctx, ADROM_ERR_ARG, "bt_solve: too many levels");
    LevelBufs& N = lv[nl + 1];
    N.n = P;
    N.sys = nsys;
    N.rhs = nrhs;
    N.sign = 1.0;
    N.sol = nsol;
    ++nl;
    if (P == 1) break;
  }
  // backward: level nl holds the 1-row solution; substitute upwards
  for (int l = nl - 1; l >= 0; --l) {
    const LevelBufs& L = lv[l];
    int64_t gb = (L.n + 255) / 256;
    if (gb > (int64_t)ctx->num_sms * 16) gb = (int64_t)ctx->num_sms * 16;
    backsub_kernel<NV><<<(int)gb, 256, 0, ctx->stream>>>(L.n, cyclic, L.Y, L.V, L.W,
                                                         lv[l + 1].sol, L.sol,
                                                         l == 0 ? add_to : nullptr);
    ADROM_LAUNCH_CK(ctx);
  }
  return ADROM_OK;
}

int bt_solve(adrom_ctx* ctx, const double* sys, const double* rhs, double rhs_sign, int64_t n,
             int nv, bool cyclic, double* out, void* ws, int* flag, const double* add_to) {
  if (nv == 1) return bt_solve_t<1>(ctx, sys, rhs, rhs_sign, n, cyclic, out, ws, flag, add_to);
  if (nv == 3) return bt_solve_t<3>(ctx, sys, rhs, rhs_sign, n, cyclic, out, ws, flag, add_to);
  // configuration-4 reacting model: 13 x 13 blocks, half-warp per partition
  if (nv == 13) return bt_solve_t<13>(ctx, sys, rhs, rhs_sign, n, cyclic, out, ws, flag, add_to);
  return set_error(ctx, ADROM_ERR_ARG, "bt_solve: unsupported block size %d", nv);
}

}  // namespace adrom
