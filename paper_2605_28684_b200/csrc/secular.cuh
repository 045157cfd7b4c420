// SVD of the iSVD core matrix by the secular equation (one thread block).
//
// The core matrix of the Brand update (tracking.py:166-173) is
//
//     K = [[lam Sigma, p], [0, rho]]   ((r+1) x (r+1))  =  [D | z],
//
// D = [lam Sigma; 0] and z = [p; rho], so K K^T = diag(d^2) + z z^T with
// d = (lam sigma_1 .. lam sigma_r, 0): a rank-one modification of a diagonal
// matrix.  Its eigenpairs are the squared singular values and the left
// singular vectors of K — everything the update needs (the rotation factors
// U[:, :r], sigma' and the dropped direction).  This is the merge step of
// LAPACK's divide-and-conquer SVD (the dlasd2 / dlasd4 / dlasd8 sequence that
// gesdd itself runs on larger matrices), restated for one block:
//
//  1. deflation (thread 0): |z_i| <= eps d_i gives the eigenpair
//     (d_i^2, e_i); d_a - d_b <= eps d_a rotates z_b into z_a (Givens) and
//     deflates b.  Both thresholds are relative (dlasd2's are absolute,
//     8 eps max(d, z)) so that rounding-level singular values keep their
//     vectors, as one-sided Jacobi's do;
//  2. one warp per remaining root: the secular equation
//         1 + sum_i z_i^2 / (d_i^2 - mu) = 0,  mu in (D_k, D_k+1),
//     solved for tau = mu - D_origin from the nearer pole (origin shift:
//     every d_i^2 - mu is formed as (d_i - d_o)(d_i + d_o) - tau, so tiny
//     singular values keep their relative accuracy), by the "middle way"
//     rational iteration (the two-pole model of dlaed4) with a bisection
//     safeguard;
//  3. Gu-Eisenstat: z^ is recomputed from the computed roots (Loewner), and
//     u_k = (z^_i / (d_i^2 - mu_k))_i / norm — numerically orthogonal
//     vectors whatever the clustering of the roots;
//  4. the deflation rotations are undone on the rows.
//
// The caller verifies the result (residual of K K^T u = s^2 u on every kept
// column and orthonormality) and falls back to one-sided Jacobi otherwise.
// O(r^2) work with r-way parallelism instead of the O(r^3) sweeps of Jacobi.
#pragma once

#include "common.cuh"

namespace adrom {

constexpr int SEC_MAXN = 136;  // n = r + 1 <= 129

struct SecularShared {
  double d[SEC_MAXN];    // sorted (descending) d of the slots
  double z[SEC_MAXN];    // z of the slots (rotated by the deflation)
  double zh[SEC_MAXN];   // z^ (Loewner), ascending secular index
  double tau[SEC_MAXN];  // per root: mu_k - D_origin
  double sv[SEC_MAXN];   // singular value of every slot's column
  double gc[SEC_MAXN], gs[SEC_MAXN];  // deflation rotations
  int perm[SEC_MAXN];    // slot -> original index
  int sec[SEC_MAXN];     // ascending secular index -> slot
  int org[SEC_MAXN];     // per root: origin (ascending secular index)
  int ga[SEC_MAXN], gb[SEC_MAXN];     // rotated slot pairs
  int m, nrot, ok;
};

// D_l - D_i = d_l^2 - d_i^2 without cancellation
__device__ __forceinline__ double sec_dd(double dl, double di) { return (dl - di) * (dl + di); }

// Fills Vcols (column j of U at Vcols + j*ld, rows = original indices
// 0..n-1) and s[j] (unsorted); returns false if a root did not converge.
// d = (lam sigma_0 .. lam sigma_{n-2}, 0), z = [p; rho].  All threads call.
// Dm: scratch of n x ldd doubles (ldd >= n; the differences D_i - mu_k).
__device__ inline bool secular_core_svd(const double* __restrict__ sigma, double lam,
                                        const double* __restrict__ p, double rho, int n,
                                        double* Vcols, int ld, double* s, double* Dm, int ldd,
                                        SecularShared& S) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  constexpr double EPS = 2.220446049250313e-16;
  // --- sort slots by d descending (ties: lower index first)
  for (int i = tid; i < n; i += blockDim.x) {
    const double di = (i < n - 1) ? lam * sigma[i] : 0.0;
    int rank = 0;
    for (int k = 0; k < n; ++k) {
      const double dk = (k < n - 1) ? lam * sigma[k] : 0.0;
      if (dk > di || (dk == di && k < i)) ++rank;
    }
    S.perm[rank] = i;
    S.d[rank] = di;
    S.z[rank] = (i < n - 1) ? p[i] : rho;
  }
  __syncthreads();
  // --- deflation (one thread; n <= 129)
  if (tid == 0) {
    double dmax = 0.0, zmax = 0.0;
    for (int i = 0; i < n; ++i) {
      dmax = fmax(dmax, fabs(S.d[i]));
      zmax = fmax(zmax, fabs(S.z[i]));
    }
    // relative deflation thresholds (a relative perturbation of K's entries):
    // the core's trailing singular values sit at rounding level of sigma_1,
    // and an absolute tolerance (8 eps max(d, z), dlasd2's) would rotate
    // those directions arbitrarily — one-sided Jacobi and the reference's
    // gesdd resolve them, and QDEIM's pivots follow them
    const double tiny = 1e-150 * fmax(dmax, zmax);
    int m = 0, nrot = 0, last = -1;
    for (int i = 0; i < n; ++i) {
      S.sv[i] = -1.0;  // -1: secular root (set later)
      if (fabs(S.z[i]) <= fmax(EPS * S.d[i], tiny)) {
        S.sv[i] = S.d[i];  // eigenpair (d_i^2, e_i)
        S.z[i] = 0.0;
        continue;
      }
      if (last >= 0 && S.d[last] - S.d[i] <= EPS * S.d[last]) {
        const double h = hypot(S.z[last], S.z[i]);
        const double c = S.z[last] / h, sn = S.z[i] / h;
        S.ga[nrot] = last;
        S.gb[nrot] = i;
        S.gc[nrot] = c;
        S.gs[nrot] = sn;
        ++nrot;
        S.z[last] = h;
        S.z[i] = 0.0;
        S.sv[i] = S.d[i];  // deflated: eigvector -s e_last + c e_i (rotated coordinates)
        continue;
      }
      last = i;
      ++m;
    }
    // ascending secular order = descending slots reversed
    int k = m;
    for (int i = 0; i < n; ++i)
      if (S.sv[i] < 0.0) S.sec[--k] = i;
    S.m = m;
    S.nrot = nrot;
    S.ok = 1;
  }
  __syncthreads();
  const int m = S.m;
  // --- roots: warp per root, ascending secular index k (0-based), mu_k in
  // (D_k, D_k+1) for k < m-1, mu_{m-1} in (D_{m-1}, D_{m-1} + ||z||^2)
  double znorm2 = 0.0;
  for (int i = 0; i < m; ++i) znorm2 += S.z[S.sec[i]] * S.z[S.sec[i]];
  for (int k = warp; k < m; k += nw) {
    double* drow = Dm + (size_t)k * ldd;
    const bool lastroot = (k == m - 1);
    double tau, lo, hi;
    int o;
    if (m == 1) {  // one pole: mu = D + z^2
      const int sl = S.sec[0];
      if (lane == 0) {
        S.tau[0] = S.z[sl] * S.z[sl];
        S.org[0] = 0;
        drow[0] = -S.tau[0];
      }
      continue;
    }
    if (lastroot) {
      o = k;
      lo = 0.0;
      hi = znorm2;
    } else {
      // f at the midpoint with origin k decides the nearer pole
      const double dk = S.d[S.sec[k]], dk1 = S.d[S.sec[k + 1]];
      const double half = 0.5 * sec_dd(dk1, dk);
      double f = 0.0;
      for (int i = lane; i < m; i += 32) {
        const double di = S.d[S.sec[i]], zi = S.z[S.sec[i]];
        f += zi * zi / (sec_dd(di, dk) - half);
      }
      f = 1.0 + warp_sum(f);
      if (f >= 0.0) {
        o = k;
        lo = 0.0;
        hi = half;
      } else {
        o = k + 1;
        lo = -half;
        hi = 0.0;
      }
    }
    const double dorg = S.d[S.sec[o]];
    tau = 0.5 * (lo + hi);
    // pole pair of the two-pole model: (k, k+1), or (m-2, m-1) for the last root
    const int pl = lastroot ? m - 2 : k, pu = pl + 1;
    bool conv = false;
    for (int it = 0; it < 100; ++it) {
      double psi = 0.0, phi = 0.0, dpsi = 0.0, dphi = 0.0;
      for (int i = lane; i < m; i += 32) {
        const int sl = S.sec[i];
        const double del = sec_dd(S.d[sl], dorg) - tau;
        const double t = S.z[sl] / del;
        if (i <= pl) {
          psi += S.z[sl] * t;
          dpsi += t * t;
        } else {
          phi += S.z[sl] * t;
          dphi += t * t;
        }
      }
      psi = warp_sum(psi);
      phi = warp_sum(phi);
      dpsi = warp_sum(dpsi);
      dphi = warp_sum(dphi);
      const double w = 1.0 + psi + phi;
      const double dw = dpsi + dphi;
      const double err = 8.0 * (fabs(psi) + fabs(phi)) + 3.0 + fabs(tau) * dw;
      if (fabs(w) <= EPS * err) {
        conv = true;
        break;
      }
      if (w < 0.0) lo = tau;
      else hi = tau;
      if (hi - lo <= 4.0 * EPS * fmax(fabs(lo), fabs(hi))) {
        conv = true;
        break;
      }
      const double dl = sec_dd(S.d[S.sec[pl]], dorg) - tau;
      const double du = sec_dd(S.d[S.sec[pu]], dorg) - tau;
      const double c = w - dl * dpsi - du * dphi;
      const double a = (dl + du) * w - dl * du * dw;
      const double b = dl * du * w;
      double eta;
      if (c == 0.0) {
        eta = (a != 0.0) ? b / a : -w / dw;
      } else {
        const double disc = sqrt(fabs(a * a - 4.0 * b * c));
        if (!lastroot) eta = (a <= 0.0) ? (a - disc) / (2.0 * c) : 2.0 * b / (a + disc);
        else eta = (a >= 0.0) ? (a + disc) / (2.0 * c) : 2.0 * b / (a - disc);
      }
      if (!(w * eta < 0.0) || !isfinite(eta)) eta = -w / dw;  // Newton
      double tn = tau + eta;
      if (!(tn > lo && tn < hi)) tn = 0.5 * (lo + hi);         // bisection
      if (tn == tau) {
        conv = true;
        break;
      }
      tau = tn;
    }
    for (int i = lane; i < m; i += 32) drow[i] = sec_dd(S.d[S.sec[i]], dorg) - tau;
    if (lane == 0) {
      S.tau[k] = tau;
      S.org[k] = o;
      if (!conv) S.ok = 0;
    }
  }
  __syncthreads();
  // --- Loewner z^ (thread per secular index i)
  for (int i = tid; i < m; i += blockDim.x) {
    const double di = S.d[S.sec[i]];
    double prod = -Dm[(size_t)(m - 1) * ldd + i];
    for (int k = 0; k < m - 1; ++k) {
      const double num = -Dm[(size_t)k * ldd + i];
      const double den = (k < i) ? sec_dd(S.d[S.sec[k]], di) : sec_dd(S.d[S.sec[k + 1]], di);
      prod *= num / den;
    }
    const double zi = S.z[S.sec[i]];
    S.zh[i] = copysign(sqrt(fabs(prod)), zi);
  }
  __syncthreads();
  // --- columns: slot-space vectors (column c of slot sc = root's slot)
  // zero all, deflated columns = unit vectors; singular values
  for (int e = tid; e < n * n; e += blockDim.x) {
    const int c = e / n, rr = e - c * n;
    Vcols[(size_t)c * ld + rr] = (S.sv[c] >= 0.0 && rr == c) ? 1.0 : 0.0;
  }
  __syncthreads();
  // secular column k lives in column slot S.sec[k]; entries over the slots
  for (int k = warp; k < m; k += nw) {
    const int cs = S.sec[k];
    const double* drow = Dm + (size_t)k * ldd;
    double nr = 0.0;
    for (int i = lane; i < m; i += 32) {
      const double v = S.zh[i] / drow[i];
      nr += v * v;
    }
    nr = warp_sum(nr);
    const double inv = 1.0 / sqrt(nr);
    for (int i = lane; i < m; i += 32) Vcols[(size_t)cs * ld + S.sec[i]] = S.zh[i] / drow[i] * inv;
    if (lane == 0) {
      const double dorg = S.d[S.sec[S.org[k]]];
      S.sv[cs] = sqrt(dorg * dorg + S.tau[k]);
    }
  }
  __syncthreads();
  // --- undo the deflation rotations (reverse order) on the rows:
  // x_a = c y_a - s y_b, x_b = s y_a + c y_b
  for (int t = S.nrot - 1; t >= 0; --t) {
    const int a = S.ga[t], b = S.gb[t];
    const double c = S.gc[t], sn = S.gs[t];
    for (int col = tid; col < n; col += blockDim.x) {
      const double ya = Vcols[(size_t)col * ld + a], yb = Vcols[(size_t)col * ld + b];
      Vcols[(size_t)col * ld + a] = c * ya - sn * yb;
      Vcols[(size_t)col * ld + b] = sn * ya + c * yb;
    }
    __syncthreads();
  }
  // --- slots -> original row indices (permute within each column via Dm scratch)
  for (int e = tid; e < n * n; e += blockDim.x) {
    const int c = e / n, rr = e - c * n;
    Dm[(size_t)c * ldd + S.perm[rr]] = Vcols[(size_t)c * ld + rr];
  }
  __syncthreads();
  for (int e = tid; e < n * n; e += blockDim.x) {
    const int c = e / n, rr = e - c * n;
    Vcols[(size_t)c * ld + rr] = Dm[(size_t)c * ldd + rr];
  }
  for (int c = tid; c < n; c += blockDim.x) s[c] = S.sv[c];
  __syncthreads();
  return S.ok != 0;
}

}  // namespace adrom
