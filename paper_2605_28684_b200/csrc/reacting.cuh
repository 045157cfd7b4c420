// Configuration-4 reacting Euler model, pointwise physics shared by every
// kernel that evaluates its residual (full rhs and FD Jacobian in
// reacting.cu, gathered / sampled residuals in fom.cu and sampled.cu).  The
// reference has no such model; oracle/reacting.py defines it and
// these functions mirror its floating-point order.  Translation units that
// include this header are compiled with --fmad=false (see physics.cuh).
#pragma once

#include "physics.cuh"

namespace adrom {

// ZD: divisions through zdiv (full-grid residuals: uniform regions have zero
// numerators) or plain IEEE division (perturbed FD states: the zero test
// would only cost instructions); both are bitwise the same quotient
template <bool ZD>
__device__ __forceinline__ double rx_div(double a, double b) {
  if (ZD) return zdiv(a, b);
  return a / b;
}

constexpr int RX_NS = 10;          // species
constexpr int RX_NR = 12;          // reactions
constexpr int RX_NV = 3 + RX_NS;   // conserved variables
constexpr int RX_TILE = 128;       // cells per tile
constexpr int RX_NT = 128;

// primitives (fom.py:204-210 semantics)
template <bool ZD = true>
__device__ __forceinline__ void rx_prim(const double* c, double gamma, double& rho, double& vel,
                                        double& p) {
  rho = np_max(c[0], PRIM_FLOOR);
  vel = rx_div<ZD>(c[1], rho);
  const double kin = (0.5 * rho) * (vel * vel);
  p = np_max((gamma - 1.0) * (c[2] - kin), PRIM_FLOOR);
}

// Rusanov interface flux between conserved states l and r -> f[13]
template <bool ZD = true>
__device__ __forceinline__ void rx_rusanov(const double* l, const double* r, double gamma,
                                           double* f) {
  double rl, vl, pl, rr, vr, pr;
  rx_prim<ZD>(l, gamma, rl, vl, pl);
  rx_prim<ZD>(r, gamma, rr, vr, pr);
  const double s = np_max(fabs(vl) + sqrt((gamma * pl) / rl), fabs(vr) + sqrt((gamma * pr) / rr));
  const double hs = 0.5 * s;
  double fl, fr;
  fl = l[1];
  fr = r[1];
  f[0] = 0.5 * (fl + fr) - hs * (r[0] - l[0]);
  fl = l[1] * vl + pl;
  fr = r[1] * vr + pr;
  f[1] = 0.5 * (fl + fr) - hs * (r[1] - l[1]);
  fl = vl * (l[2] + pl);
  fr = vr * (r[2] + pr);
  f[2] = 0.5 * (fl + fr) - hs * (r[2] - l[2]);
#pragma unroll
  for (int k = 0; k < RX_NS; ++k) {
    fl = l[1] * rx_div<ZD>(l[3 + k], rl);
    fr = r[1] * rx_div<ZD>(r[3 + k], rr);
    f[3 + k] = 0.5 * (fl + fr) - hs * (r[3 + k] - l[3 + k]);
  }
}

// sources of one cell (12 first-order Arrhenius reactions)
template <bool ZD = true>
__device__ __forceinline__ void rx_sources(const double* c, double gamma, const double* mk,
                                           double* s) {
#pragma unroll
  for (int v = 0; v < RX_NV; ++v) s[v] = 0.0;
  double rho, vel, p;
  rx_prim<ZD>(c, gamma, rho, vel, p);
  const double temp = p / rho;
#pragma unroll 1
  for (int j = 0; j < RX_NR; ++j) {
    const int a = (int)mk[j], b = (int)mk[RX_NR + j];
    const double w = (mk[2 * RX_NR + j] * exp(-mk[3 * RX_NR + j] / temp)) * np_max(c[3 + a], 0.0);
#pragma unroll
    for (int k = 0; k < RX_NS; ++k) {
      if (k == a) s[3 + k] = s[3 + k] - w;
      if (k == b) s[3 + k] = s[3 + k] + w;
    }
    s[2] = s[2] + mk[4 * RX_NR + j] * w;
  }
}

// residual of a cell from its two face fluxes and its sources
template <bool ZD = true>
__device__ __forceinline__ double rx_combine(double fr, double fl, double s, double dx) {
  return rx_div<ZD>(-(fr - fl), dx) + s;
}

// residual of one cell from its stencil (l, c, r): -(F(c,r) - F(l,c))/dx + S(c),
// the same operations as the full kernel (faces computed identically)
template <bool ZD = true>
__device__ __forceinline__ void rx_cell_res(const double* l, const double* c, const double* r,
                                            double gamma, double dx, const double* mk,
                                            double* out) {
  double fl[RX_NV], fr[RX_NV];
  rx_rusanov<ZD>(l, c, gamma, fl);
  rx_rusanov<ZD>(c, r, gamma, fr);
  double s[RX_NV];
  rx_sources<ZD>(c, gamma, mk, s);
#pragma unroll
  for (int v = 0; v < RX_NV; ++v) out[v] = rx_combine<ZD>(fr[v], fl[v], s[v], dx);
}


// residual of one cell, mechanism entries read through `mk` (5 x RX_NR:
// a, b, A, Ta, q), stencil values fetched by `get(slot, var)`, slot 0/1/2 =
// left / centre / right
template <bool ZD = true, class Get>
__device__ __forceinline__ void rx_cell_res_get(const Get& get, double gamma, double dx,
                                                const double* mk, double* out) {
  double l[RX_NV], c[RX_NV], r[RX_NV];
#pragma unroll
  for (int v = 0; v < RX_NV; ++v) {
    l[v] = get(0, v);
    c[v] = get(1, v);
    r[v] = get(2, v);
  }
  rx_cell_res<ZD>(l, c, r, gamma, dx, mk, out);
}

}  // namespace adrom
