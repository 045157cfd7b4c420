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
  return div_h(-(fr - fl), dx) + s;
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

// Cell residual with every cell's primitives, wave speed and physical flux
// evaluated once (rx_cell_res evaluates the centre cell's twice, once per
// face): the same operations on the same operands as rx_rusanov /
// rx_sources / rx_combine, so bitwise equal to rx_cell_res.  Values are
// fetched through get(slot, var) (slot 0/1/2 = left / centre / right), which
// lets the caller keep the stencil in shared memory instead of registers.
template <bool ZD, class Get>
__device__ __forceinline__ void rx_cell_res_once(const Get& get, double gamma, double dx,
                                                 const double* mk, double* out) {
  // centre: primitives, speed, physical flux
  double cu[3];
  cu[0] = get(1, 0);
  cu[1] = get(1, 1);
  cu[2] = get(1, 2);
  double rc, vc, pc;
  rx_prim<ZD>(cu, gamma, rc, vc, pc);
  const double ac = fabs(vc) + sqrt((gamma * pc) / rc);
  double fc[RX_NV];
  fc[0] = cu[1];
  fc[1] = cu[1] * vc + pc;
  fc[2] = vc * (cu[2] + pc);
#pragma unroll
  for (int k = 0; k < RX_NS; ++k) fc[3 + k] = cu[1] * rx_div<ZD>(get(1, 3 + k), rc);
  // left face (l, c): flo
  double flo[RX_NV];
  {
    double lu[3] = {get(0, 0), get(0, 1), get(0, 2)};
    double rl, vl, pl;
    rx_prim<ZD>(lu, gamma, rl, vl, pl);
    const double hs = 0.5 * np_max(fabs(vl) + sqrt((gamma * pl) / rl), ac);
    flo[0] = 0.5 * (lu[1] + fc[0]) - hs * (cu[0] - lu[0]);
    flo[1] = 0.5 * ((lu[1] * vl + pl) + fc[1]) - hs * (cu[1] - lu[1]);
    flo[2] = 0.5 * ((vl * (lu[2] + pl)) + fc[2]) - hs * (cu[2] - lu[2]);
#pragma unroll
    for (int k = 0; k < RX_NS; ++k) {
      const double lk = get(0, 3 + k);
      flo[3 + k] = 0.5 * ((lu[1] * rx_div<ZD>(lk, rl)) + fc[3 + k]) - hs * (get(1, 3 + k) - lk);
    }
  }
  // right face (c, r) -> out = -(fhi - flo) / dx (sources added below)
  {
    double ru[3] = {get(2, 0), get(2, 1), get(2, 2)};
    double rr, vr, pr;
    rx_prim<ZD>(ru, gamma, rr, vr, pr);
    const double hs = 0.5 * np_max(ac, fabs(vr) + sqrt((gamma * pr) / rr));
    out[0] = div_h(-((0.5 * (fc[0] + ru[1]) - hs * (ru[0] - cu[0])) - flo[0]), dx);
    out[1] = div_h(-((0.5 * (fc[1] + (ru[1] * vr + pr)) - hs * (ru[1] - cu[1])) - flo[1]), dx);
    out[2] = div_h(-((0.5 * (fc[2] + (vr * (ru[2] + pr))) - hs * (ru[2] - cu[2])) - flo[2]), dx);
#pragma unroll
    for (int k = 0; k < RX_NS; ++k) {
      const double rk = get(2, 3 + k), ck = get(1, 3 + k);
      const double fhi = 0.5 * (fc[3 + k] + (ru[1] * rx_div<ZD>(rk, rr))) - hs * (rk - ck);
      out[3 + k] = div_h(-(fhi - flo[3 + k]), dx);
    }
  }
  // sources of the centre cell, accumulated from zero in rx_sources' order
  // (T = p / rho from the same primitives), then added like rx_combine
  double sv[RX_NV];
#pragma unroll
  for (int v = 0; v < RX_NV; ++v) sv[v] = 0.0;
  const double temp = pc / rc;
#pragma unroll 1
  for (int j = 0; j < RX_NR; ++j) {
    const int a = (int)mk[j], b = (int)mk[RX_NR + j];
    double ya = 0.0;
#pragma unroll
    for (int k = 0; k < RX_NS; ++k)
      if (k == a) ya = get(1, 3 + k);
    const double w = (mk[2 * RX_NR + j] * exp(-mk[3 * RX_NR + j] / temp)) * np_max(ya, 0.0);
#pragma unroll
    for (int k = 0; k < RX_NS; ++k) {
      if (k == a) sv[3 + k] = sv[3 + k] - w;
      if (k == b) sv[3 + k] = sv[3 + k] + w;
    }
    sv[2] = sv[2] + mk[4 * RX_NR + j] * w;
  }
#pragma unroll
  for (int v = 0; v < RX_NV; ++v) out[v] = out[v] + sv[v];
}

}  // namespace adrom
