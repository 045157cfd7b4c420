// Pointwise full-order physics shared by every kernel that evaluates the
// residual (full rhs, sampled rhs, FD Jacobian).  One definition backs all
// of them, so the full and the gathered residual agree bit for bit, as the
// reference's do.
//
// IMPORTANT: translation units including this header are compiled with
// --fmad=false: numpy never contracts a*b+c into an FMA, and a single FMA
// changes the last bit (2.8e-11 pointwise error otherwise).
#pragma once

#include "common.cuh"

namespace adrom {

constexpr double PRIM_FLOOR = 1e-10;  // fom.py:36
constexpr double FD_EPS = 1e-7;       // fom.py:39

// IEEE division a / b with a shortcut for an exact-zero numerator: for
// b finite and nonzero, 0 / b is +-0 (sign = sign(a) xor sign(b)), which is
// what div.rn.f64 returns — but its software sequence routes a zero
// numerator through the slow path (a subroutine call per division).  Uniform
// regions (zero velocity, zero flux differences) hit that case on every
// cell.  Bitwise identical to a / b for every input.
__device__ __forceinline__ double zdiv(double a, double b) {
  if (a == 0.0 && b != 0.0 && isfinite(b))
    return __longlong_as_double((__double_as_longlong(a) ^ __double_as_longlong(b)) &
                                (long long)0x8000000000000000ull);
  return a / b;
}

// a / h for a grid spacing h.  Every BASELINE grid has n_elem = 2^k cells on
// a unit domain, so h = 2^-k (and h**2 = 2^-2k) exactly; then a / h and
// a * (1 / h) are the same exactly-scaled real number rounded once, i.e.
// bitwise identical for every a (zeros, subnormals, overflow included), and
// the multiply replaces div.rn.f64's ~10-instruction sequence.  Any other h
// takes the IEEE division.  The power-of-two test is on the kernel
// parameter, so it is warp-uniform and hoisted out of the cell loops.
__device__ __forceinline__ double div_h(double a, double h) {
  const long long b = __double_as_longlong(h);
  const int e = (int)((b >> 52) & 0x7ff);
  if ((b & 0xFFFFFFFFFFFFFll) == 0 && b > 0 && e > 0 && e < 2046)
    return a * __longlong_as_double((long long)(2046 - e) << 52);
  return zdiv(a, h);
}

struct BurgersParams {
  double dx, nu, dx2;  // dx2 = dx**2 (fom.py:187)
};

// fom.py:184-188 / fom.py:194-198
__device__ __forceinline__ double burgers_cell(double um, double u, double up,
                                               const BurgersParams& p) {
  // np.where(u > 0, back, fwd): only the selected one-sided difference is
  // divided (same value bit for bit, one division instead of two)
  // plain IEEE division: the Burgers states are smooth (zdiv's test costs
  // more than the rare zero-numerator slow path; measured 0.064 vs 0.074 ms)
  const double conv = (-u) * ((u > 0.0) ? div_h(u - um, p.dx) : div_h(up - u, p.dx));
  const double lap = (um - 2.0 * u) + up;
  const double diff = div_h(p.nu * lap, p.dx2);
  return conv + diff;
}

struct Cons {
  double m0, m1, m2;  // rho, rho*v, E
};

// fom.py:204-210
__device__ __forceinline__ void euler_prim(const Cons& c, double gamma, double& rho,
                                           double& vel, double& p) {
  rho = np_max(c.m0, PRIM_FLOOR);
  vel = zdiv(c.m1, rho);
  const double kinetic = (0.5 * rho) * (vel * vel);
  p = np_max((gamma - 1.0) * (c.m2 - kinetic), PRIM_FLOOR);
}

// fom.py:222-236 (rusanov_flux) with fom.py:213-219 (_euler_flux)
__device__ __forceinline__ Cons rusanov(const Cons& l, const Cons& r, double gamma) {
  double rl, vl, pl, rr, vr, pr;
  euler_prim(l, gamma, rl, vl, pl);
  euler_prim(r, gamma, rr, vr, pr);
  const double cl = sqrt((gamma * pl) / rl);
  const double cr = sqrt((gamma * pr) / rr);
  const double s = np_max(fabs(vl) + cl, fabs(vr) + cr);
  // physical fluxes
  const double fl0 = l.m1, fl1 = l.m1 * vl + pl, fl2 = vl * (l.m2 + pl);
  const double fr0 = r.m1, fr1 = r.m1 * vr + pr, fr2 = vr * (r.m2 + pr);
  const double hs = 0.5 * s;
  Cons f;
  f.m0 = 0.5 * (fl0 + fr0) - hs * (r.m0 - l.m0);
  f.m1 = 0.5 * (fl1 + fr1) - hs * (r.m1 - l.m1);
  f.m2 = 0.5 * (fl2 + fr2) - hs * (r.m2 - l.m2);
  return f;
}

// fom.py:269 / fom.py:277:  -(F_hi - F_lo) / dx
__device__ __forceinline__ Cons sod_cell_from_faces(const Cons& lo, const Cons& hi, double dx) {
  Cons o;
  o.m0 = div_h(-(hi.m0 - lo.m0), dx);
  o.m1 = div_h(-(hi.m1 - lo.m1), dx);
  o.m2 = div_h(-(hi.m2 - lo.m2), dx);
  return o;
}

__device__ __forceinline__ Cons sod_cell(const Cons& l, const Cons& c, const Cons& r,
                                         double gamma, double dx) {
  return sod_cell_from_faces(rusanov(l, c, gamma), rusanov(c, r, gamma), dx);
}

__device__ __forceinline__ Cons load_cons(const double* q, int64_t cell) {
  Cons c;
  c.m0 = q[3 * cell];
  c.m1 = q[3 * cell + 1];
  c.m2 = q[3 * cell + 2];
  return c;
}

__device__ __forceinline__ double cons_get(const Cons& c, int v) {
  return v == 0 ? c.m0 : (v == 1 ? c.m1 : c.m2);
}

__device__ __forceinline__ void cons_set(Cons& c, int v, double x) {
  if (v == 0) c.m0 = x;
  else if (v == 1) c.m1 = x;
  else c.m2 = x;
}

// fom.py:92-97 — neighbour with the model's boundary rule
__device__ __forceinline__ int64_t left_of(int64_t c, int64_t n, bool periodic) {
  return periodic ? (c == 0 ? n - 1 : c - 1) : (c == 0 ? 0 : c - 1);
}
__device__ __forceinline__ int64_t right_of(int64_t c, int64_t n, bool periodic) {
  return periodic ? (c == n - 1 ? 0 : c + 1) : (c == n - 1 ? n - 1 : c + 1);
}

// fom.py:317 — eps_j = 1e-7 * max(1, |q_j|)
__device__ __forceinline__ double fd_eps(double qj) { return FD_EPS * np_max(1.0, fabs(qj)); }

}  // namespace adrom
