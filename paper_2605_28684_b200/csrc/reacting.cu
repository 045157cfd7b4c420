// Configuration-4 reacting Euler model: 13 conserved
// variables per cell, [rho, m, E, rho Y_0..rho Y_9], periodic grid, Rusanov
// interfaces as the Sod model (fom.py:204-236) plus the sources of 12
// first-order Arrhenius reactions.  The reference has no such model
// (SPEC.md:8); oracle/reacting.py defines it and this kernel mirrors its
// floating-point order (compiled with --fmad=false like fom.cu).
//
// Residual kernel: tiles of RX_TILE cells staged in shared memory with a
// one-cell halo on each side (periodic wrap), one interface flux per face,
// 13 x 8 B read + 13 x 8 B written per cell (208 B/cell, HBM bound).
#include "reacting.cuh"
#include "fom_internal.cuh"

namespace adrom {

// mech (device, 5 x 12): a, b (as doubles), A, Ta, q
__global__ void __launch_bounds__(RX_NT) reacting_rhs_kernel(const double* __restrict__ q,
                                                             double* __restrict__ out, int64_t n,
                                                             double dx, double gamma,
                                                             const double* __restrict__ mech) {
  __shared__ double cells[RX_NV * (RX_TILE + 2)];
  __shared__ double faces[RX_NV * (RX_TILE + 1)];
  __shared__ double mk[5 * RX_NR];
  for (int e = threadIdx.x; e < 5 * RX_NR; e += RX_NT) mk[e] = mech[e];
  const int64_t ntiles = (n + RX_TILE - 1) / RX_TILE;
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int64_t base = t * RX_TILE;
    const int cnt = (int)((n - base < RX_TILE) ? (n - base) : RX_TILE);
    __syncthreads();
    // local cell j in [0, cnt+1] = global cell base - 1 + j (periodic wrap)
    {
      const double* src = q + base * RX_NV;
      for (int e = threadIdx.x; e < RX_NV * cnt; e += RX_NT) cells[RX_NV + e] = src[e];
      if (threadIdx.x < RX_NV) {
        const int64_t gl = (base == 0) ? n - 1 : base - 1;
        const int64_t gr = (base + cnt == n) ? 0 : base + cnt;
        cells[threadIdx.x] = q[gl * RX_NV + threadIdx.x];
        cells[RX_NV * (cnt + 1) + threadIdx.x] = q[gr * RX_NV + threadIdx.x];
      }
    }
    __syncthreads();
    // face f between local cells f and f+1
    for (int f = threadIdx.x; f <= cnt; f += RX_NT)
      rx_rusanov(cells + RX_NV * f, cells + RX_NV * (f + 1), gamma, faces + RX_NV * f);
    __syncthreads();
    // cell c (local c+1): -(F_hi - F_lo)/dx + S; results overwrite the face
    // slots only after every thread is done reading them (outs in registers)
    double res[RX_NV];
    const int c = threadIdx.x;
    if (c < cnt) {
      const double* u = cells + RX_NV * (c + 1);
      double s[RX_NV];
#pragma unroll
      for (int v = 0; v < RX_NV; ++v) s[v] = 0.0;
      double rho, vel, p;
      rx_prim(u, gamma, rho, vel, p);
      const double temp = p / rho;
#pragma unroll 1
      for (int j = 0; j < RX_NR; ++j) {
        const int a = (int)mk[j], b = (int)mk[RX_NR + j];
        const double w = (mk[2 * RX_NR + j] * exp(-mk[3 * RX_NR + j] / temp)) * np_max(u[3 + a], 0.0);
        // s[3+a] -= w; s[3+b] += w (dynamic index into registers via a switch-free loop)
#pragma unroll
        for (int k = 0; k < RX_NS; ++k) {
          if (k == a) s[3 + k] = s[3 + k] - w;
          if (k == b) s[3 + k] = s[3 + k] + w;
        }
        s[2] = s[2] + mk[4 * RX_NR + j] * w;
      }
#pragma unroll
      for (int v = 0; v < RX_NV; ++v) {
        const double div = div_h(-(faces[RX_NV * (c + 1) + v] - faces[RX_NV * c + v]), dx);
        res[v] = div + s[v];
      }
    }
    __syncthreads();
    if (c < cnt) {
#pragma unroll
      for (int v = 0; v < RX_NV; ++v) faces[RX_NV * c + v] = res[v];
    }
    __syncthreads();
    double* dst = out + base * RX_NV;
    for (int e = threadIdx.x; e < RX_NV * cnt; e += RX_NT) dst[e] = faces[e];
  }
}


// Banded FD Jacobian (fom.py:301-328 generalised; oracle/physics.py
// fd_jacobian_blocks): column (cell g, var v) with eps = 1e-7 max(1, |q|)
// touches rows g-1 (right block), g (centre), g+1 (left block).  Perturbing
// cell g changes only the faces g-1/2, g+1/2 and the sources of g, so each
// column evaluates 2 fluxes + 1 source term and reuses the tile's base faces
// and sources for the rest of the three rows — the same operations on the
// same operands as re-evaluating whole cell residuals (bitwise equal).
// apply_dt: A = I - dt J (fom.py:343-344).
constexpr int RJ_T = 32;

// per-cell physical flux and wave speed (the side terms of rx_rusanov)
__device__ __forceinline__ void rx_side(const double* u, double gamma, double* f, double& a) {
  double rho, vel, p;
  rx_prim<true>(u, gamma, rho, vel, p);
  a = fabs(vel) + sqrt((gamma * p) / rho);
  f[0] = u[1];
  f[1] = u[1] * vel + p;
  f[2] = vel * (u[2] + p);
#pragma unroll
  for (int k = 0; k < RX_NS; ++k) f[3 + k] = u[1] * rx_div<true>(u[3 + k], rho);
}
// rx_rusanov from precomputed sides (same operations, bitwise)
__device__ __forceinline__ double rx_face_v(double fl, double fr, double hs, double ur, double ul) {
  return 0.5 * (fl + fr) - hs * (ur - ul);
}

__global__ void __launch_bounds__(128) reacting_jac_kernel(const double* __restrict__ q, int64_t n,
                                                            double dx, double gamma,
                                                            const double* __restrict__ mech,
                                                            double* __restrict__ blocks,
                                                            bool apply_dt, double dt,
                                                            int* __restrict__ flag) {
  __shared__ double cs[RX_NV * (RJ_T + 4)];   // cells base-2 .. base+T+1
  __shared__ double fp[RX_NV * (RJ_T + 4)];   // their physical fluxes
  __shared__ double av[RJ_T + 4];             // their wave speeds |u| + c
  __shared__ double ff[RX_NV * (RJ_T + 3)];   // base faces: face j between cs cells j and j+1
  __shared__ double sb[RX_NV * (RJ_T + 2)];   // base sources of cs cells 1 .. T+2
  __shared__ double fb[RX_NV * (RJ_T + 2)];   // base residuals of cs cells 1 .. T+2
  __shared__ double mk[5 * RX_NR];
  for (int e = threadIdx.x; e < 5 * RX_NR; e += blockDim.x) mk[e] = mech[e];
  constexpr int NV2 = RX_NV * RX_NV;
  const int64_t ntiles = (n + RJ_T - 1) / RJ_T;
  bool bad = false;
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int64_t base = t * RJ_T;
    const int cnt = (int)((n - base < RJ_T) ? (n - base) : RJ_T);
    __syncthreads();
    for (int e = threadIdx.x; e < RX_NV * (cnt + 4); e += blockDim.x) {
      const int j = e / RX_NV, v = e - j * RX_NV;
      int64_t g = base - 2 + j;
      g = ((g % n) + n) % n;
      cs[e] = q[g * RX_NV + v];
    }
    __syncthreads();
    for (int j = threadIdx.x; j < cnt + 4; j += blockDim.x)
      rx_side(cs + RX_NV * j, gamma, fp + RX_NV * j, av[j]);
    __syncthreads();
    for (int e = threadIdx.x; e < RX_NV * (cnt + 3); e += blockDim.x) {
      const int j = e / RX_NV, v = e - j * RX_NV;
      const double hs = 0.5 * np_max(av[j], av[j + 1]);
      ff[e] = rx_face_v(fp[RX_NV * j + v], fp[RX_NV * (j + 1) + v], hs, cs[RX_NV * (j + 1) + v],
                        cs[RX_NV * j + v]);
    }
    __syncthreads();
    // base residuals of rows base-1 .. base+cnt (cs cells 1 .. cnt+2)
    for (int c = threadIdx.x; c < cnt + 2; c += blockDim.x) {
      double s0[RX_NV];
      rx_sources<true>(cs + RX_NV * (c + 1), gamma, mk, s0);
#pragma unroll
      for (int v = 0; v < RX_NV; ++v) {
        sb[RX_NV * c + v] = s0[v];
        fb[RX_NV * c + v] = rx_combine<true>(ff[RX_NV * (c + 1) + v], ff[RX_NV * c + v], s0[v], dx);
      }
    }
    __syncthreads();
    for (int item = threadIdx.x; item < cnt * RX_NV; item += blockDim.x) {
      const int il = item / RX_NV, v = item - il * RX_NV;  // cell base+il, var v
      const int jc = il + 2;                                // its index in cs
      const double qv = cs[RX_NV * jc + v];
      const double eps = fd_eps(qv);
      double pc[RX_NV];
#pragma unroll
      for (int a = 0; a < RX_NV; ++a) pc[a] = cs[RX_NV * jc + a];
      pc[v] = qv + eps;
      double fpc[RX_NV], apc;
      rx_side(pc, gamma, fpc, apc);
      double sp[RX_NV];
      rx_sources<true>(pc, gamma, mk, sp);
      const double hl = 0.5 * np_max(av[jc - 1], apc);
      const double hr = 0.5 * np_max(apc, av[jc + 1]);
      const int64_t g = base + il;
      const double* ul = cs + RX_NV * (jc - 1);
      const double* ur = cs + RX_NV * (jc + 1);
      const double* fl0 = fp + RX_NV * (jc - 1);
      const double* fr0 = fp + RX_NV * (jc + 1);
      // rows g-1 (slot 2), g (slot 1), g+1 (slot 0); the row of cs cell m
      // has faces m-1 (lo) and m (hi), sources and base residual fb[m-1]
#pragma unroll 1
      for (int rr = 0; rr < 3; ++rr) {
        const int m = jc - 1 + rr;
        int64_t row = g - 1 + rr;
        row = ((row % n) + n) % n;
        const int slot = 2 - rr;
        double* B = blocks + ((row * 3 + slot) * NV2);
#pragma unroll
        for (int a = 0; a < RX_NV; ++a) {
          const double Fl = rx_face_v(fl0[a], fpc[a], hl, pc[a], ul[a]);  // face g-1/2
          const double Fr = rx_face_v(fpc[a], fr0[a], hr, ur[a], pc[a]);  // face g+1/2
          const double Flo = (rr == 0) ? ff[RX_NV * (m - 1) + a] : (rr == 1 ? Fl : Fr);
          const double Fhi = (rr == 0) ? Fl : (rr == 1 ? Fr : ff[RX_NV * m + a]);
          const double S = (rr == 1) ? sp[a] : sb[RX_NV * (m - 1) + a];
          const double f0 = fb[RX_NV * (m - 1) + a];
          const double fpv = rx_combine<true>(Fhi, Flo, S, dx);
          const double jv = (fpv - f0) / eps;
          bad |= !isfinite(jv);
          B[a * RX_NV + v] = apply_dt ? ((slot == 1 && a == v) ? 1.0 : 0.0) - dt * jv : jv;
        }
      }
    }
  }
  if (bad) atomicOr(flag, 4);
}

int reacting_jacobian(adrom_ctx* ctx, const adrom_model& m, const double* q, double* blocks,
                      bool apply_dt, double dt, int* flag) {
  if (!m.mech) return set_error(ctx, ADROM_ERR_ARG, "reacting model: mechanism pointer is null");
  const int64_t ntiles = (m.n_elem + RJ_T - 1) / RJ_T;
  int64_t g = (int64_t)ctx->num_sms * 8;
  if (g > ntiles) g = ntiles;
  reacting_jac_kernel<<<(int)(g < 1 ? 1 : g), 128, 0, ctx->stream>>>(q, m.n_elem, m.dx, m.gamma,
                                                                    m.mech, blocks, apply_dt, dt,
                                                                    flag);
  ADROM_LAUNCH_CK(ctx);
  return ADROM_OK;
}

int reacting_rhs(adrom_ctx* ctx, const adrom_model& m, const double* q, double* f) {
  if (!m.mech) return set_error(ctx, ADROM_ERR_ARG, "reacting model: mechanism pointer is null");
  const int64_t ntiles = (m.n_elem + RX_TILE - 1) / RX_TILE;
  int64_t g = (int64_t)ctx->num_sms * 12;
  if (g > ntiles) g = ntiles;
  reacting_rhs_kernel<<<(int)(g < 1 ? 1 : g), RX_NT, 0, ctx->stream>>>(q, f, m.n_elem, m.dx,
                                                                       m.gamma, m.mech);
  ADROM_LAUNCH_CK(ctx);
  return ADROM_OK;
}

}  // namespace adrom
