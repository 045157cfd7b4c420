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
#include "physics.cuh"
#include "fom_internal.cuh"

namespace adrom {

constexpr int RX_NS = 10;          // species
constexpr int RX_NR = 12;          // reactions
constexpr int RX_NV = 3 + RX_NS;   // conserved variables
constexpr int RX_TILE = 128;       // cells per tile
constexpr int RX_NT = 128;

// primitives (fom.py:204-210 semantics)
__device__ __forceinline__ void rx_prim(const double* c, double gamma, double& rho, double& vel,
                                        double& p) {
  rho = np_max(c[0], PRIM_FLOOR);
  vel = c[1] / rho;
  const double kin = (0.5 * rho) * (vel * vel);
  p = np_max((gamma - 1.0) * (c[2] - kin), PRIM_FLOOR);
}

// Rusanov interface flux between conserved states l and r -> f[13]
__device__ __forceinline__ void rx_rusanov(const double* l, const double* r, double gamma,
                                           double* f) {
  double rl, vl, pl, rr, vr, pr;
  rx_prim(l, gamma, rl, vl, pl);
  rx_prim(r, gamma, rr, vr, pr);
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
    fl = l[1] * (l[3 + k] / rl);
    fr = r[1] * (r[3 + k] / rr);
    f[3 + k] = 0.5 * (fl + fr) - hs * (r[3 + k] - l[3 + k]);
  }
}

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
        const double div = (-(faces[RX_NV * (c + 1) + v] - faces[RX_NV * c + v])) / dx;
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
