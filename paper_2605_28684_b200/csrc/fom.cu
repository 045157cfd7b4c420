// Full-order model kernels: residual (kernel 1), gathered / sampled residual
// (kernel 2), banded FD Jacobian and the backward-Euler Newton driver.
//
// Compiled with --fmad=false (see physics.cuh): every residual value and
// every Jacobian entry is bitwise equal to the reference's numpy evaluation.
#include "physics.cuh"
#include "reacting.cuh"
#include "fom_internal.cuh"
#include "btsolve.cuh"

#include <math.h>
#include <string.h>

namespace adrom {

// ---------------------------------------------------------------------------
// kernel 1a: Burgers residual, register-streamed: a lane owns 4 consecutive
// cells (two 16-byte loads), neighbours come from the adjacent lanes by
// shuffle and, at the warp edges, from one scalar load each (periodic wrap).
// No shared memory, no block barriers: 2 warp-chunks in flight per warp.
// ---------------------------------------------------------------------------
constexpr int BURG_NT = 256;
constexpr int BURG_VPT = 4;                    // cells per lane
constexpr int BURG_WCH = 32 * BURG_VPT;        // cells per warp chunk
constexpr int BURG_U = 1;                      // warp chunks in flight
constexpr int BURG_TILE = BURG_NT * BURG_VPT * BURG_U;  // cells per block iteration

// MODE 0: out = f(q)                                     (fom.py:180-188)
// MODE 1: out = (q - qprev) - dt * f(q)                  (fom.py:340-341)
//         + per-block partial sums of out^2 + non-finite flag (dense.py:153)
template <int MODE>
__global__ void __launch_bounds__(BURG_NT, 4) burgers_rhs_kernel(
    const double* __restrict__ q, double* __restrict__ out, int64_t n, BurgersParams p,
    const double* __restrict__ qprev, double dt, double* __restrict__ partial,
    int* __restrict__ flag) {
  __shared__ double red[BURG_NT / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t nchunks = (n + BURG_WCH - 1) / BURG_WCH;
  const int64_t wstride = (int64_t)gridDim.x * (BURG_NT / 32) * BURG_U;
  double acc = 0.0;
  bool bad = false;
  for (int64_t c0 = ((int64_t)blockIdx.x * (BURG_NT / 32) + warp) * BURG_U; c0 < nchunks;
       c0 += wstride) {
    double v[BURG_U][BURG_VPT], pv[BURG_U][BURG_VPT], lft[BURG_U], rgt[BURG_U];
#pragma unroll
    for (int u = 0; u < BURG_U; ++u) {
      const int64_t ch = c0 + u;
      const int64_t i0 = ch * BURG_WCH + (int64_t)lane * BURG_VPT;
      const bool full = (ch + 1) * BURG_WCH <= n;
      if (ch < nchunks && full) {
        const double2 a = *reinterpret_cast<const double2*>(q + i0);
        const double2 b = *reinterpret_cast<const double2*>(q + i0 + 2);
        v[u][0] = a.x; v[u][1] = a.y; v[u][2] = b.x; v[u][3] = b.y;
        if (MODE == 1) {
          const double2 c = *reinterpret_cast<const double2*>(qprev + i0);
          const double2 d = *reinterpret_cast<const double2*>(qprev + i0 + 2);
          pv[u][0] = c.x; pv[u][1] = c.y; pv[u][2] = d.x; pv[u][3] = d.y;
        }
      } else {
#pragma unroll
        for (int k = 0; k < BURG_VPT; ++k) {
          const bool ok = ch < nchunks && i0 + k < n;
          v[u][k] = ok ? q[i0 + k] : 0.0;
          if (MODE == 1) pv[u][k] = ok ? qprev[i0 + k] : 0.0;
        }
      }
      // warp-edge neighbours (periodic)
      const int64_t cs = ch * BURG_WCH;
      const int64_t ce = ((cs + BURG_WCH < n) ? cs + BURG_WCH : n);  // one past the chunk
      lft[u] = (ch < nchunks && lane == 0) ? q[cs == 0 ? n - 1 : cs - 1] : 0.0;
      rgt[u] = (ch < nchunks && lane == 31) ? q[ce == n ? 0 : ce] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < BURG_U; ++u) {
      const int64_t ch = c0 + u;
      const int64_t i0 = ch * BURG_WCH + (int64_t)lane * BURG_VPT;
      const double up_from = __shfl_down_sync(0xffffffffu, v[u][0], 1);  // next lane's first
      const double dn_from = __shfl_up_sync(0xffffffffu, v[u][3], 1);    // prev lane's last
      if (ch >= nchunks) continue;
      const int64_t cs = ch * BURG_WCH;
      const int64_t ce = ((cs + BURG_WCH < n) ? cs + BURG_WCH : n);
      // neighbours of this lane's first / last cell
      const double left0 = (lane == 0) ? lft[u] : dn_from;
      double right3;
      if (i0 + BURG_VPT < ce) right3 = (lane == 31) ? rgt[u] : up_from;
      else right3 = q[ce == n ? 0 : ce];  // ragged tail: the cell after the chunk's last
      double res[BURG_VPT];
#pragma unroll
      for (int k = 0; k < BURG_VPT; ++k) {
        res[k] = 0.0;
        if (i0 + k < n) {
          const double um = (k == 0) ? left0 : v[u][k - 1];
          // the right neighbour of the chunk's last valid cell wraps at n
          double up;
          if (k < BURG_VPT - 1) up = (i0 + k + 1 < n) ? v[u][k + 1] : q[0];
          else up = right3;
          double f = burgers_cell(um, v[u][k], up, p);
          if (MODE == 1) {
            f = (v[u][k] - pv[u][k]) - dt * f;
            acc += f * f;
            bad |= !isfinite(f);
          }
          res[k] = f;
        }
      }
      if ((ch + 1) * BURG_WCH <= n) {
        *reinterpret_cast<double2*>(out + i0) = make_double2(res[0], res[1]);
        *reinterpret_cast<double2*>(out + i0 + 2) = make_double2(res[2], res[3]);
      } else {
#pragma unroll
        for (int k = 0; k < BURG_VPT; ++k)
          if (i0 + k < n) out[i0 + k] = res[k];
      }
    }
  }
  if (MODE == 1) {
    const double s = block_sum<BURG_NT>(acc, red);
    if (threadIdx.x == 0) partial[blockIdx.x] = s;
    if (bad) atomicOr(flag, 1);
  }
}

// ---------------------------------------------------------------------------
// kernel 1b: Sod residual — each interface flux evaluated once, smem staged
// ---------------------------------------------------------------------------
constexpr int SOD_NT = 256;
constexpr int SOD_TILE = 256;  // cells per tile

template <int MODE>
__global__ void __launch_bounds__(SOD_NT) sod_rhs_kernel(
    const double* __restrict__ q, double* __restrict__ out, int64_t n, double dx, double gamma,
    const double* __restrict__ qprev, double dt, double* __restrict__ partial,
    int* __restrict__ flag) {
  __shared__ double cells[3 * (SOD_TILE + 2)];
  __shared__ double faces[3 * (SOD_TILE + 1)];
  __shared__ double outs[3 * SOD_TILE];
  __shared__ double red[SOD_NT / 32];
  const int64_t ntiles = (n + SOD_TILE - 1) / SOD_TILE;
  double acc = 0.0;
  bool bad = false;
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int64_t base = t * SOD_TILE;
    const int cnt = (int)((n - base < SOD_TILE) ? (n - base) : SOD_TILE);
    __syncthreads();
    // local cell j in [0, cnt+1] holds global cell clamp(base - 1 + j):
    // the clamp IS the ghost copy of fom.py:267
    for (int e = threadIdx.x; e < 3 * (cnt + 2); e += SOD_NT) {
      const int j = e / 3, v = e - 3 * j;
      int64_t g = base - 1 + j;
      g = g < 0 ? 0 : (g > n - 1 ? n - 1 : g);
      cells[e] = q[3 * g + v];
    }
    __syncthreads();
    // face f sits between local cells f and f+1
    for (int f = threadIdx.x; f <= cnt; f += SOD_NT) {
      const Cons l{cells[3 * f], cells[3 * f + 1], cells[3 * f + 2]};
      const Cons r{cells[3 * f + 3], cells[3 * f + 4], cells[3 * f + 5]};
      const Cons fl = rusanov(l, r, gamma);
      faces[3 * f] = fl.m0;
      faces[3 * f + 1] = fl.m1;
      faces[3 * f + 2] = fl.m2;
    }
    __syncthreads();
    for (int c = threadIdx.x; c < cnt; c += SOD_NT) {
      const Cons lo{faces[3 * c], faces[3 * c + 1], faces[3 * c + 2]};
      const Cons hi{faces[3 * c + 3], faces[3 * c + 4], faces[3 * c + 5]};
      Cons o = sod_cell_from_faces(lo, hi, dx);
      if (MODE == 1) {
        const int64_t g = base + c;
        o.m0 = (cells[3 * c + 3] - qprev[3 * g]) - dt * o.m0;
        o.m1 = (cells[3 * c + 4] - qprev[3 * g + 1]) - dt * o.m1;
        o.m2 = (cells[3 * c + 5] - qprev[3 * g + 2]) - dt * o.m2;
        acc += o.m0 * o.m0 + o.m1 * o.m1 + o.m2 * o.m2;
        bad |= !(isfinite(o.m0) && isfinite(o.m1) && isfinite(o.m2));
      }
      outs[3 * c] = o.m0;
      outs[3 * c + 1] = o.m1;
      outs[3 * c + 2] = o.m2;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < 3 * cnt; e += SOD_NT) out[3 * base + e] = outs[e];
  }
  if (MODE == 1) {
    const double s = block_sum<SOD_NT>(acc, red);
    if (threadIdx.x == 0) partial[blockIdx.x] = s;
    if (bad) atomicOr(flag, 1);
  }
}


// Warp-contiguous form (replaces the tile/shared-memory kernel for the full
// grid): lane l of a warp owns cell 32 ch + l; each cell's primitives, sound
// speed and physical flux are computed once and handed to the left
// neighbour's face by shuffles (the reference's rusanov_flux evaluates them
// once per face side: the same operations on the same operands, bitwise).
// No shared memory, no barriers: 16 warps / SM keep the loads in flight.
struct SodQ {
  double f0, f1, f2, a;  // physical flux and |u| + c
};
__device__ __forceinline__ SodQ sod_q(const Cons& u, double gamma) {
  double rho, vel, p;
  euler_prim(u, gamma, rho, vel, p);
  const double c = sqrt((gamma * p) / rho);
  SodQ q;
  q.f0 = u.m1;
  q.f1 = u.m1 * vel + p;
  q.f2 = vel * (u.m2 + p);
  q.a = fabs(vel) + c;
  return q;
}
__device__ __forceinline__ Cons sod_face(const Cons& l, const SodQ& ql, const Cons& r,
                                         const SodQ& qr) {
  const double hs = 0.5 * np_max(ql.a, qr.a);
  Cons f;
  f.m0 = 0.5 * (ql.f0 + qr.f0) - hs * (r.m0 - l.m0);
  f.m1 = 0.5 * (ql.f1 + qr.f1) - hs * (r.m1 - l.m1);
  f.m2 = 0.5 * (ql.f2 + qr.f2) - hs * (r.m2 - l.m2);
  return f;
}
constexpr int SODW_NT = 256;
constexpr int SODW_CELLS = 30;  // output cells per warp chunk (lanes 1..30; 0 and 31 are halo)
// Lane l of a chunk holds cell c0 - 1 + l (clamped to the grid: the clamp IS
// the zero-gradient ghost copy of fom.py:267), so every lane evaluates its
// primitives / physical flux once, faces come from the right neighbour by a
// shuffle, and no lane runs a divergent halo branch (the former 32-cell form
// recomputed the halo cells' primitives in lanes 0 and 31, tripling the
// FP64 latency chain).  Halo cells are evaluated by both neighbouring chunks
// (2 of 32 lanes): the same operations on the same operands, bitwise.
template <int MODE>
__global__ void __launch_bounds__(SODW_NT) sod_rhs_warp_kernel(
    const double* __restrict__ q, double* __restrict__ out, int64_t n, double dx, double gamma,
    const double* __restrict__ qprev, double dt, double* __restrict__ partial,
    int* __restrict__ flag) {
  __shared__ double red[SODW_NT / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t nchunks = (n + SODW_CELLS - 1) / SODW_CELLS;
  const int64_t wstride = (int64_t)gridDim.x * (SODW_NT / 32);
  double acc = 0.0;
  bool bad = false;
  constexpr unsigned FULL = 0xffffffffu;
  auto process = [&](int64_t ch, const Cons& u) {
    const int64_t c = ch * SODW_CELLS - 1 + lane;  // this lane's cell (unclamped)
    const SodQ qu = sod_q(u, gamma);
    // face between this lane's cell and the next lane's
    Cons ur;
    SodQ qr;
    ur.m0 = __shfl_down_sync(FULL, u.m0, 1);
    ur.m1 = __shfl_down_sync(FULL, u.m1, 1);
    ur.m2 = __shfl_down_sync(FULL, u.m2, 1);
    qr.f0 = __shfl_down_sync(FULL, qu.f0, 1);
    qr.f1 = __shfl_down_sync(FULL, qu.f1, 1);
    qr.f2 = __shfl_down_sync(FULL, qu.f2, 1);
    qr.a = __shfl_down_sync(FULL, qu.a, 1);
    const Cons fr = sod_face(u, qu, ur, qr);  // lane 31: unused
    Cons fl;
    fl.m0 = __shfl_up_sync(FULL, fr.m0, 1);
    fl.m1 = __shfl_up_sync(FULL, fr.m1, 1);
    fl.m2 = __shfl_up_sync(FULL, fr.m2, 1);
    if (lane >= 1 && lane <= SODW_CELLS && c < n) {
      Cons o = sod_cell_from_faces(fl, fr, dx);
      if (MODE == 1) {
        o.m0 = (u.m0 - qprev[3 * c]) - dt * o.m0;
        o.m1 = (u.m1 - qprev[3 * c + 1]) - dt * o.m1;
        o.m2 = (u.m2 - qprev[3 * c + 2]) - dt * o.m2;
        acc += o.m0 * o.m0 + o.m1 * o.m1 + o.m2 * o.m2;
        bad |= !(isfinite(o.m0) && isfinite(o.m1) && isfinite(o.m2));
      }
      out[3 * c] = o.m0;
      out[3 * c + 1] = o.m1;
      out[3 * c + 2] = o.m2;
    }
  };
  auto cell_of = [&](int64_t ch) {
    const int64_t c = ch * SODW_CELLS - 1 + lane;
    return c < 0 ? (int64_t)0 : (c > n - 1 ? n - 1 : c);
  };
  // two chunks per iteration: both chunks' loads are in flight before either
  // is evaluated (memory-level parallelism for the latency-bound loads)
  int64_t ch = (int64_t)blockIdx.x * (SODW_NT / 32) + warp;
  for (; ch + wstride < nchunks; ch += 2 * wstride) {
    const Cons u0 = load_cons(q, cell_of(ch));
    const Cons u1 = load_cons(q, cell_of(ch + wstride));
    process(ch, u0);
    process(ch + wstride, u1);
  }
  if (ch < nchunks) process(ch, load_cons(q, cell_of(ch)));
  if (MODE == 1) {
    const double s = block_sum<SODW_NT>(acc, red);
    if (threadIdx.x == 0) partial[blockIdx.x] = s;
    if (bad) atomicOr(flag, 1);
  }
}

// deterministic final sum of per-block partials (one block)
__global__ void sum_partials_kernel(const double* __restrict__ partial, int n,
                                    double* __restrict__ out) {
  __shared__ double red[32];
  double a = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) a += partial[i];
  a = block_sum<256>(a, red);
  if (threadIdx.x == 0) out[0] = a;
}

// ---------------------------------------------------------------------------
// kernel 2: gathered residual (rhs_at_cells, fom.py:190-198 / 271-277)
// ---------------------------------------------------------------------------
__global__ void cells_kernel(int kind, const double* __restrict__ g, int64_t k,
                             BurgersParams bp, double gamma, const double* __restrict__ mech,
                             double* __restrict__ out) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < k;
       c += (int64_t)gridDim.x * blockDim.x) {
    if (kind == ADROM_BURGERS) {
      out[c] = burgers_cell(g[3 * c], g[3 * c + 1], g[3 * c + 2], bp);
    } else if (kind == ADROM_REACTING) {
      const double* s = g + 3 * RX_NV * c;
      rx_cell_res(s, s + RX_NV, s + 2 * RX_NV, gamma, bp.dx, mech, out + RX_NV * c);
    } else {
      const double* s = g + 9 * c;
      const Cons l{s[0], s[1], s[2]}, m{s[3], s[4], s[5]}, r{s[6], s[7], s[8]};
      const Cons o = sod_cell(l, m, r, gamma, bp.dx);
      out[3 * c] = o.m0;
      out[3 * c + 1] = o.m1;
      out[3 * c + 2] = o.m2;
    }
  }
}

// SamplingPlan.evaluate (fom.py:154-158) batched over n_dir FD directions:
// values = closure + h[d] * dirs[:, d]   (projection.py:185, product then sum)
__device__ __forceinline__ double plan_value(const double* __restrict__ cv,
                                             const double* __restrict__ dirs, int64_t ld,
                                             int d, double hd, int64_t pos) {
  if (dirs == nullptr) return cv[pos];
  return cv[pos] + hd * dirs[pos * ld + d];
}

__global__ void plan_kernel(int kind, const int64_t* __restrict__ gather,
                            const int64_t* __restrict__ out_cell,
                            const int64_t* __restrict__ out_var, int64_t n_s,
                            const double* __restrict__ cv, const double* __restrict__ h,
                            const double* __restrict__ dirs, int64_t ld, int n_dir,
                            BurgersParams bp, double gamma, const double* __restrict__ mech,
                            double* __restrict__ out) {
  const int nd = n_dir > 0 ? n_dir : 1;
  const int64_t total = n_s * nd;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int d = (int)(t / n_s);
    const int64_t j = t - (int64_t)d * n_s;
    const int64_t k = out_cell[j];
    const double hd = (n_dir > 0) ? h[d] : 0.0;
    const double* dd = (n_dir > 0) ? dirs : nullptr;
    double val;
    if (kind == ADROM_BURGERS) {
      const int64_t* gp = gather + 3 * k;
      val = burgers_cell(plan_value(cv, dd, ld, d, hd, gp[0]), plan_value(cv, dd, ld, d, hd, gp[1]),
                         plan_value(cv, dd, ld, d, hd, gp[2]), bp);
    } else if (kind == ADROM_REACTING) {
      const int64_t* gp = gather + 3 * RX_NV * k;
      double o[RX_NV];
      rx_cell_res_get([&](int sl, int v) { return plan_value(cv, dd, ld, d, hd, gp[sl * RX_NV + v]); },
                      gamma, bp.dx, mech, o);
      const int var = (int)out_var[j];
      val = o[0];
#pragma unroll
      for (int v = 1; v < RX_NV; ++v)
        if (v == var) val = o[v];
    } else {
      const int64_t* gp = gather + 9 * k;
      Cons s[3];
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        s[a].m0 = plan_value(cv, dd, ld, d, hd, gp[3 * a]);
        s[a].m1 = plan_value(cv, dd, ld, d, hd, gp[3 * a + 1]);
        s[a].m2 = plan_value(cv, dd, ld, d, hd, gp[3 * a + 2]);
      }
      const Cons o = sod_cell(s[0], s[1], s[2], gamma, bp.dx);
      val = cons_get(o, (int)out_var[j]);
    }
    out[t] = val;
  }
}

// ---------------------------------------------------------------------------
// banded FD Jacobian (fom.py:301-328), one thread per cell row.
// blocks[((i*3 + slot)*nv + a)*nv + b] = d rhs_{i,a} / d q_{nb(slot), b}
// apply_dt: store I - dt*J instead (fom.py:344): 1.0 - dt*J on the diagonal,
// 0.0 - dt*J elsewhere.
// ---------------------------------------------------------------------------
__device__ __forceinline__ double newton_entry(double jv, bool diag, bool apply_dt, double dt) {
  if (!apply_dt) return jv;
  return (diag ? 1.0 : 0.0) - dt * jv;
}

__global__ void burgers_jac_kernel(const double* __restrict__ q, int64_t n, BurgersParams p,
                                   double* __restrict__ blocks, bool apply_dt, double dt,
                                   int* __restrict__ flag) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t il = (i == 0) ? n - 1 : i - 1, ir = (i == n - 1) ? 0 : i + 1;
    const double um = q[il], u = q[i], up = q[ir];
    const double f0 = burgers_cell(um, u, up, p);
    const double el = fd_eps(um), ec = fd_eps(u), er = fd_eps(up);
    const double jl = (burgers_cell(um + el, u, up, p) - f0) / el;
    const double jc = (burgers_cell(um, u + ec, up, p) - f0) / ec;
    const double jr = (burgers_cell(um, u, up + er, p) - f0) / er;
    if (!(isfinite(jl) && isfinite(jc) && isfinite(jr))) atomicOr(flag, 4);
    blocks[3 * i] = newton_entry(jl, false, apply_dt, dt);
    blocks[3 * i + 1] = newton_entry(jc, true, apply_dt, dt);
    blocks[3 * i + 2] = newton_entry(jr, false, apply_dt, dt);
  }
}

__global__ void sod_jac_kernel(const double* __restrict__ q, int64_t n, double dx, double gamma,
                               double* __restrict__ blocks, bool apply_dt, double dt,
                               int* __restrict__ flag) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const bool first = (i == 0), last = (i == n - 1);
    const Cons c = load_cons(q, i);
    const Cons l = first ? c : load_cons(q, i - 1);
    const Cons r = last ? c : load_cons(q, i + 1);
    const Cons flo = rusanov(l, c, gamma), fhi = rusanov(c, r, gamma);
    const Cons f0 = sod_cell_from_faces(flo, fhi, dx);
    double* B = blocks + 27 * i;
    bool bad = false;
#pragma unroll 1
    for (int v = 0; v < 3; ++v) {
      // centre block: perturb every stencil slot that IS cell i (clamped ends)
      {
        const double e = fd_eps(cons_get(c, v));
        Cons cp = c;
        cons_set(cp, v, cons_get(c, v) + e);
        const Cons lp = first ? cp : l, rp = last ? cp : r;
        const Cons f = sod_cell(lp, cp, rp, gamma, dx);
        const double j0 = (f.m0 - f0.m0) / e, j1 = (f.m1 - f0.m1) / e, j2 = (f.m2 - f0.m2) / e;
        bad |= !(isfinite(j0) && isfinite(j1) && isfinite(j2));
        B[9 + 0 * 3 + v] = newton_entry(j0, v == 0, apply_dt, dt);
        B[9 + 1 * 3 + v] = newton_entry(j1, v == 1, apply_dt, dt);
        B[9 + 2 * 3 + v] = newton_entry(j2, v == 2, apply_dt, dt);
      }
      // left block: perturb cell i-1 (only the low face changes)
      if (!first) {
        const double e = fd_eps(cons_get(l, v));
        Cons lp = l;
        cons_set(lp, v, cons_get(l, v) + e);
        const Cons f = sod_cell_from_faces(rusanov(lp, c, gamma), fhi, dx);
        const double j0 = (f.m0 - f0.m0) / e, j1 = (f.m1 - f0.m1) / e, j2 = (f.m2 - f0.m2) / e;
        bad |= !(isfinite(j0) && isfinite(j1) && isfinite(j2));
        B[0 * 3 + v] = newton_entry(j0, false, apply_dt, dt);
        B[1 * 3 + v] = newton_entry(j1, false, apply_dt, dt);
        B[2 * 3 + v] = newton_entry(j2, false, apply_dt, dt);
      } else {
        B[0 * 3 + v] = 0.0;
        B[1 * 3 + v] = 0.0;
        B[2 * 3 + v] = 0.0;
      }
      // right block: perturb cell i+1 (only the high face changes)
      if (!last) {
        const double e = fd_eps(cons_get(r, v));
        Cons rp = r;
        cons_set(rp, v, cons_get(r, v) + e);
        const Cons f = sod_cell_from_faces(flo, rusanov(c, rp, gamma), dx);
        const double j0 = (f.m0 - f0.m0) / e, j1 = (f.m1 - f0.m1) / e, j2 = (f.m2 - f0.m2) / e;
        bad |= !(isfinite(j0) && isfinite(j1) && isfinite(j2));
        B[18 + 0 * 3 + v] = newton_entry(j0, false, apply_dt, dt);
        B[18 + 1 * 3 + v] = newton_entry(j1, false, apply_dt, dt);
        B[18 + 2 * 3 + v] = newton_entry(j2, false, apply_dt, dt);
      } else {
        B[18 + 0 * 3 + v] = 0.0;
        B[18 + 1 * 3 + v] = 0.0;
        B[18 + 2 * 3 + v] = 0.0;
      }
    }
    if (bad) atomicOr(flag, 4);
  }
}

// x += delta
__global__ void axpy1_kernel(double* __restrict__ x, const double* __restrict__ d, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    x[i] = x[i] + d[i];
}

// ---------------------------------------------------------------------------
// host wrappers
// ---------------------------------------------------------------------------
static inline int grid_for(adrom_ctx* ctx, int64_t work, int per_block, int max_per_sm = 8) {
  int64_t g = (work + per_block - 1) / per_block;
  const int64_t cap = (int64_t)ctx->num_sms * max_per_sm;
  if (g > cap) g = cap;
  return (int)(g < 1 ? 1 : g);
}

static inline BurgersParams burgers_params(const adrom_model& m) {
  BurgersParams p;
  p.dx = m.dx;
  p.nu = m.nu;
  p.dx2 = m.dx * m.dx;  // Python float dx**2 == correctly rounded dx*dx
  return p;
}

// the reacting model (kind 3) runs the residual, the FD Jacobian and the
// implicit step; its sampled-residual paths are round-2 work
static int check_model_fom(adrom_ctx* ctx, const adrom_model& m) {
  if (m.kind == ADROM_REACTING) {
    if (m.n_var != 13 || m.n_elem < 4 || !m.mech)
      return set_error(ctx, ADROM_ERR_ARG, "reacting model needs n_var=13, n_elem>=4, mech");
    return ADROM_OK;
  }
  return ADROM_OK;
}

static int check_model(adrom_ctx* ctx, const adrom_model& m) {
  if (m.kind == ADROM_BURGERS && m.n_var == 1 && m.n_elem >= 4) return ADROM_OK;
  if (m.kind == ADROM_SOD && m.n_var == 3 && m.n_elem >= 4) return ADROM_OK;
  if (m.kind == ADROM_REACTING && m.n_var == 13 && m.n_elem >= 4 && m.mech) return ADROM_OK;
  return set_error(ctx, ADROM_ERR_ARG, "unsupported model (kind=%d, n_var=%d, n_elem=%lld)",
                   m.kind, m.n_var, (long long)m.n_elem);
}

// residual launch; MODE 1 writes per-block partials into `partial`
__global__ void __launch_bounds__(256) newton_resid_kernel(const double* __restrict__ x,
                                                            const double* __restrict__ qprev,
                                                            double dt, double* __restrict__ out,
                                                            int64_t n, double* __restrict__ partial,
                                                            int* __restrict__ flag) {
  __shared__ double red[8];
  double acc = 0.0;
  bool bad = false;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double f = (x[i] - qprev[i]) - dt * out[i];
    out[i] = f;
    acc += f * f;
    bad |= !isfinite(f);
  }
  const double s2 = block_sum<256>(acc, red);
  if (threadIdx.x == 0) partial[blockIdx.x] = s2;
  if (bad) atomicOr(flag, 1);
}

static int launch_residual(adrom_ctx* ctx, const adrom_model& m, const double* x, double* out,
                           bool newton, const double* qprev, double dt, double* partial,
                           int* flag, int* nblocks_out) {
  int nb;
  if (m.kind == ADROM_REACTING) {
    int st = reacting_rhs(ctx, m, x, out);
    if (st) return st;
    nb = 0;
    if (newton) {  // r = (x - q) - dt f(x), per-block sums of r^2 (fom.py:340-341)
      nb = grid_for(ctx, m.n_elem * 13, 256);
      newton_resid_kernel<<<nb, 256, 0, ctx->stream>>>(x, qprev, dt, out, m.n_elem * 13, partial,
                                                       flag);
    }
    if (nblocks_out) *nblocks_out = nb;
    ADROM_LAUNCH_CK(ctx);
    return ADROM_OK;
  }
  if (m.kind == ADROM_BURGERS) {
    nb = grid_for(ctx, m.n_elem, BURG_TILE);
    if (newton)
      burgers_rhs_kernel<1><<<nb, BURG_NT, 0, ctx->stream>>>(x, out, m.n_elem, burgers_params(m),
                                                            qprev, dt, partial, flag);
    else
      burgers_rhs_kernel<0><<<nb, BURG_NT, 0, ctx->stream>>>(x, out, m.n_elem, burgers_params(m),
                                                            nullptr, 0.0, nullptr, nullptr);
  } else {
    nb = grid_for(ctx, m.n_elem, (SODW_NT / 32) * SODW_CELLS);
    if (newton)
      sod_rhs_warp_kernel<1><<<nb, SODW_NT, 0, ctx->stream>>>(x, out, m.n_elem, m.dx, m.gamma,
                                                            qprev, dt, partial, flag);
    else
      sod_rhs_warp_kernel<0><<<nb, SODW_NT, 0, ctx->stream>>>(x, out, m.n_elem, m.dx, m.gamma,
                                                            nullptr, 0.0, nullptr, nullptr);
  }
  if (nblocks_out) *nblocks_out = nb;
  ADROM_LAUNCH_CK(ctx);
  return ADROM_OK;
}

int fom_rhs(adrom_ctx* ctx, const adrom_model& m, const double* q, double* f) {
  if (m.kind == ADROM_REACTING) {
    if (m.n_var != 13 || m.n_elem < 4)
      return set_error(ctx, ADROM_ERR_ARG, "reacting model needs n_var=13, n_elem>=4");
    const int pr = prof_begin(ctx, PROBE_FOM_RESIDUAL);
    const int st = reacting_rhs(ctx, m, q, f);
    prof_end(ctx, pr);
    return st;
  }
  int st = check_model(ctx, m);
  if (st) return st;
  const int pr = prof_begin(ctx, PROBE_FOM_RESIDUAL);
  st = launch_residual(ctx, m, q, f, false, nullptr, 0.0, nullptr, nullptr, nullptr);
  prof_end(ctx, pr);
  return st;
}

int fom_rhs_at_cells(adrom_ctx* ctx, const adrom_model& m, const double* gathered, int64_t k,
                     double* out) {
  int st = check_model(ctx, m);
  if (st) return st;
  if (k <= 0) return ADROM_OK;
  cells_kernel<<<grid_for(ctx, k, 256), 256, 0, ctx->stream>>>(m.kind, gathered, k,
                                                               burgers_params(m), m.gamma, m.mech,
                                                               out);
  ADROM_LAUNCH_CK(ctx);
  return ADROM_OK;
}

int fom_plan_evaluate(adrom_ctx* ctx, const adrom_model& m, const int64_t* gather,
                      int64_t n_cells, const int64_t* out_cell, const int64_t* out_var,
                      int64_t n_s, const double* closure_values, const double* h,
                      const double* dirs, int64_t ld_dirs, int n_dir, double* out) {
  int st = check_model(ctx, m);
  if (st) return st;
  (void)n_cells;
  if (n_s <= 0) return ADROM_OK;
  if (n_dir > 0 && (h == nullptr || dirs == nullptr))
    return set_error(ctx, ADROM_ERR_ARG, "plan_evaluate: n_dir > 0 needs h and dirs");
  const int64_t total = n_s * (n_dir > 0 ? n_dir : 1);
  plan_kernel<<<grid_for(ctx, total, 256), 256, 0, ctx->stream>>>(
      m.kind, gather, out_cell, out_var, n_s, closure_values, h, dirs, ld_dirs, n_dir,
      burgers_params(m), m.gamma, m.mech, out);
  ADROM_LAUNCH_CK(ctx);
  return ADROM_OK;
}

static int launch_jacobian(adrom_ctx* ctx, const adrom_model& m, const double* q, double* blocks,
                           bool apply_dt, double dt, int* flag) {
  if (m.kind == ADROM_REACTING) return reacting_jacobian(ctx, m, q, blocks, apply_dt, dt, flag);
  if (m.kind == ADROM_BURGERS)
    burgers_jac_kernel<<<grid_for(ctx, m.n_elem, 256), 256, 0, ctx->stream>>>(
        q, m.n_elem, burgers_params(m), blocks, apply_dt, dt, flag);
  else
    sod_jac_kernel<<<grid_for(ctx, m.n_elem, 128), 128, 0, ctx->stream>>>(
        q, m.n_elem, m.dx, m.gamma, blocks, apply_dt, dt, flag);
  ADROM_LAUNCH_CK(ctx);
  return ADROM_OK;
}

int fom_fd_jacobian(adrom_ctx* ctx, const adrom_model& m, const double* q, double* blocks,
                    bool apply_dt, double dt) {
  int st = (m.kind == ADROM_REACTING) ? check_model_fom(ctx, m) : check_model(ctx, m);
  if (st) return st;
  st = ensure_scratch(ctx, 256);
  if (st) return st;
  int* flag = ctx->dflags + 8;
  ADROM_CK(ctx, cudaMemsetAsync(flag, 0, sizeof(int), ctx->stream));
  return launch_jacobian(ctx, m, q, blocks, apply_dt, dt, flag);
}

// ---------------------------------------------------------------------------
// backward-Euler Newton (dense.py:140-171 with fom.py:331-347)
// ---------------------------------------------------------------------------
size_t fom_newton_workspace(const adrom_model& m) {
  const int64_t N = m.n_elem * m.n_var;
  size_t b = 0;
  b += align_up(sizeof(double) * N);                               // residual r
  b += align_up(sizeof(double) * N);                               // delta
  b += align_up(sizeof(double) * m.n_elem * 3 * m.n_var * m.n_var);  // A blocks
  b += align_up(sizeof(double) * 4096);                            // partials + sums
  b += bt_workspace_bytes(m.n_elem, m.n_var);
  return b;
}

int fom_implicit_step(adrom_ctx* ctx, const adrom_model& m, const double* q, double dt,
                      double tol, int max_iter, double* x, adrom_newton_info* info) {
  int st = (m.kind == ADROM_REACTING) ? check_model_fom(ctx, m) : check_model(ctx, m);
  if (st) return st;
  if (!(tol > 0)) return set_error(ctx, ADROM_ERR_DENSE, "newton_solve requires tol > 0");
  const int64_t N = m.n_elem * m.n_var;
  st = ensure_scratch(ctx, fom_newton_workspace(m));
  if (st) return st;
  st = ensure_pinned(ctx, 64);
  if (st) return st;
  char* w = (char*)ctx->scratch;
  double* r = (double*)w;
  w += align_up(sizeof(double) * N);
  double* delta = (double*)w;
  w += align_up(sizeof(double) * N);
  double* A = (double*)w;
  w += align_up(sizeof(double) * m.n_elem * 3 * m.n_var * m.n_var);
  double* partial = (double*)w;
  double* sums = partial + 4000;
  w += align_up(sizeof(double) * 4096);
  void* btws = w;
  int* flag = ctx->dflags;
  double* hp = (double*)ctx->pinned;
  int* hflag = (int*)(hp + 2);

  ADROM_CK(ctx, cudaMemsetAsync(flag, 0, sizeof(int), ctx->stream));
  if (x != q) ADROM_CK(ctx, cudaMemcpyAsync(x, q, sizeof(double) * N, cudaMemcpyDeviceToDevice,
                                            ctx->stream));

  auto residual_norm = [&](double* rn) -> int {
    int nb = 0;
    const int pr = prof_begin(ctx, PROBE_FOM_RESIDUAL);
    int s2 = launch_residual(ctx, m, x, r, true, q, dt, partial, flag, &nb);
    prof_end(ctx, pr);
    if (s2) return s2;
    sum_partials_kernel<<<1, 256, 0, ctx->stream>>>(partial, nb, sums);
    ADROM_LAUNCH_CK(ctx);
    ADROM_CK(ctx, cudaMemcpyAsync(hp, sums, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    ADROM_CK(ctx, cudaMemcpyAsync(hflag, flag, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    ADROM_CK(ctx, cudaStreamSynchronize(ctx->stream));
    *rn = sqrt(hp[0]);
    return ADROM_OK;
  };

  double rn = 0.0;
  st = residual_norm(&rn);
  if (st) return st;
  if (*hflag & 1) return set_error(ctx, ADROM_ERR_NONFINITE, "newton residual contains non-finite entries");
  for (int it = 0; it < max_iter; ++it) {
    if (rn <= tol) {
      if (info) *info = adrom_newton_info{1, it, rn};
      return ADROM_OK;
    }
    int pr = prof_begin(ctx, PROBE_FOM_JACOBIAN);
    st = launch_jacobian(ctx, m, x, A, true, dt, flag);
    prof_end(ctx, pr);
    if (st) return st;
    // solve (I - dt J) delta = -r, then x += delta
    pr = prof_begin(ctx, PROBE_FOM_SOLVE);
    // x += delta fused into the solver's last back-substitution
    st = bt_solve(ctx, A, r, -1.0, m.n_elem, m.n_var, m.kind != ADROM_SOD, x, btws, flag, x);
    prof_end(ctx, pr);
    if (st) return st;
    (void)delta;
    st = residual_norm(&rn);
    if (st) return st;
    if (*hflag & 4)
      return set_error(ctx, ADROM_ERR_NONFINITE, "newton jacobian contains non-finite entries");
    if (*hflag & 2) return set_error(ctx, ADROM_ERR_SINGULAR, "singular Jacobian at Newton iteration %d", it);
    if (*hflag & 1)
      return set_error(ctx, ADROM_ERR_NONFINITE, "newton residual contains non-finite entries");
  }
  if (info) *info = adrom_newton_info{rn <= tol ? 1 : 0, max_iter, rn};
  return ADROM_OK;
}

}  // namespace adrom

namespace adrom {
namespace {
// fom.py:222-236 on batches of interface states (triplets), bitwise numpy
__global__ void rusanov_batch_kernel(const double* __restrict__ ul, const double* __restrict__ ur,
                                     int64_t n, double gamma, double* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const Cons l{ul[3 * i], ul[3 * i + 1], ul[3 * i + 2]};
    const Cons r{ur[3 * i], ur[3 * i + 1], ur[3 * i + 2]};
    const Cons f = rusanov(l, r, gamma);
    out[3 * i] = f.m0;
    out[3 * i + 1] = f.m1;
    out[3 * i + 2] = f.m2;
  }
}
}  // namespace
}  // namespace adrom

extern "C" int adrom_rusanov_flux(adrom_ctx* ctx, const double* ul, const double* ur, int64_t n,
                                  double gamma, double* out) {
  if (!ctx || n < 0) return ADROM_ERR_ARG;
  if (n == 0) return ADROM_OK;
  int64_t g = (n + 255) / 256;
  if (g > ctx->num_sms * 8) g = ctx->num_sms * 8;
  adrom::rusanov_batch_kernel<<<(int)g, 256, 0, ctx->stream>>>(ul, ur, n, gamma, out);
  ADROM_LAUNCH_CK(ctx);
  return ADROM_OK;
}
