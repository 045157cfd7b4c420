// Shared helpers for the adrom B200 kernels (sm_100a, fp64).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <math.h>

#include "../../include/adrom_b200.h"

#define ADROM_WARP 32

namespace adrom {

// numpy.maximum semantics: NaN in either operand propagates; otherwise max.
// (fmax() returns the non-NaN operand, which numpy does not.)
__device__ __forceinline__ double np_max(double a, double b) {
  if (a != a) return a;
  if (b != b) return b;
  return a >= b ? a : b;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Deterministic block sum (fixed reduction tree); result valid in all threads.
template <int NT>
__device__ __forceinline__ double block_sum(double v, double* sh /* >= NT/32 */) {
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x < 32) {
    t = (lane < NT / 32) ? sh[lane] : 0.0;
    t = warp_sum(t);
    if (lane == 0) sh[0] = t;
  }
  __syncthreads();
  t = sh[0];
  __syncthreads();
  return t;
}

// Runtime-sized variant (blockDim.x multiple of 32).
__device__ __forceinline__ double block_sum_dyn(double v, double* sh) {
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  __syncthreads();
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x < 32) {
    t = (lane < nw) ? sh[lane] : 0.0;
    t = warp_sum(t);
    if (lane == 0) sh[0] = t;
  }
  __syncthreads();
  t = sh[0];
  __syncthreads();
  return t;
}

// Block max (values >= 0 or NaN-free); result valid in all threads.
__device__ __forceinline__ double block_max_dyn(double v, double* sh) {
  v = warp_max(v);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  __syncthreads();
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  double t = -INFINITY;
  if (threadIdx.x < 32) {
    t = (lane < nw) ? sh[lane] : -INFINITY;
    t = warp_max(t);
    if (lane == 0) sh[0] = t;
  }
  __syncthreads();
  t = sh[0];
  __syncthreads();
  return t;
}

}  // namespace adrom

// ---------------------------------------------------------------------------
// host-side context
// ---------------------------------------------------------------------------
struct adrom_ctx {
  cudaStream_t stream = nullptr;
  int device = 0;
  int num_sms = 148;
  // growable device scratch
  void* scratch = nullptr;
  size_t scratch_bytes = 0;
  // second growable device area for internal multi-kernel stages (large
  // sampling sets: FGS ranking, plan building); never handed to callers
  void* aux = nullptr;
  size_t aux_bytes = 0;
  // device status words: [0] error code, [1] aux int, ...
  int* dflags = nullptr;
  // pinned host staging for small results
  void* pinned = nullptr;
  size_t pinned_bytes = 0;
  char err[512] = {0};
  // kernel timing probes (CUDA events on ctx->stream), see adrom_prof_*
  bool prof = false;
  int prof_used = 0;
  cudaEvent_t* prof_ev = nullptr;  // 2 * ADROM_PROF_SLOTS events
  int* prof_id = nullptr;          // probe id per slot
  long long launches = 0;          // kernels launched through this context
  // a helper context (own stream) that records its probes into the parent's
  // probe table, e.g. the session's coarse-step stream
  adrom_ctx* prof_parent = nullptr;
  // small device -> pinned-host copies that ride on the NEXT host
  // synchronisation of this stream instead of forcing their own (the
  // session's per-event status words): ride_add() registers one,
  // ride_flush() enqueues them (called right before a stream synchronise and
  // before the device words are reset); ride_done counts flushed batches
  struct Ride {
    const void* src;
    void* dst;
    size_t bytes;
  };
  Ride rides[4];
  int n_rides = 0;
  long long ride_done = 0;
};

#define ADROM_PROF_SLOTS 8192
#define ADROM_PROF_IDS 16

namespace adrom {

int set_error(adrom_ctx* ctx, int code, const char* fmt, ...);
int check_cuda(adrom_ctx* ctx, cudaError_t e, const char* where);
// scratch sub-allocation: returns a 256-byte aligned device pointer into the
// context scratch area (grown if needed; growing synchronises the stream).
void* scratch(adrom_ctx* ctx, size_t bytes, size_t offset_bytes = 0);
int ensure_scratch(adrom_ctx* ctx, size_t bytes);
int ensure_aux(adrom_ctx* ctx, size_t bytes);
int ensure_pinned(adrom_ctx* ctx, size_t bytes);
inline void ride_flush(adrom_ctx* ctx);
inline void ride_add(adrom_ctx* ctx, const void* src, void* dst, size_t bytes) {
  if (ctx->n_rides == 4) ride_flush(ctx);  // (a full table is enqueued at once, never dropped)
  ctx->rides[ctx->n_rides++] = adrom_ctx::Ride{src, dst, bytes};
}
// enqueue the registered copies on the context's stream (no synchronisation)
inline void ride_flush(adrom_ctx* ctx) {
  if (!ctx->n_rides) return;
  for (int i = 0; i < ctx->n_rides; ++i)
    cudaMemcpyAsync(ctx->rides[i].dst, ctx->rides[i].src, ctx->rides[i].bytes,
                    cudaMemcpyDeviceToHost, ctx->stream);
  ctx->n_rides = 0;
  ++ctx->ride_done;
}
inline size_t align_up(size_t x, size_t a = 256) { return (x + a - 1) / a * a; }
// upper bound on the blocks of any reduction kernel (rows of a partials buffer)
inline int partial_rows(const adrom_ctx* ctx) { return ctx->num_sms * 4; }

// probe ids (adrom_prof_read)
enum ProbeId {
  PROBE_ISVD_ROTATE = 0,
  PROBE_ISVD_PROJECT = 1,
  PROBE_ISVD_RESID = 2,
  PROBE_ISVD_CORE = 3,
  PROBE_FOM_RESIDUAL = 4,
  PROBE_FOM_JACOBIAN = 5,
  PROBE_FOM_SOLVE = 6,
  PROBE_QDEIM_ROUND = 7,
  PROBE_ROM_STEP = 8,
  PROBE_DECODE = 9,
  PROBE_OPERATOR = 10,
  PROBE_ENCODE = 11,
  PROBE_ISVD_SMALL = 12,    // least squares p = G^-1 p1, refinement, W', seeds (the r x r chain)
  PROBE_ISVD_REANCHOR = 13, // A = X W every FACT_KQ events
};
// record a begin / end event for probe `id` (no-op unless profiling)
int prof_begin(adrom_ctx* ctx, int id);
void prof_end(adrom_ctx* ctx, int slot);

}  // namespace adrom

#define ADROM_CK(ctx, call)                                          \
  do {                                                               \
    cudaError_t _e = (call);                                         \
    if (_e != cudaSuccess) return adrom::check_cuda(ctx, _e, #call); \
  } while (0)

#define ADROM_STR2(x) #x
#define ADROM_STR(x) ADROM_STR2(x)
#define ADROM_LAUNCH_CK(ctx)                                                            \
  do {                                                                                  \
    ++(ctx)->launches;                                                                  \
    cudaError_t _le = cudaGetLastError();                                               \
    if (_le != cudaSuccess)                                                             \
      return adrom::check_cuda(ctx, _le, "kernel launch at " __FILE__ ":" ADROM_STR(__LINE__)); \
  } while (0)
