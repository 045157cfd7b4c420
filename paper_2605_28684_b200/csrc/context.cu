// Context management: stream, device scratch, pinned staging, error text.
#include "common.cuh"

#include <stdarg.h>
#include <stdio.h>
#include <string.h>

namespace adrom {

int set_error(adrom_ctx* ctx, int code, const char* fmt, ...) {
  if (ctx) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(ctx->err, sizeof(ctx->err), fmt, ap);
    va_end(ap);
  }
  return code;
}

int check_cuda(adrom_ctx* ctx, cudaError_t e, const char* where) {
  return set_error(ctx, ADROM_ERR_CUDA, "CUDA error %s (%s) at %s", cudaGetErrorName(e),
                   cudaGetErrorString(e), where);
}

int ensure_scratch(adrom_ctx* ctx, size_t bytes) {
  if (bytes <= ctx->scratch_bytes && ctx->scratch) return ADROM_OK;
  size_t want = bytes < 1 << 20 ? (1 << 20) : bytes;
  want = want + want / 4;
  if (ctx->scratch) {
    ADROM_CK(ctx, cudaStreamSynchronize(ctx->stream));
    ADROM_CK(ctx, cudaFree(ctx->scratch));
    ctx->scratch = nullptr;
    ctx->scratch_bytes = 0;
  }
  ADROM_CK(ctx, cudaMalloc(&ctx->scratch, want));
  ctx->scratch_bytes = want;
  return ADROM_OK;
}

int ensure_aux(adrom_ctx* ctx, size_t bytes) {
  if (bytes <= ctx->aux_bytes && ctx->aux) return ADROM_OK;
  size_t want = bytes < 1 << 20 ? (1 << 20) : bytes;
  want = want + want / 4;
  if (ctx->aux) {
    ADROM_CK(ctx, cudaStreamSynchronize(ctx->stream));
    ADROM_CK(ctx, cudaFree(ctx->aux));
    ctx->aux = nullptr;
    ctx->aux_bytes = 0;
  }
  ADROM_CK(ctx, cudaMalloc(&ctx->aux, want));
  ctx->aux_bytes = want;
  return ADROM_OK;
}

void* scratch(adrom_ctx* ctx, size_t bytes, size_t offset_bytes) {
  (void)bytes;
  return (char*)ctx->scratch + offset_bytes;
}

int ensure_pinned(adrom_ctx* ctx, size_t bytes) {
  if (bytes <= ctx->pinned_bytes && ctx->pinned) return ADROM_OK;
  if (ctx->pinned) {
    ADROM_CK(ctx, cudaStreamSynchronize(ctx->stream));
    ADROM_CK(ctx, cudaFreeHost(ctx->pinned));
    ctx->pinned = nullptr;
  }
  size_t want = bytes < 4096 ? 4096 : bytes;
  ADROM_CK(ctx, cudaMallocHost(&ctx->pinned, want));
  ctx->pinned_bytes = want;
  return ADROM_OK;
}

int prof_begin(adrom_ctx* ctx, int id) {
  adrom_ctx* P = ctx->prof_parent ? ctx->prof_parent : ctx;
  if (!P->prof) return -1;
  // helper contexts may record from their own host thread
  const int slot = __atomic_fetch_add(&P->prof_used, 1, __ATOMIC_RELAXED);
  if (slot >= ADROM_PROF_SLOTS) return -1;
  P->prof_id[slot] = id;
  cudaEventRecord(P->prof_ev[2 * slot], ctx->stream);
  return slot;
}

void prof_end(adrom_ctx* ctx, int slot) {
  if (slot < 0) return;
  adrom_ctx* P = ctx->prof_parent ? ctx->prof_parent : ctx;
  cudaEventRecord(P->prof_ev[2 * slot + 1], ctx->stream);
}

}  // namespace adrom

extern "C" {

int adrom_prof_enable(adrom_ctx* ctx, int enable) {
  if (!ctx) return ADROM_ERR_ARG;
  if (enable && !ctx->prof_ev) {
    ctx->prof_ev = new cudaEvent_t[2 * ADROM_PROF_SLOTS];
    ctx->prof_id = new int[ADROM_PROF_SLOTS];
    for (int i = 0; i < 2 * ADROM_PROF_SLOTS; ++i)
      ADROM_CK(ctx, cudaEventCreate(&ctx->prof_ev[i]));
  }
  ctx->prof = enable != 0;
  ctx->prof_used = 0;
  return ADROM_OK;
}

int adrom_prof_read(adrom_ctx* ctx, double* host_ms, int32_t* host_count) {
  if (!ctx) return ADROM_ERR_ARG;
  for (int i = 0; i < ADROM_PROF_IDS; ++i) {
    host_ms[i] = 0.0;
    host_count[i] = 0;
  }
  if (!ctx->prof_ev) return ADROM_OK;
  ADROM_CK(ctx, cudaStreamSynchronize(ctx->stream));
  const int used = ctx->prof_used < ADROM_PROF_SLOTS ? ctx->prof_used : ADROM_PROF_SLOTS;
  for (int s = 0; s < used; ++s) {
    ADROM_CK(ctx, cudaEventSynchronize(ctx->prof_ev[2 * s + 1]));  // probes of helper streams
    float ms = 0.f;
    ADROM_CK(ctx, cudaEventElapsedTime(&ms, ctx->prof_ev[2 * s], ctx->prof_ev[2 * s + 1]));
    const int id = ctx->prof_id[s];
    if (id >= 0 && id < ADROM_PROF_IDS) {
      host_ms[id] += ms;
      host_count[id] += 1;
    }
  }
  ctx->prof_used = 0;
  return ADROM_OK;
}


int adrom_abi_version(void) { return ADROM_ABI_VERSION; }

int64_t adrom_ctx_launch_count(const adrom_ctx* ctx) { return ctx ? (int64_t)ctx->launches : 0; }

int adrom_ctx_create(adrom_ctx** out, void* stream) {
  if (!out) return ADROM_ERR_ARG;
  adrom_ctx* ctx = new adrom_ctx();
  ctx->stream = (cudaStream_t)stream;
  cudaError_t e = cudaGetDevice(&ctx->device);
  if (e != cudaSuccess) {
    delete ctx;
    *out = nullptr;
    return ADROM_ERR_CUDA;
  }
  cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, ctx->device);
  e = cudaMalloc(&ctx->dflags, 64 * sizeof(int));
  if (e != cudaSuccess) {
    delete ctx;
    *out = nullptr;
    return ADROM_ERR_CUDA;
  }
  cudaMemset(ctx->dflags, 0, 64 * sizeof(int));
  int st = adrom::ensure_pinned(ctx, 1 << 16);
  if (st) {
    cudaFree(ctx->dflags);
    delete ctx;
    *out = nullptr;
    return st;
  }
  *out = ctx;
  return ADROM_OK;
}

int adrom_ctx_set_stream(adrom_ctx* ctx, void* stream) {
  if (!ctx) return ADROM_ERR_ARG;
  ctx->stream = (cudaStream_t)stream;
  return ADROM_OK;
}

void adrom_ctx_destroy(adrom_ctx* ctx) {
  if (!ctx) return;
  cudaStreamSynchronize(ctx->stream);
  if (ctx->scratch) cudaFree(ctx->scratch);
  if (ctx->aux) cudaFree(ctx->aux);
  if (ctx->dflags) cudaFree(ctx->dflags);
  if (ctx->pinned) cudaFreeHost(ctx->pinned);
  if (ctx->prof_ev) {
    for (int i = 0; i < 2 * ADROM_PROF_SLOTS; ++i) cudaEventDestroy(ctx->prof_ev[i]);
    delete[] ctx->prof_ev;
    delete[] ctx->prof_id;
  }
  delete ctx;
}

const char* adrom_ctx_last_error(const adrom_ctx* ctx) { return ctx ? ctx->err : "null context"; }

int adrom_ctx_synchronize(adrom_ctx* ctx) {
  if (!ctx) return ADROM_ERR_ARG;
  ADROM_CK(ctx, cudaStreamSynchronize(ctx->stream));
  return ADROM_OK;
}

}  // extern "C"
