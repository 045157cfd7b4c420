// Device-resident online loop of the adaptive ROM (driver.py:291-410) and the
// C-ABI entry points for sampling, reduced operators and reduced steps.
//
// One fine step = rom_step (one block, whole Gauss-Newton loop) + decode; no
// host round-trip.  Every z steps an adaptation event runs on the device:
// coarse backward-Euler Newton of the lookahead trajectory, preprocess,
// iSVD update, QDEIM / FGS sampling, operator rebuild, state transfer.  An
// event that fails keeps the previous basis and operator (driver.py:384-385):
// the new basis / operator are built into second buffers and swapped in only
// when every stage succeeded.
#include "common.cuh"
#include "fom_internal.cuh"
#include "linalg_internal.cuh"
#include "rom_internal.cuh"
#include "sampling_internal.cuh"
#include "factored_internal.cuh"

#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <thread>
#include <vector>

using namespace adrom;

namespace {

// flags[0] also folds in dflags[PASS_A_FLAG] (written by the factored pass 1
// on the coarse-step stream, reset there before the pass)
constexpr int PASS_A_FLAG = 20;

// pinned staging slots of the status words that ride on a later
// synchronisation (ride_add): iSVD statistics, iSVD flags, reduced-step flag
constexpr size_t PIN_STATS = 512, PIN_ISVD_FLAGS = 1024, PIN_FAIL_STEP = 1280;

int read_flags(adrom_ctx* ctx, int* host_flags) {
  ADROM_CK(ctx, cudaMemcpyAsync(ctx->pinned, ctx->dflags, sizeof(int) * 24,
                                cudaMemcpyDeviceToHost, ctx->stream));
  ride_flush(ctx);
  ADROM_CK(ctx, cudaStreamSynchronize(ctx->stream));
  int tmp[24];
  memcpy(tmp, ctx->pinned, sizeof(int) * 24);
  memcpy(host_flags, tmp, sizeof(int) * 16);
  host_flags[0] |= tmp[PASS_A_FLAG];
  return ADROM_OK;
}

int reset_flags(adrom_ctx* ctx) {
  ride_flush(ctx);  // pending copies of the words read them before the reset
  ADROM_CK(ctx, cudaMemsetAsync(ctx->dflags, 0, sizeof(int) * 16, ctx->stream));
  return ADROM_OK;
}

// map device flag bits of the sampling / operator stages to reference errors
int sampling_flag_error(adrom_ctx* ctx, int f) {
  if (f & 16) return set_error(ctx, ADROM_ERR_DENSE, "not enough distinct rows to satisfy the sampling budget");
  if (f & 32) return set_error(ctx, ADROM_ERR_ARG, "sampling indices must be distinct");
  if (f & 64) return set_error(ctx, ADROM_ERR_SINGULAR, "sampled basis is rank deficient");
  if (f & 128)
    return set_error(ctx, ADROM_ERR_DENSE,
                     "sampled basis too ill-conditioned for the large-sample pseudo-inverse "
                     "(CholeskyQR2 certificate cond <= 1e8 failed)");
  if (f & 8) return set_error(ctx, ADROM_ERR_NOCONV, "SVD did not converge");
  if (f & 1) return set_error(ctx, ADROM_ERR_NONFINITE, "thin_svd input contains non-finite entries");
  return ADROM_OK;
}

__global__ void preprocess_kernel(const double* __restrict__ y, const double* __restrict__ q_ref,
                                  const double* __restrict__ d, int64_t n,
                                  double* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = d[i] * (y[i] - q_ref[i]);  // snapshots.py:47-48
}

__global__ void copy_i64_kernel(const int64_t* __restrict__ a, int64_t* __restrict__ b, int n) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) b[i] = a[i];
}

// rom-step log: per step [converged, iterations, residual]; status -> first failing step
__global__ void log_step_kernel(const double* __restrict__ info, double* __restrict__ log,
                                int64_t step, int* __restrict__ fail_step) {
  log[0] = info[0];
  log[1] = info[1];
  log[2] = info[2];
  if (info[4] != 0.0) atomicCAS(fail_step, -1, (int)step);
}

}  // namespace

// ---------------------------------------------------------------------------
// session
// ---------------------------------------------------------------------------
struct adrom_session {
  adrom_ctx* ctx = nullptr;
  adrom_session_config cfg{};
  int64_t N = 0;
  int r = 0;
  // state (device)
  double *phi[2] = {nullptr, nullptr}, *sigma[2] = {nullptr, nullptr};
  double* gram[2] = {nullptr, nullptr};  // tracked Phi^T Phi of each basis buffer
  int cur = 0;
  double *q_ref = nullptr, *d = nullptr;
  double *y_corr = nullptr, *y_next = nullptr, *y_hat = nullptr, *q_tilde = nullptr;
  double *a = nullptr;
  adrom_rom_op op[2]{};
  int opcur = 0;
  // large sampled sets (n_s > 4096, configuration 4): grid-wide plan, FGS,
  // CholeskyQR2 pseudo-inverse and Gauss-Newton step (bigsample.cu)
  bool big = false;
  BigOp bigop[2]{};
  double* rom_work = nullptr;
  double* rom_info = nullptr;
  double* isvd_stats = nullptr;
  void* isvd_ws = nullptr;
  void* qd_ws = nullptr;
  double* enc_partial = nullptr;  // fused encode partial sums (rotation epilogue)
  // factored basis (factored.cu): Phi = [phi[acur] | Qb[:, :kf]] W, W = Wd[cur]
  // (identity while w_id); sigma / gram / Wd / nrm2 are indexed by cur, the
  // anchor by acur (it only changes on a re-anchor)
  bool fact = false;
  int kf = 0, acur = 0;
  bool w_id = true;
  double* Qb = nullptr;
  // fp32 shadows of phi[b] (A32[b]), gathered by the QDEIM refresh
  float* A32[2] = {nullptr, nullptr};
  double* Wd[2] = {nullptr, nullptr};
  double* nrm2[2] = {nullptr, nullptr};
  double* vdrop[2] = {nullptr, nullptr};  // dropped direction of the event that made cur
  bool nrm2_exact = true;                 // nrm2[cur] exact (else apply vdrop[cur])
  double* fact_small = nullptr;
  double* fact_partial = nullptr;
  double* fact_rows = nullptr;
  double* fact_qv = nullptr;
  double* fact_partial_a = nullptr;
  // coarse-step stream: the advance_signal Newton solve only depends on the
  // previous coarse state, so it runs concurrently with the reduced step
  adrom_ctx* fctx = nullptr;
  cudaStream_t fstream = nullptr;
  cudaEvent_t main_mark = nullptr, fom_done = nullptr;
  // the session's own stream at the device's greatest priority: the reduced
  // steps and adaptation events (the critical path) win SM slots over the
  // coarse Newton step overlapping them on the default-priority fstream.
  // Entry points run on it with event hand-offs to and from the caller's
  // stream (ADROM_SESSION_PRIORITY=0 keeps everything on the caller's stream)
  cudaStream_t hstream = nullptr;
  cudaEvent_t ev_in = nullptr, ev_out = nullptr;
  // host_out of advance() as a ring of this many states (0 = linear)
  int64_t host_slots = 0;
  // factored path: the next event's coarse Newton solve runs on a host thread
  // (its host-side convergence checks would otherwise block the issue of this
  // event's work), started as soon as its input y_corr exists
  std::thread fom_thread;
  bool fom_pending = false;  // thread running
  bool fom_ready = false;    // finished, result not consumed yet
  int fom_status = 0;
  adrom_newton_info fom_ni{};
  // trajectory download: q~ is staged (D2D) into one of two device buffers
  // and copied to host memory on its own stream, overlapping the next steps
  cudaStream_t cstream = nullptr;
  double* stage[2] = {nullptr, nullptr};
  cudaEvent_t st_ready[2] = {nullptr, nullptr}, st_done[2] = {nullptr, nullptr};
  int64_t n_down = 0;
  double* step_log = nullptr;    // n_t_online x 3
  int* fail_step = nullptr;
  bool fail_step_read = false;  // the last event brought fail_step back with its status words
  int64_t n_online = 0;          // steps done
  int64_t cap_steps = 0;
  std::vector<adrom_event_record> events;
  std::vector<void*> allocs;

  double* alloc_d(size_t n) {
    void* p = nullptr;
    if (cudaMalloc(&p, sizeof(double) * (n ? n : 1)) != cudaSuccess) return nullptr;
    allocs.push_back(p);
    return (double*)p;
  }
  template <typename T>
  T* alloc_t(size_t n) {
    void* p = nullptr;
    if (cudaMalloc(&p, sizeof(T) * (n ? n : 1)) != cudaSuccess) return nullptr;
    allocs.push_back(p);
    return (T*)p;
  }
};

namespace {

adrom_model model_of(const adrom_session* s) { return s->cfg.model; }

// the current basis as a factored view (W = null: phi[acur] itself)
FactBasis basis_view(const adrom_session* s) {
  return FactBasis{s->phi[s->acur], s->Qb, s->r, s->w_id ? 0 : s->kf,
                   s->w_id ? nullptr : s->Wd[s->cur], s->N, s->A32[s->acur]};
}

__global__ void to_f32_kernel(const double* __restrict__ x, int64_t n, float* __restrict__ y) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    y[i] = (float)x[i];
}

__global__ void row_norms_kernel(const double* __restrict__ phi, int64_t n, int r,
                                 double* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int c = 0; c < r; ++c) s += phi[i * r + c] * phi[i * r + c];
    out[i] = s;
  }
}

// runs an entry point on the session's high-priority stream
struct HiPrio {
  adrom_session* s;
  cudaStream_t user;
  explicit HiPrio(adrom_session* ss) : s(ss), user(ss->ctx->stream) {
    if (!s->hstream) return;
    cudaEventRecord(s->ev_in, user);
    cudaStreamWaitEvent(s->hstream, s->ev_in, 0);
    s->ctx->stream = s->hstream;
  }
  ~HiPrio() {
    if (!s->hstream) return;
    cudaEventRecord(s->ev_out, s->hstream);
    cudaStreamWaitEvent(user, s->ev_out, 0);
    s->ctx->stream = user;
  }
};

int alloc_op(adrom_session* s, adrom_rom_op& op, BigOp& big) {
  const int ns = s->cfg.n_s, nv = s->cfg.model.n_var, r = s->r;
  const int64_t ne = s->cfg.model.n_elem;
  op.r = r;
  op.n_var = nv;
  op.ns_cap = ns;
  // sampled cells: at most n_s, the grid, and for FGS (whole cells on top of
  // n_base QDEIM rows) 2 n_base + ceil(n_extra / n_var) + 1; at most 3
  // stencil cells per sampled cell
  int64_t cells = (ns < ne) ? ns : ne;
  if (s->cfg.sampling == 1) {
    const int64_t nb = ns - s->cfg.n_extra;
    const int64_t fc = 2 * nb + (s->cfg.n_extra + nv - 1) / nv + 1;
    if (fc < cells) cells = fc;
  }
  const int64_t cells_c = (3 * cells < ne) ? 3 * cells : ne;
  op.nc_cap = (int32_t)(cells_c * nv);
  op.ncell_cap = (int32_t)cells;
  if (s->big) {
    big.cell_start = s->alloc_t<int64_t>(op.ncell_cap);
    big.cell_cnt = s->alloc_t<int32_t>(op.ncell_cap);
    big.rows = s->alloc_t<int32_t>(ns);
  }
  op.idx = s->alloc_t<int64_t>(ns);
  op.closure = s->alloc_t<int64_t>(op.nc_cap);
  op.gather = s->alloc_t<int64_t>((size_t)op.ncell_cap * 3 * nv);
  op.out_cell = s->alloc_t<int64_t>(ns);
  op.out_var = s->alloc_t<int64_t>(ns);
  op.sample_pos = s->alloc_t<int64_t>(ns);
  op.sizes = s->alloc_t<int32_t>(4);
  op.pinv = s->alloc_d((size_t)r * ns);
  op.d_s = s->alloc_d(ns);
  op.q_ref_c = s->alloc_d(op.nc_cap);
  op.dinv_phi_c = s->alloc_d((size_t)op.nc_cap * r);
  op.phi_s = s->alloc_d((size_t)ns * r);
  if (!op.phi_s) return set_error(s->ctx, ADROM_ERR_CUDA, "session: device allocation failed");
  return ADROM_OK;
}

// sampling (driver.py:264-273) + closure + operator for basis `phi` into op
int build_sampling_operator(adrom_session* s, const double* phi, adrom_rom_op& op,
                            const double* y_corr, bool seeded = false,
                            const FactBasis* fb = nullptr, const double* nrmb = nullptr) {
  adrom_ctx* ctx = s->ctx;
  const adrom_model m = model_of(s);
  const int n_s = s->cfg.n_s;
  int st;
  int it = 0;
  const int n_q = (s->cfg.sampling == 1) ? n_s - s->cfg.n_extra : n_s;  // QDEIM rows
  if (fb && fb->W && n_q > s->r) {
    // restarted QDEIM on a factored basis: materialise Phi into the spare
    // anchor buffer and run the explicit path (unseeded)
    st = fact_reanchor(ctx, *fb, s->phi[1 - s->acur], nullptr);
    if (st) return st;
    phi = s->phi[1 - s->acur];
    fb = nullptr;
    seeded = false;
  }
  // factored rows that stall the certification: materialise and rerun
  auto qdeim = [&](int count) -> int {
    int st2 = qdeim_pool_select(ctx, phi, s->N, s->r, count, op.idx, s->qd_ws, &it, seeded, fb, nrmb);
    if (st2 != QDEIM_NEEDS_EXPLICIT) return st2;
    st2 = fact_reanchor(ctx, *fb, s->phi[1 - s->acur], nullptr);
    if (st2) return st2;
    phi = s->phi[1 - s->acur];
    fb = nullptr;
    seeded = false;
    return qdeim_pool_select(ctx, phi, s->N, s->r, count, op.idx, s->qd_ws, &it, false);
  };
  if (s->cfg.sampling == 1) {
    const int n_base = n_s - s->cfg.n_extra;
    if (n_base > 0) {
      st = qdeim(n_base);
      if (st) return st;
    }
    st = reset_flags(ctx);
    if (st) return st;
    st = fgs_extend(ctx, m, y_corr, s->cfg.feature, op.idx, n_base, s->cfg.n_extra, nullptr);
    if (st) return st;
  } else {
    st = qdeim(n_s);
    if (st) return st;
    st = reset_flags(ctx);
    if (st) return st;
  }
  const int pr = prof_begin(ctx, PROBE_OPERATOR);
  st = s->big ? plan_build_big(ctx, m, op, s->bigop[&op == &s->op[0] ? 0 : 1], n_s, ctx->dflags)
              : plan_build(ctx, m, op, n_s, ctx->dflags);
  if (st) return st;
  st = operator_fill(ctx, op, phi, s->q_ref, s->d, n_s, ctx->dflags, fb, s->fact_rows,
                     s->big ? s->rom_work : nullptr);
  prof_end(ctx, pr);
  if (st) return st;
  int flags[16];
  st = read_flags(ctx, flags);
  if (st) return st;
  return sampling_flag_error(ctx, flags[0]);
}

int encode_into(adrom_session* s, const double* phi, const double* q, double* a) {
  adrom_ctx* ctx = s->ctx;
  double* partial = (double*)s->isvd_ws;  // first region of the iSVD workspace
  double* out = s->rom_info + 16;         // r+1 doubles after the info block
  const int pr = prof_begin(ctx, PROBE_ENCODE);
  int st = ts_project(ctx, phi, s->N, s->r, 2, q, s->q_ref, s->d, out, partial, nullptr);
  prof_end(ctx, pr);
  if (st) return st;
  ADROM_CK(ctx, cudaMemcpyAsync(a, out, sizeof(double) * s->r, cudaMemcpyDeviceToDevice,
                                ctx->stream));
  return ADROM_OK;
}

int rom_step(adrom_session* s) {
  RomStepArgs A{};
  A.op = s->op[s->opcur];
  A.kind = s->cfg.model.kind;
  A.bp = make_bp(s->cfg.model);
  A.gamma = s->cfg.model.gamma;
  A.mech = s->cfg.model.mech;
  A.a_prev = s->a;
  A.a_out = s->a;
  A.dt = s->cfg.dt;
  A.tol = s->cfg.newton_tol;
  A.max_iter = s->cfg.newton_max_iter;
  A.work = s->rom_work;
  A.info = s->rom_info;
  int st;
  if (s->big)
    st = (s->cfg.projection == 0)
             ? lspg_step_big(s->ctx, A, s->bigop[s->opcur], s->cfg.n_s)
             : set_error(s->ctx, ADROM_ERR_ARG, "galerkin on n_s > 4096 sampled rows is not supported");
  else
    st = rom_step_async(s->ctx, A, s->cfg.projection == 0);
  if (st) return st;
  if (s->n_online < s->cap_steps) {
    log_step_kernel<<<1, 1, 0, s->ctx->stream>>>(s->rom_info, s->step_log + 3 * s->n_online,
                                                 s->n_online, s->fail_step);
    ADROM_LAUNCH_CK(s->ctx);
  }
  return ADROM_OK;
}

// q~ = q_ref + (Phi a) / d with the current basis (projection.py:104)
int decode_state(adrom_session* s) {
  adrom_ctx* ctx = s->ctx;
  const int pr = prof_begin(ctx, PROBE_DECODE);
  int st;
  if (s->fact && !s->w_id)
    st = fact_decode(ctx, basis_view(s), s->a, s->q_ref, s->d, s->q_tilde, s->fact_small,
                     s->fact_partial);
  else
    st = ts_decode(ctx, s->phi[s->acur], s->N, s->r, s->a, s->q_ref, s->d, s->q_tilde);
  prof_end(ctx, pr);
  return st;
}

// Copy q~ to (pinned) host memory without stalling the loop: D2D into a
// staging slot on the main stream, D2H on the copy stream.
int download_state(adrom_session* s, double* host_dst) {
  adrom_ctx* ctx = s->ctx;
  const size_t bytes = sizeof(double) * (size_t)s->N;
  if (!s->cstream) {
    if (cudaStreamCreateWithFlags(&s->cstream, cudaStreamNonBlocking) != cudaSuccess)
      return set_error(ctx, ADROM_ERR_CUDA, "session: copy stream creation failed");
    for (int b = 0; b < 2; ++b) {
      s->stage[b] = s->alloc_d((size_t)s->N);
      if (!s->stage[b] || cudaEventCreateWithFlags(&s->st_ready[b], cudaEventDisableTiming) ||
          cudaEventCreateWithFlags(&s->st_done[b], cudaEventDisableTiming))
        return set_error(ctx, ADROM_ERR_CUDA, "session: staging allocation failed");
    }
  }
  const int b = (int)(s->n_down & 1);
  if (s->n_down >= 2) ADROM_CK(ctx, cudaStreamWaitEvent(ctx->stream, s->st_done[b], 0));
  ADROM_CK(ctx, cudaMemcpyAsync(s->stage[b], s->q_tilde, bytes, cudaMemcpyDeviceToDevice,
                                ctx->stream));
  ADROM_CK(ctx, cudaEventRecord(s->st_ready[b], ctx->stream));
  ADROM_CK(ctx, cudaStreamWaitEvent(s->cstream, s->st_ready[b], 0));
  ADROM_CK(ctx, cudaMemcpyAsync(host_dst, s->stage[b], bytes, cudaMemcpyDeviceToHost, s->cstream));
  ADROM_CK(ctx, cudaEventRecord(s->st_done[b], s->cstream));
  ++s->n_down;
  return ADROM_OK;
}

int drain_downloads(adrom_session* s) {
  if (s->cstream) ADROM_CK(s->ctx, cudaStreamSynchronize(s->cstream));
  return ADROM_OK;
}

void fom_launch_async(adrom_session* s) {
  if (s->fom_pending || s->fom_ready) return;
  const adrom_model m = model_of(s);
  const double* in = s->y_corr;
  double* out = s->y_next;
  // the coarse-step stream first waits for everything enqueued on the main
  // stream so far (the input y_corr may come from it, and the output buffer
  // was last read by it)
  cudaEventRecord(s->main_mark, s->ctx->stream);
  cudaStreamWaitEvent(s->fctx->stream, s->main_mark, 0);
  s->fom_pending = true;
  s->fom_thread = std::thread([s, m, in, out]() {
    s->fom_status = fom_implicit_step(s->fctx, m, in, s->cfg.z * s->cfg.dt, s->cfg.newton_tol,
                                      s->cfg.newton_max_iter, out, &s->fom_ni);
  });
}

void fom_wait(adrom_session* s) {
  if (!s->fom_pending) return;
  s->fom_thread.join();
  s->fom_pending = false;
  s->fom_ready = true;
}

// result of the started coarse step (consumed)
int fom_join(adrom_session* s, adrom_newton_info* ni) {
  fom_wait(s);
  s->fom_ready = false;
  *ni = s->fom_ni;
  return s->fom_status;
}

// the rest of an event on the factored basis (after the coarse step and
// preprocess): no rotation — the residual becomes column kf of Qb and
// W' = [[W, 0], [0, 1/||q||]] B; committed only if every stage succeeds
int run_event_factored(adrom_session* s, adrom_event_record& ev, bool* decoded) {
  adrom_ctx* ctx = s->ctx;
  adrom_ctx* fc = s->fctx;
  int st;
  // on the coarse-step stream, still overlapping the reduced step: snapshot
  // preprocess, re-anchor when due, pass 1 (X^T y, exact row norms)
  preprocess_kernel<<<(int)((s->N + 255) / 256 < ctx->num_sms * 8 ? (s->N + 255) / 256
                                                                   : ctx->num_sms * 8),
                      256, 0, fc->stream>>>(s->y_corr, s->q_ref, s->d, s->N, s->y_hat);
  ADROM_LAUNCH_CK(fc);
  if (s->kf == FACT_KQ) {  // re-anchor: A = X W (same basis), exact row norms
    st = fact_reanchor(fc, basis_view(s), s->phi[1 - s->acur], s->nrm2[s->cur],
                       s->A32[1 - s->acur]);
    if (st) return st;
    s->acur = 1 - s->acur;
    s->kf = 0;
    s->w_id = true;
    s->nrm2_exact = true;
  }
  const int nxt = 1 - s->cur;
  const FactBasis b = basis_view(s);
  FactEventArgs e{};
  e.y = s->y_hat;
  e.a = s->a;
  e.q_ref = s->q_ref;
  e.d = s->d;
  e.q_tilde = s->q_tilde;
  e.Qw = s->Qb;
  e.qv = s->fact_qv;
  e.sigma = s->sigma[s->cur];
  e.G = s->gram[s->cur];
  e.lam = s->cfg.lam;
  e.partial = s->fact_partial;
  e.partial_a = s->fact_partial_a;
  e.flag_a = ctx->dflags + PASS_A_FLAG;
  e.small = s->fact_small;
  e.W_out = s->Wd[nxt];
  e.sigma_out = s->sigma[nxt];
  e.G_out = s->gram[nxt];
  double* a_new = s->rom_info + 16;
  e.a_out = a_new;
  e.stats = s->isvd_stats;
  e.flag = ctx->dflags;
  e.nrm2_inout = s->nrm2[s->cur];
  e.vdrop_in = s->nrm2_exact ? nullptr : s->vdrop[s->cur];
  e.vdrop_out = s->vdrop[nxt];
  e.nrm2_out = s->nrm2[nxt];
  qdeim_seed_buffers(s->qd_ws, s->N, &e.seed_res2, &e.seed_bnd2, &e.seed_ver);
  ADROM_CK(ctx, cudaMemsetAsync(e.flag_a, 0, sizeof(int), fc->stream));
  const long long l0 = fc->launches;
  st = fact_event_pass_a(fc, b, e);
  ctx->launches += fc->launches - l0;
  if (st) {
    snprintf(ctx->err, sizeof(ctx->err), "%s", fc->err);
    return st;
  }
  ADROM_CK(ctx, cudaEventRecord(s->fom_done, fc->stream));
  ADROM_CK(ctx, cudaStreamWaitEvent(ctx->stream, s->fom_done, 0));
  // the next event's coarse step only needs this y_corr: start it now (it
  // queues behind pass 1 on the coarse-step stream)
  fom_launch_async(s);
  st = reset_flags(ctx);
  if (st) return st;
  st = fact_event_pass_b(ctx, b, e);
  if (st) return st;
  *decoded = true;
  s->nrm2_exact = true;  // pass 1 made nrm2[cur] exact for the current basis
  // the iSVD's status words ride on the sampling stage's first host
  // synchronisation (a QDEIM round); the sampling and the operator write only
  // spare buffers, so a failed update costs nothing but their time
  ride_add(ctx, s->isvd_stats, (char*)ctx->pinned + PIN_STATS, sizeof(double) * 8);
  ride_add(ctx, ctx->dflags, (char*)ctx->pinned + PIN_ISVD_FLAGS, sizeof(int) * 24);
  const FactBasis b2{s->phi[s->acur], s->Qb,     s->r,           b.k + 1,
                     s->Wd[nxt],       s->N,      s->A32[s->acur],
                     getenv("ADROM_QDEIM_NO_VDROP") ? nullptr : s->vdrop[nxt]};
  const int onx = 1 - s->opcur;
  // the reduced step's failure flag shares the operator's final read
  ride_add(ctx, s->fail_step, (char*)ctx->pinned + PIN_FAIL_STEP, sizeof(int));
  st = build_sampling_operator(s, nullptr, s->op[onx], s->y_corr, true, &b2, s->nrm2[nxt]);
  if (st == ADROM_ERR_CUDA) return st;
  if (st) {  // an error return may precede the stage's synchronisation
    ride_flush(ctx);
    ADROM_CK(ctx, cudaStreamSynchronize(ctx->stream));
  }
  s->fail_step_read = true;  // pinned + PIN_FAIL_STEP holds this step's flag
  const double* hs = (const double*)((char*)ctx->pinned + PIN_STATS);
  int iflags[24];
  memcpy(iflags, (char*)ctx->pinned + PIN_ISVD_FLAGS, sizeof(iflags));
  iflags[0] |= iflags[PASS_A_FLAG];
  if (iflags[0] & 1) {
    ev.error = ADROM_ERR_NONFINITE;
    return ADROM_OK;
  }
  if (iflags[0] & 8) {
    ev.error = ADROM_ERR_NOCONV;
    return ADROM_OK;
  }
  ev.residual_norm = hs[2];
  if (getenv("ADROM_DEBUG_CORE"))
    fprintf(stderr, "core: sweeps %g converged %g fallback %g\n", hs[5], hs[6], hs[7]);
  if (st) {
    ev.error = st;
    return ADROM_OK;
  }
  ADROM_CK(ctx, cudaMemcpyAsync(s->a, a_new, sizeof(double) * s->r, cudaMemcpyDeviceToDevice,
                                ctx->stream));
  s->kf = b.k + 1;
  s->w_id = false;
  s->cur = nxt;
  s->opcur = onx;
  s->nrm2_exact = false;  // nrm2[cur] is the seed bound; vdrop[cur] corrects it
  return ADROM_OK;
}

// one adaptation event (driver.py:351-387, history-aware branch).  The
// decode of the reduced state (driver.py:345) rides on the iSVD's first pass
// over the old basis (*decoded = true); the state transfer (encode, :376) and
// the QDEIM seed bounds ride on the rotation that writes the new basis.
int run_event(adrom_session* s, adrom_event_record& ev, bool* decoded) {
  adrom_ctx* ctx = s->ctx;
  const adrom_model m = model_of(s);
  *decoded = false;
  ev.error = 0;
  ev.residual_norm = 0.0;
  // advance_signal: coarse backward-Euler step of size z*dt (driver.py:354-358)
  // on the coarse-step stream, after every main-stream operation that came
  // before this step's reduced step (main_mark), overlapping that step
  adrom_newton_info ni{};
  adrom_ctx* fc = s->fctx;
  const long long l0 = fc->launches;
  int st;
  // started early on a host thread (fom_launch_async, right after the
  // previous event) unless this is the first event or the previous coarse
  // step failed; it then overlapped the last z reduced steps
  fom_launch_async(s);  // no-op when already started / finished
  st = fom_join(s, &ni);
  ctx->launches += fc->launches - l0;
  if (st || !s->fact) {  // (the factored path joins after its pass 1)
    ADROM_CK(ctx, cudaEventRecord(s->fom_done, fc->stream));
    ADROM_CK(ctx, cudaStreamWaitEvent(ctx->stream, s->fom_done, 0));
  }
  if (st) {
    snprintf(ctx->err, sizeof(ctx->err), "%s", fc->err);
    if (st == ADROM_ERR_CUDA) return st;
    ev.error = st;
    return ADROM_OK;
  }
  std::swap(s->y_corr, s->y_next);
  ev.coarse_converged = ni.converged;
  ev.coarse_iterations = ni.iterations;
  ev.pad = 1;  // coarse advance done (event dict carries coarse_* keys)
  if (s->fact) return run_event_factored(s, ev, decoded);
  // y_hat = D (y - q_ref)
  preprocess_kernel<<<(int)((s->N + 255) / 256 < ctx->num_sms * 8 ? (s->N + 255) / 256
                                                                   : ctx->num_sms * 8),
                      256, 0, ctx->stream>>>(s->y_corr, s->q_ref, s->d, s->N, s->y_hat);
  ADROM_LAUNCH_CK(ctx);
  // iSVD into the spare buffers
  const int nxt = 1 - s->cur;
  const bool fused = rot_fusable(s->r, s->r);
  RotFuse fz;
  if (fused) {
    fz.enc_x = s->q_tilde;
    fz.enc_q_ref = s->q_ref;
    fz.enc_d = s->d;
    fz.enc_partial = s->enc_partial;
    qdeim_seed_buffers(s->qd_ws, s->N, &fz.seed_res2, &fz.seed_bnd2, &fz.seed_ver);
  }
  st = reset_flags(ctx);
  if (st) return st;
  st = isvd_update_async(ctx, s->phi[s->cur], s->sigma[s->cur], s->y_hat, s->N, s->r, s->r,
                         s->cfg.lam, s->phi[nxt], s->sigma[nxt], s->gram[s->cur], s->gram[nxt],
                         s->isvd_ws, ctx->dflags, ISVD_REORTH_RATIO, s->isvd_stats, s->a,
                         s->q_ref, s->d, s->q_tilde, fused ? &fz : nullptr);
  if (st) return st;
  *decoded = true;
  int flags[16];
  ADROM_CK(ctx, cudaMemcpyAsync((char*)ctx->pinned + 512, s->isvd_stats, sizeof(double) * 8,
                                cudaMemcpyDeviceToHost, ctx->stream));
  st = read_flags(ctx, flags);
  if (st) return st;
  const double* hs = (const double*)((char*)ctx->pinned + 512);
  if (flags[0] & 1) {
    ev.error = ADROM_ERR_NONFINITE;
    return ADROM_OK;
  }
  if (flags[0] & 8) {
    ev.error = ADROM_ERR_NOCONV;
    return ADROM_OK;
  }
  ev.residual_norm = hs[2];  // ||y - Phi Phi^T y|| with the old basis (driver.py:366-367)
  // sampling + operator for the new basis (driver.py:369-374)
  const int onx = 1 - s->opcur;
  st = build_sampling_operator(s, s->phi[nxt], s->op[onx], s->y_corr, fused);
  if (st == ADROM_ERR_CUDA) return st;
  if (st) {
    ev.error = st;
    return ADROM_OK;
  }
  // state transfer a = Phi'^T D (q~ - q_ref)  (driver.py:376)
  if (fused) {
    const int pr = prof_begin(ctx, PROBE_ENCODE);
    st = rot_encode_finish(ctx, fz, s->N, s->r, s->rom_info + 16);
    prof_end(ctx, pr);
    if (st) return st;
    ADROM_CK(ctx, cudaMemcpyAsync(s->a, s->rom_info + 16, sizeof(double) * s->r,
                                  cudaMemcpyDeviceToDevice, ctx->stream));
  } else {
    st = encode_into(s, s->phi[nxt], s->q_tilde, s->a);
    if (st) return st;
  }
  s->cur = nxt;
  s->acur = nxt;
  s->opcur = onx;
  return ADROM_OK;
}

}  // namespace

extern "C" {

int adrom_session_create(adrom_ctx* ctx, const adrom_session_config* cfg, adrom_session** out) {
  if (!ctx || !cfg || !out) return ADROM_ERR_ARG;
  adrom_session* s = new adrom_session();
  s->ctx = ctx;
  s->cfg = *cfg;
  s->N = cfg->model.n_elem * cfg->model.n_var;
  s->r = cfg->r;
  if (cfg->r < 1 || cfg->r > 128 || cfg->n_s < cfg->r || cfg->z < 1) {
    delete s;
    return set_error(ctx, ADROM_ERR_ARG, "session: bad r/n_s/z");
  }
  const int64_t N = s->N;
  const int r = s->r;
  for (int b = 0; b < 2; ++b) {
    s->phi[b] = s->alloc_d((size_t)N * r);
    s->sigma[b] = s->alloc_d(r);
    s->gram[b] = s->alloc_d((size_t)r * r);
  }
  s->q_ref = s->alloc_d(N);
  s->d = s->alloc_d(N);
  s->y_corr = s->alloc_d(N);
  s->y_next = s->alloc_d(N);
  s->y_hat = s->alloc_d(N);
  s->q_tilde = s->alloc_d(N);
  s->a = s->alloc_d(r);
  {
    // grid-wide reduced operator (bigsample.cu) from 256 sampled rows: the
    // one-block kernels win below that (cfg 0: 16 rows, cfg 3: 64 rows) and
    // lose above (cfg 1, 615 rows: 635 -> 1429 steps/s); they cannot hold
    // more than 4096 rows.  ADROM_BIG_SAMPLES=0/1 overrides (tests)
    const char* ev = getenv("ADROM_BIG_SAMPLES");
    s->big = ev ? (atoi(ev) != 0 || cfg->n_s > 4096) : (cfg->n_s >= 256);
    // the grid-wide path implements LSPG only (Galerkin keeps the one-block
    // kernels up to their 4096-row limit)
    if (cfg->projection != 0 && cfg->n_s <= 4096) s->big = false;
  }
  int st = alloc_op(s, s->op[0], s->bigop[0]);
  if (!st) st = alloc_op(s, s->op[1], s->bigop[1]);
  {
    size_t w = rom_step_work_doubles(s->op[0]);
    if (s->big) {
      const size_t wb = big_work_doubles(s->op[0]);
      const size_t wp = deim_pinv_big_work_doubles(cfg->n_s, r);
      w = wb > wp ? wb : wp;
    }
    s->rom_work = s->alloc_d(w);
  }
  s->rom_info = s->alloc_d(16 + r + 1 + 16);
  s->isvd_stats = s->alloc_d(16);
  const size_t iws = isvd_workspace_bytes(ctx, N, r, r);
  cudaMalloc(&s->isvd_ws, iws);
  s->allocs.push_back(s->isvd_ws);
  {
    // QDEIM picks n_s rows (qdeim) or the n_s - n_extra base rows (fgs)
    const int n_q = (cfg->sampling == 1) ? cfg->n_s - cfg->n_extra : cfg->n_s;
    cudaMalloc(&s->qd_ws, qdeim_pool_workspace_bytes(N, r, n_q > 0 ? n_q : 1));
  }
  s->allocs.push_back(s->qd_ws);
  s->enc_partial = s->alloc_d(rot_fuse_partial_doubles(ctx, r));
  {
    // factored basis: r in {32, 64} at scale (ADROM_FACTORED=0/1 overrides)
    const char* ev = getenv("ADROM_FACTORED");
    const bool shape_ok = (r == 32 || r == 64);
    s->fact = shape_ok && !s->big && (ev ? atoi(ev) != 0 : N >= (1 << 18));
  }
  if (s->fact) {
    s->Qb = s->alloc_d((size_t)N * FACT_KQ);
    for (int b = 0; b < 2; ++b) {
      s->Wd[b] = s->alloc_d((size_t)(r + FACT_KQ + 1) * r);
      s->nrm2[b] = s->alloc_d((size_t)N);
      s->vdrop[b] = s->alloc_d((size_t)(r + FACT_KQ + 1));
    }
    s->fact_small = s->alloc_d(fact_small_doubles(r));
    s->fact_partial = s->alloc_d(fact_partial_doubles(ctx, N, r));
    s->fact_partial_a = s->alloc_d(fact_partial_doubles(ctx, N, r));
    s->fact_rows = s->alloc_d((size_t)(3 * cfg->n_s * cfg->model.n_var + cfg->n_s) * r);
    s->fact_qv = s->alloc_d((size_t)N);
    if (s->Qb) cudaMemsetAsync(s->Qb, 0, sizeof(double) * (size_t)N * FACT_KQ, ctx->stream);
    if (!getenv("ADROM_NO_SHADOW") || !atoi(getenv("ADROM_NO_SHADOW"))) {
      // fp32 anchor shadows for the QDEIM refresh (optional: null -> fp64 gathers)
      for (int b = 0; b < 2; ++b) s->A32[b] = s->alloc_t<float>((size_t)N * r);
      if (!s->A32[0] || !s->A32[1]) {
        s->A32[0] = s->A32[1] = nullptr;
        cudaGetLastError();
      }
    }
  }
  s->cap_steps = cfg->n_t > cfg->w_init ? cfg->n_t - cfg->w_init : 1;
  s->step_log = s->alloc_d((size_t)s->cap_steps * 3);
  s->fail_step = s->alloc_t<int>(1);
  if (s->fact && (!s->Qb || !s->nrm2[1] || !s->fact_rows || !s->fact_partial || !s->fact_qv ||
                  !s->fact_partial_a))
    st = set_error(ctx, ADROM_ERR_CUDA, "session: device allocation failed (factored basis)");
  if (st || !s->phi[1] || !s->step_log || !s->fail_step || !s->qd_ws || !s->isvd_ws) {
    for (void* p : s->allocs) cudaFree(p);
    delete s;
    return set_error(ctx, ADROM_ERR_CUDA, "session: device allocation failed (N=%lld r=%d)",
                     (long long)N, r);
  }
  cudaMemsetAsync(s->fail_step, 0xff, sizeof(int), ctx->stream);  // -1
  size_t need = fom_newton_workspace(cfg->model) + 4096;
  st = ensure_scratch(ctx, need);
  if (!st && cudaStreamCreateWithFlags(&s->fstream, cudaStreamNonBlocking) != cudaSuccess)
    st = set_error(ctx, ADROM_ERR_CUDA, "session: stream creation failed");
  if (!st) st = adrom_ctx_create(&s->fctx, s->fstream);
  if (!st) {
    s->fctx->prof_parent = ctx;
    st = ensure_scratch(s->fctx, need);
    if (st) set_error(ctx, st, "session: coarse-step workspace (%zu bytes): %s", need, s->fctx->err);
  }
  if (!st && (cudaEventCreateWithFlags(&s->main_mark, cudaEventDisableTiming) != cudaSuccess ||
              cudaEventCreateWithFlags(&s->fom_done, cudaEventDisableTiming) != cudaSuccess))
    st = set_error(ctx, ADROM_ERR_CUDA, "session: event creation failed");
  if (!st) {
    const char* ev = getenv("ADROM_SESSION_PRIORITY");
    if (!ev || atoi(ev) != 0) {
      int least = 0, greatest = 0;
      cudaDeviceGetStreamPriorityRange(&least, &greatest);
      if (cudaStreamCreateWithPriority(&s->hstream, cudaStreamNonBlocking, greatest) != cudaSuccess ||
          cudaEventCreateWithFlags(&s->ev_in, cudaEventDisableTiming) != cudaSuccess ||
          cudaEventCreateWithFlags(&s->ev_out, cudaEventDisableTiming) != cudaSuccess)
        st = set_error(ctx, ADROM_ERR_CUDA, "session: priority stream creation failed");
    }
  }
  if (st) {
    adrom_session_destroy(s);
    return st;
  }
  *out = s;
  return ADROM_OK;
}

void adrom_session_destroy(adrom_session* s) {
  if (!s) return;
  fom_wait(s);
  cudaStreamSynchronize(s->ctx->stream);
  if (s->fctx) adrom_ctx_destroy(s->fctx);
  if (s->fstream) cudaStreamDestroy(s->fstream);
  if (s->main_mark) cudaEventDestroy(s->main_mark);
  if (s->fom_done) cudaEventDestroy(s->fom_done);
  if (s->ev_in) cudaEventDestroy(s->ev_in);
  if (s->ev_out) cudaEventDestroy(s->ev_out);
  if (s->hstream) {
    cudaStreamSynchronize(s->hstream);
    cudaStreamDestroy(s->hstream);
  }
  if (s->cstream) {
    cudaStreamSynchronize(s->cstream);
    cudaStreamDestroy(s->cstream);
  }
  for (int b = 0; b < 2; ++b) {
    if (s->st_ready[b]) cudaEventDestroy(s->st_ready[b]);
    if (s->st_done[b]) cudaEventDestroy(s->st_done[b]);
  }
  for (void* p : s->allocs) cudaFree(p);
  delete s;
}

// offline results (device pointers): q_ref, row scale d, basis phi0 (N x r),
// sigma0 (r), q_last (= training[w_init]).  Copied into the session.
int adrom_session_load(adrom_session* s, const double* q_ref, const double* d, const double* phi0,
                       const double* sigma0, const double* q_last) {
  if (!s) return ADROM_ERR_ARG;
  adrom_ctx* ctx = s->ctx;
  const size_t N = s->N;
  ADROM_CK(ctx, cudaMemcpyAsync(s->q_ref, q_ref, 8 * N, cudaMemcpyDeviceToDevice, ctx->stream));
  ADROM_CK(ctx, cudaMemcpyAsync(s->d, d, 8 * N, cudaMemcpyDeviceToDevice, ctx->stream));
  ADROM_CK(ctx, cudaMemcpyAsync(s->phi[0], phi0, 8 * N * s->r, cudaMemcpyDeviceToDevice,
                                ctx->stream));
  ADROM_CK(ctx, cudaMemcpyAsync(s->sigma[0], sigma0, 8 * s->r, cudaMemcpyDeviceToDevice,
                                ctx->stream));
  int st = ts_gram(ctx, s->phi[0], s->N, s->r, s->gram[0], (double*)s->isvd_ws,
                   isvd_partial_doubles(ctx, s->r));
  if (st) return st;
  ADROM_CK(ctx, cudaMemcpyAsync(s->q_tilde, q_last, 8 * N, cudaMemcpyDeviceToDevice,
                                ctx->stream));
  ADROM_CK(ctx, cudaMemcpyAsync(s->y_corr, q_last, 8 * N, cudaMemcpyDeviceToDevice, ctx->stream));
  fom_wait(s);
  s->fom_ready = false;  // a coarse step of a previous run is discarded
  s->cur = 0;
  s->acur = 0;
  s->kf = 0;
  s->w_id = true;
  s->nrm2_exact = true;
  s->opcur = 0;
  s->n_online = 0;
  if (s->fact) {
    int64_t g = (s->N + 255) / 256;
    if (g > (int64_t)ctx->num_sms * 8) g = (int64_t)ctx->num_sms * 8;
    row_norms_kernel<<<(int)g, 256, 0, ctx->stream>>>(s->phi[0], s->N, s->r, s->nrm2[0]);
    ADROM_LAUNCH_CK(ctx);
    if (s->A32[0]) {
      to_f32_kernel<<<(int)g, 256, 0, ctx->stream>>>(s->phi[0], s->N * s->r, s->A32[0]);
      ADROM_LAUNCH_CK(ctx);
    }
  }
  s->events.clear();
  ADROM_CK(ctx, cudaMemsetAsync(s->fail_step, 0xff, sizeof(int), ctx->stream));
  return ADROM_OK;
}

// driver.py:321-331: initial lookahead (adaptive or FGS), sampling, operator,
// encode(q_last).  Errors here propagate (they are outside the event try).
int adrom_session_start(adrom_session* s) {
  if (!s) return ADROM_ERR_ARG;
  HiPrio hp(s);
  adrom_ctx* ctx = s->ctx;
  const adrom_model m = model_of(s);
  const bool needs_signal = s->cfg.adaptive || s->cfg.sampling == 1;
  if (needs_signal) {
    adrom_newton_info ni{};
    int st = fom_implicit_step(ctx, m, s->y_corr, s->cfg.z * s->cfg.dt, s->cfg.newton_tol,
                               s->cfg.newton_max_iter, s->y_next, &ni);
    if (st) return st;
    std::swap(s->y_corr, s->y_next);
  }
  int st = build_sampling_operator(s, s->phi[s->acur], s->op[s->opcur], s->y_corr);
  if (st) return st;
  return encode_into(s, s->phi[s->acur], s->q_tilde, s->a);
}

// Advance n_steps online steps (driver.py:337-387).  For saved steps (every
// `save_every`-th, counted from the first online step) the decoded state is
// copied to dev_out (device, row-major) and/or host_out (pinned host).
int adrom_session_advance(adrom_session* s, int64_t n_steps, int64_t save_every, double* dev_out,
                          double* host_out, int64_t* n_saved) {
  if (!s) return ADROM_ERR_ARG;
  HiPrio hp(s);
  adrom_ctx* ctx = s->ctx;
  int64_t saved = 0;
  const int64_t N = s->N;
  for (int64_t k = 0; k < n_steps; ++k) {
    const int64_t n = s->cfg.w_init + s->n_online;  // driver loop index
    ADROM_CK(ctx, cudaEventRecord(s->main_mark, ctx->stream));
    int st = rom_step(s);
    if (st) return st;
    ++s->n_online;
    const bool save = save_every > 0 && (s->n_online % save_every == 0 || k == n_steps - 1);
    const bool at_event = s->cfg.adaptive && ((n + 1 - s->cfg.w_init) % s->cfg.z == 0);
    adrom_event_record ev{};
    bool decoded = false;
    if (at_event) {
      ev.step = n + 1;
      st = run_event(s, ev, &decoded);  // decodes q~ in its first basis pass
      if (st) return st;
      // explicit basis: the next event's coarse step only needs this y_corr;
      // start it now so it overlaps the next z reduced steps (the factored
      // path starts it inside the event, after its pass 1)
      if (!s->fact && ev.pad) fom_launch_async(s);
    }
    if (!decoded) {
      st = decode_state(s);
      if (st) return st;
    }
    if (save) {
      if (dev_out)
        ADROM_CK(ctx, cudaMemcpyAsync(dev_out + saved * N, s->q_tilde, 8 * N,
                                      cudaMemcpyDeviceToDevice, ctx->stream));
      if (host_out) {
        const int64_t slot = s->host_slots > 0 ? saved % s->host_slots : saved;
        st = download_state(s, host_out + slot * N);
        if (st) return st;
      }
      ++saved;
    }
    if (at_event) {
      s->events.push_back(ev);
      // a failed reduced step aborts the run like the reference (driver.py:338)
      int fs = -1;
      if (s->fail_step_read) {  // came back with the event's own status words
        memcpy(&fs, (char*)ctx->pinned + PIN_FAIL_STEP, sizeof(int));
        s->fail_step_read = false;
      } else {
        ADROM_CK(ctx, cudaMemcpyAsync(ctx->pinned, s->fail_step, sizeof(int),
                                      cudaMemcpyDeviceToHost, ctx->stream));
        ADROM_CK(ctx, cudaStreamSynchronize(ctx->stream));
        memcpy(&fs, ctx->pinned, sizeof(int));
      }
      if (fs >= 0)
        return set_error(ctx, ADROM_ERR_ROMSTEP, "rank-deficient sampled Jacobian at online step %d",
                         fs + (int)s->cfg.w_init + 1);
    }
  }
  if (n_saved) *n_saved = saved;
  // a coarse step started for the next event is finished before returning
  // (its result is kept: fom_pending stays false, the output is consumed by
  // the next event through fom_join's saved status)
  fom_wait(s);
  // host_out is complete when advance returns (the copies overlapped the steps)
  return drain_downloads(s);
}

int adrom_session_finish(adrom_session* s) {
  if (!s) return ADROM_ERR_ARG;
  HiPrio hp(s);
  adrom_ctx* ctx = s->ctx;
  int st = drain_downloads(s);
  if (st) return st;
  int fs = -1;
  ADROM_CK(ctx, cudaMemcpyAsync(ctx->pinned, s->fail_step, sizeof(int), cudaMemcpyDeviceToHost,
                                ctx->stream));
  ADROM_CK(ctx, cudaStreamSynchronize(ctx->stream));
  memcpy(&fs, ctx->pinned, sizeof(int));
  if (fs >= 0)
    return set_error(ctx, ADROM_ERR_ROMSTEP, "rank-deficient sampled Jacobian at online step %d",
                     fs + (int)s->cfg.w_init + 1);
  return ADROM_OK;
}

int adrom_session_read(adrom_session* s, double* host_step_log, int64_t max_steps,
                       adrom_event_record* host_events, int64_t max_events, int64_t* n_steps,
                       int64_t* n_events, double* dev_a, double* dev_phi, double* dev_sigma,
                       double* dev_q_tilde) {
  if (!s) return ADROM_ERR_ARG;
  adrom_ctx* ctx = s->ctx;
  const int64_t ns = s->n_online < max_steps ? s->n_online : max_steps;
  if (host_step_log && ns > 0)
    ADROM_CK(ctx, cudaMemcpyAsync(host_step_log, s->step_log, sizeof(double) * 3 * ns,
                                  cudaMemcpyDeviceToHost, ctx->stream));
  if (dev_a)
    ADROM_CK(ctx, cudaMemcpyAsync(dev_a, s->a, 8 * s->r, cudaMemcpyDeviceToDevice, ctx->stream));
  if (dev_phi)
    if (s->fact && !s->w_id) {
      int st = fact_reanchor(ctx, basis_view(s), dev_phi, nullptr);
      if (st) return st;
    } else
    ADROM_CK(ctx, cudaMemcpyAsync(dev_phi, s->phi[s->acur], 8 * (size_t)s->N * s->r,
                                  cudaMemcpyDeviceToDevice, ctx->stream));
  if (dev_sigma)
    ADROM_CK(ctx, cudaMemcpyAsync(dev_sigma, s->sigma[s->cur], 8 * s->r, cudaMemcpyDeviceToDevice,
                                  ctx->stream));
  if (dev_q_tilde)
    ADROM_CK(ctx, cudaMemcpyAsync(dev_q_tilde, s->q_tilde, 8 * (size_t)s->N,
                                  cudaMemcpyDeviceToDevice, ctx->stream));
  ADROM_CK(ctx, cudaStreamSynchronize(ctx->stream));
  const int64_t ne = (int64_t)s->events.size() < max_events ? (int64_t)s->events.size() : max_events;
  if (host_events)
    for (int64_t i = 0; i < ne; ++i) host_events[i] = s->events[i];
  if (n_steps) *n_steps = s->n_online;
  if (n_events) *n_events = (int64_t)s->events.size();
  return ADROM_OK;
}

int adrom_session_set_host_ring(adrom_session* s, int64_t slots) {
  if (!s || slots < 0) return ADROM_ERR_ARG;
  s->host_slots = slots;
  return ADROM_OK;
}

int adrom_session_signal(adrom_session* s, double* dev_y) {
  if (!s || !dev_y) return ADROM_ERR_ARG;
  ADROM_CK(s->ctx, cudaMemcpyAsync(dev_y, s->y_corr, sizeof(double) * s->N,
                                   cudaMemcpyDeviceToDevice, s->ctx->stream));
  return ADROM_OK;
}

int adrom_session_sampling(adrom_session* s, int64_t* dev_idx) {
  if (!s) return ADROM_ERR_ARG;
  ADROM_CK(s->ctx, cudaMemcpyAsync(dev_idx, s->op[s->opcur].idx, sizeof(int64_t) * s->cfg.n_s,
                                   cudaMemcpyDeviceToDevice, s->ctx->stream));
  return ADROM_OK;
}

// ---- stateless entry points ---------------------------------------------
int adrom_qdeim(adrom_ctx* ctx, const double* phi, int64_t n, int32_t r, int32_t n_s,
                int64_t* idx) {
  if (!ctx) return ADROM_ERR_ARG;
  int st = ensure_scratch(ctx, qdeim_pool_workspace_bytes(n, r, n_s) + 4096);
  if (st) return st;
  return qdeim_pool_select(ctx, phi, n, r, n_s, idx, ctx->scratch, nullptr);
}

int adrom_fgs(adrom_ctx* ctx, const adrom_model* m, const double* phi, int32_t r,
              const double* y_corr, int32_t n_s, int32_t n_extra, int32_t feature, int64_t* idx) {
  if (!ctx || !m) return ADROM_ERR_ARG;
  if (n_extra > n_s) return set_error(ctx, ADROM_ERR_ARG, "n_extra cannot exceed the total number of sampling points");
  const int64_t N = m->n_elem * m->n_var;
  const int n_base = n_s - n_extra;
  int st = ensure_scratch(ctx, qdeim_pool_workspace_bytes(N, r, n_s) + 4096);
  if (st) return st;
  if (n_base > 0) {
    st = qdeim_pool_select(ctx, phi, N, r, n_base, idx, ctx->scratch, nullptr);
    if (st) return st;
  }
  st = reset_flags(ctx);
  if (st) return st;
  st = fgs_extend(ctx, *m, y_corr, feature, idx, n_base, n_extra, nullptr);
  if (st) return st;
  int flags[16];
  st = read_flags(ctx, flags);
  if (st) return st;
  return sampling_flag_error(ctx, flags[0]);
}

int adrom_deim_operator(adrom_ctx* ctx, const double* phi, int64_t n, int32_t r, const int64_t* idx,
                        int32_t n_s, double* pinv) {
  if (!ctx) return ADROM_ERR_ARG;
  (void)n;
  int st = ensure_scratch(ctx, sizeof(double) * (size_t)n_s * r + 4096);
  if (st) return st;
  st = reset_flags(ctx);
  if (st) return st;
  st = deim_pinv_only(ctx, phi, idx, n_s, r, (double*)ctx->scratch, pinv, ctx->dflags);
  if (st) return st;
  int flags[16];
  st = read_flags(ctx, flags);
  if (st) return st;
  return sampling_flag_error(ctx, flags[0]);
}

int adrom_rom_operator_build(adrom_ctx* ctx, const adrom_model* m, const double* phi, int64_t n,
                             const double* q_ref, const double* d, const int64_t* idx,
                             int32_t n_s, adrom_rom_op* op) {
  if (!ctx || !m || !op) return ADROM_ERR_ARG;
  (void)n;
  if (n_s < 1 || n_s > op->ns_cap || op->nc_cap < 3 * n_s * m->n_var)
    return set_error(ctx, ADROM_ERR_ARG, "rom_operator_build: capacities too small");
  int st = reset_flags(ctx);
  if (st) return st;
  if (idx && idx != op->idx) {
    copy_i64_kernel<<<1, 256, 0, ctx->stream>>>(idx, op->idx, n_s);
    ADROM_LAUNCH_CK(ctx);
  }
  st = plan_build(ctx, *m, *op, n_s, ctx->dflags);
  if (st) return st;
  st = operator_fill(ctx, *op, phi, q_ref, d, n_s, ctx->dflags);
  if (st) return st;
  int flags[16];
  st = read_flags(ctx, flags);
  if (st) return st;
  return sampling_flag_error(ctx, flags[0]);
}

int adrom_rom_step(adrom_ctx* ctx, const adrom_model* m, const adrom_rom_op* op, int32_t kind,
                   const double* a_prev, double dt, double tol, int32_t max_iter, double* a_out,
                   adrom_rom_step_info* host_info) {
  if (!ctx || !m || !op) return ADROM_ERR_ARG;
  const size_t wd = rom_step_work_doubles(*op);
  int st = ensure_scratch(ctx, sizeof(double) * (wd + 64));
  if (st) return st;
  RomStepArgs A{};
  A.op = *op;
  A.kind = m->kind;
  A.bp = make_bp(*m);
  A.gamma = m->gamma;
  A.mech = m->mech;
  A.a_prev = a_prev;
  A.a_out = a_out;
  A.dt = dt;
  A.tol = tol;
  A.max_iter = max_iter;
  A.work = (double*)ctx->scratch;
  A.info = A.work + wd;
  st = rom_step_async(ctx, A, kind == 0);
  if (st) return st;
  ADROM_CK(ctx, cudaMemcpyAsync(ctx->pinned, A.info, sizeof(double) * 8, cudaMemcpyDeviceToHost,
                                ctx->stream));
  ADROM_CK(ctx, cudaStreamSynchronize(ctx->stream));
  const double* hi = (const double*)ctx->pinned;
  if (hi[4] != 0.0) {
    if (kind == 0)
      return set_error(ctx, ADROM_ERR_ROMSTEP,
                       "rank-deficient sampled Jacobian at iteration %d (condition number %.3e)",
                       (int)hi[1], hi[3]);
    return set_error(ctx, ADROM_ERR_ROMSTEP, "singular reduced Jacobian at iteration %d", (int)hi[1]);
  }
  if (host_info) {
    host_info->converged = (int)hi[0];
    host_info->iterations = (int)hi[1];
    host_info->residual_norm = hi[2];
  }
  return ADROM_OK;
}

}  // extern "C"
