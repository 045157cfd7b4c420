// Host-side internal API of the factored basis (factored.cu), see its header.
#pragma once

#include "common.cuh"

namespace adrom {

constexpr int FACT_KQ = 16;  // residual columns kept before re-anchoring

// Q (the residual columns) is stored as FACT_KQ / 4 panels of 4 columns:
// panel P holds columns 4P..4P+3 as n rows of 32 bytes (one DRAM sector).
// A pass over the basis with k live columns reads ceil(k / 4) sectors per
// row instead of the whole 128-byte row of a row-major n x 16 store, and a
// gathered row still costs ceil(k / 4) sectors.
__host__ __device__ __forceinline__ int64_t qpanel(int64_t i, int j, int64_t n) {
  return ((int64_t)(j >> 2) * n + i) * 4 + (j & 3);
}

// Phi = [A | Q_0 .. Q_{k-1}] W;  W == nullptr means W = I (then k == 0)
struct FactBasis {
  const double* A;  // n x r row-major anchor
  const double* Q;  // n x FACT_KQ residual columns, 4-column panels (qpanel)
  int r, k;
  const double* W;  // (r + k) x r row-major, or null
  int64_t n;
  // optional fp32 shadow of A (the QDEIM refresh gathers it)
  const float* A32 = nullptr;
  // optional: the direction the last iSVD event dropped, in X coordinates
  // (r + k entries).  The event's QDEIM seed ||Phi_i||^2 + q^_i^2 exceeds the
  // new row norm by exactly (X_i . vdrop)^2; the bound refresh subtracts it
  const double* vdrop = nullptr;
};

struct FactEventArgs {
  const double* y;        // snapshot y_hat
  const double* a;        // reduced state to decode
  const double* q_ref;
  const double* d;
  double* q_tilde;        // decoded state (out)
  double* Qw;             // Q (column k is written)
  double* qv;             // N-vector: the residual q, contiguous (seed bounds)
  const double* sigma;    // current sigma (r)
  const double* G;        // tracked Phi^T Phi (r x r)
  double lam;
  double* partial;        // fact_partial_doubles (pass 2)
  double* partial_a;      // fact_partial_doubles (pass 1; may equal partial if serial)
  int* flag_a;            // flags of pass 1 (its stream's)
  double* small;          // fact_small_doubles
  double* W_out;          // (r + k + 1) x r
  double* sigma_out;
  double* G_out;
  double* a_out;          // state transfer a' = Phi'^T D (q~ - q_ref)
  double* stats;          // isvd stats (>= 8 doubles)
  int* flag;
  // row norms: nrm2_inout holds bounds of ||Phi_i||^2 for the current basis;
  // with vdrop_in (the previous event's dropped direction in the current X
  // coordinates) pass 1 turns them into exact norms (in place).  vdrop_out
  // receives this event's dropped direction for the next one.
  double* nrm2_inout;
  const double* vdrop_in;
  double* vdrop_out;      // r + k + 1
  // QDEIM k = 0 bounds of the new basis (optional)
  double* nrm2_out;
  double* seed_res2;
  double* seed_bnd2;
  unsigned char* seed_ver;
};

inline size_t fact_small_doubles(int r) {
  return 8 * (size_t)(r + FACT_KQ + 2) + 2 * (size_t)(r + 1) * r + 3 * (size_t)r + 256;
}
size_t fact_partial_doubles(adrom_ctx* ctx, int64_t n, int r);

// one history-aware iSVD event on the factored basis (tracking.py:141-178):
// decode, both passes, core SVD, W', state transfer, QDEIM seed bounds.
// Asynchronous; flags as isvd_update_async.
int fact_isvd_event(adrom_ctx* ctx, const FactBasis& b, const FactEventArgs& e);
// the same in two halves: pass 1 (X^T y, row norms; needs y only) and the rest
// (needs the reduced state a).  The session runs them on two streams.
int fact_event_pass_a(adrom_ctx* ctx, const FactBasis& b, const FactEventArgs& e);
int fact_event_pass_b(adrom_ctx* ctx, const FactBasis& b, const FactEventArgs& e);

// q~ = q_ref + (X (W a)) / d   (projection.py:104 on the factored basis)
int fact_decode(adrom_ctx* ctx, const FactBasis& b, const double* a, const double* q_ref,
                const double* d, double* q_tilde, double* small, double* partial);

// out (n x r) = X W (tensor cores); exact row norms into nrm2 (optional)
// (out32: optional fp32 copy of out)
int fact_reanchor(adrom_ctx* ctx, const FactBasis& b, double* out, double* nrm2,
                  float* out32 = nullptr);

// rows_out[p] = Phi_{rows[p]} (r doubles each) for p < min(count, *dcount)
// (rows[p] < 0 -> zeros; dcount: optional device-side count)
int fact_gather_rows(adrom_ctx* ctx, const FactBasis& b, const int64_t* rows, int64_t count,
                     double* rows_out, const int* dcount = nullptr);

}  // namespace adrom
