// Host-side internal API: QDEIM / FGS sampling, stencil closure + gather plan,
// reduced operator assembly.
#pragma once

#include "common.cuh"

namespace adrom {

// Exact greedy via a certified candidate pool (qdeim.cu): the path used by
// the session and the C-ABI.  Blocking (one sync per pass).
size_t qdeim_pool_workspace_bytes(int64_t n, int r, int count);
// seeded: the workspace's res2/bnd2/ver already hold the k = 0 bounds
// (||phi_i||^2, written by the rotation epilogue: qdeim_seed_buffers)
// fb (factored basis Phi = X W, factored.cu): rows are read through it and
// nrmb holds bounds of ||Phi_i||^2 (then seeded and count <= r are required)
struct FactBasis;
// qdeim_pool_select on factored rows could not certify a pivot (bound slack):
// not an error, rerun on the materialised basis
constexpr int QDEIM_NEEDS_EXPLICIT = 100;
int qdeim_pool_select(adrom_ctx* ctx, const double* phi, int64_t n, int r, int count,
                      int64_t* out_idx, void* ws, int* passes_out, bool seeded = false,
                      const FactBasis* fb = nullptr, const double* nrmb = nullptr);
void qdeim_seed_buffers(void* ws, int64_t n, double** res2, double** bnd2, unsigned char** ver);
// FGS (sampling.py:117-159): idx[0..n_base) must already hold the QDEIM
// rows; appends n_extra rows ranked by |grad feature(y_corr)|.
int fgs_extend(adrom_ctx* ctx, const adrom_model& m, const double* y_corr, int feature_kind,
               int64_t* idx, int n_base, int n_extra, void* ws);
size_t fgs_workspace_bytes(const adrom_model& m);

// Device layout of a reduced operator (projection.py:57-87) with capacities.
using DevOp = adrom_rom_op;

// plan + closure from idx (device, n_s rows) — fom.py:127-152, sampling.py:178-189
int plan_build(adrom_ctx* ctx, const adrom_model& m, DevOp& op, int n_s, int* flag);
// gathers + DEIM pseudo-inverse (sampling.py:162-175, projection.py:69-80)
// fb (factored basis): rows are materialised into fact_rows
// (>= (nc_cap + ns_cap) * r doubles) first
// big_work (large sampled sets): the pseudo-inverse by CholeskyQR2
// (bigsample.cu, deim_pinv_big_work_doubles) instead of the one-block QR
int operator_fill(adrom_ctx* ctx, DevOp& op, const double* phi, const double* q_ref,
                  const double* d, int n_s, int* flag, const FactBasis* fb = nullptr,
                  double* fact_rows = nullptr, double* big_work = nullptr);

int deim_pinv_only(adrom_ctx* ctx, const double* phi, const int64_t* idx, int n_s, int r,
                   double* phi_s, double* pinv, int* flag);

}  // namespace adrom
