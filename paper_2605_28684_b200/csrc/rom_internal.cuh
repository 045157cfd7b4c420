// Host-side internal API of the reduced steppers (sampled.cu).
#pragma once

#include "physics.cuh"
#include "sampling_internal.cuh"

namespace adrom {

struct RomStepArgs {
  DevOp op;              // reduced operator (device pointers, sizes on device)
  int kind;              // ADROM_BURGERS / ADROM_SOD / ADROM_REACTING
  BurgersParams bp;      // dx, nu, dx^2
  double gamma;
  const double* mech;    // ADROM_REACTING: 5 x 12 mechanism (device), else NULL
  const double* a_prev;  // device [r]
  double* a_out;         // device [r] (may alias a_prev)
  double dt, tol;
  int max_iter;
  double* work;          // device scratch: rom_step_work_doubles(op)
  double* info;          // device [8]: converged, iterations, residual, cond, status
};

size_t rom_step_work_doubles(const DevOp& op);

// ---- large sampled sets (bigsample.cu) -----------------------------------
// physics of the sampled residual
struct PlanParams {
  BurgersParams bp;
  double gamma;
  const double* mech;
};
// sampled rows grouped by sampled cell (slot ks of op.gather): rows
// rows[cell_start[ks] .. + cell_cnt[ks]) in variable order
struct BigOp {
  int64_t* cell_start;  // [ncell_cap]
  int32_t* cell_cnt;    // [ncell_cap]
  int32_t* rows;        // [ns_cap]
};
int fgs_extend_big(adrom_ctx* ctx, const adrom_model& m, const double* y_corr, int feature_kind,
                   int64_t* idx, int n_base, int n_extra);
int plan_build_big(adrom_ctx* ctx, const adrom_model& m, DevOp& op, const BigOp& big, int n_s,
                   int* flag);
size_t deim_pinv_big_work_doubles(int n_s, int r);
// flag bit 128: Cholesky failed or cond bound > 1e8
int deim_pinv_big(adrom_ctx* ctx, DevOp& op, int n_s, double* work, int* flag);
size_t big_work_doubles(const DevOp& op);
// enqueues the Gauss-Newton loop; synchronises once per iteration to stop
int lspg_step_big(adrom_ctx* ctx, const RomStepArgs& A, const BigOp& big, int n_s);
// sampled.cu: r x r update of the large-sample LSPG step.  C = [jac | rho]
// (r x (r+1), column-major); st = [a (r), h (r), it, done, gnorm, status]
int lspg_update_launch(adrom_ctx* ctx, const double* C, int r, double* st, double tol,
                       int max_iter);
int lspg_finish_launch(adrom_ctx* ctx, const double* st, int r, double tol, double* a_out,
                       double* info);
// Asynchronous: enqueues one reduced step; status (RomStepError) in info[4].
int rom_step_async(adrom_ctx* ctx, const RomStepArgs& args, bool lspg);

inline BurgersParams make_bp(const adrom_model& m) {
  BurgersParams p;
  p.dx = m.dx;
  p.nu = m.nu;
  p.dx2 = m.dx * m.dx;
  return p;
}

}  // namespace adrom
