// Host-side internal API of the FOM kernels (used by capi.cu and session.cu).
#pragma once

#include "common.cuh"

namespace adrom {

int fom_rhs(adrom_ctx* ctx, const adrom_model& m, const double* q, double* f);
// configuration-4 reacting Euler residual (reacting.cu)
int reacting_rhs(adrom_ctx* ctx, const adrom_model& m, const double* q, double* f);
int reacting_jacobian(adrom_ctx* ctx, const adrom_model& m, const double* q, double* blocks,
                      bool apply_dt, double dt, int* flag);
int fom_rhs_at_cells(adrom_ctx* ctx, const adrom_model& m, const double* gathered, int64_t k,
                     double* out);
int fom_plan_evaluate(adrom_ctx* ctx, const adrom_model& m, const int64_t* gather,
                      int64_t n_cells, const int64_t* out_cell, const int64_t* out_var,
                      int64_t n_s, const double* closure_values, const double* h,
                      const double* dirs, int64_t ld_dirs, int n_dir, double* out);
// J (apply_dt = false) or A = I - dt*J (apply_dt = true) in block storage
int fom_fd_jacobian(adrom_ctx* ctx, const adrom_model& m, const double* q, double* blocks,
                    bool apply_dt, double dt);
// backward-Euler Newton (fom.py:331-347 + dense.py:140-171).  Blocking.
int fom_implicit_step(adrom_ctx* ctx, const adrom_model& m, const double* q, double dt,
                      double tol, int max_iter, double* x, adrom_newton_info* info);
// workspace bytes needed by fom_implicit_step at this size
size_t fom_newton_workspace(const adrom_model& m);

}  // namespace adrom
