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
