// Partitioned block-tridiagonal solver (cyclic or open chain) for the Newton
// systems (I - dt J) delta = -r of the backward-Euler step.
#pragma once

#include "common.cuh"

namespace adrom {

// bytes of workspace bt_solve needs for n block rows of size nv
size_t bt_workspace_bytes(int64_t n, int nv);

// Solve sys * x = rhs_sign * rhs where sys is block tridiagonal in the layout
// sys[((i*3 + slot)*nv + a)*nv + b], slot 0 = coupling to the left
// neighbour, 1 = diagonal, 2 = right neighbour.  cyclic: row 0's left
// neighbour is row n-1 and row n-1's right neighbour is row 0.  A zero pivot
// sets bit 2 of *flag.  Asynchronous (no host sync).
int bt_solve(adrom_ctx* ctx, const double* sys, const double* rhs, double rhs_sign, int64_t n,
             int nv, bool cyclic, double* out, void* ws, int* flag,
             const double* add_to = nullptr);

}  // namespace adrom
