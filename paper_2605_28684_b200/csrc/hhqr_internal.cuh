// Householder QR / Q application (hhqr.cu) and the device POD (offline.cu).
#pragma once
#include "common.cuh"

namespace adrom {

// work doubles for hh_qr (w = m) or hh_apply (w = nc) on N rows
size_t hh_work_doubles(int64_t N, int w);

// In-place Householder QR of the column-major N x m matrix A (N >= m): R in
// the upper triangle, reflector vectors below the diagonal, the reflectors'
// leading entries in vk[m] and v^T v in vtv[m] (0: identity).
int hh_qr(adrom_ctx* ctx, int64_t N, int m, double* A, int64_t lda, double* vk, double* vtv,
          double* work);

// X (N x nc, column-major, ldx) <- Q X (transpose = false) or Q^T X, with
// Q = H_0 ... H_{m-1} from hh_qr.
int hh_apply(adrom_ctx* ctx, int64_t N, int m, const double* A, int64_t lda, const double* vk,
             const double* vtv, double* X, int64_t ldx, int nc, bool transpose, double* work);

}  // namespace adrom
