// FP64 tensor-core GEMMs of the large-sample reduced operator (dgemm.cu).
#pragma once
#include "common.cuh"

namespace adrom {

constexpr int DMMA_TN_MAX_M = 128;  // output rows (basis rank)
constexpr int DMMA_TN_MAX_N = 136;  // output columns (rank + 1 right-hand side)

// blocks (= K chunks = partials) dmma_tn launches at most
int dmma_tn_blocks(const adrom_ctx* ctx);

// C (m x n, column-major) = sum_k A(k, i) B(k, c) with A row-major K x m
// (A[k * lda + i]) or, if a_kmajor, K-major (A[i * lda + k]); B row-major
// K x n (B[k * ldb + c]).  `part` holds max(dmma_tn_blocks, max_blocks) m x n
// partials; the split-K sum is in a fixed order (deterministic).
int dmma_tn(adrom_ctx* ctx, int m, int n, int64_t K, const double* A, int64_t lda, bool a_kmajor,
            const double* B, int64_t ldb, double* C, double* part, int max_blocks = 0);

// out = A M with A row-major K x m (lda), M column-major m x n (row-major if
// m_rowmajor); out row-major K x n (out[k * ldo + c]) or, if out_kmajor,
// n x K (out[c * ldo + k]).
int dmma_apply(adrom_ctx* ctx, int64_t K, int m, int n, const double* A, int64_t lda,
               const double* M, double* out, int64_t ldo, bool out_kmajor,
               bool m_rowmajor = false);

// C-ABI helpers (scratch for the split-K partials from the context)
int ts_tn(adrom_ctx* ctx, int64_t K, int m, int n, const double* A, int64_t lda, bool a_kmajor,
          const double* B, int64_t ldb, double* C);

}  // namespace adrom
