// train_f64.h -- host entry points of the FP64 tensor-core (DMMA) train
// kernels (train_f64.cu).  Internal C++; everything runs on the given stream.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace csb {

// C = alpha op(A) op(B) + beta C on the DMMA GEMM (flags: DgemmFlags in
// dmma_f64.cuh -- transposes, triangular operand structure, lower-only C).
void dmma_gemm(cudaStream_t st, int flags, int M, int N, int K, double alpha, const double* A, int64_t lda,
               const double* B, int64_t ldb, double beta, double* C, int64_t ldc);

// Gram matrix of the normalised memory vectors (mset.cpp:151-152) in GEMM
// form on DMMA with the similarity map, exact unit diagonal and near-zero
// recompute fused in the epilogue; G is m x m, full (mirrored), ld m.
void dmma_gram(cudaStream_t st, const double* Dn, int64_t n, int64_t m, int kind, double h, double* G);

// G^-1 of an SPD matrix by a recursive blocked Cholesky factorisation whose
// leaves factor and invert 128-blocks in one CTA and whose off-diagonal work
// is grouped DMMA GEMMs, then G^-1 = L^-T L^-1 (full symmetric, ld m).
// Returns false when a pivot is not positive (G not numerically SPD).
bool dmma_chol_inverse(cudaStream_t st, const double* G, int64_t m, double* out);

}  // namespace csb
