// Tensor-core (tcgen05, sm_100a) GEMM for the dense compression's mode-1
// contraction: Z[m, n] = sum_k A[m, k] * X[k + K n] with fp32 operands split
// into TF32 hi/lo parts (3 MMAs per k-step: hi*hi + hi*lo + lo*hi), fp32
// accumulation in TMEM.  Returns false when the shape/alignment is not
// supported (or OCTEN_DISABLE_TCGEN05 is set), so the caller can use the SIMT
// path.
#pragma once

#include <cuda_runtime.h>

namespace octen {

bool tc_gemm_available();
// A_hi / A_lo: M x K row-major (leading dimension lda >= K, lda % 4 == 0);
// X: K x N column-major (K contiguous); Z: M x N row-major (ld N).
bool tc_gemm_tf32x3(const float* Ahi, const float* Alo, int lda, const float* X, float* Z, int M, long long N, int K,
                    cudaStream_t st);

}  // namespace octen
