// Tensor-core (tcgen05, sm_100a) GEMM for the dense compression's mode-1
// contraction: Z[m, n] = sum_k A[m, k] * X[k + K n] with fp32 operands split
// into TF32 hi/lo parts (3 MMAs per k-step: hi*hi + hi*lo + lo*hi), fp32
// accumulation in TMEM.  Returns false when the shape is not supported, so the
// caller can use the SIMT path.
#pragma once

#include <cuda_runtime.h>

namespace octen {

bool tc_gemm_f32_nt(const float* A, const float* X, float* Z, int M, long long N, int K, cudaStream_t st);

}  // namespace octen
