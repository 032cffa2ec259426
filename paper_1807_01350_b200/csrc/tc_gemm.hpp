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
// cuTensorMapEncodeTiled through the runtime's driver entry point (nullptr if absent).
void* tc_tensor_map_encoder();
// A_hi / A_lo: M x K row-major (leading dimension lda >= K, lda % 4 == 0);
// X: K x N column-major (K contiguous); Z: M x N row-major (ld N).
// scatter_p > 0: output row m of the deduplicated stack is written to the
// replica rows p * scatter_q + a (shared rows m < scatter_sh to every replica),
// so Z is scatter_p * scatter_q x N.
// nonfinite (optional): set to 1 when X holds a non-finite value (the
// conversion warps check every element they pass).
// max_ctas > 0 caps the persistent grid (default: one CTA per SM).
bool tc_gemm_tf32x3(const float* Ahi, const float* Alo, int lda, const float* X, float* Z, int M, long long N, int K,
                    cudaStream_t st, int scatter_p = 0, int scatter_q = 0, int scatter_sh = 0, int* nonfinite = nullptr,
                    int max_ctas = 0);
// Mode-2 contraction batched over (replica, slice):
//   Z2[p * zstride + a + Q b + Q^2 k] = sum_j Z1[p Q + a][k J + j] V_p[j, b]
// Z1: P*Q x N1 row-major (N1 = J * tc); Vhi/Vlo: TF32 hi/lo split of V,
// P*Q x ldv row-major (row p Q + b holds V_p[:, b]).  Requires Q <= 112.
bool tc_mode2_tf32x3(const float* Z1, long long N1, int J, int tc, const float* Vhi, const float* Vlo, int ldv, int P,
                     int Q, float* Z2, long long zstride, cudaStream_t st);

}  // namespace octen
