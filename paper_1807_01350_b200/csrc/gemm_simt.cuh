// Batched SIMT GEMM with functor-addressed operands, used for the many small
// and oddly-strided contractions of the ALS / merge stages (fp64) and as the
// fp64-input compression path.  C(b,m,n) <- sum_k A(b,m,k) * B(b,k,n), the
// store functor decides assign/accumulate.  Optional deterministic split-K:
// partial sums go to a workspace and are reduced in fixed split order, so the
// result is bit-reproducible run to run (the reference's determinism
// contract, tests/test_streaming.cpp:188-203).
#pragma once

#include <cuda_runtime.h>

#include "octen_common.cuh"

namespace octen {

// Tile: BM x BN outputs per block, BK deep, TM x TN per thread.
// A_KFAST / B_KFAST choose the global->shared load order (the unit-stride
// operand index should vary fastest across threads).
template <typename TIn, typename Acc, int BM, int BN, int BK, int TM, int TN, bool A_KFAST, bool B_KFAST,
          class AF, class BF, class CF>
__global__ void __launch_bounds__((BM / TM) * (BN / TN))
    gemm_simt_kernel(int M, int N, int K, int ksplit, int kchunk, AF af, BF bf, CF cf, Acc* partial,
                     int lower_only) {
    constexpr int NT = (BM / TM) * (BN / TN);
    // lower_only: skip output tiles strictly above the diagonal (m < n everywhere)
    if (lower_only && (int)(blockIdx.x * BN) >= (int)(blockIdx.y * BM + BM)) return;
    __shared__ Acc As[BK][BM + 1];
    __shared__ Acc Bs[BK][BN + 1];
    const int tid = threadIdx.x;
    const int zb = blockIdx.z;
    const int batch = zb / ksplit;
    const int ks = zb % ksplit;
    const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
    const int kbeg = ks * kchunk;
    const int kend = min(K, kbeg + kchunk);
    const int tm = (tid / (BN / TN)) * TM;
    const int tn = (tid % (BN / TN)) * TN;
    Acc acc[TM][TN];
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = Acc(0);

    for (int k0 = kbeg; k0 < kend; k0 += BK) {
        for (int e = tid; e < BM * BK; e += NT) {
            int mm, kk;
            if (A_KFAST) {
                kk = e % BK;
                mm = e / BK;
            } else {
                mm = e % BM;
                kk = e / BM;
            }
            const int gm = m0 + mm, gk = k0 + kk;
            As[kk][mm] = (gm < M && gk < kend) ? Acc(af(batch, gm, gk)) : Acc(0);
        }
        for (int e = tid; e < BN * BK; e += NT) {
            int nn, kk;
            if (B_KFAST) {
                kk = e % BK;
                nn = e / BK;
            } else {
                nn = e % BN;
                kk = e / BN;
            }
            const int gn = n0 + nn, gk = k0 + kk;
            Bs[kk][nn] = (gn < N && gk < kend) ? Acc(bf(batch, gk, gn)) : Acc(0);
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < BK; ++kk) {
            Acc a[TM], b[TN];
#pragma unroll
            for (int i = 0; i < TM; ++i) a[i] = As[kk][tm + i];
#pragma unroll
            for (int j = 0; j < TN; ++j) b[j] = Bs[kk][tn + j];
#pragma unroll
            for (int i = 0; i < TM; ++i)
#pragma unroll
                for (int j = 0; j < TN; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) {
            const int gm = m0 + tm + i, gn = n0 + tn + j;
            if (gm < M && gn < N) {
                if (ksplit == 1)
                    cf(batch, gm, gn, acc[i][j]);
                else
                    partial[(((size_t)batch * ksplit + ks) * M + gm) * N + gn] = acc[i][j];
            }
        }
}

template <typename Acc, class CF>
__global__ void gemm_splitk_reduce(int batches, int M, int N, int ksplit, const Acc* partial, CF cf) {
    const size_t total = (size_t)batches * M * N;
    for (size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x; idx < total;
         idx += (size_t)gridDim.x * blockDim.x) {
        const int n = (int)(idx % N);
        const int m = (int)((idx / N) % M);
        const int b = (int)(idx / ((size_t)M * N));
        Acc s = Acc(0);
        for (int k = 0; k < ksplit; ++k) s += partial[(((size_t)b * ksplit + k) * M + m) * N + n];
        cf(b, m, n, s);
    }
}

// Host launcher.  workspace must hold batches*ksplit*M*N Acc when ksplit > 1.
template <typename TIn, typename Acc, bool A_KFAST, bool B_KFAST, class AF, class BF, class CF>
void gemm_simt(int batches, int M, int N, int K, AF af, BF bf, CF cf, cudaStream_t st, int ksplit = 1,
               Acc* workspace = nullptr, int lower_only = 0) {
    if (batches <= 0 || M <= 0 || N <= 0) return;
    if (K <= 0) {
        ksplit = 1;
    }
    if (ksplit < 1) ksplit = 1;
    int kchunk = (K + ksplit - 1) / ksplit;
    if (kchunk < 1) kchunk = 1;
    constexpr int BM = 64, BN = 64, BK = 16, TM = 4, TN = 4;
    dim3 grid((N + BN - 1) / BN, (M + BM - 1) / BM, batches * ksplit);
    gemm_simt_kernel<TIn, Acc, BM, BN, BK, TM, TN, A_KFAST, B_KFAST>
        <<<grid, (BM / TM) * (BN / TN), 0, st>>>(M, N, K, ksplit, kchunk, af, bf, cf, workspace,
                                                              lower_only); OCTEN_LAUNCHED(1);
    if (ksplit > 1) {
        const size_t total = (size_t)batches * M * N;
        int blocks = (int)((total + 255) / 256);
        if (blocks > 148 * 16) blocks = 148 * 16;
        gemm_splitk_reduce<Acc><<<blocks, 256, 0, st>>>(batches, M, N, ksplit, workspace, cf); OCTEN_LAUNCHED(1);
    }
}

// Pick a split factor that gives roughly `target` blocks.
inline int pick_ksplit(int batches, int M, int N, int K, int target = 296, int min_chunk = 256) {
    const long tiles = (long)batches * ((M + 63) / 64) * ((N + 63) / 64);
    int ks = 1;
    while (tiles * ks < target && K / (ks * 2) >= min_chunk) ks *= 2;
    return ks;
}

}  // namespace octen
