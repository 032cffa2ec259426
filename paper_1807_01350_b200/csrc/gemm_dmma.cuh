// Batched fp64 GEMM on the FP64 tensor cores (mma.sync.m8n8k4.f64, the only
// fp64 MMA on sm_100a: tcgen05 has no f64 kind), with functor-addressed
// operands so the ALS / merge contractions run on their native layouts.
//
//   C(b,m,n) <- sum_k A(b,m,k) B(b,k,n)     (store functor decides = or +=)
//
// 64x64 block tile, BK = 16, 8 warps each owning a 32x16 sub-tile (4 x 2
// m8n8 accumulators), register-staged double buffering of the shared tiles.
// Deterministic split-K (fixed-order reduction) as in gemm_simt.cuh.
#pragma once

#include <cuda_runtime.h>

#include "gemm_simt.cuh"
#include "octen_common.cuh"

namespace octen {

// Launch `k` as a programmatic dependent of the previous work on `st` (the
// kernel must call pdl_wait() before reading its predecessor's output).
template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    OCTEN_CUDA(cudaLaunchKernelEx(&cfg, k, static_cast<KArgs>(args)...));
    OCTEN_LAUNCHED(1);
}

__device__ __forceinline__ void dmma_m8n8k4(double& d0, double& d1, double a, double b) {
    asm volatile(
        "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
        : "+d"(d0), "+d"(d1)
        : "d"(a), "d"(b));
}

template <bool A_KFAST, bool B_KFAST, class AF, class BF, class CF>
__global__ void __launch_bounds__(256)
    gemm_dmma_kernel(int M, int N, int K, int ksplit, int kchunk, AF af, BF bf, CF cf, double* partial,
                     int lower_only) {
    constexpr int BM = 64, BN = 64, BK = 16, PAD = 4;
    __shared__ double As[2][BK][BM + PAD];
    __shared__ double Bs[2][BK][BN + PAD];
    if (lower_only && (int)(blockIdx.x * BN) >= (int)(blockIdx.y * BM + BM)) return;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g = lane >> 2, t4 = lane & 3;
    const int wm = (warp & 1) * 32, wn = (warp >> 1) * 16;
    const int zb = blockIdx.z;
    const int batch = zb / ksplit, ks = zb % ksplit;
    const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
    const int kbeg = ks * kchunk;
    const int kend = min(K, kbeg + kchunk);

    double acc[4][2][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

    double ra[4], rb[4];
    auto load = [&](int k0) {
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const int e = tid + r * 256;
            int mm, kk;
            if (A_KFAST) {
                kk = e % BK;
                mm = e / BK;
            } else {
                mm = e % BM;
                kk = e / BM;
            }
            const int gm = m0 + mm, gk = k0 + kk;
            ra[r] = (gm < M && gk < kend) ? (double)af(batch, gm, gk) : 0.0;
            int nn, kb;
            if (B_KFAST) {
                kb = e % BK;
                nn = e / BK;
            } else {
                nn = e % BN;
                kb = e / BN;
            }
            const int gn = n0 + nn, gk2 = k0 + kb;
            rb[r] = (gn < N && gk2 < kend) ? (double)bf(batch, gk2, gn) : 0.0;
        }
    };
    auto store = [&](int buf) {
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const int e = tid + r * 256;
            int mm, kk;
            if (A_KFAST) {
                kk = e % BK;
                mm = e / BK;
            } else {
                mm = e % BM;
                kk = e / BM;
            }
            As[buf][kk][mm] = ra[r];
            int nn, kb;
            if (B_KFAST) {
                kb = e % BK;
                nn = e / BK;
            } else {
                nn = e % BN;
                kb = e / BN;
            }
            Bs[buf][kb][nn] = rb[r];
        }
    };

    int buf = 0;
    if (kbeg < kend) {
        load(kbeg);
        store(0);
    }
    __syncthreads();
    for (int k0 = kbeg; k0 < kend; k0 += BK) {
        const bool more = k0 + BK < kend;
        if (more) load(k0 + BK);
#pragma unroll
        for (int kk = 0; kk < BK; kk += 4) {
            double a[4], b[2];
#pragma unroll
            for (int i = 0; i < 4; ++i) a[i] = As[buf][kk + t4][wm + i * 8 + g];
#pragma unroll
            for (int j = 0; j < 2; ++j) b[j] = Bs[buf][kk + t4][wn + j * 8 + g];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 2; ++j) dmma_m8n8k4(acc[i][j][0], acc[i][j][1], a[i], b[j]);
        }
        if (more) {
            store(buf ^ 1);
            __syncthreads();
            buf ^= 1;
        }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
            for (int v = 0; v < 2; ++v) {
                const int gm = m0 + wm + i * 8 + g, gn = n0 + wn + j * 8 + 2 * t4 + v;
                if (gm < M && gn < N) {
                    if (ksplit == 1)
                        cf(batch, gm, gn, acc[i][j][v]);
                    else
                        partial[(((size_t)batch * ksplit + ks) * M + gm) * N + gn] = acc[i][j][v];
                }
            }
}

// ---------------------------------------------------------------------------
// Block-cooperative small fp64 GEMM from shared (or global) memory on the
// FP64 tensor cores: C(m, n) = sum_k A(m, k) B(k, n) with element strides
//   A(m, k) = A[m * sam + k * sak],  B(k, n) = B[k * sbk + n * sbn],
//   C(m, n) = C[m * scm + n * scn].
// The block's warps take 8 x 8 output tiles round-robin and step k by 4
// (DMMA m8n8k4); indices past M / N / K read as zero.  For the R x R and
// Q x R products of the ALS update (Q <= 256, R <= 64).  No barrier inside:
// callers synchronize before reading C.
// ---------------------------------------------------------------------------
__device__ inline void block_dmma_small(int M, int N, int K, const double* A, int sam, int sak, const double* B,
                                        int sbk, int sbn, double* C, int scm, int scn) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int g = lane >> 2, t4 = lane & 3;
    const int tm = (M + 7) >> 3, tn = (N + 7) >> 3;
    for (int tile = warp; tile < tm * tn; tile += nw) {
        const int m0 = (tile % tm) * 8, n0 = (tile / tm) * 8;
        double c0 = 0.0, c1 = 0.0;
        const int am = m0 + g, bn = n0 + g;
        for (int k0 = 0; k0 < K; k0 += 4) {
            const int k = k0 + t4;
            const double a = (am < M && k < K) ? A[am * sam + k * sak] : 0.0;
            const double b = (bn < N && k < K) ? B[k * sbk + bn * sbn] : 0.0;
            dmma_m8n8k4(c0, c1, a, b);
        }
        const int cm = m0 + g, cn = n0 + 2 * t4;
        if (cm < M) {
            if (cn < N) C[cm * scm + cn * scn] = c0;
            if (cn + 1 < N) C[cm * scm + (cn + 1) * scn] = c1;
        }
    }
}

// ---------------------------------------------------------------------------
// Pipelined variant for operands with 16-byte contiguous pairs along the
// fast dimension: the functors return element POINTERS (A(b, m, k), B(b, k, n))
// and tiles move by cp.async 16 B chunks through a 3-stage shared-memory
// ring, so global latency overlaps the DMMAs.  128 x 64 CTA tile, BK = 16,
// 8 warps of 32 x 32 (16 DMMA per 8 fragment loads).  A is M-fast
// (A_KFAST = false: pairs (m, m+1)) or K-fast (pairs (k, k+1)); B is K-fast.
// Requirements (checked by the caller): the pair start addresses are 16-byte
// aligned, M (M-fast A) or K is even, the K chunk of a split is a multiple of
// 16.  Rows/columns/k past the ranges are zero-filled (src-size 0).
// ---------------------------------------------------------------------------
namespace pipe {
constexpr int BM = 128, BN = 64, BK = 16, ST = 3, PAD = 4;
constexpr int A_M_FAST_ELEMS = BK * (BM + PAD);  // [k][m]
constexpr int A_K_FAST_ELEMS = BM * (BK + PAD);  // [m][k]
constexpr int B_ELEMS = BN * (BK + PAD);         // [n][k] (K-fast B) or [k][n] with BK * (BN + PAD) <= B_ELEMS
template <bool A_KFAST>
constexpr int a_elems() {
    return A_KFAST ? A_K_FAST_ELEMS : A_M_FAST_ELEMS;
}
template <bool A_KFAST>
constexpr size_t smem_bytes() {
    return (size_t)ST * (a_elems<A_KFAST>() + B_ELEMS) * sizeof(double);
}
__device__ __forceinline__ void cp16(void* dst, const void* src, bool valid) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    const int n = valid ? 16 : 0;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(src), "r"(n) : "memory");
}
__device__ __forceinline__ void commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}
}  // namespace pipe

template <bool A_KFAST, class AF, class BF, class CF, bool B_KFAST = true>
__global__ void __launch_bounds__(256)
    gemm_dmma_pipe_kernel(int M, int N, int K, int ksplit, int kchunk, AF af, BF bf, CF cf, double* partial) {
    using namespace pipe;
    pdl_trigger();
    pdl_wait();
    extern __shared__ double pipe_smem[];
    constexpr int AE = a_elems<A_KFAST>();
    double* As = pipe_smem;                 // ST x AE
    double* Bs = pipe_smem + ST * AE;       // ST x B_ELEMS
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g = lane >> 2, t4 = lane & 3;
    const int wm = (warp & 3) * 32, wn = (warp >> 2) * 32;
    const int zb = blockIdx.z;
    const int batch = zb / ksplit, ks = zb % ksplit;
    const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
    const int kbeg = ks * kchunk;
    const int kend = min(K, kbeg + kchunk);
    const int ntiles = kend > kbeg ? (kend - kbeg + BK - 1) / BK : 0;
    const double* dummy = af(batch, 0, 0);

    auto load = [&](int kt, int stg) {
        const int k0 = kbeg + kt * BK;
        double* as = As + stg * AE;
        double* bs = Bs + stg * B_ELEMS;
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const int c = tid + r * 256;  // 1024 chunks
            if (A_KFAST) {
                const int mm = c >> 3, kk = (c & 7) * 2;
                const int gm = m0 + mm, gk = k0 + kk;
                const bool v = gm < M && gk < kend;
                cp16(as + mm * (BK + PAD) + kk, v ? af(batch, gm, gk) : dummy, v);
            } else {
                const int kk = c >> 6, mm = (c & 63) * 2;
                const int gm = m0 + mm, gk = k0 + kk;
                const bool v = gm < M && gk < kend;
                cp16(as + kk * (BM + PAD) + mm, v ? af(batch, gm, gk) : dummy, v);
            }
        }
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            const int c = tid + r * 256;  // 512 chunks
            if (B_KFAST) {
                const int nn = c >> 3, kk = (c & 7) * 2;
                const int gn = n0 + nn, gk = k0 + kk;
                const bool v = gn < N && gk < kend;
                cp16(bs + nn * (BK + PAD) + kk, v ? bf(batch, gk, gn) : dummy, v);
            } else {  // pairs (n, n+1): [k][n] layout
                const int kk = c >> 5, nn = (c & 31) * 2;
                const int gn = n0 + nn, gk = k0 + kk;
                const bool v = gn < N && gk < kend;
                cp16(bs + kk * (BN + PAD) + nn, v ? bf(batch, gk, gn) : dummy, v);
            }
        }
    };

    double acc[4][4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

#pragma unroll
    for (int s = 0; s < ST - 1; ++s) {
        if (s < ntiles) load(s, s);
        commit();
    }
    for (int kt = 0; kt < ntiles; ++kt) {
        wait<ST - 2>();
        __syncthreads();
        if (kt + ST - 1 < ntiles) load(kt + ST - 1, (kt + ST - 1) % ST);
        commit();
        const double* as = As + (kt % ST) * AE;
        const double* bs = Bs + (kt % ST) * B_ELEMS;
        const int kvalid = kend - (kbeg + kt * BK);  // < BK only on a ragged last tile (uniform)
#pragma unroll
        for (int kk = 0; kk < BK; kk += 4) {
            if (kk >= kvalid) break;
            double fa[4], fb[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int m = wm + i * 8 + g;
                fa[i] = A_KFAST ? as[m * (BK + PAD) + kk + t4] : as[(kk + t4) * (BM + PAD) + m];
            }
#pragma unroll
            for (int j = 0; j < 4; ++j)
                fb[j] = B_KFAST ? bs[(wn + j * 8 + g) * (BK + PAD) + kk + t4] : bs[(kk + t4) * (BN + PAD) + wn + j * 8 + g];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) dmma_m8n8k4(acc[i][j][0], acc[i][j][1], fa[i], fb[j]);
        }
    }
    wait<0>();
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int v = 0; v < 2; ++v) {
                const int gm = m0 + wm + i * 8 + g, gn = n0 + wn + j * 8 + 2 * t4 + v;
                if (gm < M && gn < N) {
                    if (ksplit == 1)
                        cf(batch, gm, gn, acc[i][j][v]);
                    else
                        partial[(((size_t)batch * ksplit + ks) * M + gm) * N + gn] = acc[i][j][v];
                }
            }
}

template <bool A_KFAST, class AF, class BF, class CF, bool B_KFAST = true>
void gemm_f64_pipe(int batches, int M, int N, int K, AF af, BF bf, CF cf, cudaStream_t st, int ksplit = 1,
                   double* workspace = nullptr, bool pdl = false) {
    if (batches <= 0 || M <= 0 || N <= 0) return;
    if (K <= 0) ksplit = 1;
    if (ksplit < 1) ksplit = 1;
    int kchunk = (K + ksplit - 1) / ksplit;
    kchunk = ((kchunk + pipe::BK - 1) / pipe::BK) * pipe::BK;
    const size_t smem = pipe::smem_bytes<A_KFAST>();
    static PerDevice attr;
    attr.once([&] {
        OCTEN_CUDA(cudaFuncSetAttribute(gemm_dmma_pipe_kernel<A_KFAST, AF, BF, CF, B_KFAST>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    });
    dim3 grid((N + pipe::BN - 1) / pipe::BN, (M + pipe::BM - 1) / pipe::BM, batches * ksplit);
    if (pdl) {
        launch_pdl(gemm_dmma_pipe_kernel<A_KFAST, AF, BF, CF, B_KFAST>, grid, dim3(256), smem, st, M, N, K, ksplit,
                   kchunk, af, bf, cf, workspace);
    } else {
        gemm_dmma_pipe_kernel<A_KFAST, AF, BF, CF, B_KFAST><<<grid, 256, smem, st>>>(M, N, K, ksplit, kchunk, af, bf,
                                                                                     cf, workspace);
        OCTEN_LAUNCHED(1);
    }
    if (ksplit > 1) {
        const size_t total = (size_t)batches * M * N;
        int blocks = (int)((total + 255) / 256);
        if (blocks > 148 * 16) blocks = 148 * 16;
        gemm_splitk_reduce<double><<<blocks, 256, 0, st>>>(batches, M, N, ksplit, workspace, cf);
        OCTEN_LAUNCHED(1);
    }
}

// Same interface as gemm_simt (fp64 only).
template <bool A_KFAST, bool B_KFAST, class AF, class BF, class CF>
void gemm_f64(int batches, int M, int N, int K, AF af, BF bf, CF cf, cudaStream_t st, int ksplit = 1,
              double* workspace = nullptr, int lower_only = 0) {
    if (batches <= 0 || M <= 0 || N <= 0) return;
    if (K <= 0) ksplit = 1;
    if (ksplit < 1) ksplit = 1;
    int kchunk = (K + ksplit - 1) / ksplit;
    kchunk = ((kchunk + 15) / 16) * 16;
    if (kchunk < 16) kchunk = 16;
    dim3 grid((N + 63) / 64, (M + 63) / 64, batches * ksplit);
    gemm_dmma_kernel<A_KFAST, B_KFAST><<<grid, 256, 0, st>>>(M, N, K, ksplit, kchunk, af, bf, cf, workspace,
                                                             lower_only);
    OCTEN_LAUNCHED(1);
    if (ksplit > 1) {
        const size_t total = (size_t)batches * M * N;
        int blocks = (int)((total + 255) / 256);
        if (blocks > 148 * 16) blocks = 148 * 16;
        gemm_splitk_reduce<double><<<blocks, 256, 0, st>>>(batches, M, N, ksplit, workspace, cf);
        OCTEN_LAUNCHED(1);
    }
}

}  // namespace octen
