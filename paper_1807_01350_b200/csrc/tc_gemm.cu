// tcgen05 split-TF32 GEMM for the dense compression's mode-1 contraction
// (reference: the mode-0 product of compress(), compression.cpp:117-128 /
// tensor.cpp:168-178, batched over all replicas with the shared columns
// deduplicated):
//
//     Z[m, n] = sum_k A[m, k] * X[k + K n]        (A: Meff x K, X: K x N, fp32)
//
// fp32 accuracy from the TF32 tensor cores: A = A_hi + A_lo (pre-split once
// per stream from the fp64 projections), X = X_hi + X_lo (split in shared
// memory right after the TMA lands), D += A_hi X_hi + A_hi X_lo + A_lo X_hi,
// fp32 accumulation in TMEM.  Per CTA one 128 x 256 output tile:
//   warp 0      TMA producer (A_hi, A_lo, X tiles; 128B swizzle, 2 stages)
//   warp 1      TMEM allocation + single-thread tcgen05.mma issue
//   warps 2..7  split X into hi/lo in place (same swizzled layout)
//   warps 4..7  epilogue: tcgen05.ld 32x32b.x32 -> fp32 stores
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdlib>

#include <cstdint>
#include <cstring>
#include <mutex>

#include "errors.hpp"
#include "octen_common.cuh"
#include "tc_gemm.hpp"

namespace octen {

namespace {

constexpr int BM = 128, BN = 256, BKB = 128;  // BK in bytes (32 fp32), 128 B swizzle (mode-2 kernel)
constexpr int BK = BKB / 4;
// GEMM1: 16-wide k-blocks (64 B rows, 64 B swizzle) in a 4-deep ring: the
// same 192 KB of shared memory as two 32-wide stages, but three k-blocks are
// in flight while one is consumed, which covers the TMA latency
constexpr int G1_BKB = 64;
constexpr int G1_BK = G1_BKB / 4;
constexpr int STAGES = 4;
constexpr int A_BYTES = BM * G1_BKB;           // 8 KB
constexpr int B_BYTES = BN * G1_BKB;           // 16 KB
constexpr int STAGE_BYTES = 2 * A_BYTES + 2 * B_BYTES;  // A_hi, A_lo, B(hi in place), B_lo
constexpr int NUM_THREADS = 256;
constexpr int CONVERT_WARP0 = 2, CONVERT_WARPS = 6;
// kind::tf32 reads the fp32 container and ignores its 13 low mantissa bits,
// so the raw tile already is the hi part: the converters only write lo
// (one 16 B store per 4 elements instead of two; shared memory bandwidth is
// the converters' limit).  Set true to store the masked hi explicitly.
constexpr bool kWriteHi = false;
constexpr uint32_t TMEM_COLS = 256;

// ---- PTX helpers ----
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// Bounded wait: a protocol bug traps (kernel error) instead of hanging the GPU.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    const uint32_t addr = smem_u32(bar);
    for (uint32_t it = 0;; ++it) {
        uint32_t ok;
        asm volatile(
            "{\n"
            ".reg .pred P1;\n"
            "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n"
            "selp.u32 %0, 1, 0, P1;\n"
            "}\n"
            : "=r"(ok)
            : "r"(addr), "r"(phase)
            : "memory");
        if (ok) return;
        if (it > (1u << 26)) asm volatile("trap;");
    }
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
            smem_u32(dst)),
        "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
        : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// UMMA shared-memory descriptor: K-major, 64B swizzle, 8-row groups 512 B apart.
__device__ __forceinline__ uint64_t make_desc_sw64(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);        // start address
    d |= (uint64_t)1 << 16;                         // leading byte offset (unused for swizzled K-major)
    d |= (uint64_t)(512 >> 4) << 32;                // stride byte offset
    d |= (uint64_t)1 << 46;                         // descriptor version (sm_100)
    d |= (uint64_t)4 << 61;                         // layout: SWIZZLE_64B
    return d;
}
// UMMA shared-memory descriptor: K-major, 128B swizzle, 8-row groups 1024 B apart.
__device__ __forceinline__ uint64_t make_desc_sw128(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);        // start address
    d |= (uint64_t)1 << 16;                         // leading byte offset (unused for SW128 K-major)
    d |= (uint64_t)(1024 >> 4) << 32;               // stride byte offset
    d |= (uint64_t)1 << 46;                         // descriptor version (sm_100)
    d |= (uint64_t)2 << 61;                         // layout: SWIZZLE_128B
    return d;
}

// Instruction descriptor: kind::tf32, fp32 accumulate, A/B K-major, M=128, N=256.
constexpr uint32_t make_idesc() {
    return (1u << 4)                // D format F32
           | (2u << 7)              // A format TF32
           | (2u << 10)             // B format TF32
           | ((uint32_t)(BN >> 3) << 17)  // N
           | ((uint32_t)(BM >> 4) << 24); // M
}

__device__ __forceinline__ void mma_tf32(uint32_t dtmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t acc) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n"
        "}\n" ::"r"(dtmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}

// Row scatter of the epilogue (scP > 0): output row m of the deduplicated
// stack goes to replica rows p*Q + a -- the `sh` shared rows to every replica,
// private row m = sh + p (Q - sh) + (a - sh) to its own -- so the next
// contraction reads each replica's Q rows contiguously.
__device__ __forceinline__ void store_row_chunk(float* Z, long long ldz, int row, long long nb, long long N,
                                                const uint32_t* r, int scP, int scQ, int scSh) {
    auto put = [&](float* zrow) {
        if (nb + 32 <= N && (ldz % 4) == 0) {
            float4* dst = (float4*)(zrow + nb);
#pragma unroll
            for (int j = 0; j < 8; ++j)
                dst[j] = make_float4(__uint_as_float(r[4 * j]), __uint_as_float(r[4 * j + 1]),
                                     __uint_as_float(r[4 * j + 2]), __uint_as_float(r[4 * j + 3]));
        } else {
            for (int j = 0; j < 32; ++j)
                if (nb + j < N) zrow[nb + j] = __uint_as_float(r[j]);
        }
    };
    if (scP <= 0) {
        put(Z + (size_t)row * ldz);
    } else if (row < scSh) {
        for (int p = 0; p < scP; ++p) put(Z + ((size_t)p * scQ + row) * ldz);
    } else {
        const int pr = scQ - scSh;
        const int p = (row - scSh) / pr, a = scSh + (row - scSh) % pr;
        put(Z + ((size_t)p * scQ + a) * ldz);
    }
}

__global__ void __launch_bounds__(NUM_THREADS, 1)
    tc_gemm_tf32x3_kernel(const __grid_constant__ CUtensorMap map_ahi, const __grid_constant__ CUtensorMap map_alo,
                          const __grid_constant__ CUtensorMap map_x, float* __restrict__ Z, int M, long long N, int K,
                          long long ldz, int scP, int scQ, int scSh) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    // 1024-align the stage buffers (SW128 atoms)
    uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    uint64_t* full_bar = (uint64_t*)(smem + STAGES * STAGE_BYTES);
    uint64_t* conv_bar = full_bar + STAGES;
    uint64_t* empty_bar = conv_bar + STAGES;
    uint64_t* done_bar = empty_bar + STAGES;
    uint32_t* tmem_slot = (uint32_t*)(done_bar + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // m-tiles fastest: the CTAs sharing one X slab (all m-tiles of an n-tile)
    // run back to back, so X comes from DRAM once and from L2 thereafter
    const int m_tile = blockIdx.x, n_tile = blockIdx.y;
    const int m0 = m_tile * BM;
    const long long n0 = (long long)n_tile * BN;
    const int num_kb = (K + G1_BK - 1) / G1_BK;

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full_bar[s], 1);
            mbar_init(&conv_bar[s], CONVERT_WARPS * 32);
            mbar_init(&empty_bar[s], 1);
        }
        mbar_init(done_bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            // ---- TMA producer ----
            for (int kb = 0; kb < num_kb; ++kb) {
                const int s = kb % STAGES;
                const uint32_t ph = (kb / STAGES) & 1;
                if (kb >= STAGES) mbar_wait(&empty_bar[s], ph ^ 1);
                uint8_t* st = smem + s * STAGE_BYTES;
                mbar_arrive_expect_tx(&full_bar[s], 2 * A_BYTES + B_BYTES);
                tma_load_2d(st, &map_ahi, &full_bar[s], kb * G1_BK, m0);
                tma_load_2d(st + A_BYTES, &map_alo, &full_bar[s], kb * G1_BK, m0);
                tma_load_2d(st + 2 * A_BYTES, &map_x, &full_bar[s], kb * G1_BK, (int)n0);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            // ---- MMA issuer ----
            constexpr uint32_t idesc = make_idesc();
            for (int kb = 0; kb < num_kb; ++kb) {
                const int s = kb % STAGES;
                const uint32_t ph = (kb / STAGES) & 1;
                mbar_wait(&conv_bar[s], ph);
                tc_fence_after();
                uint8_t* st = smem + s * STAGE_BYTES;
                const uint32_t a_hi = smem_u32(st), a_lo = smem_u32(st + A_BYTES);
                const uint32_t b_hi = smem_u32(st + 2 * A_BYTES), b_lo = smem_u32(st + 2 * A_BYTES + B_BYTES);
#pragma unroll
                for (int k = 0; k < G1_BK / 8; ++k) {
                    const uint32_t off = k * 32;  // 8 tf32 = 32 bytes along K inside the swizzle atom
                    const uint32_t acc0 = (kb > 0 || k > 0) ? 1u : 0u;
                    mma_tf32(tmem_base, make_desc_sw64(a_hi + off), make_desc_sw64(b_hi + off), idesc, acc0);
                    mma_tf32(tmem_base, make_desc_sw64(a_hi + off), make_desc_sw64(b_lo + off), idesc, 1u);
                    mma_tf32(tmem_base, make_desc_sw64(a_lo + off), make_desc_sw64(b_hi + off), idesc, 1u);
                }
                mma_commit(&empty_bar[s]);
            }
            mma_commit(done_bar);
        }
    } else {
        // ---- X hi/lo split (warps 2..7) ----
        const int ct = threadIdx.x - CONVERT_WARP0 * 32;
        for (int kb = 0; kb < num_kb; ++kb) {
            const int s = kb % STAGES;
            const uint32_t ph = (kb / STAGES) & 1;
            mbar_wait(&full_bar[s], ph);
            uint8_t* st = smem + s * STAGE_BYTES;
            float4* bx = (float4*)(st + 2 * A_BYTES);
            float4* bl = (float4*)(st + 2 * A_BYTES + B_BYTES);
            for (int i = ct; i < B_BYTES / 16; i += CONVERT_WARPS * 32) {
                float4 v = bx[i];
                float4 h, l;
                h.x = __uint_as_float(__float_as_uint(v.x) & 0xFFFFE000u);
                h.y = __uint_as_float(__float_as_uint(v.y) & 0xFFFFE000u);
                h.z = __uint_as_float(__float_as_uint(v.z) & 0xFFFFE000u);
                h.w = __uint_as_float(__float_as_uint(v.w) & 0xFFFFE000u);
                l.x = v.x - h.x;
                l.y = v.y - h.y;
                l.z = v.z - h.z;
                l.w = v.w - h.w;
                if (kWriteHi) bx[i] = h;
                bl[i] = l;
            }
            fence_proxy_async();
            mbar_arrive(&conv_bar[s]);
        }
        if (warp >= 4) {
            // ---- epilogue ----
            mbar_wait(done_bar, 0);
            tc_fence_after();
            const int q = warp & 3;
            const int row = m0 + q * 32 + lane;
#pragma unroll 1
            for (int c0 = 0; c0 < BN; c0 += 32) {
                uint32_t r[32];
                const uint32_t taddr = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)c0;
                asm volatile(
                    "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                    "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                    : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                      "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
                      "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
                      "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
                      "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
                    : "r"(taddr));
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                if (row < M) store_row_chunk(Z, ldz, row, n0 + c0, N, r, scP, scQ, scSh);
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TMEM_COLS));
    }
}

// ---------------------------------------------------------------------------
// Persistent GEMM1: one CTA per SM loops over the output tiles (m-tiles
// fastest, tile L = blockIdx.x + i * gridDim.x, so the CTAs running at the
// same time share X slabs in L2).  The accumulator is double-buffered in
// TMEM (2 x 256 of the 512 columns): four dedicated epilogue warps (8..11)
// drain tile i while the MMA warp accumulates tile i+1, and the stage ring
// (TMA -> converters -> MMA) runs on across tile boundaries.  The per-tile
// prologue (TMEM alloc, barrier init, pipeline fill) and the epilogue's
// 128 KB of stores no longer sit between mainloops.
//   warp 0: TMA producer    warp 1: TMEM alloc + MMA issuer
//   warps 2..7: X lo split   warps 8..11: epilogue (TMEM lanes 32 (w % 4) ..)
// ---------------------------------------------------------------------------
constexpr int G1P_THREADS = 384;
constexpr int G1P_EPI_WARP0 = 8;
constexpr uint32_t G1P_TMEM_COLS = 512;
constexpr size_t G1P_EPI_BYTES = 4 * 32 * 33 * sizeof(float);

__global__ void __launch_bounds__(G1P_THREADS, 1)
    tc_gemm_tf32x3_persistent_kernel(const __grid_constant__ CUtensorMap map_ahi,
                                     const __grid_constant__ CUtensorMap map_alo,
                                     const __grid_constant__ CUtensorMap map_x, float* __restrict__ Z, int M,
                                     long long N, int K, long long ldz, int scP, int scQ, int scSh, int mt,
                                     long long ntiles, int two_mma, int* __restrict__ nonfinite) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    uint64_t* full_bar = (uint64_t*)(smem + STAGES * STAGE_BYTES);
    uint64_t* conv_bar = full_bar + STAGES;
    uint64_t* empty_bar = conv_bar + STAGES;
    uint64_t* tfull_bar = empty_bar + STAGES;  // [2] MMA -> epilogue
    uint64_t* tempty_bar = tfull_bar + 2;      // [2] epilogue -> MMA
    uint32_t* tmem_slot = (uint32_t*)(tempty_bar + 2);
    float* epi = (float*)(smem + STAGES * STAGE_BYTES + 256);  // 4 warps x 32 x 33 epilogue staging

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int num_kb = (K + G1_BK - 1) / G1_BK;

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full_bar[s], 1);
            mbar_init(&conv_bar[s], CONVERT_WARPS * 32);
            mbar_init(&empty_bar[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&tfull_bar[b], 1);
            mbar_init(&tempty_bar[b], 4 * 32);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(G1P_TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            // ---- TMA producer ----
            uint32_t it = 0;
            for (long long L = blockIdx.x; L < ntiles; L += gridDim.x) {
                const int m0 = (int)(L % mt) * BM;
                const long long n0 = (L / mt) * BN;
                for (int kb = 0; kb < num_kb; ++kb, ++it) {
                    const int s = it % STAGES;
                    const uint32_t ph = (it / STAGES) & 1;
                    if (it >= STAGES) mbar_wait(&empty_bar[s], ph ^ 1);
                    uint8_t* st = smem + s * STAGE_BYTES;
                    mbar_arrive_expect_tx(&full_bar[s], 2 * A_BYTES + B_BYTES);
                    tma_load_2d(st, &map_ahi, &full_bar[s], kb * G1_BK, m0);
                    tma_load_2d(st + A_BYTES, &map_alo, &full_bar[s], kb * G1_BK, m0);
                    tma_load_2d(st + 2 * A_BYTES, &map_x, &full_bar[s], kb * G1_BK, (int)n0);
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            // ---- MMA issuer ----
            constexpr uint32_t idesc = make_idesc();
            uint32_t it = 0, ti = 0;
            for (long long L = blockIdx.x; L < ntiles; L += gridDim.x, ++ti) {
                const uint32_t acc = ti & 1, use = ti >> 1;
                if (ti >= 2) mbar_wait(&tempty_bar[acc], (use - 1) & 1);  // tile ti-2 drained
                tc_fence_after();
                const uint32_t dt = tmem_base + acc * 256;
                for (int kb = 0; kb < num_kb; ++kb, ++it) {
                    const int s = it % STAGES;
                    const uint32_t ph = (it / STAGES) & 1;
                    mbar_wait(&conv_bar[s], ph);
                    tc_fence_after();
                    uint8_t* st = smem + s * STAGE_BYTES;
                    const uint32_t a_hi = smem_u32(st), a_lo = smem_u32(st + A_BYTES);
                    const uint32_t b_hi = smem_u32(st + 2 * A_BYTES), b_lo = smem_u32(st + 2 * A_BYTES + B_BYTES);
#pragma unroll
                    for (int k = 0; k < G1_BK / 8; ++k) {
                        const uint32_t off = k * 32;
                        const uint32_t acc0 = (kb > 0 || k > 0) ? 1u : 0u;
                        mma_tf32(dt, make_desc_sw64(a_hi + off), make_desc_sw64(b_hi + off), idesc, acc0);
                        if (!two_mma)
                            mma_tf32(dt, make_desc_sw64(a_hi + off), make_desc_sw64(b_lo + off), idesc, 1u);
                        mma_tf32(dt, make_desc_sw64(a_lo + off), make_desc_sw64(b_hi + off), idesc, 1u);
                    }
                    mma_commit(&empty_bar[s]);
                }
                mma_commit(&tfull_bar[acc]);
            }
        }
    } else if (warp < G1P_EPI_WARP0) {
        // ---- X hi/lo split (warps 2..7); with `nonfinite` the batch's
        // non-finite scan rides along (every X element passes through here) ----
        const int ct = threadIdx.x - CONVERT_WARP0 * 32;
        uint32_t it = 0;
        uint32_t bad = 0;
        auto nf = [](float f) { return (__float_as_uint(f) & 0x7f800000u) == 0x7f800000u ? 1u : 0u; };
        for (long long L = blockIdx.x; L < ntiles; L += gridDim.x) {
            for (int kb = 0; kb < num_kb; ++kb, ++it) {
                const int s = it % STAGES;
                const uint32_t ph = (it / STAGES) & 1;
                mbar_wait(&full_bar[s], ph);
                uint8_t* st = smem + s * STAGE_BYTES;
                float4* bx = (float4*)(st + 2 * A_BYTES);
                float4* bl = (float4*)(st + 2 * A_BYTES + B_BYTES);
                if (two_mma) {
                    // X rounded to the nearest TF32 in place (the MMAs then
                    // read it exactly): round half away from zero on the
                    // magnitude bits
                    for (int i = ct; i < B_BYTES / 16; i += CONVERT_WARPS * 32) {
                        const float4 v = bx[i];
                        bad |= nf(v.x) | nf(v.y) | nf(v.z) | nf(v.w);
                        float4 h;
                        h.x = __uint_as_float((__float_as_uint(v.x) + 0x1000u) & 0xFFFFE000u);
                        h.y = __uint_as_float((__float_as_uint(v.y) + 0x1000u) & 0xFFFFE000u);
                        h.z = __uint_as_float((__float_as_uint(v.z) + 0x1000u) & 0xFFFFE000u);
                        h.w = __uint_as_float((__float_as_uint(v.w) + 0x1000u) & 0xFFFFE000u);
                        bx[i] = h;
                    }
                } else {
                    for (int i = ct; i < B_BYTES / 16; i += CONVERT_WARPS * 32) {
                        const float4 v = bx[i];
                        bad |= nf(v.x) | nf(v.y) | nf(v.z) | nf(v.w);
                        float4 l;
                        l.x = v.x - __uint_as_float(__float_as_uint(v.x) & 0xFFFFE000u);
                        l.y = v.y - __uint_as_float(__float_as_uint(v.y) & 0xFFFFE000u);
                        l.z = v.z - __uint_as_float(__float_as_uint(v.z) & 0xFFFFE000u);
                        l.w = v.w - __uint_as_float(__float_as_uint(v.w) & 0xFFFFE000u);
                        bl[i] = l;
                    }
                }
                fence_proxy_async();
                mbar_arrive(&conv_bar[s]);
            }
        }
        if (nonfinite && __any_sync(0xffffffffu, bad) && lane == 0) atomicOr(nonfinite, 1);
    } else {
        // ---- epilogue (warps 8..11) ----
        const int q = warp & 3;
        uint32_t ti = 0;
        for (long long L = blockIdx.x; L < ntiles; L += gridDim.x, ++ti) {
            const uint32_t acc = ti & 1, use = ti >> 1;
            const int m0 = (int)(L % mt) * BM;
            const long long n0 = (L / mt) * BN;
            mbar_wait(&tfull_bar[acc], use & 1);
            tc_fence_after();
            // staged through shared memory so every store instruction writes
            // whole 128 B lines (8 lanes per row): lane-per-row stores left
            // half-written sectors in L2 that were evicted early under the
            // concurrent mainloop (ECC read-modify-write, 1.7x DRAM traffic)
            float* tile = epi + q * 32 * 33;
#pragma unroll 1
            for (int c0 = 0; c0 < BN; c0 += 32) {
                uint32_t r[32];
                const uint32_t taddr = tmem_base + acc * 256 + ((uint32_t)(q * 32) << 16) + (uint32_t)c0;
                asm volatile(
                    "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                    "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                    : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                      "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
                      "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
                      "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
                      "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
                    : "r"(taddr));
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                for (int j = 0; j < 32; ++j) tile[lane * 33 + j] = __uint_as_float(r[j]);
                __syncwarp();
                const int cc = (lane & 7) * 4;
                const long long col = n0 + c0 + cc;
#pragma unroll 1
                for (int it2 = 0; it2 < 8; ++it2) {
                    const int rr = it2 * 4 + (lane >> 3);
                    const int row = m0 + q * 32 + rr;
                    if (row >= M) continue;
                    const float v0 = tile[rr * 33 + cc], v1 = tile[rr * 33 + cc + 1], v2 = tile[rr * 33 + cc + 2],
                                v3 = tile[rr * 33 + cc + 3];
                    auto put = [&](float* zrow) {
                        if (col + 4 <= N && (ldz % 4) == 0) {
                            *(float4*)(zrow + col) = make_float4(v0, v1, v2, v3);
                        } else {
                            if (col < N) zrow[col] = v0;
                            if (col + 1 < N) zrow[col + 1] = v1;
                            if (col + 2 < N) zrow[col + 2] = v2;
                            if (col + 3 < N) zrow[col + 3] = v3;
                        }
                    };
                    if (scP <= 0) {
                        put(Z + (size_t)row * ldz);
                    } else if (row < scSh) {
                        for (int p = 0; p < scP; ++p) put(Z + ((size_t)p * scQ + row) * ldz);
                    } else {
                        const int pr = scQ - scSh;
                        const int p = (row - scSh) / pr, a = scSh + (row - scSh) % pr;
                        put(Z + ((size_t)p * scQ + a) * ldz);
                    }
                }
                __syncwarp();
            }
            // every thread's TMEM reads of this buffer are complete
            tc_fence_before();
            mbar_arrive(&tempty_bar[acc]);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(G1P_TMEM_COLS));
    }
}

// ---------------------------------------------------------------------------
// Mode-2 contraction of the compression, batched over (replica p, slice k):
//   Z2[p][a + Q b + Q^2 k] = sum_j Z1[p Q + a][k J + j] * V_p[j, b]
// One CTA per (p, k): M = 128 rows of Z1 (a < Q used), N = 112 columns
// (b < Q used), K = J in 32-wide blocks.  Z1 (replica-contiguous rows, the
// scattered GEMM1 output) is split hi/lo in shared memory like X in GEMM1;
// V_p comes pre-split (Vhi/Vlo, P*Q x ldv, rows b, K = j contiguous).  Rows
// or columns past the tensors are TMA zero-filled; A columns past slice k
// meet zero B rows (j >= J), so they contribute nothing.
// ---------------------------------------------------------------------------
// N tile (columns b of V_p): 112 covers Q <= 112 (c3: Q = 100), 128 covers
// Q <= 128 (c5); the stage size follows it
constexpr int M2_BN_MAX = 128;
constexpr int M2_STAGES = 3;
constexpr int M2_A_BYTES = BM * BKB;                      // 16 KB
template <int BN2>
constexpr int m2_b_bytes() { return BN2 * BKB; }          // 14 / 16 KB
template <int BN2>
constexpr int m2_stage_bytes() { return 2 * M2_A_BYTES + 2 * m2_b_bytes<BN2>(); }
constexpr uint32_t M2_TMEM_COLS = 128;

template <int BN2>
constexpr uint32_t make_idesc_m2() {
    return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(BN2 >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
}

template <int BN2>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    tc_mode2_tf32x3_kernel(const __grid_constant__ CUtensorMap map_z1, const __grid_constant__ CUtensorMap map_vhi,
                           const __grid_constant__ CUtensorMap map_vlo, float* __restrict__ Z2, int Q, int J, int tc,
                           long long zstride) {
    constexpr int M2_BN = BN2;
    constexpr int M2_B_BYTES = m2_b_bytes<BN2>();
    constexpr int M2_STAGE_BYTES = m2_stage_bytes<BN2>();
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    uint64_t* full_bar = (uint64_t*)(smem + M2_STAGES * M2_STAGE_BYTES);
    uint64_t* conv_bar = full_bar + M2_STAGES;
    uint64_t* empty_bar = conv_bar + M2_STAGES;
    uint64_t* done_bar = empty_bar + M2_STAGES;
    uint32_t* tmem_slot = (uint32_t*)(done_bar + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int p = blockIdx.x / tc, k = blockIdx.x % tc;
    const int num_kb = (J + BK - 1) / BK;

    if (threadIdx.x == 0) {
        for (int s = 0; s < M2_STAGES; ++s) {
            mbar_init(&full_bar[s], 1);
            mbar_init(&conv_bar[s], CONVERT_WARPS * 32);
            mbar_init(&empty_bar[s], 1);
        }
        mbar_init(done_bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(M2_TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            for (int kb = 0; kb < num_kb; ++kb) {
                const int s = kb % M2_STAGES;
                const uint32_t ph = (kb / M2_STAGES) & 1;
                if (kb >= M2_STAGES) mbar_wait(&empty_bar[s], ph ^ 1);
                uint8_t* st = smem + s * M2_STAGE_BYTES;
                mbar_arrive_expect_tx(&full_bar[s], M2_A_BYTES + 2 * M2_B_BYTES);
                tma_load_2d(st, &map_z1, &full_bar[s], k * J + kb * BK, p * Q);
                tma_load_2d(st + 2 * M2_A_BYTES, &map_vhi, &full_bar[s], kb * BK, p * Q);
                tma_load_2d(st + 2 * M2_A_BYTES + M2_B_BYTES, &map_vlo, &full_bar[s], kb * BK, p * Q);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            constexpr uint32_t idesc = make_idesc_m2<BN2>();
            for (int kb = 0; kb < num_kb; ++kb) {
                const int s = kb % M2_STAGES;
                const uint32_t ph = (kb / M2_STAGES) & 1;
                mbar_wait(&conv_bar[s], ph);
                tc_fence_after();
                uint8_t* st = smem + s * M2_STAGE_BYTES;
                const uint32_t a_hi = smem_u32(st), a_lo = smem_u32(st + M2_A_BYTES);
                const uint32_t b_hi = smem_u32(st + 2 * M2_A_BYTES), b_lo = smem_u32(st + 2 * M2_A_BYTES + M2_B_BYTES);
#pragma unroll
                for (int kk = 0; kk < BK / 8; ++kk) {
                    const uint32_t off = kk * 32;
                    const uint32_t acc0 = (kb > 0 || kk > 0) ? 1u : 0u;
                    mma_tf32(tmem_base, make_desc_sw128(a_hi + off), make_desc_sw128(b_hi + off), idesc, acc0);
                    mma_tf32(tmem_base, make_desc_sw128(a_hi + off), make_desc_sw128(b_lo + off), idesc, 1u);
                    mma_tf32(tmem_base, make_desc_sw128(a_lo + off), make_desc_sw128(b_hi + off), idesc, 1u);
                }
                mma_commit(&empty_bar[s]);
            }
            mma_commit(done_bar);
        }
    } else {
        // ---- Z1 tile hi/lo split (warps 2..7) ----
        const int ct = threadIdx.x - CONVERT_WARP0 * 32;
        for (int kb = 0; kb < num_kb; ++kb) {
            const int s = kb % M2_STAGES;
            const uint32_t ph = (kb / M2_STAGES) & 1;
            mbar_wait(&full_bar[s], ph);
            uint8_t* st = smem + s * M2_STAGE_BYTES;
            float4* ah = (float4*)st;
            float4* al = (float4*)(st + M2_A_BYTES);
            for (int i = ct; i < M2_A_BYTES / 16; i += CONVERT_WARPS * 32) {
                const float4 v = ah[i];
                float4 h, l;
                h.x = __uint_as_float(__float_as_uint(v.x) & 0xFFFFE000u);
                h.y = __uint_as_float(__float_as_uint(v.y) & 0xFFFFE000u);
                h.z = __uint_as_float(__float_as_uint(v.z) & 0xFFFFE000u);
                h.w = __uint_as_float(__float_as_uint(v.w) & 0xFFFFE000u);
                l.x = v.x - h.x;
                l.y = v.y - h.y;
                l.z = v.z - h.z;
                l.w = v.w - h.w;
                if (kWriteHi) ah[i] = h;
                al[i] = l;
            }
            fence_proxy_async();
            mbar_arrive(&conv_bar[s]);
        }
        if (warp >= 4) {
            // ---- epilogue: lanes are rows a; each column b is one coalesced 128 B store per warp ----
            mbar_wait(done_bar, 0);
            tc_fence_after();
            const int q = warp & 3;
            const int a = q * 32 + lane;
            const size_t q2 = (size_t)Q * Q;
            float* zb = Z2 + (size_t)p * zstride + q2 * k;
#pragma unroll 1
            for (int c0 = 0; c0 < M2_BN; c0 += 32) {
                uint32_t r[32];
                const uint32_t taddr = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)c0;
                asm volatile(
                    "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                    "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                    : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                      "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
                      "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
                      "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
                      "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
                    : "r"(taddr));
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                if (a < Q) {
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        const int b = c0 + j;
                        if (b < Q) zb[a + (size_t)Q * b] = __uint_as_float(r[j]);
                    }
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(M2_TMEM_COLS));
    }
}

// ---- host: tensor maps through the driver entry point (no libcuda link) ----
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn get_encode() {
    static EncodeTiledFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = (EncodeTiledFn)p;
    });
    return fn;
}

bool make_map(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer, uint64_t row_bytes,
              uint32_t box_inner, uint32_t box_outer,
              CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B) {
    EncodeTiledFn enc = get_encode();
    if (!enc) return false;
    // keep every extent and stride a whole number of 16-byte units
    if ((inner * 4) % 16 != 0 || row_bytes % 16 != 0) return false;
    cuuint64_t dims[2] = {inner, outer};
    cuuint64_t strides[1] = {row_bytes};
    cuuint32_t box[2] = {box_inner, box_outer};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(base), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

bool g_disabled = false;

}  // namespace

void* tc_tensor_map_encoder() { return (void*)get_encode(); }

bool tc_gemm_available() {
    if (g_disabled) return false;
    if (std::getenv("OCTEN_DISABLE_TCGEN05")) return false;
    int dev = 0, major = 0, minor = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return false;
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
    cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
    return major == 10 && minor == 0 && get_encode() != nullptr;
}

bool tc_gemm_tf32x3(const float* Ahi, const float* Alo, int lda, const float* X, float* Z, int M, long long N, int K,
                    cudaStream_t st, int scatter_p, int scatter_q, int scatter_sh, int* nonfinite, int max_ctas) {
    if (!tc_gemm_available()) return false;
    if ((K % 4) != 0 || (lda % 4) != 0 || ((uintptr_t)X % 16) != 0 || ((uintptr_t)Ahi % 16) != 0 ||
        ((uintptr_t)Alo % 16) != 0 || N > (1LL << 31) - 1 || M <= 0 || N <= 0 || K <= 0)
        return false;
    CUtensorMap mhi, mlo, mx;
    // inner extents in whole 16-byte units: the zero padding of A (lda >= K)
    // stands in for the tail (X's own extent is K, TMA zero-fills past it)
    if (!make_map(&mhi, Ahi, (uint64_t)lda, (uint64_t)M, (uint64_t)lda * 4, G1_BK, BM, CU_TENSOR_MAP_SWIZZLE_64B))
        return false;
    if (!make_map(&mlo, Alo, (uint64_t)lda, (uint64_t)M, (uint64_t)lda * 4, G1_BK, BM, CU_TENSOR_MAP_SWIZZLE_64B))
        return false;
    if (!make_map(&mx, X, (uint64_t)K, (uint64_t)N, (uint64_t)K * 4, G1_BK, BN, CU_TENSOR_MAP_SWIZZLE_64B))
        return false;
    const size_t smem = STAGES * STAGE_BYTES + 1024 + 256;
    static const bool classic = std::getenv("OCTEN_G1_CLASSIC") != nullptr;  // diagnostics: one CTA per tile
    if (!classic) {
        static PerDevice pattr;
        pattr.once([&] {
            OCTEN_CUDA(cudaFuncSetAttribute(tc_gemm_tf32x3_persistent_kernel,
                                            cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(smem + G1P_EPI_BYTES)));
        });
        int nsm = 0, dev = 0;
        OCTEN_CUDA(cudaGetDevice(&dev));
        OCTEN_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
        const int mt = (M + BM - 1) / BM;
        const long long ntiles = (long long)mt * ((N + BN - 1) / BN);
        if (max_ctas > 0) nsm = std::min(nsm, max_ctas);
        const int grid = (int)std::min<long long>(ntiles, nsm);
        // two MMAs per k-step (A_hi X_rn + A_lo X_rn, X rounded to the
        // nearest TF32) unless OCTEN_G1_3MMA asks for the A_hi X_hi +
        // A_hi X_lo + A_lo X_hi split
        static const int two_mma = std::getenv("OCTEN_G1_3MMA") ? 0 : 1;
        tc_gemm_tf32x3_persistent_kernel<<<grid, G1P_THREADS, smem + G1P_EPI_BYTES, st>>>(
            mhi, mlo, mx, Z, M, N, K, N, scatter_p, scatter_q, scatter_sh, mt, ntiles, two_mma, nonfinite);
        OCTEN_LAUNCHED(1);
        OCTEN_CUDA(cudaGetLastError());
        return true;
    }
    static PerDevice attr;
    attr.once([&] {
        OCTEN_CUDA(cudaFuncSetAttribute(tc_gemm_tf32x3_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    });
    if ((N + BN - 1) / BN > 65535 || nonfinite) return false;  // (diagnostics path: no fused scan)
    dim3 grid((unsigned)((M + BM - 1) / BM), (unsigned)((N + BN - 1) / BN));
    tc_gemm_tf32x3_kernel<<<grid, NUM_THREADS, smem, st>>>(mhi, mlo, mx, Z, M, N, K, N, scatter_p, scatter_q,
                                                           scatter_sh);
    OCTEN_LAUNCHED(1);
    OCTEN_CUDA(cudaGetLastError());
    return true;
}

bool tc_mode2_tf32x3(const float* Z1, long long N1, int J, int tc, const float* Vhi, const float* Vlo, int ldv, int P,
                     int Q, float* Z2, long long zstride, cudaStream_t st) {
    if (!tc_gemm_available()) return false;
    // the A box of slice k starts at column k J: TMA needs that inner
    // coordinate on a 16-byte boundary, hence J % 4 == 0
    if (Q > M2_BN_MAX || Q < 1 || (J % 4) != 0 || (N1 % 4) != 0 || (ldv % 4) != 0 || ((uintptr_t)Z1 % 16) != 0 ||
        ((uintptr_t)Vhi % 16) != 0 || ((uintptr_t)Vlo % 16) != 0 || (long long)P * tc > 2147483647LL)
        return false;
    const int bn2 = Q <= 112 ? 112 : 128;
    CUtensorMap mz, mh, ml;
    if (!make_map(&mz, Z1, (uint64_t)N1, (uint64_t)P * Q, (uint64_t)N1 * 4, BK, BM)) return false;
    // inner extent ldv (zero-padded past J, a whole number of 16-byte units)
    if (!make_map(&mh, Vhi, (uint64_t)ldv, (uint64_t)P * Q, (uint64_t)ldv * 4, BK, bn2)) return false;
    if (!make_map(&ml, Vlo, (uint64_t)ldv, (uint64_t)P * Q, (uint64_t)ldv * 4, BK, bn2)) return false;
    auto launch = [&](auto kern, size_t stage_bytes, PerDevice& attr) {
        const size_t smem = M2_STAGES * stage_bytes + 1024 + 256;
        attr.once([&] {
            OCTEN_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        });
        kern<<<P * tc, NUM_THREADS, smem, st>>>(mz, mh, ml, Z2, Q, J, tc, zstride);
    };
    static PerDevice attr112, attr128;
    if (bn2 == 112)
        launch(tc_mode2_tf32x3_kernel<112>, (size_t)m2_stage_bytes<112>(), attr112);
    else
        launch(tc_mode2_tf32x3_kernel<128>, (size_t)m2_stage_bytes<128>(), attr128);
    OCTEN_LAUNCHED(1);
    OCTEN_CUDA(cudaGetLastError());
    return true;
}

}  // namespace octen
