// fp64 CP-ALS partial contractions on the int8 tensor cores (tcgen05
// kind::i8) by exact digit splitting; see ozaki.hpp for the arithmetic.
//
// Reference: the MTTKRP of cp_als.cpp:296-303 (Y_(n) times the Khatri-Rao
// product of the other factors, Eigen fp64 GEMM); als.cu forms it as
// T = Y x_n F (one GEMM shared by two mode updates) and contracts T with the
// remaining factor.  This kernel is that T GEMM:
//     T[p][m + Q^2 n] = sum_k A_o(p; m, k) F(p; k, n)
// M = Q^2 rows (tile 128), N = S R columns (tile 64), K = Q <= 128 (one
// 128-byte row of digits, TMA zero-fills k >= Q).
//
// Per CTA (one 128 x 64 output tile, 256 threads, one CTA per SM):
//   thread 0     TMA: the 7 digit slices of the A tile (128 rows x 128 B
//                each, 128 B swizzle), pre-sliced once per CP-ALS run
//   all threads  the 7 digit slices of the factor columns, written straight
//                into shared memory in the same swizzled K-major layout
//   thread 32    TMEM (512 columns: 8 diagonals x 64) and the MMAs: for
//                every A slice i, B slices j <= min(7, 9 - i) in runs of up to 4
//                (N = 64 per slice), accumulating into diagonal d = i + j
//   all warps    epilogue: 8 int32 diagonals per output -> fp64 -> T
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <string>

#include "errors.hpp"
#include "gemm_dmma.cuh"
#include "octen_common.cuh"
#include "ozaki.hpp"
#include "ozaki_digits.cuh"
#include "tc_gemm.hpp"

namespace octen {

namespace {

constexpr int NS = kOzSlices;       // digit slices per operand
using oz::kBadExp;
using oz::oz_exponent;
using oz::pow2i;
using oz::oz_scales;
using oz::oz_digits;
constexpr int DMAX = NS + 2;        // pairs kept: i + j <= DMAX
constexpr int ND = DMAX - 1;        // diagonals d = 2 .. DMAX
constexpr int BM = 128;             // rows per tile
constexpr int NG = 64;              // columns per CTA (two halves)
constexpr int NH = 32;              // columns per half (one TMEM buffer)
constexpr int KB = 128;             // bytes of K per row (K <= 128)
constexpr int KH = 64;              // bytes of K per A stage (64 B swizzle)
constexpr int A_SLICE = BM * KH;    // 8 KB: one digit slice of a K-half A tile
constexpr int A_STAGE = NS * A_SLICE;  // 56 KB
#ifndef OCTEN_OZ_NSLOT
#define OCTEN_OZ_NSLOT 2
#endif
constexpr int NSLOT = OCTEN_OZ_NSLOT;  // A stages in flight (ring; 2 measured 11.66 vs 3: 11.77 ms per c3 step)
constexpr int BH_SLICE = NH * KB;   // 4 KB
#ifndef OCTEN_OZ_EPI_WARPS
#define OCTEN_OZ_EPI_WARPS 8
#endif
constexpr int EPI_WARPS = OCTEN_OZ_EPI_WARPS;  // 8: one per (TMEM lane quarter, half); 16: two, 16 columns each
constexpr int EPI_COLS = NH * 8 / EPI_WARPS;  // columns of a half per epilogue warp
constexpr int PW = EPI_WARPS;       // the MMA warp
constexpr int LW = EPI_WARPS + 1;   // the TMA warp
constexpr int THREADS = (EPI_WARPS + 2) * 32;
constexpr uint32_t TMEM_COLS = 512; // 2 halves x ND diagonals x NH
constexpr size_t SMEM_BYTES = (size_t)NSLOT * A_STAGE + 2 * NS * BH_SLICE + 128 + 1024;

static_assert(2 * ND * NH <= (int)TMEM_COLS, "diagonals must fit TMEM");

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
// bounded wait: a protocol bug traps instead of hanging the GPU
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    const uint32_t addr = smem_u32(bar);
    for (uint32_t it = 0;; ++it) {
        uint32_t ok;
        asm volatile(
            "{\n"
            ".reg .pred P1;\n"
            "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2, %3;\n"
            "selp.u32 %0, 1, 0, P1;\n"
            "}\n"
            : "=r"(ok)
            : "r"(addr), "r"(phase), "r"(0x989680u)
            : "memory");
        if (ok) return;
        if (it > (1u << 20)) asm volatile("trap;");
    }
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                            int c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], "
        "[%2];" ::"r"(smem_u32(dst)),
        "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
        : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// UMMA shared-memory descriptor: K-major, 128 B swizzle, 8-row groups 1024 B apart.
__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)1 << 16;
    d |= (uint64_t)(1024 >> 4) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)2 << 61;
    return d;
}
// UMMA shared-memory descriptor: K-major, 64 B swizzle, 8-row groups 512 B apart.
__device__ __forceinline__ uint64_t desc_sw64(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)1 << 16;
    d |= (uint64_t)(512 >> 4) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)4 << 61;
    return d;
}
// Instruction descriptor, kind::i8: S32 accumulate, A/B signed or unsigned
// bytes, both K-major, M = 128.
__device__ __forceinline__ uint32_t idesc_i8(bool a_signed, bool b_signed, int n) {
    return (2u << 4) | ((a_signed ? 1u : 0u) << 7) | ((b_signed ? 1u : 0u) << 10) | ((uint32_t)(n >> 3) << 17) |
           ((uint32_t)(BM >> 4) << 24);
}
__device__ __forceinline__ void mma_i8(uint32_t dtmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n"
        "}\n" ::"r"(dtmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}

// Four values' digit words -> one 32-bit word per slice (byte t of word i-1
// = d_i of value t), by byte permutes.
__device__ __forceinline__ void oz_pack4(const unsigned long long (&g)[4], uint32_t (&w)[NS]) {
    const uint32_t l0 = (uint32_t)g[0], l1 = (uint32_t)g[1], l2 = (uint32_t)g[2], l3 = (uint32_t)g[3];
    const uint32_t h0 = (uint32_t)(g[0] >> 32), h1 = (uint32_t)(g[1] >> 32), h2 = (uint32_t)(g[2] >> 32),
                   h3 = (uint32_t)(g[3] >> 32);
    // bytes 0..3 (slices 7..4), bytes 4..6 (slices 3..1)
    const uint32_t a01 = __byte_perm(l0, l1, 0x5140), b01 = __byte_perm(l0, l1, 0x7362);
    const uint32_t a23 = __byte_perm(l2, l3, 0x5140), b23 = __byte_perm(l2, l3, 0x7362);
    const uint32_t c01 = __byte_perm(h0, h1, 0x5140), e01 = __byte_perm(h0, h1, 0x7362);
    const uint32_t c23 = __byte_perm(h2, h3, 0x5140), e23 = __byte_perm(h2, h3, 0x7362);
    w[6] = __byte_perm(a01, a23, 0x5410);  // byte 0: slice 7
    w[5] = __byte_perm(a01, a23, 0x7632);  // byte 1: slice 6
    w[4] = __byte_perm(b01, b23, 0x5410);  // byte 2
    w[3] = __byte_perm(b01, b23, 0x7632);  // byte 3
    w[2] = __byte_perm(c01, c23, 0x5410);  // byte 4
    w[1] = __byte_perm(c01, c23, 0x7632);  // byte 5
    w[0] = __byte_perm(e01, e23, 0x5410);  // byte 6: slice 1 (top)
}

// 32 rows m of one (orientation, replica) per 128-thread CTA: the rows are
// staged in shared memory with coalesced loads (along k when the row is
// contiguous, orientation 0; along m otherwise), then four threads per row
// form its exponent (a shuffle max) and its digits, 16 bytes at a time.
constexpr int SL_ROWS = 32;
__global__ void __launch_bounds__(128) oz_slice_y_kernel(const double* __restrict__ Y, int P, int Q, int pitch,
                                                         uint8_t* __restrict__ As, int* __restrict__ Ea) {
    extern __shared__ double tile[];  // SL_ROWS x (Q + 1)
    const int o = blockIdx.z, p = blockIdx.y;
    const int q2 = Q * Q, ld = Q + 1;
    const int m0 = blockIdx.x * SL_ROWS;
    size_t s0, s1, sk;
    if (o == 2) {
        s0 = 1, s1 = (size_t)Q, sk = (size_t)q2;
    } else if (o == 1) {
        s0 = 1, s1 = (size_t)q2, sk = (size_t)Q;
    } else {
        s0 = (size_t)Q, s1 = (size_t)q2, sk = 1;
    }
    const double* Yp = Y + (size_t)p * q2 * Q;
    const int tid = threadIdx.x;
    if (sk == 1) {  // row-contiguous: a warp per row, lanes along k
        for (int r = tid >> 5; r < SL_ROWS; r += 4) {
            const int m = m0 + r;
            const double* row = Yp + (size_t)(m % Q) * s0 + (size_t)(m / Q) * s1;
            for (int k = tid & 31; k < Q; k += 32) tile[r * ld + k] = m < q2 ? __ldg(row + k) : 0.0;
        }
    } else {  // m-contiguous: lanes along m
        const int r = tid & 31;
        const int m = m0 + r;
        const double* row = Yp + (size_t)(m % Q) * s0 + (size_t)(m / Q) * s1;
        for (int k = tid >> 5; k < Q; k += 4) tile[r * ld + k] = m < q2 ? __ldg(row + k * sk) : 0.0;
    }
    __syncthreads();
    const int r = tid >> 2, part = tid & 3;  // four threads per row, 32 k each
    const int m = m0 + r;
    const double* trow = tile + r * ld;
    double mx = 0.0;
    int bad = 0;
    for (int k = part * 32; k < min(Q, part * 32 + 32); ++k) {
        const double v = trow[k];
        bad |= !isfinite(v);
        mx = fmax(mx, fabs(v));
    }
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
    bad |= __shfl_xor_sync(0xffffffffu, bad, 1);
    bad |= __shfl_xor_sync(0xffffffffu, bad, 2);
    const int e = oz_exponent(mx, bad != 0);
    if (m >= q2) return;
    const size_t plane = (size_t)o * P + p;
    if (part == 0) Ea[plane * q2 + m] = e;
    double c1 = 0.0, c2 = 0.0;
    if (e != kBadExp) oz_scales(e, c1, c2);
    const size_t splane = (size_t)q2 * pitch;
    uint8_t* out = As + plane * NS * splane + (size_t)m * pitch;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int k0 = part * 32 + h * 16;
        if (k0 >= pitch) break;
        uint32_t w[4][NS];
#pragma unroll
        for (int qd = 0; qd < 4; ++qd) {
            unsigned long long g[4];
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                const int k = k0 + 4 * qd + t;
                g[t] = (k < Q && e != kBadExp) ? oz_digits(trow[k], c1, c2) : 0ull;
            }
            oz_pack4(g, w[qd]);
        }
#pragma unroll
        for (int i = 0; i < NS; ++i)
            *reinterpret_cast<uint4*>(out + i * splane + k0) = make_uint4(w[0][i], w[1][i], w[2][i], w[3][i]);
    }
}

// Persistent over the m-tiles of one (replica, 64-column group): CTA c of
// the group takes tiles c, c + cpg, ...  The group's 64 columns are two
// halves of 32, each with its own TMEM buffer (8 diagonals x 32 columns), so
// the epilogue of one half overlaps the MMAs of the other.  The A tiles come
// as K-halves (64 B swizzle) through a ring of NSLOT stages, so the next
// tile's loads overlap this tile's MMAs and epilogue.
//   warps 0..7   epilogue (TMEM lane quarter w & 3, half w >> 2)
//   warp 8       MMA issue (one thread)
//   warp 9       TMA producer (one thread)
__global__ void __launch_bounds__(THREADS, 1)
    oz_tgemm_kernel(const __grid_constant__ CUtensorMap amap, const __grid_constant__ CUtensorMap bmap,
                    const int* __restrict__ Ea, const double* __restrict__ Fcs, double* __restrict__ T, int Q, int S,
                    int R, int mode, int G) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    uint8_t* sA = smem;                      // NSLOT stages x NS slices x 128 rows x 64 B
    uint8_t* sB = smem + NSLOT * A_STAGE;
    __shared__ double sCs[NG];  // 2^eb per column (NaN: non-finite column)
    uint64_t* bars = (uint64_t*)(sB + 2 * NS * BH_SLICE);
    uint64_t* done_bar = bars;                // [2] MMAs of half h complete
    uint64_t* empty_bar = bars + 2;           // [2] TMEM buffer h drained
    uint64_t* bfull_bar = bars + 4;           // the factor digits landed
    uint64_t* full_bar = bars + 5;            // [NSLOT] A stage landed
    uint64_t* sfree_bar = bars + 5 + NSLOT;   // [NSLOT] A stage consumed
    uint32_t* tmem_slot = (uint32_t*)(bars + 5 + 2 * NSLOT);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int p = blockIdx.z, cpg = gridDim.x;
    const int q2 = Q * Q, SR = S * R;
    const int mtiles = (q2 + BM - 1) / BM;
    const int n0 = blockIdx.y * NG;

    pdl_trigger();
    if (threadIdx.x == 0) {
        for (int i = 0; i < NSLOT; ++i) {
            mbar_init(&full_bar[i], 1);
            mbar_init(&sfree_bar[i], 1);
        }
        mbar_init(bfull_bar, 1);
        mbar_init(&done_bar[0], 1);
        mbar_init(&done_bar[1], 1);
        mbar_init(&empty_bar[0], EPI_WARPS / 2 * 32);
        mbar_init(&empty_bar[1], EPI_WARPS / 2 * 32);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == PW) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    // the digit slices of Y were written before this CP-ALS run began (a
    // normal launch, no programmatic trigger): safe to load ahead of pdl_wait
    const size_t bplane = oz::factor_plane(p, mode, blockIdx.y, G);
    pdl_wait();  // the factor digits are the previous mode update's output
    if (threadIdx.x == LW * 32 && (int)blockIdx.x < mtiles) {
        mbar_arrive_expect_tx(bfull_bar, 2 * NS * BH_SLICE);
        tma_load_3d(sB, &bmap, bfull_bar, 0, 0, (int)bplane);
        tma_load_3d(sB + NS * BH_SLICE, &bmap, bfull_bar, 0, NS * NH, (int)bplane);
    }
    if (threadIdx.x < NG) sCs[threadIdx.x] = __ldg(Fcs + bplane * NG + threadIdx.x);
    fence_proxy_async();
    __syncthreads();

    if (warp == LW) {
        // TMA producer: the K-halves of the CTA's A tiles through the ring
        // (the digit slices of Y were written before this CP-ALS run began,
        // by a normal launch, so they may be read ahead of pdl_wait too)
        if (lane == 0) {
            int stage = 0;
#pragma unroll 1
            for (int mt = blockIdx.x; mt < mtiles; mt += cpg) {
#pragma unroll 1
                for (int kh = 0; kh < 2; ++kh, ++stage) {
                    const int slot = stage % NSLOT;
                    if (stage >= NSLOT) mbar_wait(&sfree_bar[slot], ((stage / NSLOT) - 1) & 1);
                    uint8_t* dst = sA + slot * A_STAGE;
                    mbar_arrive_expect_tx(&full_bar[slot], A_STAGE);
#pragma unroll 1
                    for (int i = 0; i < NS; ++i)
                        tma_load_3d(dst + i * A_SLICE, &amap, &full_bar[slot], kh * KH, mt * BM, p * NS + i);
                }
            }
        }
        __syncwarp();
    } else if (warp == PW) {
        if (lane == 0) {
            const uint32_t a0 = smem_u32(sA);
            const uint64_t db = desc_sw128(smem_u32(sB));
            const int nks = (Q + 31) / 32;
            mbar_wait(bfull_bar, 0);
            int it = 0, stage = 0;
#pragma unroll 1
            for (int mt = blockIdx.x; mt < mtiles; mt += cpg, ++it) {
#pragma unroll 1
                for (int kh = 0; kh < 2; ++kh, ++stage) {
                    const int slot = stage % NSLOT;
                    mbar_wait(&full_bar[slot], (stage / NSLOT) & 1);
                    const uint64_t da = desc_sw64(a0 + slot * A_STAGE);
#pragma unroll 1
                    for (int h = 0; h < 2; ++h) {
                        if (kh == 0 && it > 0) mbar_wait(&empty_bar[h], (it - 1) & 1);
                        tc_fence_after();
                        const uint32_t dt = tmem_base + (uint32_t)(h * ND * NH);
#pragma unroll 1
                        for (int kl = 0; kl < 2; ++kl) {
                            const int ks = 2 * kh + kl;
                            if (ks >= nks) break;
                            // diagonals [0, inited) already hold this tile's
                            // partial sums (compile-time bookkeeping: the loop
                            // is unrolled); A slice i against B slices 1 .. jmax
                            // in one MMA
                            int inited = 0;
#pragma unroll
                            for (int i = 1; i <= NS; ++i) {
                                const int jmax = NS < DMAX - i ? NS : DMAX - i;
                                const uint64_t ad = da + (uint64_t)(((i - 1) * A_SLICE + kl * 32) >> 4);
                                const uint64_t bd = db + (uint64_t)(((h * NS) * BH_SLICE + ks * 32) >> 4);
                                const int b0d = i - 1;
                                const int k = b0d >= inited ? 0 : (inited - b0d < jmax ? inited - b0d : jmax);
                                if (k > 0) mma_i8(dt + (uint32_t)(b0d * NH), ad, bd, idesc_i8(true, true, k * NH), 1u);
                                if (jmax > k)
                                    mma_i8(dt + (uint32_t)((b0d + k) * NH), ad, bd + (uint64_t)((k * BH_SLICE) >> 4),
                                           idesc_i8(true, true, (jmax - k) * NH), ks > 0 ? 1u : 0u);
                                inited = inited > b0d + jmax ? inited : b0d + jmax;
                            }
                        }
                        if (kh == 1) {
                            mma_commit(&done_bar[h]);
                        }
                    }
                    mma_commit(&sfree_bar[slot]);
                }
            }
        }
        __syncwarp();
    } else {
        const int q = warp & 3, h = (warp >> 2) & 1, sub = warp >> 3;
        const int r = q * 32 + lane;
        const uint32_t trow = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(h * ND * NH);
        const int ncol = min(NH, SR - n0 - h * NH);  // valid columns of this half
        double* Tp = T + (size_t)p * q2 * SR + (size_t)q2 * (n0 + h * NH);
        const double* cs = sCs + h * NH;
        int it = 0;
        // the row exponent of the next tile is loaded one tile ahead
        int ea_next = (int)blockIdx.x * BM + r < q2 ? __ldg(Ea + (size_t)p * q2 + blockIdx.x * BM + r) : 0;
#pragma unroll 1
        for (int mt = blockIdx.x; mt < mtiles; mt += cpg, ++it) {
            const int m = mt * BM + r;
            const int ea = ea_next;
            if (mt + cpg < mtiles)
                ea_next = m + cpg * BM < q2 ? __ldg(Ea + (size_t)p * q2 + m + cpg * BM) : 0;
            // row weights: the two Horner groups weigh 2^(ea - 36), 2^(ea - 68)
            const bool fast = ea >= -1022 + 68 && ea <= 1023 + 36;  // (false for kBadExp)
            const double w0 = fast ? pow2i(ea - 36) : 0.0;
            const double w1 = fast ? pow2i(ea - 68) : 0.0;
            const bool all_fast = __all_sync(0xffffffffu, fast);
            const bool row_ok = m < q2;
            double* trow_out = Tp + m;
            mbar_wait(&done_bar[h], it & 1);
            tc_fence_after();
            // chunks of 8 columns; the TMEM loads of chunk c + 1 are in flight
            // while chunk c is converted and stored
#ifndef OCTEN_OZ_TMEM_DB
#define OCTEN_OZ_TMEM_DB 1
#endif
            constexpr int NBUF = OCTEN_OZ_TMEM_DB ? 2 : 1;  // TMEM load buffers (double: next chunk in flight)
            uint32_t a[NBUF][ND][8];
            auto tload = [&](int buf, int c0) {
#pragma unroll
                for (int d = 0; d < ND; ++d)
                    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                                 : "=r"(a[buf][d][0]), "=r"(a[buf][d][1]), "=r"(a[buf][d][2]), "=r"(a[buf][d][3]),
                                   "=r"(a[buf][d][4]), "=r"(a[buf][d][5]), "=r"(a[buf][d][6]), "=r"(a[buf][d][7])
                                 : "r"(trow + (uint32_t)(d * NH + c0)));
            };
            tload(0, sub * EPI_COLS);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
            for (int ch = 0; ch < EPI_COLS / 8; ++ch) {
                const int c0 = sub * EPI_COLS + ch * 8, buf = NBUF == 2 ? (ch & 1) : 0;
                if (NBUF == 2 && ch + 1 < EPI_COLS / 8) tload(buf ^ 1, c0 + 8);
                if (NBUF == 1 && ch > 0) {
                    tload(0, c0);
                    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                }
                double val[8];
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    // diagonal b weighs 2^(-12 - 8 b): two exact int64 Horner
                    // groups (|H| < 2^49), converted to fp64 exactly via 2^52 + 2^51
                    const long long h0 = (long long)(int)a[buf][0][j] * 16777216LL +
                                         (long long)(int)a[buf][1][j] * 65536LL + (long long)(int)a[buf][2][j] * 256LL +
                                         (long long)(int)a[buf][3][j];
                    const long long h1 = (long long)(int)a[buf][4][j] * 16777216LL +
                                         (long long)(int)a[buf][5][j] * 65536LL + (long long)(int)a[buf][6][j] * 256LL +
                                         (long long)(int)a[buf][7][j];
                    const double d0 = __longlong_as_double(h0 + 0x4338000000000000LL) - 6755399441055744.0;
                    const double d1 = __longlong_as_double(h1 + 0x4338000000000000LL) - 6755399441055744.0;
                    val[j] = fma(d0, w0, d1 * w1) * cs[c0 + j];
                }
                if (!all_fast && !fast) {  // rows at the ends of the exponent range, non-finite rows
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        const long long h0 = (long long)(int)a[buf][0][j] * 16777216LL +
                                             (long long)(int)a[buf][1][j] * 65536LL +
                                             (long long)(int)a[buf][2][j] * 256LL + (long long)(int)a[buf][3][j];
                        const long long h1 = (long long)(int)a[buf][4][j] * 16777216LL +
                                             (long long)(int)a[buf][5][j] * 65536LL +
                                             (long long)(int)a[buf][6][j] * 256LL + (long long)(int)a[buf][7][j];
                        val[j] = ea == kBadExp ? __longlong_as_double(0x7ff8000000000000LL)
                                               : ldexp((double)h0 * 0x1p-36 + (double)h1 * 0x1p-68, ea) * cs[c0 + j];
                    }
                }
                if (row_ok) {
                    double* o = trow_out + (size_t)q2 * c0;
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        if (c0 + j < ncol) *o = val[j];
                        o += q2;
                    }
                }
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            }
            tc_fence_before();
            mbar_arrive(&empty_bar[h]);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == PW) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TMEM_COLS));
    }
}

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

}  // namespace

bool ozaki_supported(int Q) { return Q >= 1 && Q <= KB && tc_gemm_available(); }

bool ozaki_selected(int Q) {
    // The sweeps' T-GEMM engine: this kernel unless OCTEN_ALS_TGEMM=dmma
    // (measured at c3, pipelined step: 12.47 ms against 12.95 ms on DMMA)
    const char* e = std::getenv("OCTEN_ALS_TGEMM");  // (read per CP-ALS run)
    return !(e && std::string(e) == "dmma") && ozaki_supported(Q);
}

int ozaki_pitch(int Q) { return (Q + 15) / 16 * 16; }

void ozaki_slice_y(const double* Y, int P, int Q, uint8_t* As, int* Ea, cudaStream_t st) {
    const int q2 = Q * Q;
    dim3 grid((unsigned)((q2 + SL_ROWS - 1) / SL_ROWS), (unsigned)P, 3);
    const size_t smem = (size_t)SL_ROWS * (Q + 1) * sizeof(double);
    if (smem > 48 * 1024) {
        static PerDevice attr;
        attr.once([] {
            OCTEN_CUDA(cudaFuncSetAttribute(oz_slice_y_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            (int)(SL_ROWS * 129 * sizeof(double))));
        });
    }
    oz_slice_y_kernel<<<grid, 128, smem, st>>>(Y, P, Q, ozaki_pitch(Q), As, Ea);
    OCTEN_LAUNCHED(1);
    OCTEN_CUDA(cudaGetLastError());
}

bool ozaki_make_map(CUtensorMap* map, const uint8_t* As, int P, int Q, int o, int p0, int pn) {
    EncodeTiledFn enc = (EncodeTiledFn)tc_tensor_map_encoder();
    if (!enc) return false;
    const uint64_t q2 = (uint64_t)Q * Q, pitch = (uint64_t)ozaki_pitch(Q);
    const uint8_t* base = As + ((uint64_t)o * P + p0) * NS * q2 * pitch;
    cuuint64_t dims[3] = {(cuuint64_t)Q, (cuuint64_t)q2, (cuuint64_t)pn * NS};
    cuuint64_t strides[2] = {(cuuint64_t)pitch, (cuuint64_t)(q2 * pitch)};
    cuuint32_t box[3] = {KH, BM, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    return enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<uint8_t*>(base), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool ozaki_make_fmap(CUtensorMap* map, const uint8_t* Fd, int Q, int G, int p0, int pn) {
    EncodeTiledFn enc = (EncodeTiledFn)tc_tensor_map_encoder();
    if (!enc) return false;
    const uint64_t rows = 2 * NS * NH;
    const uint8_t* base = Fd + oz::factor_plane(p0, 0, 0, G) * rows * KB;
    cuuint64_t dims[3] = {(cuuint64_t)Q, (cuuint64_t)rows, (cuuint64_t)pn * 3 * G};
    cuuint64_t strides[2] = {(cuuint64_t)KB, (cuuint64_t)(rows * KB)};
    cuuint32_t box[3] = {KB, NS * NH, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    return enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<uint8_t*>(base), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

int ozaki_groups(int S, int R) { return (S * R + NG - 1) / NG; }
size_t ozaki_fd_bytes(int P, int S, int R) { return (size_t)P * 3 * ozaki_groups(S, R) * 2 * NS * NH * KB; }
size_t ozaki_fcs_count(int P, int S, int R) { return (size_t)P * 3 * ozaki_groups(S, R) * NG; }

namespace {
// One warp per factor column of every (problem, mode): the digits the
// T-GEMM reads for the factors as they stand (after initialisation).
__global__ void __launch_bounds__(256) oz_slice_factors_kernel(const double* __restrict__ F, int S, int Q, int R,
                                                               int NPS, uint8_t* __restrict__ Fd,
                                                               double* __restrict__ Fcs, int G) {
    const int warp = (int)(blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)), lane = threadIdx.x & 31;
    if (warp >= NPS * 3 * R) return;
    const int r = warp % R, mode = (warp / R) % 3, prob = warp / (3 * R);
    oz::factor_column_digits(Fd, Fcs, G, S, R, Q, prob, mode, r, F + ((size_t)prob * 3 + mode) * Q * R + (size_t)Q * r,
                             lane);
}
}  // namespace

void ozaki_slice_factors(const double* F, int P, int S, int Q, int R, uint8_t* Fd, double* Fcs, cudaStream_t st) {
    const int warps = P * S * 3 * R;
    oz_slice_factors_kernel<<<(warps + 7) / 8, 256, 0, st>>>(F, S, Q, R, P * S, Fd, Fcs, ozaki_groups(S, R));
    OCTEN_LAUNCHED(1);
    OCTEN_CUDA(cudaGetLastError());
}

void ozaki_tgemm(const CUtensorMap& amap, const CUtensorMap& bmap, const int* Ea_lane, const double* Fcs_lane,
                 double* T, int pn, int Q, int S, int R, int mode, cudaStream_t st, bool pdl) {
    static PerDevice attr;
    attr.once([] {
        OCTEN_CUDA(cudaFuncSetAttribute(oz_tgemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM_BYTES));
    });
    const int q2 = Q * Q, SR = S * R, G = ozaki_groups(S, R);
    // m-tiles per CTA
    static const int per_cta = [] {
        const char* e = std::getenv("OCTEN_OZ_TILES");
        return e ? std::max(1, std::atoi(e)) : 4;  // measured 2/3/4/5: 12.8/12.57/12.47/12.47 ms per c3 step
    }();
    const int mtiles = (q2 + BM - 1) / BM;
    dim3 grid((unsigned)((mtiles + per_cta - 1) / per_cta), (unsigned)G, (unsigned)pn);
    if (pdl) {
        launch_pdl(oz_tgemm_kernel, grid, dim3(THREADS), SMEM_BYTES, st, amap, bmap, Ea_lane, Fcs_lane, T, Q, S, R,
                   mode, G);
    } else {
        oz_tgemm_kernel<<<grid, THREADS, SMEM_BYTES, st>>>(amap, bmap, Ea_lane, Fcs_lane, T, Q, S, R, mode, G);
        OCTEN_LAUNCHED(1);
    }
    path_counter(kTcgen05Als).fetch_add(1, std::memory_order_relaxed);
    OCTEN_CUDA(cudaGetLastError());
}

}  // namespace octen
