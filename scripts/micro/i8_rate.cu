// tcgen05 issue-rate probe: kind::i8 / kind::f16 / kind::tf32 MMAs (M = 128,
// N = 64 .. 256, one 128-byte K row per operand, 128 B swizzle) from one
// thread per SM on all SMs; prints dense Tops/s per (kind, N).  Also the
// diagonal pattern of ozaki.cu (A slice i against B slices j, accumulating
// into column block i + j).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o i8_rate i8_rate.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc_sw128(uint32_t a) {
    return (uint64_t)((a >> 4) & 0x3FFF) | (1ull << 16) | ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61);
}
template <int KIND>  // 0 i8, 1 f16, 2 tf32
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    if (KIND == 0)
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc));
    else if (KIND == 1)
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc));
    else
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
template <int KIND>
__host__ __device__ constexpr uint32_t idesc(int n) {
    return KIND == 0 ? ((2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | (8u << 24))
         : KIND == 1 ? ((1u << 4) | (0u << 7) | (0u << 10) | ((uint32_t)(n >> 3) << 17) | (8u << 24))
                     : ((1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(n >> 3) << 17) | (8u << 24));
}

// mode 0: N-wide MMAs into one accumulator; mode 1: the ozaki diagonal pattern
template <int KIND>
__global__ void __launch_bounds__(128, 1) rate(int iters, int n, int mode, float* out) {
    extern __shared__ __align__(1024) uint8_t sm_raw[];
    uint8_t* sm = (uint8_t*)(((uintptr_t)sm_raw + 1023) & ~(uintptr_t)1023);
    uint8_t* As = sm;               // 7 x 16 KB
    uint8_t* Bs = sm + 7 * 16384;   // 7 x 8 KB
    __shared__ __align__(8) uint64_t bar;
    __shared__ uint32_t tslot;
    for (int i = threadIdx.x; i < (7 * 16384 + 7 * 8192) / 4; i += blockDim.x) ((uint32_t*)sm)[i] = 0;
    if (threadIdx.x == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tslot)), "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = tslot;
    if (threadIdx.x == 0) {
        const uint32_t a0 = smem_u32(As), b0 = smem_u32(Bs);
        for (int it = 0; it < iters; ++it) {
            if (mode == 0) {
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    mma<KIND>(tmem, desc_sw128(a0 + 32 * k), desc_sw128(b0 + 32 * k), idesc<KIND>(n), 1u);
            } else {
#pragma unroll
                for (int k = 0; k < 4; ++k) {
#pragma unroll
                    for (int i = 1; i <= 7; ++i) {
                        const int jmax = (9 - i) < 7 ? 9 - i : 7;
                        const uint64_t ad = desc_sw128(a0 + (i - 1) * 16384 + 32 * k);
                        // all-signed: one run of slices j = 1 .. jmax, N <= 256 per MMA
                        for (int j0 = 1; j0 <= jmax; j0 += 4) {
                            const int nb = (jmax - j0 + 1) < 4 ? jmax - j0 + 1 : 4;
                            mma<KIND>(tmem + (uint32_t)((i + j0 - 2) * 64), ad, desc_sw128(b0 + (j0 - 1) * 8192 + 32 * k),
                                      idesc<KIND>(nb * 64), 1u);
                        }
                    }
                }
            }
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)) : "memory");
        uint32_t ok = 0;
        while (!ok)
            asm volatile("{\n.reg .pred P1;\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], 0;\nselp.u32 %0, 1, 0, P1;\n}\n"
                         : "=r"(ok) : "r"(smem_u32(&bar)) : "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (threadIdx.x < 32) {
        uint32_t v;
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(v) : "r"(tmem));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        out[blockIdx.x * 32 + threadIdx.x] = (float)v;
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
    }
}

template <int KIND>
void run(const char* name, int sms, float* buf) {
    const size_t smem = 7 * 16384 + 7 * 8192 + 1024;
    cudaFuncSetAttribute(rate<KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int kbytes = 32;  // K bytes per MMA: i8 32 elems, f16 16, tf32 8
    const int kel = KIND == 0 ? 32 : KIND == 1 ? 16 : 8;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int mode = 0; mode < 2; ++mode)
        for (int n : {64, 128, 256}) {
            if (mode == 1 && n != 64) continue;
            const int iters = mode == 0 ? 20000 : 1000;
            float best = 1e30f;
            for (int r = 0; r < 3; ++r) {
                cudaEventRecord(e0);
                rate<KIND><<<sms, 128, smem>>>(iters, n, mode, buf);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                if (ms < best) best = ms;
            }
            // MACs per iteration: mode 0: 4 x 128 x n x kel; mode 1: 4 x 128 x (34 x 64) x kel
            const double macs = mode == 0 ? 4.0 * 128 * n * kel : 4.0 * 128 * (34 * 64) * kel;
            const double tops = 2.0 * macs * iters * sms / (best * 1e-3) / 1e12;
            std::printf("%s mode=%d N=%d: %.1f Tops/s (%.3f ms)\n", name, mode, n, tops, best);
            (void)kbytes;
        }
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float* buf;
    cudaMalloc(&buf, sms * 32 * sizeof(float));
    run<0>("i8  ", sms, buf);
    run<1>("f16 ", sms, buf);
    run<2>("tf32", sms, buf);
    std::printf("status %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
