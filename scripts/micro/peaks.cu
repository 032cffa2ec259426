// Measured arithmetic peaks of this part for the per-stage rooflines
// (bench.py reads profiles/peaks_b200.json, written by this program):
//   * tcgen05.mma kind::tf32, M=128 N=256 K=8, one issuing thread per SM,
//     operands in shared memory, fp32 accumulators in TMEM
//     (the dense compression's GEMM1 / mode-2 pipe);
//   * DMMA (mma.sync m8n8k4 f64, the only fp64 MMA on sm_100a: CP-ALS, merge);
//   * FP32 FFMA (the sparse slice kernel) and FP64 DFMA.
// Each is a register/shared-only loop over all 148 SMs timed with CUDA events
// (best of 5 after a warm-up launch).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o peaks peaks.cu && ./peaks out.json
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t desc_sw64(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)1 << 16;
    d |= (uint64_t)(512 >> 4) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)4 << 61;
    return d;
}

constexpr int TM = 128, TN = 256;
constexpr uint32_t kIdesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(TN >> 3) << 17) | ((uint32_t)(TM >> 4) << 24);

__global__ void __launch_bounds__(128, 1) tc_tf32_rate(int iters, float* out) {
    __shared__ __align__(1024) float As[TM * 16];
    __shared__ __align__(1024) float Bs[TN * 16];
    __shared__ __align__(8) uint64_t bar;
    __shared__ uint32_t tslot;
    for (int i = threadIdx.x; i < TM * 16; i += blockDim.x) As[i] = 0.f;
    for (int i = threadIdx.x; i < TN * 16; i += blockDim.x) Bs[i] = 0.f;
    if (threadIdx.x == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tslot)),
                     "r"(256));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = tslot;
    if (threadIdx.x == 0) {
        const uint64_t a0 = desc_sw64(smem_u32(As)), b0 = desc_sw64(smem_u32(Bs));
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                asm volatile(
                    "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                    "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
                    "l"(a0 + 2 * k), "l"(b0 + 2 * k), "r"(kIdesc), "r"(it | k));
            }
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                         smem_u32(&bar))
                     : "memory");
        uint32_t ok = 0;
        while (!ok)
            asm volatile(
                "{\n.reg .pred P1;\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], 0;\nselp.u32 %0, 1, 0, P1;\n}\n"
                : "=r"(ok)
                : "r"(smem_u32(&bar))
                : "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (threadIdx.x < 32) {
        uint32_t v;
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(v) : "r"(tmem));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        out[blockIdx.x * 32 + threadIdx.x] = __uint_as_float(v);
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256));
    }
}

__global__ void dmma_rate(int iters, double* out) {
    double a = threadIdx.x * 1e-3, b = 1.0 + blockIdx.x * 1e-6;
    double c[8][2];
#pragma unroll
    for (int u = 0; u < 8; ++u) c[u][0] = c[u][1] = 0.0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 8; ++u)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
                         : "+d"(c[u][0]), "+d"(c[u][1])
                         : "d"(a), "d"(b));
    }
    double s = 0;
#pragma unroll
    for (int u = 0; u < 8; ++u) s += c[u][0] + c[u][1];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void ffma_rate(int iters, float x, float y, float* out) {
    float c[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) c[u] = threadIdx.x + u;
    const float a = x + threadIdx.x, b = y;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 16; ++u) c[u] = fmaf(a, c[u], b);
#pragma unroll
        for (int u = 0; u < 16; ++u) c[u] = fmaf(b, c[u], a);
    }
    float s = 0;
#pragma unroll
    for (int u = 0; u < 16; ++u) s += c[u];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void dfma_rate(int iters, double x, double y, double* out) {
    double c[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) c[u] = threadIdx.x + u;
    const double a = x + threadIdx.x, b = y;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 8; ++u) c[u] = fma(a, c[u], b);
#pragma unroll
        for (int u = 0; u < 8; ++u) c[u] = fma(b, c[u], a);
    }
    double s = 0;
#pragma unroll
    for (int u = 0; u < 8; ++u) s += c[u];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <class F>
static float best_ms(F launch) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    launch();
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0);
        launch();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return best;
}

int main(int argc, char** argv) {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int clk_khz = 0;
    cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
    void* buf;
    cudaMalloc(&buf, (size_t)sms * 16 * 1024 * sizeof(double));
    // tcgen05 tf32: 2 MMAs of 2*128*256*8 flop per iteration per SM
    const int tc_iters = 200000;
    const float tc_ms = best_ms([&] { tc_tf32_rate<<<sms, 128>>>(tc_iters, (float*)buf); });
    const double tc_tf = 2.0 * 2 * TM * TN * 8 * (double)tc_iters * sms / (tc_ms * 1e-3) / 1e12;
    double dmma_tf = 0, ffma_tf = 0, dfma_tf = 0;
    for (int bps : {2, 4, 8}) {
        const int it = 20000;
        const dim3 g(sms * bps), b(256);
        float ms = best_ms([&] { dmma_rate<<<g, b>>>(it, (double*)buf); });
        const double t1 = 2.0 * 8 * 8 * 4 * 8.0 * it * (g.x * 8.0) / (ms * 1e-3) / 1e12;
        ms = best_ms([&] { ffma_rate<<<g, b>>>(it, 1.0001f, 0.999f, (float*)buf); });
        const double t2 = 2.0 * 32 * it * (double)g.x * 256 / (ms * 1e-3) / 1e12;
        ms = best_ms([&] { dfma_rate<<<g, b>>>(it / 4, 1.0001, 0.999, (double*)buf); });
        const double t3 = 2.0 * 16 * (it / 4) * (double)g.x * 256 / (ms * 1e-3) / 1e12;
        if (t1 > dmma_tf) dmma_tf = t1;
        if (t2 > ffma_tf) ffma_tf = t2;
        if (t3 > dfma_tf) dfma_tf = t3;
    }
    const cudaError_t err = cudaGetLastError();
    char json[1024];
    std::snprintf(json, sizeof(json),
                  "{\"tcgen05_tf32_tflops\": %.2f, \"dmma_f64_tflops\": %.3f, \"ffma_f32_tflops\": %.2f, "
                  "\"dfma_f64_tflops\": %.3f, \"sms\": %d, \"sm_clock_mhz_attr\": %d, \"status\": \"%s\", "
                  "\"how\": \"scripts/micro/peaks.cu: register/shared-only loops on all SMs, CUDA events, best of 5; "
                  "tcgen05 kind::tf32 M128 N256 K8 from one thread per SM\"}\n",
                  tc_tf, dmma_tf, ffma_tf, dfma_tf, sms, clk_khz / 1000, cudaGetErrorString(err));
    std::fputs(json, stdout);
    if (argc > 1) {
        FILE* f = std::fopen(argv[1], "w");
        if (f) {
            std::fputs(json, f);
            std::fclose(f);
        }
    }
    return err == cudaSuccess ? 0 : 1;
}
