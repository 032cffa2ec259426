// Throughput of warp-level mma.sync (TF32 m16n8k8, BF16 m16n8k16) and of
// 3-register FFMA on this part, to choose the arithmetic of the sparse
// slice kernel's rank-update phase.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 mma_rate.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void mma_tf32(float* out, int iters) {
    unsigned a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, b0 = a0 * 3, b1 = a0 * 5;
    float c[8][4] = {};
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 8; ++u)
            asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                         : "+f"(c[u][0]), "+f"(c[u][1]), "+f"(c[u][2]), "+f"(c[u][3])
                         : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }
    float s = 0;
    for (int u = 0; u < 8; ++u) s += c[u][0] + c[u][1] + c[u][2] + c[u][3];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void mma_bf16(float* out, int iters) {
    unsigned a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, b0 = a0 * 3, b1 = a0 * 5;
    float c[8][4] = {};
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 8; ++u)
            asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                         : "+f"(c[u][0]), "+f"(c[u][1]), "+f"(c[u][2]), "+f"(c[u][3])
                         : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }
    float s = 0;
    for (int u = 0; u < 8; ++u) s += c[u][0] + c[u][1] + c[u][2] + c[u][3];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void ffma(float* out, int iters, float x, float y) {
    float c[16];
    for (int u = 0; u < 16; ++u) c[u] = threadIdx.x + u;
    float a = x + threadIdx.x, b = y;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 16; ++u) c[u] = fmaf(a, c[u], b);
#pragma unroll
        for (int u = 0; u < 16; ++u) c[u] = fmaf(b, c[u], a);
    }
    float s = 0;
    for (int u = 0; u < 16; ++u) s += c[u];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
    float* out;
    cudaMalloc(&out, 148 * 8 * 1024 * sizeof(float));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    int sms = 148;
    for (int blocksPerSm : {2, 4}) {
        const int iters = 20000;
        dim3 grid(sms * blocksPerSm), block(256);
        float ms;
        mma_tf32<<<grid, block>>>(out, 10);
        cudaEventRecord(e0);
        mma_tf32<<<grid, block>>>(out, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        double fl = 2.0 * 16 * 8 * 8 * 8.0 * iters * (grid.x * 8.0);
        printf("blocks/SM %d  mma.sync tf32 m16n8k8: %.1f TFLOP/s\n", blocksPerSm, fl / ms / 1e9);
        mma_bf16<<<grid, block>>>(out, 10);
        cudaEventRecord(e0);
        mma_bf16<<<grid, block>>>(out, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        fl = 2.0 * 16 * 8 * 16 * 8.0 * iters * (grid.x * 8.0);
        printf("blocks/SM %d  mma.sync bf16 m16n8k16: %.1f TFLOP/s\n", blocksPerSm, fl / ms / 1e9);
        ffma<<<grid, block>>>(out, 10, 1.0001f, 0.999f);
        cudaEventRecord(e0);
        ffma<<<grid, block>>>(out, iters, 1.0001f, 0.999f);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        fl = 2.0 * 32 * iters * (double)grid.x * 256;
        printf("blocks/SM %d  FFMA: %.1f TFLOP/s\n", blocksPerSm, fl / ms / 1e9);
    }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
