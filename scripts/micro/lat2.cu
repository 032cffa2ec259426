// Dependent-chain latency per op (unrolled x64 in a loop of 16).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, long long* t, double seed) {
    double x = seed + threadIdx.x, y = 1.000001;
    float xf = (float)x;
    long long t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < 16; ++i) {
#pragma unroll
        for (int j = 0; j < 64; ++j) x = fma(x, y, 1e-9);
    }
    long long t1 = clock64();
#pragma unroll 1
    for (int i = 0; i < 16; ++i) {
#pragma unroll
        for (int j = 0; j < 64; ++j) xf = fmaf(xf, 1.0001f, 1e-6f);
    }
    long long t2 = clock64();
    double r = x;
#pragma unroll 1
    for (int i = 0; i < 16; ++i) {
#pragma unroll
        for (int j = 0; j < 16; ++j) { double q; asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(q) : "d"(r)); r = q + 1.0; }
    }
    long long t3 = clock64();
    out[threadIdx.x] = x + xf + r;
    if (threadIdx.x == 0) { t[0] = t1 - t0; t[1] = t2 - t1; t[2] = t3 - t2; }
}
int main() {
    double* o; long long* t; cudaMalloc(&o, 4096 * 8); cudaMallocManaged(&t, 64 * 8);
    for (int rep = 0; rep < 2; ++rep) {
        k<<<1, 32>>>(o, t, 1.0); cudaDeviceSynchronize();
        printf("DFMA %.1f  FFMA %.1f  (MUFU.RSQ64H + DADD) %.1f cycles\n", t[0] / 1024.0, t[1] / 1024.0, t[2] / 256.0);
    }
}
