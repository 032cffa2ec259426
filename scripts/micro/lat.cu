// Latency microbenchmarks (one warp): dependent DFMA / DMUL / FFMA chains,
// shared-memory load->use, rsqrt(double), __syncwarp, __syncthreads.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, long long* t, double seed) {
    __shared__ double sm[1024];
    __shared__ int idx[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) { sm[i] = 1.0 + i * 1e-9; idx[i] = (i + 1) & 1023; }
    __syncthreads();
    double x = seed + threadIdx.x, y = 1.000001;
    long long t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < 1024; ++i) x = fma(x, y, 1e-9);
    long long t1 = clock64();
#pragma unroll 1
    for (int i = 0; i < 1024; ++i) x = x * y;
    long long t2 = clock64();
    float xf = (float)x;
#pragma unroll 1
    for (int i = 0; i < 1024; ++i) xf = fmaf(xf, 1.0001f, 1e-6f);
    long long t3 = clock64();
    int j = threadIdx.x & 1;
#pragma unroll 1
    for (int i = 0; i < 1024; ++i) j = idx[j];
    long long t4 = clock64();
    double r = x;
#pragma unroll 1
    for (int i = 0; i < 256; ++i) r = rsqrt(r + 1.0);
    long long t5 = clock64();
#pragma unroll 1
    for (int i = 0; i < 1024; ++i) { __syncwarp(); sm[threadIdx.x & 31] += 1.0; }
    long long t6 = clock64();
#pragma unroll 1
    for (int i = 0; i < 1024; ++i) { __syncthreads(); }
    long long t7 = clock64();
    double z = x;
#pragma unroll 1
    for (int i = 0; i < 1024; ++i) { sm[threadIdx.x] = z; __syncwarp(); z = sm[(threadIdx.x + 1) & 31] * 1.0000001; }
    long long t8 = clock64();
    out[threadIdx.x] = x + xf + j + r + z;
    if (threadIdx.x == 0) {
        t[0] = t1 - t0; t[1] = t2 - t1; t[2] = t3 - t2; t[3] = t4 - t3; t[4] = t5 - t4; t[5] = t6 - t5; t[6] = t7 - t6; t[7] = t8 - t7;
    }
}
int main() {
    double* o; long long* t; cudaMalloc(&o, 4096 * 8); cudaMallocManaged(&t, 64 * 8);
    for (int bs : {32, 128, 256}) {
        k<<<1, bs>>>(o, t, 1.0); cudaDeviceSynchronize();
        k<<<1, bs>>>(o, t, 1.0); cudaDeviceSynchronize();
        printf("block %3d: DFMA %.1f  DMUL %.1f  FFMA %.1f  LDS->use %.1f  rsqrt(f64) %.1f  syncwarp+STS %.1f  syncthreads %.1f  STS-syncwarp-LDS-DMUL %.1f  (cycles per op)\n",
               bs, t[0] / 1024.0, t[1] / 1024.0, t[2] / 1024.0, t[3] / 1024.0, t[4] / 256.0, t[5] / 1024.0, t[6] / 1024.0, t[7] / 1024.0);
    }
    return 0;
}
