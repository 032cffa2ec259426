// Per-SM throughput of the epilogue's candidate instructions (dependent
// chains interleaved 8-wide, 16 warps per SM): cycles per warp-instruction.
#include <cstdio>
#include <cuda_runtime.h>
template <int OP>
__global__ void k(int iters, long long* out, int seed) {
    long long acc[8];
    double dacc[8];
    int ia[8];
    for (int j = 0; j < 8; ++j) { acc[j] = seed + j + threadIdx.x; dacc[j] = (double)(seed + j); ia[j] = seed * j + threadIdx.x; }
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            if (OP == 0) acc[j] = (long long)ia[j] * 16777216LL + acc[j];            // IMAD.WIDE
            if (OP == 1) dacc[j] = dacc[j] + (double)ia[j];                           // I2F.F64 + DADD
            if (OP == 2) dacc[j] = fma(dacc[j], 1.0000001, 0.5);                      // DFMA
            if (OP == 3) acc[j] = acc[j] + (long long)ia[j];                          // IADD 64
            if (OP == 4) dacc[j] = __longlong_as_double(acc[j] + 0x4338000000000000LL) - 6755399441055744.0 + dacc[j];  // magic
            if (OP == 5) ia[j] = ia[j] * 257 + j;                                     // IMAD 32
        }
    }
    const long long t1 = clock64();
    long long s = 0;
    for (int j = 0; j < 8; ++j) s += acc[j] + (long long)dacc[j] + ia[j];
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
    if (s == 42) out[blockIdx.x + 1000] = s;
}
int main() {
    long long* d; cudaMalloc(&d, 4096 * 8);
    long long h[1];
    const char* names[] = {"IMAD.WIDE (int32*c + int64)", "I2F.F64 + DADD", "DFMA", "IADD 64", "magic cvt + 2 DADD", "IMAD 32"};
    for (int op = 0; op < 6; ++op) {
        int iters = 2000;
        auto run = [&](auto kern) { kern<<<148, 512>>>(iters, d, 3); cudaDeviceSynchronize(); cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost); };
        if (op == 0) run(k<0>); if (op == 1) run(k<1>); if (op == 2) run(k<2>); if (op == 3) run(k<3>); if (op == 4) run(k<4>); if (op == 5) run(k<5>);
        // 16 warps per SM, 8 ops per iteration per warp
        printf("%-32s %.2f cycles per warp-op per SM (16 warps)\n", names[op], (double)h[0] / (iters * 8.0 * 16));
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
