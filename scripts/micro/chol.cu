// block_chol_inv_t in isolation: cycles for one 16x16 (warp) and 32x32 / 64x64 (block) factorization.
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_1807_01350_b200/csrc/small_linalg.cuh"
#include "chol_old.cuh"
using namespace octen;
template <int kPer, int kThreads, bool kWarp, int kOld = 0>
__global__ void k(int n, long long* t, double* out) {
    extern __shared__ double dsm[]; double* A = dsm; double* X = dsm + 64 * 65; double* scr = X + 64 * 65; double* L = A;
    for (int e = threadIdx.x; e < 64 * 65; e += blockDim.x) {
        const int i = e % 65, j = e / 65;
        A[e] = (i == j) ? 100.0 + i : 1.0 / (1.0 + i + j);
    }
    __syncthreads();
    long long t0 = clock64();
    int rk = 0;
    if (kOld == 2) rk = block_chol_inv_1b<kPer, kThreads, kWarp>(A, 65, n, 1e-12, L, 65, X, 65, scr);
    else if (kOld == 1) rk = block_chol_inv_old<kPer, kThreads>(A, 65, n, 1e-12, L, 65, X, 65, scr);
    else if (!kWarp || threadIdx.x < 32) rk = block_chol_inv_t<kPer, kThreads, kWarp>(A, 65, n, 1e-12, L, 65, X, 65, scr);
    long long t1 = clock64();
    __syncthreads();
    if (threadIdx.x == 0) { t[0] = t1 - t0; out[0] = L[n - 1 + 65 * (n - 1)] + X[3] + rk; }
}
template <int a, int b, bool c, int d = 0>
void setup() { cudaFuncSetAttribute(k<a, b, c, d>, cudaFuncAttributeMaxDynamicSharedMemorySize, 80000); }
int main() {
    setup<5, 32, true>(); setup<5, 128, false>(); setup<5, 256, false>(); setup<9, 256, false>(); setup<1, 256, false>(); setup<5, 128, false, 1>(); setup<1, 256, false, 1>(); setup<5, 128, false, 2>(); setup<1, 256, false, 2>(); setup<5, 32, true, 2>(); setup<9, 256, false, 2>();
    long long* t; double* o; cudaMallocManaged(&t, 64); cudaMallocManaged(&o, 64);
    for (int rep = 0; rep < 2; ++rep) {
        k<5, 32, true><<<1, 32, 80000>>>(16, t, o); cudaDeviceSynchronize(); printf("warp 16x16: %lld cycles (%.0f/col) %g\n", t[0], t[0] / 16.0, o[0]);
        k<5, 128, false><<<1, 128, 80000>>>(32, t, o); cudaDeviceSynchronize(); printf("block128 32x32: %lld cycles (%.0f/col) %g\n", t[0], t[0] / 32.0, o[0]);
        k<5, 256, false><<<1, 256, 80000>>>(40, t, o); cudaDeviceSynchronize(); printf("block256 40x40: %lld cycles (%.0f/col)\n", t[0], t[0] / 40.0);
        k<9, 256, false><<<1, 256, 80000>>>(64, t, o); cudaDeviceSynchronize(); printf("block256 64x64: %lld cycles (%.0f/col) %g\n", t[0], t[0] / 64.0, o[0]);
        k<1, 256, false><<<1, 256, 80000>>>(20, t, o); cudaDeviceSynchronize(); printf("block256 20x20: %lld cycles (%.0f/col) %g\n", t[0], t[0] / 20.0, o[0]);
        k<5, 128, false, 1><<<1, 128, 80000>>>(32, t, o); cudaDeviceSynchronize(); printf("OLD block128 32x32: %lld cycles (%.0f/col)\n", t[0], t[0] / 32.0);
        k<1, 256, false, 1><<<1, 256, 80000>>>(20, t, o); cudaDeviceSynchronize(); printf("OLD block256 20x20: %lld cycles (%.0f/col)\n", t[0], t[0] / 20.0);
        k<5, 128, false, 2><<<1, 128, 80000>>>(32, t, o); cudaDeviceSynchronize(); printf("1B block128 32x32: %lld cycles (%.0f/col) %g\n", t[0], t[0] / 32.0, o[0]);
        k<1, 256, false, 2><<<1, 256, 80000>>>(20, t, o); cudaDeviceSynchronize(); printf("1B block256 20x20: %lld cycles (%.0f/col) %g\n", t[0], t[0] / 20.0, o[0]);
        k<5, 32, true, 2><<<1, 32, 80000>>>(16, t, o); cudaDeviceSynchronize(); printf("1B warp 16x16: %lld cycles (%.0f/col) %g\n", t[0], t[0] / 16.0, o[0]);
        k<9, 256, false, 2><<<1, 256, 80000>>>(64, t, o); cudaDeviceSynchronize(); printf("1B block256 64x64: %lld cycles (%.0f/col) %g\n", t[0], t[0] / 64.0, o[0]);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
