// Probe: can a runtime-API kernel launch go to a green-context stream
// (cuGreenCtxStreamCreate) with the primary context current, does it touch
// primary-context allocations, and is it confined to the green SM set?
// nvcc -gencode arch=compute_100a,code=sm_100a -o scripts/micro/green scripts/micro/green.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <set>
#include <vector>

__global__ void smid_kernel(int* out, int n) {
    unsigned s;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
    long long t0 = clock64();
    while (clock64() - t0 < 200000) {
    }
    if (threadIdx.x == 0 && blockIdx.x < n) out[blockIdx.x] = (int)s;
}

#define CK(x)                                                                                    \
    do {                                                                                         \
        CUresult r = (x);                                                                        \
        if (r != CUDA_SUCCESS) {                                                                 \
            const char* s = nullptr;                                                             \
            cuGetErrorString(r, &s);                                                             \
            std::printf("%s -> %d %s\n", #x, (int)r, s ? s : "?");                               \
            return 1;                                                                            \
        }                                                                                        \
    } while (0)

int run(cudaStream_t s, int* d, int n, const char* what) {
    cudaMemset(d, 0xff, n * sizeof(int));
    cudaDeviceSynchronize();
    smid_kernel<<<n, 128, 0, s>>>(d, n);
    cudaError_t e = cudaGetLastError();
    cudaError_t e2 = cudaStreamSynchronize(s);
    std::vector<int> h(n);
    cudaMemcpy(h.data(), d, n * sizeof(int), cudaMemcpyDeviceToHost);
    std::set<int> sms(h.begin(), h.end());
    std::printf("%-40s launch=%s sync=%s distinct SMs=%zu (first %d)\n", what, cudaGetErrorString(e),
                cudaGetErrorString(e2), sms.size(), h[0]);
    return 0;
}

int main() {
    cudaSetDevice(0);
    cudaFree(0);
    int* d = nullptr;
    const int n = 1024;
    cudaMalloc(&d, n * sizeof(int));
    CUdevice dev;
    CK(cuDeviceGet(&dev, 0));
    CUdevResource all, part, rest;
    CK(cuDeviceGetDevResource(dev, &all, CU_DEV_RESOURCE_TYPE_SM));
    std::printf("device SMs %u\n", all.sm.smCount);
    for (unsigned want : {32u, 48u}) {
        unsigned groups = 1;
        CK(cuDevSmResourceSplitByCount(&part, &groups, &all, &rest, 0, want));
        std::printf("split %u -> groups %u, part %u SMs, rest %u SMs\n", want, groups, part.sm.smCount,
                    rest.sm.smCount);
        CUdevResourceDesc desc;
        CK(cuDevResourceGenerateDesc(&desc, &part, 1));
        CUgreenCtx g;
        CK(cuGreenCtxCreate(&g, desc, dev, CU_GREEN_CTX_DEFAULT_STREAM));
        CUstream gs;
        CK(cuGreenCtxStreamCreate(&gs, g, CU_STREAM_NON_BLOCKING, 0));
        run(0, d, n, "primary stream");
        run((cudaStream_t)gs, d, n, "green stream, primary current");
        CUcontext gc;
        CK(cuCtxFromGreenCtx(&gc, g));
        CUcontext prev;
        CK(cuCtxGetCurrent(&prev));
        CK(cuCtxSetCurrent(gc));
        run((cudaStream_t)gs, d, n, "green stream, green current");
        int* d2 = nullptr;
        cudaError_t ea = cudaMalloc(&d2, n * sizeof(int));
        std::printf("cudaMalloc in green ctx: %s\n", cudaGetErrorString(ea));
        CK(cuCtxSetCurrent(prev));
        if (ea == cudaSuccess) run(0, d2, n, "primary stream, green-ctx allocation");
        // event ordering across the two
        cudaEvent_t ev;
        cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
        smid_kernel<<<n, 128, 0, (cudaStream_t)gs>>>(d, n);
        std::printf("record on green stream: %s\n", cudaGetErrorString(cudaEventRecord(ev, (cudaStream_t)gs)));
        std::printf("primary waits: %s\n", cudaGetErrorString(cudaStreamWaitEvent(0, ev, 0)));
        std::printf("sync: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    }
    return 0;
}
