// Common definitions for the OCTen B200 kernels and their host-side twins.
//
// OCTEN_HD marks routines compiled both for the device (nvcc, inside the
// kernels of this library) and for the host (g++, only by the CPU test
// harness tests/cpu_harness/small_linalg_host.cpp, which checks the small
// dense solvers against numpy without a GPU).
#pragma once

#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstdlib>

#if defined(__CUDACC__)
#define OCTEN_HD __host__ __device__
#define OCTEN_DEV __device__
#else
#define OCTEN_HD
#define OCTEN_DEV
#endif

#define OCTEN_LAUNCHED(n) ::octen::launch_counter().fetch_add((n), std::memory_order_relaxed)

#if defined(__CUDACC__)
#include <cuda_runtime.h>
#endif

namespace octen {

// Number of kernels this library has launched (reported by bench.py as
// gpu_launches).
inline std::atomic<long long>& launch_counter() {
    static std::atomic<long long> c{0};
    return c;
}
// Path counters (octen_kernel_counts): tcgen05 launches of the fp32 dense
// compression (GEMM1 + mode-2), chunks of it that ran on the SIMT GEMM
// instead (a shape outside the tcgen05 kernels' limits), and DMMA launches
// of the fp64-input compression, tcgen05 (kind::i8, digit-split fp64)
// launches of the CP-ALS T-GEMM.
enum PathCounter { kTcgen05Launches = 0, kSimtFallbacks = 1, kDmmaCompress = 2, kTcgen05Als = 3, kNumPathCounters = 4 };
inline std::atomic<long long>& path_counter(int i) {
    static std::atomic<long long> c[kNumPathCounters];
    return c[i];
}

#if defined(__CUDACC__)
// Stream priorities (B200: least 0 .. greatest -5).  Measured at c3 with the
// pipelined ingest (ms per step): the batch streams at the default (least)
// priority with every merge factorization chain at the greatest, 13.1; the
// batch streams one level below the greatest with the merge chain just above
// the merge's least-priority bulk updates, 13.9 (CP-ALS 9.5 ms, but the
// merge, now starved, 13.3 ms becomes the longer stage).  The first is the
// default; OCTEN_PRIO_MODE=1 selects the second (diagnostics).
inline int prio_mode() {
    static const int m = [] {
        const char* e = std::getenv("OCTEN_PRIO_MODE");
        return e ? std::atoi(e) : 0;
    }();
    return m;
}
// priority of the streams that carry a batch's compression and CP-ALS
inline int critical_stream_priority() {
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    if (prio_mode() == 1) return hi < lo ? hi + 1 : hi;
    return lo;
}
// priority of a factorization chain whose bulk updates run on `st`
inline int chain_priority_over(cudaStream_t st) {
    int lo = 0, hi = 0, p = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    if (prio_mode() != 1) return hi;
    if (cudaStreamGetPriority(st, &p) != cudaSuccess) p = lo;
    return p > hi ? p - 1 : hi;
}

// Kernel attributes (cudaFuncSetAttribute) are per device: a process that
// drives handles on several GPUs must set them once per device ordinal, not
// once per process.  `PerDevice` remembers the devices already done.
struct PerDevice {
    std::atomic<unsigned long long> done{0};
    template <class F>
    void once(F&& f) {
        int dev = 0;
        cudaGetDevice(&dev);
        const unsigned long long bit = 1ull << (dev & 63);
        if (done.load(std::memory_order_acquire) & bit) return;
        f();
        done.fetch_or(bit, std::memory_order_release);
    }
};
#endif

// A "team" is the set of threads cooperating on one small problem: a CUDA
// thread block on the device, a single thread on the host.  Team-parallel
// routines only use tid()/size()/sync() and block-strided loops, so the
// one-thread host instantiation executes exactly the same arithmetic.
#if defined(__CUDACC__)
struct TeamDev {
    __device__ int tid() const { return (int)threadIdx.x; }
    __device__ int size() const { return (int)blockDim.x; }
    __device__ void sync() const { __syncthreads(); }
};
// One warp as a team (lanes 0..31); sync is a warp barrier.
struct TeamWarp {
    __device__ int tid() const { return (int)(threadIdx.x & 31); }
    __device__ int size() const { return 32; }
    __device__ void sync() const { __syncwarp(); }
};
#endif
struct TeamHost {
    int tid() const { return 0; }
    int size() const { return 1; }
    void sync() const {}
};

// Device-side error record. Kernels that detect a reference error condition
// write the first (lowest problem index wins) record; the host turns it into
// the reference exception text.
enum StatusCode : int {
    kOk = 0,
    kAlsNonFiniteFactor = 1,   // a = sweep, b = mode            (cp_als.cpp:305-307)
    kAlsNonFiniteFit = 2,      // a = sweep                      (cp_als.cpp:335-336)
    kAlignDegenerateRef = 3,   // a = mode                       (recovery.cpp:181-183)
    kAlignDegenerateRep = 4,   // a = replica, b = mode          (recovery.cpp:253-255)
    kAlignDegenerateScale = 5, // a = replica, b = mode          (recovery.cpp:279-281)
    kRecoverRankDeficient = 6, // a = mode, b = rank, c = cols   (recovery.cpp:34-36)
    kRecoverZeroColumn = 7,    //                                 (streaming.cpp:143-144)
    kAppendRankDeficient = 8,  //                                 (recovery.cpp:398-399)
    kAppendNonFiniteGauge = 9, //                                 (recovery.cpp:402-403)
    kGevdFailed = 10,          // internal: GEVD init exhausted -> random fallback
};

struct DevStatus {
    int code;
    int problem;  // ordering key: lowest wins
    int a, b, c;
    double d;
};

OCTEN_HD inline double dsq(double x) { return x * x; }

#if defined(__CUDACC__)
// Programmatic dependent launch.  A kernel launched with launch_pdl may start
// while its predecessor on the stream is still running: it must call
// pdl_wait() before touching anything the predecessor writes (the wait returns
// once the predecessor has completed and its writes are visible; it is a no-op
// in a kernel launched normally).  pdl_trigger() lets the successor launch
// once every block of this grid has issued it.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }

// Block-wide global -> shared copy with eight independent loads in flight per
// thread (the ALS update's 2400-element M / V^-1 staging in one latency).
// (A plain `dst[e] = src[e]` loop through generic pointers makes every load
// wait for the previous shared store, since the compiler cannot rule out
// aliasing: one global latency per element per thread.)  src must not have
// been read by this SM earlier in the kernel while other blocks wrote it
// (the non-coherent load path).
__device__ __forceinline__ void g2s_copy(double* dst, const double* src, int n) {
    constexpr int U = 8;
    const int st = blockDim.x;
    int e = threadIdx.x;
    for (; e + (U - 1) * st < n; e += U * st) {
        double v[U];
#pragma unroll
        for (int j = 0; j < U; ++j) v[j] = __ldg(src + e + j * st);
#pragma unroll
        for (int j = 0; j < U; ++j) dst[e + j * st] = v[j];
    }
    {
        double v[U];
#pragma unroll
        for (int j = 0; j < U; ++j) v[j] = (e + j * st < n) ? __ldg(src + e + j * st) : 0.0;
#pragma unroll
        for (int j = 0; j < U; ++j)
            if (e + j * st < n) dst[e + j * st] = v[j];
    }
}
#endif

}  // namespace octen
