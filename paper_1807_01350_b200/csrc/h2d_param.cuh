// Small host -> device parameter uploads that bypass the copy engines.
//
// A pipelined caller keeps the next batch's 400 MB host -> device copy on a
// copy engine while the current batch runs (octen_stream_prefetch).  A small
// cudaMemcpyAsync of the current batch (CP-ALS mixture weights, seeds, merge
// flags) on another stream would queue behind that DMA on the same engine and
// stall its stream for milliseconds.  These uploads are instead staged in a
// per-thread ring of pinned, device-mapped host memory and read by a one-CTA
// kernel on the caller's stream.  A ring region is reused only after the
// event recorded behind its reader has completed.
#pragma once

#include <cuda_runtime.h>

#include <cstring>
#include <deque>
#include <vector>

#include "errors.hpp"
#include "octen_common.cuh"

namespace octen {

template <int kUnused = 0>  // a template: one definition across the translation units
__global__ void h2d_param_pull_kernel(unsigned char* __restrict__ dst, const unsigned char* __restrict__ src,
                                      size_t n) {
    size_t i = threadIdx.x;
    if (((uintptr_t)dst | (uintptr_t)src | n) % 8 == 0) {
        for (; i < n / 8; i += blockDim.x) reinterpret_cast<double*>(dst)[i] = reinterpret_cast<const double*>(src)[i];
    } else {
        for (; i < n; i += blockDim.x) dst[i] = src[i];
    }
}

class ParamStager {
public:
    static ParamStager& get() {
        static thread_local ParamStager* s = new ParamStager;  // never destroyed: outlives queued readers
        return *s;
    }
    void upload(void* dst, const void* src, size_t bytes, cudaStream_t st) {
        if (bytes == 0) return;
        const size_t need = (bytes + 255) & ~size_t(255);
        if (need > kCap) {  // not a parameter: plain copy
            OCTEN_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st));
            return;
        }
        if (!host_) {
            OCTEN_CUDA(cudaHostAlloc((void**)&host_, kCap, cudaHostAllocMapped));
            OCTEN_CUDA(cudaHostGetDevicePointer((void**)&dev_, host_, 0));
        }
        // Live regions, oldest first: those of the previous lap (above the
        // head, ascending), then this lap's (below the head).
        if (head_ + need > kCap) {  // wrap: the previous lap's remainder above the head retires first
            while (!live_.empty() && live_.front().start >= head_) retire();
            head_ = 0;
        }
        // wait for earlier readers of [head_, head_ + need)
        while (!live_.empty() && live_.front().start < head_ + need && head_ < live_.front().end) retire();
        std::memcpy(host_ + head_, src, bytes);
        h2d_param_pull_kernel<0><<<1, 256, 0, st>>>((unsigned char*)dst, dev_ + head_, bytes);
        OCTEN_LAUNCHED(1);
        OCTEN_CUDA(cudaGetLastError());
        cudaEvent_t ev;
        if (free_ev_.empty()) {
            OCTEN_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        } else {
            ev = free_ev_.back();
            free_ev_.pop_back();
        }
        OCTEN_CUDA(cudaEventRecord(ev, st));
        live_.push_back(Region{head_, head_ + need, ev});
        head_ += need;
    }

private:
    struct Region {
        size_t start, end;
        cudaEvent_t ev;
    };
    void retire() {
        OCTEN_CUDA(cudaEventSynchronize(live_.front().ev));
        free_ev_.push_back(live_.front().ev);
        live_.pop_front();
    }
    static constexpr size_t kCap = 4u << 20;
    unsigned char* host_ = nullptr;
    unsigned char* dev_ = nullptr;
    size_t head_ = 0;
    std::deque<Region> live_;
    std::vector<cudaEvent_t> free_ev_;
};

inline void h2d_param(void* dst, const void* src, size_t bytes, cudaStream_t st) {
    ParamStager::get().upload(dst, src, bytes, st);
}

}  // namespace octen
