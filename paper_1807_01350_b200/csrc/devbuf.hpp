// Minimal owning device buffer.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <vector>

#include "errors.hpp"

namespace octen {

template <class T>
struct DevBuf {
    T* p = nullptr;
    size_t n = 0;

    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() { release(); }

    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
    // Ensure capacity for `count` elements (contents not preserved).
    T* reserve(size_t count) {
        if (count <= n && p) return p;
        release();
        if (count == 0) count = 1;
        OCTEN_CUDA(cudaMalloc(&p, count * sizeof(T)));
        n = count;
        return p;
    }
    // Ensure capacity, preserving the first `keep` elements.
    T* grow(size_t count, size_t keep, cudaStream_t st) {
        if (count <= n && p) return p;
        T* q = nullptr;
        OCTEN_CUDA(cudaMalloc(&q, count * sizeof(T)));
        if (p && keep) OCTEN_CUDA(cudaMemcpyAsync(q, p, keep * sizeof(T), cudaMemcpyDeviceToDevice, st));
        OCTEN_CUDA(cudaStreamSynchronize(st));
        release();
        p = q;
        n = count;
        return p;
    }
    void zero(size_t count, cudaStream_t st) {
        OCTEN_CUDA(cudaMemsetAsync(p, 0, count * sizeof(T), st));
    }
    void upload(const T* h, size_t count, cudaStream_t st) {
        reserve(count);
        OCTEN_CUDA(cudaMemcpyAsync(p, h, count * sizeof(T), cudaMemcpyHostToDevice, st));
    }
    void download(T* h, size_t count, cudaStream_t st) const {
        OCTEN_CUDA(cudaMemcpyAsync(h, p, count * sizeof(T), cudaMemcpyDeviceToHost, st));
    }
    std::vector<T> to_host(size_t count, cudaStream_t st) const {
        std::vector<T> h(count);
        download(h.data(), count, st);
        OCTEN_CUDA(cudaStreamSynchronize(st));
        return h;
    }
};

}  // namespace octen
