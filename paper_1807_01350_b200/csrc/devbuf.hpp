// Minimal owning device buffer over a per-thread, per-device block cache.
//
// cudaFree synchronizes the whole device, so per-batch temporaries released
// with it would stall the pipeline between kernels.  Released blocks go to a
// cache instead and are reused by later reservations.  Reuse is stream-safe
// because every public entry point finishes with a stream synchronize and a
// handle is driven from one host thread (the reference's threading contract,
// SPEC.md:453): a cached block is never still in use by queued work of
// another stream when it is handed out again.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstring>
#include <map>
#include <utility>
#include <vector>

#include "errors.hpp"

namespace octen {

// Device -> host reads of small results (status words, ranks, flags) through
// a per-thread pinned staging buffer.  A pageable cudaMemcpyAsync D2H waits
// for its stream inside the driver while holding a lock that other host
// threads' CUDA calls need: the pipelined merge's worker reading a flag
// behind a long factorization stalled the next batch's enqueue on the main
// thread for ~1.5 ms per batch.  With a pinned destination the copy is truly
// asynchronous and only the calling thread waits (cudaStreamSynchronize).
inline void d2h_sync(void* dst, const void* src, size_t bytes, cudaStream_t st) {
    struct Stage {
        void* p = nullptr;
        size_t cap = 0;
    };
    static thread_local Stage* s = new Stage;  // never destroyed: may be in flight at thread exit
    if (bytes == 0) {
        OCTEN_CUDA(cudaStreamSynchronize(st));
        return;
    }
    if (bytes > s->cap) {
        OCTEN_CUDA(cudaStreamSynchronize(st));
        if (s->p) OCTEN_CUDA(cudaFreeHost(s->p));
        s->cap = bytes < (1u << 20) ? (1u << 20) : 2 * bytes;
        OCTEN_CUDA(cudaHostAlloc(&s->p, s->cap, cudaHostAllocDefault));
    }
    OCTEN_CUDA(cudaMemcpyAsync(s->p, src, bytes, cudaMemcpyDeviceToHost, st));
    OCTEN_CUDA(cudaStreamSynchronize(st));
    std::memcpy(dst, s->p, bytes);
}

struct BlockCache {
    std::multimap<size_t, void*> free_blocks[16];  // per device ordinal (bytes -> block)

    static BlockCache& get() {
        static thread_local BlockCache* c = new BlockCache;  // never destroyed: buffers may outlive it
        return *c;
    }
    void* take(size_t bytes, size_t& got) {
        int dev = 0;
        cudaGetDevice(&dev);
        auto& m = free_blocks[dev & 15];
        auto it = m.lower_bound(bytes);
        if (it != m.end() && it->first <= 2 * bytes + (1 << 20)) {
            void* p = it->second;
            got = it->first;
            m.erase(it);
            return p;
        }
        // New blocks come from the device's stream-ordered pool on a private
        // stream: unlike cudaMalloc this does not synchronize the device, so
        // a buffer that grows mid-stream (C, per-batch scratch) does not
        // stall the kernels in flight.  Freed pool memory is kept (release
        // threshold max) and the pool is reused.
        void* p = nullptr;
        cudaStream_t s = alloc_stream(dev);
        cudaError_t e = cudaMallocAsync(&p, bytes, s);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);
        if (e != cudaSuccess) {
            (void)cudaGetLastError();
            trim(dev);
            OCTEN_CUDA(cudaMallocAsync(&p, bytes, s));
            OCTEN_CUDA(cudaStreamSynchronize(s));
        }
        got = bytes;
        return p;
    }
    static cudaStream_t alloc_stream(int dev) {
        static thread_local cudaStream_t s[16] = {};
        if (!s[dev & 15]) {
            OCTEN_CUDA(cudaStreamCreateWithFlags(&s[dev & 15], cudaStreamNonBlocking));
            cudaMemPool_t pool;
            if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
                unsigned long long thr = ~0ull;
                cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
            }
        }
        return s[dev & 15];
    }
    // A block goes back to the list of the device it was allocated on (which
    // need not be the current one when the owner is released).
    void give(void* p, size_t bytes, int dev) { free_blocks[dev & 15].emplace(bytes, p); }
    void trim(int dev) {
        OCTEN_CUDA(cudaDeviceSynchronize());
        cudaStream_t s = alloc_stream(dev);
        for (auto& kv : free_blocks[dev & 15]) cudaFreeAsync(kv.second, s);
        free_blocks[dev & 15].clear();
        OCTEN_CUDA(cudaStreamSynchronize(s));
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) cudaMemPoolTrimTo(pool, 0);
    }
};

template <class T>
struct DevBuf {
    T* p = nullptr;
    size_t n = 0;
    int dev = 0;  // device ordinal the block belongs to

    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() { release(); }

    void swap(DevBuf& o) {
        std::swap(p, o.p);
        std::swap(n, o.n);
        std::swap(dev, o.dev);
    }
    void release() {
        if (p) BlockCache::get().give(p, n * sizeof(T), dev);
        p = nullptr;
        n = 0;
    }
    // Ensure capacity for `count` elements (contents not preserved).
    T* reserve(size_t count) {
        if (count <= n && p) return p;
        release();
        if (count == 0) count = 1;
        size_t got = 0;
        OCTEN_CUDA(cudaGetDevice(&dev));
        p = static_cast<T*>(BlockCache::get().take(count * sizeof(T), got));
        n = got / sizeof(T);
        return p;
    }
    // Ensure capacity, preserving the first `keep` elements.
    T* grow(size_t count, size_t keep, cudaStream_t st) {
        if (count <= n && p) return p;
        size_t got = 0;
        int qdev = 0;
        OCTEN_CUDA(cudaGetDevice(&qdev));
        T* q = static_cast<T*>(BlockCache::get().take(count * sizeof(T), got));
        if (p && keep) OCTEN_CUDA(cudaMemcpyAsync(q, p, keep * sizeof(T), cudaMemcpyDeviceToDevice, st));
        OCTEN_CUDA(cudaStreamSynchronize(st));
        release();
        p = q;
        dev = qdev;
        n = got / sizeof(T);
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
        d2h_sync(h.data(), p, count * sizeof(T), st);
        return h;
    }
};

}  // namespace octen
