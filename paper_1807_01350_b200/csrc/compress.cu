// Stage 1: multi-replica compression of one temporal batch into the summaries
// (reference compress + update_summaries, proj/src/compression.cpp:108-153,
// mode products of tensor.cpp:168-178).
//
//   GEMM1  Z1 = A X_(1)          A = deduplicated [U_1 ... U_P]^T (Meff x I):
//                                the `shared` leading columns are identical in
//                                every replica (compression.cpp:43-60), so they
//                                are contracted once: Meff = shared + P (Q - shared)
//   GEMM2  Z2_p(:,:,k) = Z1_p(:,:,k) V_p      per (replica, slice)
//   GEMM3  Y_p += Z2_p (Q^2 x t) W_p          fp64 accumulate (update_summaries)
//
// The batch is processed in chunks of temporal slices so Z1 stays bounded.
// fp32 input: GEMM1 and GEMM2 run on the tensor cores (tcgen05, split-TF32).
// A shape outside those kernels' limits (K or J not a multiple of 4, Q > 128)
// runs that chunk on the SIMT GEMM and is counted (octen_kernel_counts); the
// tcgen05 path being unavailable on the device is an error unless
// OCTEN_DISABLE_TCGEN05 / OCTEN_ALLOW_SIMT opts in (diagnostics).
// fp64 input: GEMM1 and GEMM2 on the FP64 tensor cores (DMMA).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "engine.hpp"
#include "errors.hpp"
#include "gemm_dmma.cuh"
#include "tc_gemm.hpp"

namespace octen {

namespace {

template <typename T>
struct G1A {  // A(0, m, i) = A[m*I + i]   (row-major, K contiguous)
    const T* A;
    long long I;
    __device__ T operator()(int, int m, int i) const { return A[(size_t)m * I + i]; }
};
template <typename T>
struct G1B {  // B(0, i, n) = X[i + I n]
    const T* X;
    long long I;
    __device__ T operator()(int, int i, int n) const { return X[(size_t)i + (size_t)I * n]; }
};
template <typename T>
struct G1C {  // Z1[m*N + n]
    T* Z;
    long long N;
    __device__ void operator()(int, int m, int n, T v) const { Z[(size_t)m * N + n] = v; }
};
template <typename T>
struct G2A {  // batch bt = p*tc + k : A(bt, a, j) = Z1[row(p,a)*N1 + k*J + j]
    const T* Z1;
    const int* rowmap;
    long long N1, J;
    int tc, Q;
    __device__ T operator()(int bt, int a, int j) const {
        const int p = bt / tc, k = bt % tc;
        return Z1[(size_t)rowmap[p * Q + a] * N1 + (size_t)k * J + j];
    }
};
template <typename T>
struct G2B {  // B(bt, j, b) = V[p][j + J b]
    const T* V;
    long long J;
    int tc, Q;
    __device__ T operator()(int bt, int j, int b) const {
        const int p = bt / tc;
        return V[(size_t)p * J * Q + j + (size_t)J * b];
    }
};
template <typename T>
struct G2C {  // Z2[p * zs + (a + Q b) + Q^2 k]   (zs: per-replica stride, Q^2 t for the whole batch)
    T* Z2;
    long long zs;
    int tc, Q;
    __device__ void operator()(int bt, int a, int b, T v) const {
        const int p = bt / tc, k = bt % tc;
        const size_t q2 = (size_t)Q * Q;
        Z2[(size_t)p * zs + a + (size_t)Q * b + q2 * k] = v;
    }
};
template <typename T>
struct G3A {  // A(p, m, k) = Z2[p][m + Q^2 k]
    const T* Z2;
    int tc, Q;
    __device__ double operator()(int p, int m, int k) const {
        const size_t q2 = (size_t)Q * Q;
        return (double)Z2[(size_t)p * q2 * tc + m + q2 * k];
    }
};
struct G3B {  // B(p, k, c) = W[p][(k0 + k) + t c]
    const double* W;
    long long t, k0;
    int Q;
    __device__ double operator()(int p, int k, int c) const { return W[(size_t)p * t * Q + (k0 + k) + (size_t)t * c]; }
};
struct G3C {  // Yout[p](a, b, c) = Yin[p](a, b, c) + v, m = a + Q b   (in place when Yin == Yout)
    const double* Yin;
    double* Yout;
    int Q;
    // element strides of (non-temporal slot 0, slot 1, temporal) in the
    // summaries, which keep the stream's original mode order
    // (compression.cpp:117-127): (1, Q, Q^2) when the temporal mode is last
    int s0, s1, st;
    __device__ void operator()(int p, int m, int c, double v) const {
        const size_t q3 = (size_t)Q * Q * Q;
        const int a = m % Q, b = m / Q;
        const size_t e = (size_t)p * q3 + (size_t)a * s0 + (size_t)b * s1 + (size_t)c * st;
        Yout[e] = Yin[e] + v;
    }
};

__global__ void nonfinite_chunk_kernel(const float* x32, const double* x64, size_t n, int* flag) {
    int bad = 0;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        if (!isfinite(x32 ? (double)x32[i] : x64[i])) bad = 1;
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flag, 1);
}

// Modes 1 and 2 of the compression for the whole batch, slice chunk by
// slice chunk: Z2[p][a + Q b + Q^2 k] = (X x1 U_p^T x2 V_p^T)(a, b, k).
// With `ready` the chunk waits for its host->device copy event first, so the
// copies of later chunks overlap the contractions of earlier ones; with
// `flag` every chunk is also scanned for non-finite values (the batch must
// be rejected before the summaries change).
bool simt_opt_in() {
    return std::getenv("OCTEN_DISABLE_TCGEN05") != nullptr || std::getenv("OCTEN_ALLOW_SIMT") != nullptr;
}

template <typename T>
void run_project(CompressEngine& e, const T* dX, std::int64_t t, T* Z1, T* Z2, const T* A, const T* V,
                 std::int64_t tc_max, cudaStream_t st, bool use_tc, const cudaEvent_t* ready, int* flag) {
    const int Q = e.Q, P = e.P;
    const long long zs = (long long)Q * Q * t;
    for (std::int64_t k0 = 0, ci = 0; k0 < t; k0 += tc_max, ++ci) {
        const int tc = (int)std::min<std::int64_t>(tc_max, t - k0);
        const long long N1 = e.J * tc;
        const T* Xc = dX + (size_t)e.I * e.J * k0;
        if (ready) OCTEN_CUDA(cudaStreamWaitEvent(st, ready[ci], 0));
        // the non-finite scan: fused into the tcgen05 GEMM1's conversion
        // warps when it runs, else a separate pass
        bool scanned = false;
        auto scan = [&] {
            if (!flag || scanned) return;
            scanned = true;
            const size_t n = (size_t)e.I * e.J * tc;
            size_t blocks = (n + 255) / 256;
            if (blocks > 148 * 8) blocks = 148 * 8;
            if constexpr (std::is_same<T, float>::value)
                nonfinite_chunk_kernel<<<(int)blocks, 256, 0, st>>>(Xc, nullptr, n, flag);
            else
                nonfinite_chunk_kernel<<<(int)blocks, 256, 0, st>>>(nullptr, Xc, n, flag);
            OCTEN_LAUNCHED(1);
        };
        bool done = false;
        OCTEN_CUDA(cudaEventRecord(e.event(2 * e.g1_used), st));
        if constexpr (std::is_same<T, float>::value) {
            // tensor-core path: GEMM1 scatters its rows replica-contiguously
            // (P*Q x N1) for the batched tcgen05 mode-2 contraction
            if (use_tc) {
                if (!tc_gemm_available()) {
                    if (!simt_opt_in())
                        throw CudaError("octen: the tcgen05 compression kernels are unavailable on this device "
                                        "(sm_100a required; set OCTEN_ALLOW_SIMT=1 to run the SIMT GEMMs)");
                } else {
                    done = tc_gemm_tf32x3(e.Ahi.p, e.Alo.p, e.lda_tc, Xc, Z1, (int)e.Meff, (long long)N1, (int)e.I,
                                          st, P, Q, e.shared, flag, e.g1_ctas);
                    if (done) scanned = true;
                    if (done)
                        path_counter(kTcgen05Launches).fetch_add(1);
                    else
                        path_counter(kSimtFallbacks).fetch_add(1);
                }
            }
            e.used_tc = done;
        }
        if (!done) {
            scan();
            if constexpr (std::is_same<T, double>::value) {
                gemm_f64<true, true>(1, (int)e.Meff, (int)N1, (int)e.I, G1A<T>{A, e.I}, G1B<T>{Xc, e.I},
                                     G1C<T>{Z1, N1}, st);
                path_counter(kDmmaCompress).fetch_add(1);
            } else {
                gemm_simt<T, T, true, true>(1, (int)e.Meff, (int)N1, (int)e.I, G1A<T>{A, e.I}, G1B<T>{Xc, e.I},
                                            G1C<T>{Z1, N1}, st);
            }
        }
        OCTEN_CUDA(cudaEventRecord(e.event(2 * e.g1_used + 1), st));
        ++e.g1_used;
        ++e.gemm1_launches;
        e.gemm1_flops += 2.0 * (double)e.Meff * (double)N1 * (double)e.I;
        T* Z2c = Z2 + (size_t)Q * Q * k0;
        bool done2 = false;
        if constexpr (std::is_same<T, float>::value) {
            static const bool no_m2 = std::getenv("OCTEN_DISABLE_TC_MODE2") != nullptr;
            if (done && !no_m2) {
                done2 = tc_mode2_tf32x3(Z1, N1, (int)e.J, tc, e.Vhi.p, e.Vlo.p, e.ldv_tc, P, Q, Z2c, zs, st);
                path_counter(done2 ? kTcgen05Launches : kSimtFallbacks).fetch_add(1);
            }
        }
        if (!done2) {
            if constexpr (std::is_same<T, double>::value) {
                gemm_f64<true, true>(P * tc, Q, Q, (int)e.J, G2A<T>{Z1, e.rowmap.p, N1, e.J, tc, Q},
                                     G2B<T>{V, e.J, tc, Q}, G2C<T>{Z2c, zs, tc, Q}, st);
                path_counter(kDmmaCompress).fetch_add(1);
            } else {
                gemm_simt<T, T, true, false>(P * tc, Q, Q, (int)e.J,
                                             G2A<T>{Z1, done ? e.rowmap_id.p : e.rowmap.p, N1, e.J, tc, Q},
                                             G2B<T>{V, e.J, tc, Q}, G2C<T>{Z2c, zs, tc, Q}, st);
            }
        }
    }
    OCTEN_CUDA(cudaGetLastError());
}

// Mode 3 for the whole batch, accumulated into the summaries (update_summaries):
// Y_p += Z2_p (Q^2 x t) W_p (t x Q), fp64.
template <typename T>
void run_accumulate(CompressEngine& e, std::int64_t t, const T* Z2, const double* dW, const double* dYin,
                    double* dY, cudaStream_t st) {
    const int Q = e.Q, P = e.P;
    gemm_f64<false, true>(P, Q * Q, Q, (int)t, G3A<T>{Z2, (int)t, Q}, G3B{dW, t, 0, Q},
                          G3C{dYin, dY, Q, e.ys[0], e.ys[1], e.ys[2]}, st);
    OCTEN_CUDA(cudaGetLastError());
}

}  // namespace

void accumulate_z2_f32(int P, int Q, std::int64_t t, const float* Z2, const double* dW, double* dY, cudaStream_t st) {
    gemm_f64<false, true>(P, Q * Q, Q, (int)t, G3A<float>{Z2, (int)t, Q}, G3B{dW, t, 0, Q}, G3C{dY, dY, Q, 1, Q, Q * Q},
                          st);
    OCTEN_CUDA(cudaGetLastError());
}

cudaEvent_t CompressEngine::event(int i) {
    while ((int)g1_events.size() <= i) {
        cudaEvent_t ev;
        OCTEN_CUDA(cudaEventCreate(&ev));
        g1_events.push_back(ev);
    }
    return g1_events[i];
}

double CompressEngine::collect_gemm1_ms() {
    double ms = 0.0;
    for (int i = 0; i < g1_used; ++i) {
        float t = 0.f;
        OCTEN_CUDA(cudaEventElapsedTime(&t, g1_events[2 * i], g1_events[2 * i + 1]));
        ms += t;
    }
    g1_used = 0;
    return ms;
}

CompressEngine::~CompressEngine() {
    for (cudaEvent_t e : g1_events) cudaEventDestroy(e);
}

void CompressEngine::set_projections(int P_, int Q_, int shared_, std::int64_t I_, std::int64_t J_, const double* hU,
                                     const double* hV, cudaStream_t st) {
    P = P_;
    Q = Q_;
    shared = shared_;
    set_temporal_mode(2);  // the stream sets its own after this
    I = I_;
    J = J_;
    Meff = shared + (std::int64_t)P * (Q - shared);
    std::vector<int> rm((size_t)P * Q);
    std::vector<double> a64((size_t)Meff * I);
    for (int p = 0; p < P; ++p)
        for (int a = 0; a < Q; ++a) {
            const std::int64_t row = a < shared ? a : shared + (std::int64_t)p * (Q - shared) + (a - shared);
            rm[(size_t)p * Q + a] = (int)row;
            if (a < shared && p > 0) continue;
            const double* u = hU + (size_t)p * I * Q + (size_t)I * a;
            for (std::int64_t i = 0; i < I; ++i) a64[(size_t)row * I + i] = u[i];
        }
    std::vector<float> a32(a64.begin(), a64.end());
    // TF32 hi/lo split of the fp64 projections: hi = fp32 value with the low
    // 13 mantissa bits cleared, lo = fp32(u - hi)
    lda_tc = (int)((I + 3) / 4 * 4);
    std::vector<float> ahi((size_t)Meff * lda_tc, 0.f), alo((size_t)Meff * lda_tc, 0.f);
    for (std::int64_t m = 0; m < Meff; ++m)
        for (std::int64_t i = 0; i < I; ++i) {
            const double u = a64[(size_t)m * I + i];
            float f = (float)u;
            uint32_t bits;
            std::memcpy(&bits, &f, 4);
            bits &= 0xFFFFE000u;
            float h;
            std::memcpy(&h, &bits, 4);
            ahi[(size_t)m * lda_tc + i] = h;
            alo[(size_t)m * lda_tc + i] = (float)(u - (double)h);
        }
    Ahi.upload(ahi.data(), ahi.size(), st);
    Alo.upload(alo.data(), alo.size(), st);
    // same split of V for the tensor-core mode-2 contraction: row p Q + b = V_p[:, b]
    ldv_tc = (int)((J + 3) / 4 * 4);
    {
        std::vector<float> vhi((size_t)P * Q * ldv_tc, 0.f), vlo((size_t)P * Q * ldv_tc, 0.f);
        for (int p = 0; p < P; ++p)
            for (int b = 0; b < Q; ++b)
                for (std::int64_t j = 0; j < J; ++j) {
                    const double v = hV[(size_t)p * J * Q + j + (size_t)J * b];
                    float f = (float)v;
                    uint32_t bits;
                    std::memcpy(&bits, &f, 4);
                    bits &= 0xFFFFE000u;
                    float h;
                    std::memcpy(&h, &bits, 4);
                    vhi[((size_t)p * Q + b) * ldv_tc + j] = h;
                    vlo[((size_t)p * Q + b) * ldv_tc + j] = (float)(v - (double)h);
                }
        Vhi.upload(vhi.data(), vhi.size(), st);
        Vlo.upload(vlo.data(), vlo.size(), st);
        std::vector<int> rid((size_t)P * Q);
        for (size_t i = 0; i < rid.size(); ++i) rid[i] = (int)i;
        rowmap_id.upload(rid.data(), rid.size(), st);
    }
    std::vector<float> v32(hV, hV + (size_t)P * J * Q);
    rowmap.upload(rm.data(), rm.size(), st);
    A64.upload(a64.data(), a64.size(), st);
    A32.upload(a32.data(), a32.size(), st);
    V64.upload(hV, (size_t)P * J * Q, st);
    V32.upload(v32.data(), v32.size(), st);
    // Z1 chunk of about 1 GiB
    const std::int64_t zrows = std::max<std::int64_t>(Meff, (std::int64_t)P * Q);  // scattered tc layout: P*Q rows
    chunk_slices = std::max<std::int64_t>(1, (std::int64_t)((1ULL << 28) / (unsigned long long)std::max<std::int64_t>(1, zrows * J)));
    OCTEN_CUDA(cudaStreamSynchronize(st));
}

void CompressEngine::project(const void* dX, int dtype, std::int64_t t, cudaStream_t st, const cudaEvent_t* ready,
                             std::int64_t ready_slices, int* flag) {
    std::int64_t tc = std::min(t, chunk_slices);
    if (ready) tc = ready_slices;  // chunks follow the copies
    const size_t zrows = (size_t)std::max<std::int64_t>(Meff, (std::int64_t)P * Q);
    if (dtype == 1) {
        Z1f.reserve(zrows * J * tc);
        Z2f.reserve((size_t)P * Q * Q * t);
        run_project<float>(*this, (const float*)dX, t, Z1f.p, Z2f.p, A32.p, V32.p, tc, st, true, ready, flag);
    } else {
        Z1d.reserve((size_t)Meff * J * tc);
        Z2d.reserve((size_t)P * Q * Q * t);
        run_project<double>(*this, (const double*)dX, t, Z1d.p, Z2d.p, A64.p, V64.p, tc, st, false, ready, flag);
    }
}

void CompressEngine::accumulate(int dtype, std::int64_t t, const double* dW, const double* dYin, double* dY,
                                cudaStream_t st) {
    if (dtype == 1)
        run_accumulate<float>(*this, t, Z2f.p, dW, dYin, dY, st);
    else
        run_accumulate<double>(*this, t, Z2d.p, dW, dYin, dY, st);
}

void CompressEngine::accumulate_rows(int dtype, std::int64_t t, const double* dW, std::int64_t t_total,
                                     std::int64_t k0, double* dY, cudaStream_t st) {
    if (dtype == 1)
        gemm_f64<false, true>(P, Q * Q, Q, (int)t, G3A<float>{Z2f.p, (int)t, Q}, G3B{dW, t_total, k0, Q},
                              G3C{dY, dY, Q, ys[0], ys[1], ys[2]}, st);
    else
        gemm_f64<false, true>(P, Q * Q, Q, (int)t, G3A<double>{Z2d.p, (int)t, Q}, G3B{dW, t_total, k0, Q},
                              G3C{dY, dY, Q, ys[0], ys[1], ys[2]}, st);
    OCTEN_CUDA(cudaGetLastError());
}

void CompressEngine::compress_f32(const float* dX, std::int64_t t, const double* dW, double* dY, cudaStream_t st) {
    project(dX, 1, t, st, nullptr, 0, nullptr);
    accumulate(1, t, dW, dY, dY, st);
}

void CompressEngine::compress_f64(const double* dX, std::int64_t t, const double* dW, double* dY, cudaStream_t st) {
    project(dX, 0, t, st, nullptr, 0, nullptr);
    accumulate(0, t, dW, dY, dY, st);
}

}  // namespace octen
