// On-device synthetic stream generator: the reference's
// generate_synthetic (proj/src/commands.cpp:110-134) produced slice batch by
// slice batch in HBM, so the large configs (c5: 2000 x 2000 x 4000) never
// pass through the host.
//
//   factors   U(0,1) per mode from derive(seed, {9, n}), column-major
//             (host mt19937_64: bit-identical to the reference, rng.hpp:75-79)
//   tensor    reconstruct(model) (cp_als.cpp:361-367) on the FP64 tensor cores
//   noise     N(mu, sigma) added in flat order (first index fastest) from ONE
//             mt19937_64 stream derive(seed, {10}) through the reference's
//             Box-Muller with its cached spare (rng.hpp:59-72)
//
// The noise stream is inherently sequential.  One CTA runs the mt19937_64
// recurrence in parallel across each 312-word state block (the twist splits
// into two dependency-free halves) and writes the 53-bit uniforms; a wide
// kernel then turns consecutive pairs into the two Box-Muller normals and
// adds them to the clean slices.  Batches must be drawn in order (the
// generator keeps the stream position and the pending spare across calls).
// The device's log/sqrt/sincos differ from glibc's in the last ulp at most,
// so the values match the reference's to a few ulp (tests/test_gpu_synth.py).
#include <cuda_runtime.h>

#include <cmath>
#include <vector>

#include "engine.hpp"
#include "errors.hpp"
#include "gemm_dmma.cuh"
#include "rng_host.hpp"
#include "small_linalg.cuh"
#include "synth.hpp"

namespace octen {

namespace {

constexpr int kMtN = 312, kMtM = 156;

__device__ __forceinline__ uint64_t mt_twist_word(uint64_t cur, uint64_t nxt, uint64_t far) {
    const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL, A = 0xB5026F5AA96619E9ULL;
    const uint64_t x = (cur & UM) | (nxt & LM);
    uint64_t xa = x >> 1;
    if (x & 1ULL) xa ^= A;
    return far ^ xa;
}
__device__ __forceinline__ uint64_t mt_temper(uint64_t y) {
    y ^= (y >> 29) & 0x5555555555555555ULL;
    y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
    y ^= (y << 37) & 0xFFF7EEE000000000ULL;
    y ^= y >> 43;
    return y;
}

// `need` consecutive 53-bit uniforms of the stream in `gs` (state words +
// position), in order, into u[0..need).  One CTA of 320 threads.  zero_flag
// is raised when a uniform is exactly 0 (the reference's Box-Muller would
// redraw it: probability 2^-53 per draw; reported, not emulated).
__global__ void __launch_bounds__(320) mt_uniforms_kernel(Mt64* gs, long long need, double* u, int* zero_flag) {
    __shared__ uint64_t cur[kMtN], nw[kMtN];
    __shared__ int s_idx;
    const int tid = threadIdx.x;
    for (int i = tid; i < kMtN; i += blockDim.x) cur[i] = gs->mt[i];
    if (tid == 0) s_idx = gs->idx;
    __syncthreads();
    int idx = s_idx;
    long long done = 0;
    int zero = 0;
    while (done < need) {
        if (idx >= kMtN) {
            // twist: words [0, 156) read only old words; [156, 312) read the
            // new word i - 156 and the old word i + 1 (the new word 0 for 311)
            if (tid < kMtM) nw[tid] = mt_twist_word(cur[tid], cur[tid + 1], cur[tid + kMtM]);
            __syncthreads();
            if (tid < kMtN - kMtM) {
                const int i = tid + kMtM;
                const uint64_t nxt = i + 1 < kMtN ? cur[i + 1] : nw[0];
                nw[i] = mt_twist_word(cur[i], nxt, nw[i - kMtM]);
            }
            __syncthreads();
            for (int i = tid; i < kMtN; i += blockDim.x) cur[i] = nw[i];
            __syncthreads();
            idx = 0;
        }
        const long long take = min((long long)(kMtN - idx), need - done);
        for (int i = tid; i < take; i += blockDim.x) {
            const uint64_t y = mt_temper(cur[idx + i]);
            const double v = (double)(y >> 11) * 0x1.0p-53;
            if (v <= 0.0) zero = 1;
            u[done + i] = v;
        }
        idx += (int)take;
        done += take;
    }
    __syncthreads();
    for (int i = tid; i < kMtN; i += blockDim.x) gs->mt[i] = cur[i];
    if (tid == 0) gs->idx = idx;
    if (__syncthreads_or(zero) && tid == 0) *zero_flag = 1;
}

// X[e] += mu + sigma * n_e with n the stream's normals: pair j of uniforms
// (u[2j], u[2j+1]) gives r cos(theta) then r sin(theta); `lead` = 1 when the
// stream's pending spare feeds element 0.  Writes fp64 or fp32 out.
template <typename T>
__global__ void add_noise_kernel(const double* __restrict__ X, const double* __restrict__ u, long long n, int lead,
                                 double spare, double mu, double sigma, T* __restrict__ out) {
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n;
         e += (long long)gridDim.x * blockDim.x) {
        double z;
        if (e < lead) {
            z = spare;
        } else {
            const long long q = e - lead, j = q >> 1;
            const double u1 = u[2 * j], u2 = u[2 * j + 1];
            const double r = sqrt(-2.0 * log(u1));
            const double theta = 2.0 * 3.14159265358979323846 * u2;
            double sn, cs;
            sincos(theta, &sn, &cs);
            // rng.hpp:66-71: mu + sigma * r * cos(theta) (left to right), and
            // the spare r * sin(theta) returned as mu + sigma * spare
            out[e] = (T)(X[e] + ((q & 1) ? mu + sigma * (r * sn) : mu + sigma * r * cs));
            continue;
        }
        out[e] = (T)(X[e] + (mu + sigma * z));
    }
}

template <typename T>
__global__ void copy_cast_kernel(const double* __restrict__ X, long long n, T* __restrict__ out) {
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n;
         e += (long long)gridDim.x * blockDim.x)
        out[e] = (T)X[e];
}

// reconstruct of slices [k0, k0 + t): X(i, j + J k) = sum_r A(i, r) B(j, r) C(k0 + k, r)
struct SynA {  // A(0, i, r)
    const double* A;
    long long I;
    __device__ double operator()(int, int i, int r) const { return A[i + (size_t)I * r]; }
};
struct SynB {  // B(0, r, n) = B(j, r) C(k0 + k, r), n = j + J k
    const double* B;
    const double* C;
    long long J, K, k0;
    __device__ double operator()(int, int r, int n) const {
        const long long j = n % J, k = n / J;
        return B[j + (size_t)J * r] * C[(k0 + k) + (size_t)K * r];
    }
};
struct SynStore {
    double* X;
    long long I;
    __device__ void operator()(int, int i, int n, double v) const { X[i + (size_t)I * n] = v; }
};

int grid_for_n(long long n) {
    long long b = (n + 255) / 256;
    if (b > 148 * 8) b = 148 * 8;
    return (int)(b < 1 ? 1 : b);
}

}  // namespace

SynthStream::SynthStream(const std::vector<std::int64_t>& dims_, int rank_, std::uint64_t seed_, double mu_,
                         double sigma_, int device_)
    : dims(dims_), rank(rank_), seed(seed_), mu(mu_), sigma(sigma_), device(device_) {
    // commands.cpp:110-115
    if (dims.size() < 2) throw ConfigError("gen: need at least two extents");
    for (std::int64_t d : dims)
        if (d < 1) throw ConfigError("gen: extents must be >= 1");
    if (rank < 1) throw ConfigError("gen: rank must be >= 1");
    if (sigma < 0.0) throw ConfigError("gen: noise sigma must be >= 0");
    if (dims.size() != 3) throw ConfigError("octen: the device generator produces order-3 tensors");
    OCTEN_CUDA(cudaSetDevice(device));
    OCTEN_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    // factors: U(0,1) per mode from derive(seed, {9, n}), column-major (commands.cpp:118-123)
    hF.resize(dims.size());
    for (size_t n = 0; n < dims.size(); ++n) {
        hF[n].assign((size_t)dims[n] * rank, 0.0);
        rng::Substream s(rng::derive(seed, {rng::kSynthFactor, (std::uint64_t)n}));
        s.fill_uniform(hF[n].data(), dims[n], rank, dims[n]);
    }
    for (size_t n = 0; n < dims.size(); ++n) dF[n].upload(hF[n].data(), hF[n].size(), st);
    // the noise stream derive(seed, {10}) (commands.cpp:127-130)
    noisy = sigma > 0.0 || mu != 0.0;
    Mt64 h;
    h.seed(rng::derive(seed, {rng::kSynthNoise}));
    state.upload(&h, 1, st);
    flag.reserve(1);
    flag.zero(1, st);
    OCTEN_CUDA(cudaStreamSynchronize(st));
}

SynthStream::~SynthStream() {
    if (st) {
        cudaStreamSynchronize(st);
        cudaStreamDestroy(st);
    }
}

void SynthStream::next(std::int64_t t, void* out, int dtype) {
    if (t < 1 || k_next + t > dims[2]) throw ConfigError("gen: slice range outside the tensor");
    const std::int64_t I = dims[0], J = dims[1], K = dims[2];
    const long long n = (long long)I * J * t;
    X.reserve((size_t)n);
    // clean slices on the FP64 tensor cores
    gemm_f64<false, false>(1, (int)I, (int)(J * t), rank, SynA{dF[0].p, I}, SynB{dF[1].p, dF[2].p, J, K, k_next},
                           SynStore{X.p, I}, st);
    OCTEN_CUDA(cudaGetLastError());
    if (noisy) {
        const int lead = have_spare ? 1 : 0;
        const long long pairs = (n - lead + 1) / 2;
        U.reserve((size_t)std::max<long long>(1, 2 * pairs));
        if (pairs > 0) {
            mt_uniforms_kernel<<<1, 320, 0, st>>>(state.p, 2 * pairs, U.p, flag.p);
            OCTEN_LAUNCHED(1);
        }
        if (dtype == 1)
            add_noise_kernel<float><<<grid_for_n(n), 256, 0, st>>>(X.p, U.p, n, lead, spare, mu, sigma, (float*)out);
        else
            add_noise_kernel<double><<<grid_for_n(n), 256, 0, st>>>(X.p, U.p, n, lead, spare, mu, sigma,
                                                                   (double*)out);
        OCTEN_LAUNCHED(1);
        // the spare left for the next batch: the sin half of the last pair
        // when the batch used only its cos half
        if ((n - lead) % 2 == 1) {
            double u2h[2];
            OCTEN_CUDA(cudaMemcpyAsync(u2h, U.p + 2 * (pairs - 1), 2 * sizeof(double), cudaMemcpyDeviceToHost, st));
            OCTEN_CUDA(cudaStreamSynchronize(st));
            const double r = std::sqrt(-2.0 * std::log(u2h[0]));
            spare = r * std::sin(2.0 * 3.14159265358979323846 * u2h[1]);
            have_spare = true;
        } else {
            have_spare = false;
        }
        int zf = 0;
        OCTEN_CUDA(cudaMemcpyAsync(&zf, flag.p, sizeof(int), cudaMemcpyDeviceToHost, st));
        OCTEN_CUDA(cudaStreamSynchronize(st));
        if (zf) throw NumericError("gen: a zero uniform was drawn (Box-Muller redraw not emulated on the device)");
    } else {
        if (dtype == 1)
            copy_cast_kernel<float><<<grid_for_n(n), 256, 0, st>>>(X.p, n, (float*)out);
        else
            copy_cast_kernel<double><<<grid_for_n(n), 256, 0, st>>>(X.p, n, (double*)out);
        OCTEN_LAUNCHED(1);
    }
    OCTEN_CUDA(cudaGetLastError());
    OCTEN_CUDA(cudaStreamSynchronize(st));
    k_next += t;
}

void SynthStream::truth(double* const* factors, double* lambda) const {
    // model.normalize() (cp_als.cpp:216-228): unit columns, norms into lambda
    const int order = (int)dims.size();
    std::vector<double> lam(rank, 1.0);
    for (int n = 0; n < order; ++n) {
        const std::int64_t d = dims[n];
        for (int c = 0; c < rank; ++c) {
            double s = 0.0;
            for (std::int64_t i = 0; i < d; ++i) s += hF[n][i + d * c] * hF[n][i + d * c];
            const double nrm = std::sqrt(s);
            for (std::int64_t i = 0; i < d; ++i)
                factors[n][i + d * c] = nrm > 0.0 ? hF[n][i + d * c] / nrm : hF[n][i + d * c];
            if (nrm > 0.0) lam[c] *= nrm;
        }
    }
    for (int c = 0; c < rank; ++c) lambda[c] = lam[c];
}

}  // namespace octen
