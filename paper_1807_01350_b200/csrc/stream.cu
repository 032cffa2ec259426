// Host orchestrator of the per-batch pipeline: init_stream / ingest_batch
// (reference proj/src/streaming.cpp:181-346) over device-resident state.
//
// Host work is limited to what the reference's determinism contract pins to
// the host: the seeded projection draws (gen_replicas / extend_temporal,
// compression.cpp:22-99) and the stage sequencing.  Summaries Y_p, history
// accumulators M_p, the model factors and every contraction/solve live on the
// device.
#include <cuda.h>
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <cstdlib>
#include <cstring>

#include <chrono>
#include <cmath>
#include <memory>
#include <string>
#include <vector>

#include "engine.hpp"
#include "errors.hpp"
#include "rng_host.hpp"
#include "stream.hpp"
#include "evprof.hpp"
#include "h2d_param.cuh"

namespace octen {

namespace {

using Clock = std::chrono::steady_clock;
double seconds_since(Clock::time_point t0) { return std::chrono::duration<double>(Clock::now() - t0).count(); }

__global__ void nonfinite_f32_kernel(const float* x, size_t n, int* flag) {
    int bad = 0;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        if (!isfinite(x[i])) bad = 1;
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flag, 1);
}
__global__ void nonfinite_f64_kernel(const double* x, size_t n, int* flag) {
    int bad = 0;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        if (!isfinite(x[i])) bad = 1;
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flag, 1);
}

// C_raw = C * diag(lambda) for the first K rows (ld = cap)
__global__ void scale_cols_kernel(double* C, long long K, long long cap, int R, const double* lam) {
    const size_t total = (size_t)K * R;
    for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < total; e += (size_t)gridDim.x * blockDim.x) {
        const long long k = (long long)(e % K);
        const int r = (int)(e / K);
        C[k + (size_t)cap * r] *= lam[r];
    }
}
// append t new rows (t x R col-major) at row offset K of C (ld = cap)
__global__ void append_rows_kernel(double* C, long long K, long long cap, int R, const double* rows, long long t) {
    const size_t total = (size_t)t * R;
    for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < total; e += (size_t)gridDim.x * blockDim.x) {
        const long long k = (long long)(e % t);
        const int r = (int)(e / t);
        C[(K + k) + (size_t)cap * r] = rows[k + (size_t)t * r];
    }
}
// KruskalModel::normalize over (A, B, C) for column r (cp_als.cpp:216-228).
__global__ void normalize_model_kernel(double* A, long long I, double* B, long long J, double* C, long long K,
                                       long long capC, double* lam) {
    __shared__ double red[256];
    const int r = blockIdx.x;
    double l = 1.0;
    for (int f = 0; f < 3; ++f) {
        double* col = f == 0 ? A + (size_t)I * r : (f == 1 ? B + (size_t)J * r : C + (size_t)capC * r);
        const long long n = f == 0 ? I : (f == 1 ? J : K);
        double s = 0.0;
        for (long long i = threadIdx.x; i < n; i += blockDim.x) s += col[i] * col[i];
        red[threadIdx.x] = s;
        __syncthreads();
        for (int st = blockDim.x / 2; st > 0; st >>= 1) {
            if ((int)threadIdx.x < st) red[threadIdx.x] += red[threadIdx.x + st];
            __syncthreads();
        }
        const double nrm = sqrt(red[0]);
        __syncthreads();
        if (nrm > 0.0) {
            for (long long i = threadIdx.x; i < n; i += blockDim.x) col[i] /= nrm;
            l *= nrm;
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) lam[r] = l;
}

// A batch with the temporal mode at position tm, as the I x J x t
// temporal-last block the compression contracts: out(i, j, k) =
// X(i, j, k) read with the strides of the batch's own mode order.
template <typename T>
__global__ void to_temporal_last_kernel(const T* __restrict__ X, T* __restrict__ out, long long I, long long J,
                                        long long t, long long sI, long long sJ, long long sT) {
    const long long n = I * J * t;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x) {
        const long long i = e % I, r = e / I, j = r % J, k = r / J;
        out[e] = X[i * sI + j * sJ + k * sT];
    }
}
// replica factors (P x 3 x Q x R, the stream's mode order) into slot order:
// non-temporal slot 0, slot 1, then the temporal factor
__global__ void factors_to_slots_kernel(const double* __restrict__ in, double* __restrict__ out, int P, long long qr,
                                        int m0, int m1, int mt) {
    const long long n = (long long)P * 3 * qr;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x) {
        const long long x = e % qr, r = e / qr;
        const int slot = (int)(r % 3), p = (int)(r / 3);
        const int m = slot == 0 ? m0 : (slot == 1 ? m1 : mt);
        out[e] = in[((long long)p * 3 + m) * qr + x];
    }
}

int grid1d(size_t n) {
    size_t b = (n + 255) / 256;
    if (b > 148 * 8) b = 148 * 8;
    return (int)(b < 1 ? 1 : b);
}

}  // namespace

Stream::Stream(const StreamCfg& c, int rank, int world) : cfg(c), shard_rank(rank), shard_world(world) {
    if (world < 1 || rank < 0 || rank >= world) throw ConfigError("octen: shard rank/world out of range");
    if (cfg.p >= 1 && world > cfg.p) throw ConfigError("octen: more shards than replicas");
    const int P = std::max(1, cfg.p);
    chunk = (P + world - 1) / world;
    p0 = std::min(P, rank * chunk);
    pl = std::max(0, std::min(P, p0 + chunk) - p0);
    OCTEN_CUDA(cudaSetDevice(cfg.device));
    OCTEN_CUDA(cudaStreamCreateWithPriority(&st, cudaStreamNonBlocking, critical_stream_priority()));
    OCTEN_CUDA(cudaEventCreate(&ev0));
    OCTEN_CUDA(cudaEventCreate(&ev1));
    for (auto& e : evs) OCTEN_CUDA(cudaEventCreate(&e));
}

Stream::~Stream() {
    (void)aworker.wait();
    (void)worker.wait();
    if (ast) {
        cudaStreamSynchronize(ast);
        cudaStreamDestroy(ast);
    }
    for (cudaEvent_t e : aevs)
        if (e) cudaEventDestroy(e);
    for (cudaEvent_t e : ievs)
        if (e) cudaEventDestroy(e);
    if (mst) {
        cudaStreamSynchronize(mst);
        cudaStreamDestroy(mst);
    }
    if (st) cudaStreamSynchronize(st);
    if (cp) {
        cudaStreamSynchronize(cp);
        cudaStreamDestroy(cp);
    }
    for (cudaEvent_t e : copy_ev) cudaEventDestroy(e);
    if (pcp) {
        cudaStreamSynchronize(pcp);
        cudaStreamDestroy(pcp);
    }
    for (auto& v : pf_ev)
        for (cudaEvent_t e : v) cudaEventDestroy(e);
    for (cudaEvent_t e : slot_free)
        if (e) cudaEventDestroy(e);
    if (pin_ev) cudaEventDestroy(pin_ev);
    if (pin_buf) cudaFreeHost(pin_buf);
    if (pub_pin) cudaFreeHost(pub_pin);
    if (ev0) cudaEventDestroy(ev0);
    if (ev1) cudaEventDestroy(ev1);
    for (auto& e : evs)
        if (e) cudaEventDestroy(e);
    if (st) cudaStreamDestroy(st);
}

void Stream::validate(int order) {
    // streaming.cpp:23-34
    if (order < 3) throw ConfigError("stream: tensor order must be >= 3");
    if (cfg.rank < 1) throw ConfigError("stream: rank must be >= 1");
    if (cfg.p < 1) throw ConfigError("stream: p must be >= 1");
    if (cfg.q < 1) throw ConfigError("stream: Q must be >= 1");
    if (cfg.shared < 0 || cfg.shared >= cfg.q) throw ConfigError("stream: shared must lie in [0, Q)");
    if (cfg.temporal_mode >= order) throw ConfigError("stream: temporal mode out of range");
    if (cfg.p >= 2 && cfg.shared < 1) throw ConfigError("stream: alignment across replicas needs shared >= 1");
    if (order != 3)
        throw ConfigError("octen: the device path supports order-3 streams (any temporal mode)");
}

void Stream::gen_replicas() {
    // compression.cpp:22-70 (host RNG, bit-exact draws)
    const int P = cfg.p, Q = cfg.q, sh = cfg.shared;
    const std::int64_t dimv[2] = {I, J};
    std::vector<double>* dst[2] = {&hU, &hV};
    for (int m = 0; m < 2; ++m) {
        const std::int64_t d = dimv[m];
        std::vector<double> shared_block((size_t)d * sh);
        rng::Substream s(rng::derive(cfg.seed, {rng::kNontemporalShared, (std::uint64_t)m}));
        s.fill_uniform(shared_block.data(), d, sh, d);
        dst[m]->assign((size_t)P * d * Q, 0.0);
        for (int r = 0; r < P; ++r) {
            double* mat = dst[m]->data() + (size_t)r * d * Q;
            for (size_t i = 0; i < shared_block.size(); ++i) mat[i] = shared_block[i];
            if (Q > sh) {
                rng::Substream s2(
                    rng::derive(cfg.seed, {rng::kNontemporalPrivate, (std::uint64_t)m, (std::uint64_t)r}));
                s2.fill_uniform(mat + (size_t)d * sh, d, Q - sh, d);
            }
        }
    }
    tgram.assign((size_t)sh * sh, 0.0);
    batches_drawn = 0;
}

TemporalDraw draw_temporal(std::uint64_t seed, int P, int Q, int sh, std::uint64_t key, std::int64_t t_new) {
    // compression.cpp:72-99: the shared leading columns once per batch, each
    // replica's private columns from its own substream; the batch's
    // contribution to the shared temporal Gram
    TemporalDraw d;
    d.key = key;
    d.t = t_new;
    std::vector<double> shared_rows((size_t)t_new * sh);
    {
        rng::Substream s(rng::derive(seed, {rng::kTemporalShared, key}));
        s.fill_uniform(shared_rows.data(), t_new, sh, t_new);
    }
    d.gram.assign((size_t)sh * sh, 0.0);
    for (int i = 0; i < sh; ++i)
        for (int j = 0; j < sh; ++j) {
            double acc = 0.0;
            for (std::int64_t k = 0; k < t_new; ++k)
                acc += shared_rows[k + (size_t)t_new * i] * shared_rows[k + (size_t)t_new * j];
            d.gram[i + (size_t)sh * j] = acc;
        }
    d.w.assign((size_t)P * t_new * Q, 0.0);
    for (int r = 0; r < P; ++r) {
        double* w = d.w.data() + (size_t)r * t_new * Q;
        for (size_t i = 0; i < shared_rows.size(); ++i) w[i] = shared_rows[i];
        if (Q > sh) {
            rng::Substream s2(rng::derive(seed, {rng::kTemporalPrivate, key, (std::uint64_t)r}));
            s2.fill_uniform(w + (size_t)t_new * sh, t_new, Q - sh, t_new);
        }
    }
    return d;
}

void Stream::extend_temporal(std::int64_t t_new) {
    // compression.cpp:72-99.  The draws are a pure function of (seed, batch
    // key, t_new): the next batch's rows are drawn ahead on a helper thread
    // (assuming the same t_new) so the ~0.5 ms of host RNG at c3 is off the
    // batch's critical path; a mismatched guess is discarded.
    const int P = cfg.p, Q = cfg.q, sh = cfg.shared;
    const std::uint64_t key = (std::uint64_t)batches_drawn;
    TemporalDraw d;
    if (next_draw.valid()) {
        TemporalDraw nd = next_draw.get();
        if (nd.key == key && nd.t == t_new) d = std::move(nd);
    }
    if (d.w.empty()) d = draw_temporal(cfg.seed, P, Q, sh, key, t_new);
    for (size_t e = 0; e < d.gram.size(); ++e) tgram[e] += d.gram[e];
    hW = std::move(d.w);
    next_w_slot();
    upload_mapped(dWb[wslot], hW.data(), hW.size());
    dW = dWb[wslot].p;
    ++batches_drawn;
    next_draw = std::async(std::launch::async, draw_temporal, cfg.seed, P, Q, sh, key + 1, t_new);
}

namespace {
__global__ void pull_f64_kernel(double* __restrict__ dst, const double* __restrict__ src, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        dst[i] = src[i];
}
}  // namespace

// Host -> device copy of a small per-batch array through a pinned, mapped
// staging buffer read by a kernel: it bypasses the copy engines, so it is
// not queued behind a prefetch of the next batch (octen_stream_prefetch).
void Stream::upload_mapped(DevBuf<double>& dst, const double* h, size_t n) {
    if (n > pin_cap) {
        if (pin_buf) {
            OCTEN_CUDA(cudaStreamSynchronize(st));
            OCTEN_CUDA(cudaFreeHost(pin_buf));
        }
        OCTEN_CUDA(cudaHostAlloc((void**)&pin_buf, n * sizeof(double), cudaHostAllocMapped));
        pin_cap = n;
        if (!pin_ev) OCTEN_CUDA(cudaEventCreateWithFlags(&pin_ev, cudaEventDisableTiming));
    } else if (pin_ev) {
        OCTEN_CUDA(cudaEventSynchronize(pin_ev));  // the previous pull has read the staging buffer
    }
    std::memcpy(pin_buf, h, n * sizeof(double));
    double* src = nullptr;
    OCTEN_CUDA(cudaHostGetDevicePointer((void**)&src, pin_buf, 0));
    dst.reserve(n);
    const int blocks = (int)std::min<size_t>(148, (n + 255) / 256);
    pull_f64_kernel<<<blocks > 0 ? blocks : 1, 256, 0, st>>>(dst.p, src, n);
    OCTEN_LAUNCHED(1);
    OCTEN_CUDA(cudaGetLastError());
    OCTEN_CUDA(cudaEventRecord(pin_ev, st));
}

const void* Stream::stage_input(const void* data, int dtype, int location, size_t n) {
    if (location == 1) return data;
    if (dtype == 1) {
        X32.reserve(n);
        OCTEN_CUDA(cudaMemcpyAsync(X32.p, data, n * sizeof(float), cudaMemcpyHostToDevice, st));
        return X32.p;
    }
    X64.reserve(n);
    OCTEN_CUDA(cudaMemcpyAsync(X64.p, data, n * sizeof(double), cudaMemcpyHostToDevice, st));
    return X64.p;
}

void Stream::check_finite(const void* dX, int dtype, size_t n) {
    flag.reserve(1);
    flag.zero(1, st);
    if (dtype == 1)
        nonfinite_f32_kernel<<<grid1d(n), 256, 0, st>>>((const float*)dX, n, flag.p);
    else
        nonfinite_f64_kernel<<<grid1d(n), 256, 0, st>>>((const double*)dX, n, flag.p);
    OCTEN_LAUNCHED(1);
    OCTEN_CUDA(cudaGetLastError());
    if (flag.to_host(1, st)[0]) throw NumericError("DenseTensor: non-finite value");
}

// streaming.cpp:263-269: every non-temporal extent must match (messages
// name the mode 1-based, in the stream's own mode order)
void Stream::check_extents(const std::int64_t* dims) {
    const int tm = cfg.temporal_mode;
    const std::int64_t want[2] = {I, J};
    int slot = 0;
    for (int n = 0; n < 3; ++n) {
        if (n == tm) continue;
        if (dims[n] != want[slot])
            throw ConfigError("ingest_batch: extent mismatch on mode " + std::to_string(n + 1) + " at batch " +
                              std::to_string(batches_seen));
        ++slot;
    }
    if (dims[tm] < 1) throw ConfigError("ingest_batch: batch has no temporal extent");
}

// The batch (the stream's mode order, first index fastest) as the I x J x t
// temporal-last block on the device.
const void* Stream::temporal_last(const void* data, int dtype, int location, const std::int64_t* dims) {
    const int tm = cfg.temporal_mode;
    const std::int64_t t = dims[tm];
    const size_t n = (size_t)I * J * t, esz = dtype == 1 ? sizeof(float) : sizeof(double);
    const void* src = data;
    if (location == 0) {
        void* d = dtype == 1 ? (void*)X32.reserve(n) : (void*)X64.reserve(n);
        OCTEN_CUDA(cudaMemcpyAsync(d, data, n * esz, cudaMemcpyHostToDevice, st));
        src = d;
    }
    long long stride[3] = {1, dims[0], dims[0] * dims[1]};
    const long long sI = stride[tm == 0 ? 1 : 0], sJ = stride[tm == 2 ? 1 : 2], sT = stride[tm];
    void* out;
    if (dtype == 1) {
        out = XT32.reserve(n);
        to_temporal_last_kernel<float><<<grid1d(n), 256, 0, st>>>((const float*)src, (float*)out, I, J, t, sI, sJ, sT);
    } else {
        out = XT64.reserve(n);
        to_temporal_last_kernel<double><<<grid1d(n), 256, 0, st>>>((const double*)src, (double*)out, I, J, t, sI, sJ,
                                                                   sT);
    }
    OCTEN_LAUNCHED(1);
    OCTEN_CUDA(cudaGetLastError());
    return out;
}

// strides of (slot 0, slot 1, temporal) in the summaries for the merge's
// temporal unfolding
void Stream::set_mode_strides() {
    const int Q = cfg.q, tm = cfg.temporal_mode, q2 = Q * Q;
    int s3[3];
    if (tm == 2) {
        s3[0] = 1; s3[1] = Q; s3[2] = q2;
    } else if (tm == 1) {
        s3[0] = 1; s3[1] = q2; s3[2] = Q;
    } else {
        s3[0] = Q; s3[1] = q2; s3[2] = 1;
    }
    merge.set_ystrides(s3);
}

// the model's factor of mode n (the stream's mode order): A, B are the
// non-temporal slots, C the temporal factor
int Stream::factor_slot(int mode) const {
    const int tm = cfg.temporal_mode;
    if (mode == tm) return 2;
    return mode < tm ? mode : mode - 1;
}

void Stream::ensure_c_capacity(std::int64_t rows, cudaStream_t st) {
    if (rows <= capC && C.p) return;
    std::int64_t cap = std::max<std::int64_t>(capC * 2, rows);
    cap = std::max<std::int64_t>(cap, 64);
    DevBuf<double> nc;
    nc.reserve((size_t)cap * cfg.rank);
    if (C.p && K > 0)
        OCTEN_CUDA(cudaMemcpy2DAsync(nc.p, cap * sizeof(double), C.p, capC * sizeof(double), K * sizeof(double),
                                     cfg.rank, cudaMemcpyDeviceToDevice, st));
    OCTEN_CUDA(cudaStreamSynchronize(st));
    C.swap(nc);
    capC = cap;
}

// ---- first-batch preparation (streaming.cpp:181-215) ----
void Stream::prepare(int order, const std::int64_t* dims) {
    if (cfg.temporal_mode < 0) cfg.temporal_mode = order - 1;
    validate(order);
    const int tm = cfg.temporal_mode;
    const std::int64_t t0 = dims[tm];
    if (t0 < 1) throw ConfigError("init_stream: first batch has no temporal extent");
    // the non-temporal modes in ascending order are slots 0 and 1 (A, B)
    I = dims[tm == 0 ? 1 : 0];
    J = dims[tm == 2 ? 1 : 2];
    if (cfg.enforce_bounds) {
        // replica_bound_nmode (recovery.cpp:548-557) and kruskal_check (recovery.cpp:531-541)
        if (cfg.q <= cfg.shared) throw ConfigError("replica_bound: requires Q > shared");
        double worst = (double)(I - cfg.shared) / (double)(cfg.q - cfg.shared);
        worst = std::max(worst, (double)J / cfg.q);
        worst = std::max(worst, (double)t0 / cfg.q);
        const std::int64_t need = (std::int64_t)std::ceil(worst);
        if (cfg.p < need)
            throw ConfigError("init_stream: p=" + std::to_string(cfg.p) + " below the replica bound; need p >= " +
                              std::to_string(need));
        long sum = 0;
        for (int n = 0; n < 3; ++n) sum += std::min<std::int64_t>(cfg.q, std::min<std::int64_t>(dims[n], cfg.rank));
        if (sum < 2L * cfg.rank + 2)
            throw ConfigError("init_stream: compressed decomposition fails the identifiability bound");
    }
    gen_replicas();
    const int P = cfg.p, Q = cfg.q, R = cfg.rank;
    // compression and summaries for the owned replicas only
    if (pl > 0) {
        comp.set_projections(pl, Q, cfg.shared, I, J, hU.data() + (size_t)p0 * I * Q, hV.data() + (size_t)p0 * J * Q,
                             st);
        comp.set_temporal_mode(tm);
    }
    merge.set_projections(P, Q, cfg.shared, R, I, J, hU.data(), hV.data(), st);
    set_mode_strides();
    const size_t q3 = (size_t)Q * Q * Q;
    Y.reserve((size_t)std::max(pl, 1) * q3);
    Y.zero((size_t)std::max(pl, 1) * q3, st);
    hist.reserve((size_t)P * Q * R);
    hist.zero((size_t)P * Q * R, st);
    lam.reserve(R);
    A.reserve((size_t)I * R);
    B.reserve((size_t)J * R);
    K = 0;
    batches_seen = 0;
}

// ---- phase 1: stage, compress and decompose the owned replicas ----
namespace {
// CTAs of the background pull (OCTEN_PULL_CTAS, diagnostics; default 8)
int pull_ctas() {
    static const int n = [] {
        const char* e = std::getenv("OCTEN_PULL_CTAS");
        return e ? std::max(1, std::atoi(e)) : 8;
    }();
    return n;
}

__global__ void __launch_bounds__(256) h2d_pull_kernel(int4* __restrict__ dst, const int4* __restrict__ src,
                                                       long long n16) {
    const long long stride = (long long)gridDim.x * blockDim.x;
    long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    for (; i + 7 * stride < n16; i += 8 * stride) {
        int4 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = src[i + u * stride];
#pragma unroll
        for (int u = 0; u < 8; ++u) dst[i + u * stride] = v[u];
    }
    for (; i < n16; i += stride) dst[i] = src[i];
}
}  // namespace

void Stream::prefetch(const void* data, int dtype, int order, const std::int64_t* dims) {
    if (order != 3 || dims[0] < 1 || dims[1] < 1 || dims[2] < 1)
        throw ConfigError("octen: prefetch needs an order-3 batch with positive extents");
    if (cfg.temporal_mode >= 0 && cfg.temporal_mode != 2)
        throw ConfigError("octen: prefetch needs the temporal mode last");
    if (initialized && (dims[0] != I || dims[1] != J))
        throw ConfigError("ingest_batch: extent mismatch on mode 1 at batch " + std::to_string(batches_seen));
    if (pf.size() >= 2) throw ConfigError("octen: two prefetched batches are already pending");
    if (!pcp) {
        int lo = 0, hi = 0;
        OCTEN_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        OCTEN_CUDA(cudaStreamCreateWithPriority(&pcp, cudaStreamNonBlocking, lo));  // lowest priority
        for (auto& e : slot_free) {
            OCTEN_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            OCTEN_CUDA(cudaEventRecord(e, st));
        }
    }
    Prefetch f;
    f.host = data;
    f.dtype = dtype;
    for (int i = 0; i < 3; ++i) f.dims[i] = dims[i];
    f.slot = pf.empty() ? 0 : 1 - pf.front().slot;
    const std::int64_t t = dims[2];
    const size_t plane = (size_t)dims[0] * dims[1], n = plane * t;
    const size_t esz = dtype == 1 ? sizeof(float) : sizeof(double);
    // chunking as in begin(): about five chunks, bounded by the Z1 chunk of
    // the compression once the stream knows its shapes
    const std::int64_t cs = initialized ? comp.chunk_slices : t;
    f.sub = std::max<std::int64_t>(1, std::min<std::int64_t>(cs, std::min<std::int64_t>(t, (t + 4) / 5)));
    f.nch = (t + f.sub - 1) / f.sub;
    void* dst = dtype == 1 ? (void*)PX32[f.slot].reserve(n) : (void*)PX64[f.slot].reserve(n);
    auto& evv = pf_ev[f.slot];
    while ((std::int64_t)evv.size() < f.nch) {
        cudaEvent_t e;
        OCTEN_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        evv.push_back(e);
    }
    // the slot's previous batch must have been read by the compression
    OCTEN_CUDA(cudaStreamWaitEvent(pcp, slot_free[f.slot], 0));
    // The copy runs on the low-priority copy stream through the copy engine.
    // The small per-batch H2D parameter uploads of the batch being processed
    // are read by kernels from mapped host memory (h2d_param.cuh), so they do
    // not queue behind this DMA.  With OCTEN_PREFETCH_PULL=1 a BACKGROUND copy
    // (another prefetch is pending) of pinned memory is pulled by an 8-CTA
    // kernel instead (the round-1 scheme, before the parameter bypass).
    cudaPointerAttributes at{};
    const void* mapped = nullptr;
    // Background copies go through the copy engine (55 GB/s measured; the
    // per-batch parameter uploads bypass it, h2d_param.cuh).  OCTEN_PREFETCH_PULL=1
    // pulls them with an 8-CTA kernel instead (c3 e2e 15.2 vs 14.7 ms/step).
    static const bool use_ce = [] {
        const char* e = std::getenv("OCTEN_PREFETCH_PULL");
        return !(e && e[0] == '1');
    }();
    if (!use_ce && !pf.empty() && cudaPointerGetAttributes(&at, data) == cudaSuccess &&
        at.type == cudaMemoryTypeHost && at.devicePointer)
        mapped = at.devicePointer;
    (void)cudaGetLastError();
    for (std::int64_t c = 0; c < f.nch; ++c) {
        const std::int64_t k0 = c * f.sub, kc = std::min(f.sub, t - k0);
        const size_t off = plane * k0 * esz, bytes = plane * kc * esz;
        if (mapped && (((uintptr_t)mapped + off) % 16) == 0 && (((uintptr_t)dst + off) % 16) == 0 && bytes % 16 == 0) {
            h2d_pull_kernel<<<pull_ctas(), 256, 0, pcp>>>((int4*)((char*)dst + off), (const int4*)((const char*)mapped + off),
                                                 (long long)(bytes / 16));
            OCTEN_LAUNCHED(1);
        } else {
            OCTEN_CUDA(cudaMemcpyAsync((char*)dst + off, (const char*)data + off, bytes, cudaMemcpyHostToDevice, pcp));
        }
        OCTEN_CUDA(cudaEventRecord(evv[c], pcp));
    }
    OCTEN_CUDA(cudaGetLastError());
    pf.push_back(f);
}

// ---- per-batch context, worker thread ----

BatchCtx::~BatchCtx() {
    for (cudaEvent_t& e : ev)
        if (e) cudaEventDestroy(e);
}

Worker::~Worker() {
    if (th.joinable()) {
        {
            std::lock_guard<std::mutex> lk(mu);
            quit = true;
        }
        cv.notify_all();
        th.join();
    }
}

void Worker::loop(int device) {
    cudaSetDevice(device);
    std::unique_lock<std::mutex> lk(mu);
    for (;;) {
        cv.wait(lk, [&] { return quit || (posted && !running && !done); });
        if (quit && !(posted && !done)) return;
        running = true;
        std::function<void()> f = std::move(task);
        lk.unlock();
        std::exception_ptr e;
        try {
            f();
        } catch (...) {
            e = std::current_exception();
        }
        lk.lock();
        err = e;
        running = false;
        done = true;
        cv.notify_all();
    }
}

void Worker::post(int device, std::function<void()> f) {
    if (!th.joinable()) th = std::thread([this, device] { loop(device); });
    std::lock_guard<std::mutex> lk(mu);
    task = std::move(f);
    err = nullptr;
    done = false;
    posted = true;
    cv.notify_all();
}

std::exception_ptr Worker::wait() {
    std::unique_lock<std::mutex> lk(mu);
    if (!posted) return nullptr;
    cv.wait(lk, [&] { return done; });
    posted = false;
    done = false;
    std::exception_ptr e = err;
    err = nullptr;
    return e;
}

void Stream::next_w_slot() { wslot = (wslot + 1) % 3; }

void Stream::begin_ctx(BatchCtx& b, bool first, std::int64_t t) {
    b.context = first ? std::string() : "batch " + std::to_string(batches_seen) + ": ";
    b.pending = true;
    b.first = first;
    b.compressed = false;
    b.init_failed = false;
    b.als_init_ms = 0.f;
    b.als_init_s = 0.0;
    b.Yb = nullptr;
    b.t = t;
    b.t_start = Clock::now();
    b.rec = BatchRecordC{};
    b.rec.batch_index = first ? 0 : batches_seen;
    b.rec.t_new = t;
    for (cudaEvent_t& e : b.ev)
        if (!e) OCTEN_CUDA(cudaEventCreate(&e));
    if (!b.st) b.st = st;
}

void Stream::begin(BatchCtx& b, const void* data, int dtype, int location, int order, const std::int64_t* dims,
                   double* models_out, bool out_of_place, bool run_als) {
    if (b.pending) throw ConfigError("octen: the previous batch has not finished (begin/merge/finish)");
    const bool first = !initialized;
    if (first) {
        prepare(order, dims);
    } else {
        // streaming.cpp:258-346
        if (order != 3)
            throw ConfigError("ingest_batch: batch order mismatch at batch " + std::to_string(batches_seen));
        check_extents(dims);
    }
    const int tm = cfg.temporal_mode;
    const std::int64_t t = dims[tm];
    if (tm != 2) {
        // the compression contracts temporal-last blocks: reorder the batch
        // on the device once (one pass over it)
        data = temporal_last(data, dtype, location, dims);
        location = 1;
    }
    if (!first && cfg.strict) snapshot(backup);
    begin_ctx(b, first, t);
    const int Q = cfg.q;
    // out of place (pipelined ingest): Ynext = Y + this batch's compression
    DevBuf<double>& Yout = out_of_place ? Ynext : Y;
    try {
        auto tc = Clock::now();
        const size_t n = (size_t)I * J * t;
        OCTEN_CUDA(cudaEventRecord(evs[0], st));
        if (pl > 0) {
            // modes 1-2 chunk by chunk; a host batch is copied chunk by chunk on
            // the copy stream so the transfer overlaps the contractions; every
            // chunk is scanned for non-finite values before Y is touched
            flag.reserve(1);
            flag.zero(1, st);
            const bool use_pf = location == 0 && !pf.empty() && pf.front().host == data &&
                                pf.front().dtype == dtype && order == 3 && pf.front().dims[0] == dims[0] &&
                                pf.front().dims[1] == dims[1] && pf.front().dims[2] == dims[2];
            if (location == 0 && !use_pf) pf.clear();  // stale prefetches (the caller changed course)
            if (use_pf) {
                const Prefetch f = pf.front();
                pf.erase(pf.begin());
                const void* dst = dtype == 1 ? (const void*)PX32[f.slot].p : (const void*)PX64[f.slot].p;
                // a copy that has already landed is contracted in one chunk
                // (the chunks only exist to overlap a copy still in flight)
                bool landed = true;
                for (std::int64_t c = 0; c < f.nch && landed; ++c) {
                    const cudaError_t q = cudaEventQuery(pf_ev[f.slot][c]);
                    if (q == cudaErrorNotReady) {
                        landed = false;
                        (void)cudaGetLastError();
                    } else {
                        OCTEN_CUDA(q);
                    }
                }
                if (landed)
                    comp.project(dst, dtype, t, st, nullptr, 0, flag.p);
                else
                    comp.project(dst, dtype, t, st, pf_ev[f.slot].data(), f.sub, flag.p);
                OCTEN_CUDA(cudaEventRecord(slot_free[f.slot], st));
            } else if (location == 0) {
                const std::int64_t sub = std::max<std::int64_t>(
                    1, std::min<std::int64_t>(comp.chunk_slices, std::min<std::int64_t>(t, (t + 4) / 5)));
                const std::int64_t nch = (t + sub - 1) / sub;
                const size_t esz = dtype == 1 ? sizeof(float) : sizeof(double);
                void* dst;
                if (dtype == 1)
                    dst = X32.reserve(n);
                else
                    dst = X64.reserve(n);
                if (!cp) OCTEN_CUDA(cudaStreamCreateWithPriority(&cp, cudaStreamNonBlocking, critical_stream_priority()));
                while ((std::int64_t)copy_ev.size() < nch) {
                    cudaEvent_t e;
                    OCTEN_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
                    copy_ev.push_back(e);
                }
                // the copy stream must not overwrite X while earlier work on st reads it
                OCTEN_CUDA(cudaEventRecord(copy_ev[0], st));
                OCTEN_CUDA(cudaStreamWaitEvent(cp, copy_ev[0], 0));
                const size_t plane = (size_t)I * J;
                for (std::int64_t c = 0; c < nch; ++c) {
                    const std::int64_t k0 = c * sub, kc = std::min(sub, t - k0);
                    OCTEN_CUDA(cudaMemcpyAsync((char*)dst + plane * k0 * esz, (const char*)data + plane * k0 * esz,
                                               plane * kc * esz, cudaMemcpyHostToDevice, cp));
                    OCTEN_CUDA(cudaEventRecord(copy_ev[c], cp));
                }
                comp.project(dst, dtype, t, st, copy_ev.data(), sub, flag.p);
            } else {
                comp.project(data, dtype, t, st, nullptr, 0, flag.p);
            }
            // in place, Y must not be touched by a batch with non-finite
            // values; out of place (Ynext) the mode-3 accumulation is enqueued
            // first and the scan is read once, after it
            if (!out_of_place && flag.to_host(1, st)[0]) throw NumericError("DenseTensor: non-finite value");
        } else {
            const void* dX = stage_input(data, dtype, location, n);
            check_finite(dX, dtype, n);
        }
        const std::int64_t drawn_before = batches_drawn;
        const std::vector<double> tgram_before = tgram;
        b.tgram.clear();
        extend_temporal(t);
        b.tgram = tgram;
        b.dW = dW;
        if (out_of_place) Ynext.reserve((size_t)std::max(pl, 1) * Q * Q * Q);
        if (pl > 0) comp.accumulate(dtype, t, dW + (size_t)p0 * t * Q, Y.p, Yout.p, st);
        if (pl > 0 && out_of_place && flag.to_host(1, st)[0]) {
            batches_drawn = drawn_before;  // the draw of this batch never happened
            tgram = tgram_before;
            throw NumericError("DenseTensor: non-finite value");
        }
        b.compressed = true;
        ++batches_seen;
        OCTEN_CUDA(cudaEventRecord(evs[1], st));
        OCTEN_CUDA(cudaStreamSynchronize(st));
        b.rec.compress_seconds = std::chrono::duration<double>(Clock::now() - tc).count();
        // device time of the compression (main stream)
        float cms = 0.f;
        OCTEN_CUDA(cudaEventElapsedTime(&cms, evs[0], evs[1]));
        dev_ms[0] += cms;
        dev_ms[3] += comp.collect_gemm1_ms();
        gemm1_flops = comp.gemm1_flops;
        gemm1_launches = comp.gemm1_launches;
        if (run_als) als_phase(b, Yout.p, models_out, st);
    } catch (...) {
        fail_pending(b);
    }
}

// CP-ALS of the owned replicas on the updated summaries, packed into this
// rank's models block (status header + factors + lambdas).
void Stream::als_phase(BatchCtx& b, const double* dY, double* models_out, cudaStream_t st) {
    als_init_phase(b, dY, als, st);
    als_sweep_phase(b, models_out, als, st, 1);
}

// CP-ALS, part 1: norms, GEVD starts and initial factors of the owned
// replicas on `e` (host syncs on `st`).
void Stream::als_init_phase(BatchCtx& b, const double* dY, AlsEngine& e, cudaStream_t st) {
    auto ta = Clock::now();
    for (cudaEvent_t& ev : ievs)
        if (!ev) OCTEN_CUDA(cudaEventCreate(&ev));
    OCTEN_CUDA(cudaEventRecord(ievs[0], st));
    if (pl > 0) {
        std::vector<std::uint64_t> seeds(pl);
        for (int r = 0; r < pl; ++r)
            seeds[r] = rng::derive(cfg.seed, {rng::kStreamAls, (std::uint64_t)(p0 + r), (std::uint64_t)b.rec.batch_index});
        e.run_init(pl, cfg.als_n_restarts, cfg.q, cfg.rank, cfg.als_max_iters, cfg.als_rel_tol, dY, seeds, st);
    }
    OCTEN_CUDA(cudaEventRecord(ievs[1], st));
    OCTEN_CUDA(cudaStreamSynchronize(st));
    float ms = 0.f;
    OCTEN_CUDA(cudaEventElapsedTime(&ms, ievs[0], ievs[1]));
    b.als_init_ms = ms;
    b.als_init_s = std::chrono::duration<double>(Clock::now() - ta).count();
}

// CP-ALS, part 2: the sweeps on `e` (stream `st`, ordered after part 1),
// packed into this rank's models block (status header + factors + lambdas).
// `ahead`: how many batches later the engine runs again (its host draws are
// prefetched for that batch).
void Stream::als_sweep_phase(BatchCtx& b, double* models_out, AlsEngine& e, cudaStream_t st, int ahead) {
    const int Q = cfg.q, R = cfg.rank;
    auto ta = Clock::now();
    for (cudaEvent_t& ev : aevs)
        if (!ev) OCTEN_CUDA(cudaEventCreate(&ev));
    OCTEN_CUDA(cudaEventRecord(aevs[0], st));
    double hdr[4] = {0, 0, 0, 0};
    const size_t qr = (size_t)Q * R;
    if (pl > 0) {
        try {
            e.run_sweeps(st);
            // the engine's next batch's host draws, off its critical path
            std::vector<std::uint64_t> seeds(pl);
            for (int r = 0; r < pl; ++r)
                seeds[r] = rng::derive(cfg.seed, {rng::kStreamAls, (std::uint64_t)(p0 + r),
                                                  (std::uint64_t)(b.rec.batch_index + ahead)});
            e.prefetch_host_draws(seeds, cfg.als_n_restarts, Q);
        } catch (const NumericError&) {
            // a replica's CP-ALS failed: every rank raises it after the exchange
            if (e.failure.kind == 0) throw;
            hdr[0] = e.failure.kind;
            hdr[1] = e.failure.a;
            hdr[2] = e.failure.b;
        }
        if (hdr[0] == 0.0) {
            OCTEN_CUDA(cudaMemcpyAsync(models_out + 4, e.Mf.p, sizeof(double) * pl * 3 * qr,
                                       cudaMemcpyDeviceToDevice, st));
            OCTEN_CUDA(cudaMemcpyAsync(models_out + 4 + (size_t)chunk * 3 * qr, e.Mlam.p, sizeof(double) * pl * R,
                                       cudaMemcpyDeviceToDevice, st));
        }
    }
    h2d_param(models_out, hdr, sizeof(hdr), st);
    OCTEN_CUDA(cudaEventRecord(aevs[1], st));
    OCTEN_CUDA(cudaStreamSynchronize(st));
    b.rec.als_seconds = b.als_init_s + std::chrono::duration<double>(Clock::now() - ta).count();
    // device time of CP-ALS (its streams; the compression and the merge add their own)
    float ms = 0.f;
    OCTEN_CUDA(cudaEventElapsedTime(&ms, aevs[0], aevs[1]));
    dev_ms[1] += ms + b.als_init_ms;
    OCTEN_CUDA(cudaEventRecord(b.ev[2], st));
}

namespace {
__global__ void add_f64_kernel(double* __restrict__ y, const double* __restrict__ x, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        y[i] += x[i];
}
__global__ void set_status_kernel(double* out, int G, size_t blk, const int* flag) {
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g < G) out[(size_t)g * blk + blk - 1] = *flag ? 1.0 : 0.0;
}
}  // namespace

// ---- temporal sharding, phase 1a: this rank's slices [k_off, k_off + t_local)
// of a batch of t_total slices, compressed into partial summaries of EVERY
// replica, laid out as shard_world blocks (block g: replicas of rank g,
// chunk x Q^3, then one status double = this rank's non-finite flag) for a
// reduce-scatter (sum) by the caller.  The temporal rows of the whole batch
// are drawn here (identically on every rank).
void Stream::begin_temporal(const void* data, int dtype, int location, int order, const std::int64_t* dims_local,
                            std::int64_t k_off, std::int64_t t_total, double* partial_out) {
    BatchCtx& b = cur;
    if (b.pending) throw ConfigError("octen: the previous batch has not finished (begin/merge/finish)");
    if (order != 3) throw ConfigError("ingest_batch: batch order mismatch at batch " + std::to_string(batches_seen));
    if (cfg.temporal_mode >= 0 && cfg.temporal_mode != 2)
        throw ConfigError("octen: temporal sharding needs the temporal mode last");
    const std::int64_t t_local = dims_local[2];
    if (t_total < 1 || k_off < 0 || t_local < 0 || k_off + t_local > t_total)
        throw ConfigError("octen: temporal shard outside the batch");
    const bool first = !initialized;
    if (first) {
        const std::int64_t full[3] = {dims_local[0], dims_local[1], t_total};
        prepare(order, full);
    } else {
        if (dims_local[0] != I)
            throw ConfigError("ingest_batch: extent mismatch on mode 1 at batch " + std::to_string(batches_seen));
        if (dims_local[1] != J)
            throw ConfigError("ingest_batch: extent mismatch on mode 2 at batch " + std::to_string(batches_seen));
    }
    if (!comp_all_ready) {
        comp_all.set_projections(cfg.p, cfg.q, cfg.shared, I, J, hU.data(), hV.data(), st);
        comp_all_ready = true;
    }
    if (!first && cfg.strict) snapshot(backup);
    begin_ctx(b, first, t_total);
    tshard_drawn = batches_drawn;
    tshard_tgram = tgram;
    const int P = cfg.p, Q = cfg.q;
    const size_t q3 = (size_t)Q * Q * Q, blk = (size_t)chunk * q3 + 1;
    try {
        auto tc = Clock::now();
        OCTEN_CUDA(cudaEventRecord(evs[0], st));
        extend_temporal(t_total);
        b.tgram = tgram;
        b.dW = dW;
        flag.reserve(1);
        flag.zero(1, st);
        Zpart.reserve((size_t)shard_world * chunk * q3);
        Zpart.zero((size_t)shard_world * chunk * q3, st);
        if (t_local > 0) {
            const void* dX = stage_input(data, dtype, location, (size_t)I * J * t_local);
            comp_all.project(dX, dtype, t_local, st, nullptr, 0, flag.p);
            comp_all.accumulate_rows(dtype, t_local, dW, t_total, k_off, Zpart.p, st);
        }
        // replica-contiguous partials -> per-owner blocks with a status slot
        OCTEN_CUDA(cudaMemcpy2DAsync(partial_out, blk * sizeof(double), Zpart.p, (size_t)chunk * q3 * sizeof(double),
                                     (size_t)chunk * q3 * sizeof(double), shard_world, cudaMemcpyDeviceToDevice, st));
        set_status_kernel<<<1, 32 * ((shard_world + 31) / 32), 0, st>>>(partial_out, shard_world, blk, flag.p);
        OCTEN_LAUNCHED(1);
        OCTEN_CUDA(cudaGetLastError());
        OCTEN_CUDA(cudaEventRecord(evs[1], st));
        OCTEN_CUDA(cudaStreamSynchronize(st));
        b.rec.compress_seconds = std::chrono::duration<double>(Clock::now() - tc).count();
        (void)P;
    } catch (...) {
        batches_drawn = tshard_drawn;
        tgram = tshard_tgram;
        fail_pending(b);
    }
}

// ---- temporal sharding, phase 1b: the reduced block of this rank's replicas
// (sum over ranks of their partials; last slot = number of ranks that saw a
// non-finite value) is added to the owned summaries, then CP-ALS as begin().
void Stream::begin_reduced(const double* owned_block, double* models_out) {
    BatchCtx& b = cur;
    if (!b.pending) throw ConfigError("octen: begin_reduced without begin_temporal");
    const int Q = cfg.q;
    const size_t q3 = (size_t)Q * Q * Q, blk = (size_t)chunk * q3 + 1;
    try {
        double status = 0.0;
        d2h_sync(&status, owned_block + blk - 1, sizeof(double), st);
        if (status != 0.0) {
            batches_drawn = tshard_drawn;
            tgram = tshard_tgram;
            throw NumericError("DenseTensor: non-finite value");
        }
        if (pl > 0) {
            const size_t n = (size_t)pl * q3;
            add_f64_kernel<<<(int)std::min<size_t>(148 * 8, (n + 255) / 256), 256, 0, st>>>(Y.p, owned_block, n);
            OCTEN_LAUNCHED(1);
            OCTEN_CUDA(cudaGetLastError());
        }
        b.compressed = true;
        ++batches_seen;
        float cms = 0.f;  // this rank's share of the compression (begin_temporal)
        OCTEN_CUDA(cudaEventElapsedTime(&cms, evs[0], evs[1]));
        dev_ms[0] += cms;
        dev_ms[3] += comp_all.collect_gemm1_ms();
        als_phase(b, Y.p, models_out, st);
    } catch (...) {
        fail_pending(b);
    }
}

// ---- phase 2: align, recover A and B, temporal-stack rows of the owned replicas ----
void Stream::merge_phase(BatchCtx& b, const double* models_all, double* rows_out) {
    if (!b.pending) throw ConfigError("octen: merge without a begun batch");
    cudaStream_t st = b.st;  // the merge's stream (the main one, or the pipelined ingest's merge stream)
    try {
        b.t_recover = Clock::now();
        if (st != this->st) OCTEN_CUDA(cudaStreamWaitEvent(st, b.ev[2], 0));
        OCTEN_CUDA(cudaEventRecord(b.ev[0], st));
        static thread_local EvProf sp;
        sp.mark("begin", st);
        const int P = cfg.p, Q = cfg.q, R = cfg.rank;
        const size_t qr = (size_t)Q * R, mc = models_count();
        // CP-ALS failures of any rank (lowest replica first)
        std::vector<double> hdr((size_t)shard_world * 4);
        for (int g = 0; g < shard_world; ++g)
            d2h_sync(hdr.data() + 4 * g, models_all + (size_t)g * mc, 4 * sizeof(double), st);
        for (int g = 0; g < shard_world; ++g)
            if (hdr[4 * g] != 0.0)
                throw NumericError(als_failure_message((int)hdr[4 * g], (int)hdr[4 * g + 1], (int)hdr[4 * g + 2]));
        MfAll.reserve((size_t)P * 3 * qr);
        MlamAll.reserve((size_t)P * R);
        for (int g = 0; g < shard_world; ++g) {
            const int g0 = g * chunk, gl = std::max(0, std::min(P, g0 + chunk) - g0);
            if (gl == 0) continue;
            const double* blk = models_all + (size_t)g * mc;
            OCTEN_CUDA(cudaMemcpyAsync(MfAll.p + (size_t)g0 * 3 * qr, blk + 4, sizeof(double) * gl * 3 * qr,
                                       cudaMemcpyDeviceToDevice, st));
            OCTEN_CUDA(cudaMemcpyAsync(MlamAll.p + (size_t)g0 * R, blk + 4 + (size_t)chunk * 3 * qr,
                                       sizeof(double) * gl * R, cudaMemcpyDeviceToDevice, st));
        }
        if (cfg.temporal_mode != 2) {
            // the replica models come in the stream's mode order; the merge
            // works in slot order (non-temporal 0, 1, temporal)
            const int tm = cfg.temporal_mode;
            MfSlot.reserve((size_t)P * 3 * qr);
            factors_to_slots_kernel<<<grid1d((size_t)P * 3 * qr), 256, 0, st>>>(
                MfAll.p, MfSlot.p, P, (long long)qr, tm == 0 ? 1 : 0, tm == 2 ? 1 : 2, tm);
            OCTEN_LAUNCHED(1);
            MfAll.swap(MfSlot);
        }
        AlignResultHost ar;
        sp.mark("hdr+gather", st);
        merge.align(MfAll.p, MlamAll.p, b.tgram, st, &ar);
        sp.mark("align", st);
        b.rec.min_match_similarity = ar.min_match;
        b.rec.max_offdiag_similarity = ar.max_offdiag;
        Anew.reserve((size_t)I * R);
        Bnew.reserve((size_t)J * R);
        merge.recover_ab(b.first ? nullptr : A.p, b.first ? nullptr : B.p, Anew.p, Bnew.p, st);
        sp.mark("recover_ab", st);
        if (pl > 0) merge.temporal_stack(b.Yb ? b.Yb : Y.p, p0, pl, Anew.p, Bnew.p, rows_out, true, st);
        sp.mark("temporal_stack", st);
        sp.report("merge_phase");
        OCTEN_CUDA(cudaStreamSynchronize(st));
    } catch (...) {
        fail_pending(b);
    }
}

namespace {
// rows_all (world blocks of chunk x Q x R, replica-major) -> P*Q x R stacked
__global__ void unpack_rows_kernel(const double* rows_all, size_t per_rank, int chunk, int P, int Q, int R,
                                   double* tstack) {
    const size_t total = (size_t)P * Q * R, PQ = (size_t)P * Q;
    for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < total; e += (size_t)gridDim.x * blockDim.x) {
        const size_t row = e % PQ;
        const int r = (int)(e / PQ);
        const int p = (int)(row / Q), i = (int)(row % Q);
        const int g = p / chunk, pi = p % chunk;
        tstack[row + PQ * r] = rows_all[(size_t)g * per_rank + (size_t)pi * Q * R + i + (size_t)Q * r];
    }
}
}  // namespace

// ---- phase 3: temporal append, model assembly, BatchRecord ----
void Stream::finish(BatchCtx& b, const double* rows_all) {
    if (!b.pending) throw ConfigError("octen: finish without a begun batch");
    cudaStream_t st = b.st;
    try {
        const int P = cfg.p, Q = cfg.q, R = cfg.rank;
        const std::int64_t t_new = b.t;
        tstackAll.reserve((size_t)P * Q * R);
        unpack_rows_kernel<<<grid1d((size_t)P * Q * R), 256, 0, st>>>(rows_all, rows_count(), chunk, P, Q, R,
                                                                       tstackAll.p);
        OCTEN_LAUNCHED(1);
        rows.reserve((size_t)t_new * R);
        double residual = 0.0;
        static thread_local EvProf fp;
        fp.mark("begin", st);
        merge.temporal_append(tstackAll.p, b.dW, t_new, hist.p, rows.p, &residual, st);
        fp.mark("temporal_append", st);
        fp.report("finish");
        b.rec.temporal_residual = residual;
        b.rec.warned = residual > cfg.residual_warning ? 1 : 0;
        if (b.rec.warned && cfg.strict) {
            if (b.first)
                throw NumericError("init_stream: temporal solve residual " + std::to_string(residual) +
                                   " exceeds strict threshold");
            throw NumericError("temporal solve residual " + std::to_string(residual) + " exceeds strict threshold");
        }
        // assemble_model (streaming.cpp:162-177): C_raw = [C diag(lambda); rows]
        ensure_c_capacity(K + t_new, st);
        if (!b.first && K > 0) {
            scale_cols_kernel<<<grid1d((size_t)K * R), 256, 0, st>>>(C.p, K, capC, R, lam.p);
            OCTEN_LAUNCHED(1);
        }
        append_rows_kernel<<<grid1d((size_t)t_new * R), 256, 0, st>>>(C.p, K, capC, R, rows.p, t_new);
        OCTEN_LAUNCHED(1);
        A.swap(Anew);
        B.swap(Bnew);
        normalize_model_kernel<<<R, 256, 0, st>>>(A.p, I, B.p, J, C.p, K + t_new, capC, lam.p);
        OCTEN_LAUNCHED(1);
        OCTEN_CUDA(cudaGetLastError());
        OCTEN_CUDA(cudaEventRecord(b.ev[1], st));
        const std::int64_t Kn = K + t_new;
        if (publish) {  // D2H of the batch's model (the step's result) into pinned staging
            const size_t need = (size_t)(I + J + Kn) * R + R;
            if (need > pub_cap) {
                OCTEN_CUDA(cudaStreamSynchronize(st));
                if (pub_pin) OCTEN_CUDA(cudaFreeHost(pub_pin));
                pub_cap = std::max(need, 2 * pub_cap);
                OCTEN_CUDA(cudaHostAlloc((void**)&pub_pin, pub_cap * sizeof(double), cudaHostAllocDefault));
            }
            OCTEN_CUDA(cudaMemcpyAsync(pub_pin, A.p, sizeof(double) * I * R, cudaMemcpyDeviceToHost, st));
            OCTEN_CUDA(cudaMemcpyAsync(pub_pin + I * R, B.p, sizeof(double) * J * R, cudaMemcpyDeviceToHost, st));
            OCTEN_CUDA(cudaMemcpy2DAsync(pub_pin + (I + J) * R, Kn * sizeof(double), C.p, capC * sizeof(double),
                                         Kn * sizeof(double), R, cudaMemcpyDeviceToHost, st));
            OCTEN_CUDA(cudaMemcpyAsync(pub_pin + (I + J + Kn) * R, lam.p, sizeof(double) * R, cudaMemcpyDeviceToHost,
                                       st));
        }
        OCTEN_CUDA(cudaStreamSynchronize(st));
        if (publish) {
            std::lock_guard<std::mutex> lk(pub_mu);
            pubA.assign(pub_pin, pub_pin + I * R);
            pubB.assign(pub_pin + I * R, pub_pin + (I + J) * R);
            pubC.assign(pub_pin + (I + J) * R, pub_pin + (I + J + Kn) * R);
            pubLam.assign(pub_pin + (I + J + Kn) * R, pub_pin + (I + J + Kn) * R + R);
            pub_K = Kn;
            pub_batches = (std::int64_t)log.size() + 1;
        }
        K += t_new;
        float ms = 0.f;
        OCTEN_CUDA(cudaEventElapsedTime(&ms, b.ev[0], b.ev[1]));
        dev_ms[2] += ms;
        b.rec.recover_seconds = std::chrono::duration<double>(Clock::now() - b.t_recover).count();
        b.rec.total_seconds = std::chrono::duration<double>(Clock::now() - b.t_start).count();
        log.push_back(b.rec);
        initialized = true;
        b.pending = false;
    } catch (...) {
        fail_pending(b);
    }
}

// Error inside a phase: drain the streams, roll back (strict mode), add the
// batch context (streaming.cpp:336-345) and rethrow.
void Stream::fail_pending(BatchCtx& b) {
    cudaStreamSynchronize(st);
    if (b.st && b.st != st) cudaStreamSynchronize(b.st);
    (void)cudaGetLastError();
    const bool had = b.pending;
    b.pending = false;
    const bool first = b.first;
    if (had && !first && cfg.strict) restore(backup);
    try {
        throw;
    } catch (const ConfigError& e) {
        throw ConfigError(b.context + e.what());
    } catch (const NumericError& e) {
        throw NumericError(b.context + e.what());
    }
}

void Stream::snapshot(Snapshot& s) {
    const int P = cfg.p, Q = cfg.q, R = cfg.rank;
    const size_t ny = (size_t)std::max(pl, 1) * Q * Q * Q;
    s.Y.reserve(ny);
    OCTEN_CUDA(cudaMemcpyAsync(s.Y.p, Y.p, sizeof(double) * ny, cudaMemcpyDeviceToDevice, st));
    s.hist.reserve((size_t)P * Q * R);
    OCTEN_CUDA(cudaMemcpyAsync(s.hist.p, hist.p, sizeof(double) * P * Q * R, cudaMemcpyDeviceToDevice, st));
    s.A.reserve((size_t)I * R);
    OCTEN_CUDA(cudaMemcpyAsync(s.A.p, A.p, sizeof(double) * I * R, cudaMemcpyDeviceToDevice, st));
    s.B.reserve((size_t)J * R);
    OCTEN_CUDA(cudaMemcpyAsync(s.B.p, B.p, sizeof(double) * J * R, cudaMemcpyDeviceToDevice, st));
    s.C.reserve((size_t)capC * R);
    OCTEN_CUDA(cudaMemcpyAsync(s.C.p, C.p, sizeof(double) * capC * R, cudaMemcpyDeviceToDevice, st));
    s.lam.reserve(R);
    OCTEN_CUDA(cudaMemcpyAsync(s.lam.p, lam.p, sizeof(double) * R, cudaMemcpyDeviceToDevice, st));
    s.capC = capC;
    s.K = K;
    s.batches_seen = batches_seen;
    s.batches_drawn = batches_drawn;
    s.tgram = tgram;
    s.log_len = log.size();
    OCTEN_CUDA(cudaStreamSynchronize(st));
}

void Stream::restore(Snapshot& s) {
    Y.swap(s.Y);
    hist.swap(s.hist);
    A.swap(s.A);
    B.swap(s.B);
    C.swap(s.C);
    lam.swap(s.lam);
    capC = s.capC;
    K = s.K;
    batches_seen = s.batches_seen;
    batches_drawn = s.batches_drawn;
    tgram = s.tgram;
    log.resize(s.log_len);
}

void Stream::init(const void* data, int dtype, int location, int order, const std::int64_t* dims) {
    xmodels.reserve(models_count() * shard_world);
    xrows.reserve(rows_count() * shard_world);
    begin(cur, data, dtype, location, order, dims, xmodels.p, false);
    merge_phase(cur, xmodels.p, xrows.p);
    finish(cur, xrows.p);
}

void Stream::ingest(const void* data, int dtype, int location, int order, const std::int64_t* dims) {
    if (shard_world != 1) throw ConfigError("octen: a sharded stream ingests through begin/merge/finish");
    sync();
    xmodels.reserve(models_count());
    xrows.reserve(rows_count());
    begin(cur, data, dtype, location, order, dims, xmodels.p, false);
    merge_phase(cur, xmodels.p, xrows.p);
    finish(cur, xrows.p);
}

void Stream::sync() {
    // the pipelined ingest's batches in flight: the last batch's sweeps and
    // the merge before them, then the last batch's merge
    std::exception_ptr a_err = aworker.wait();
    BatchCtx* pa = a_prev;
    a_prev = nullptr;
    std::exception_ptr m_err = worker.wait();
    m_prev = nullptr;
    if (m_err) {
        // the earlier batch failed in its merge: the reference stops there
        if (pa) {
            rollback_to(*pa);
            Y.swap(Yhold);
            pa->pending = false;
        }
        std::rethrow_exception(m_err);
    }
    if (a_err) std::rethrow_exception(a_err);
    if (pa) {
        pa->Yb = Y.p;
        post_merge(*pa, pa->models);
        std::exception_ptr e = worker.wait();
        if (e) std::rethrow_exception(e);
    }
}

void Stream::post_merge(BatchCtx& b, double* models) {
    xrows.reserve(rows_count());
    worker.post(cfg.device, [this, &b, models] {
        merge_phase(b, models, xrows.p);
        finish(b, xrows.p);
    });
}

void Stream::rollback_to(const BatchCtx& b) {
    batches_drawn = b.rb_drawn;
    batches_seen = b.rb_seen;
    tgram = b.rb_tgram;
}

namespace {
// OCTEN_MERGE_SMS=k (experiment): the pipelined merge runs on a green-context
// stream confined to k SMs, so its latency-bound factorizations cannot
// occupy the SMs the next batch's compression and CP-ALS need.  Driver
// entry points resolved at run time (libcuda is already loaded by the
// runtime).  Returns null when unavailable.
cudaStream_t green_merge_stream(int device, int sms, int priority) {
    void* h = dlopen("libcuda.so.1", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libcuda.so.1", RTLD_NOW);
    if (!h) return nullptr;
    auto devget = reinterpret_cast<CUresult (*)(CUdevice*, int)>(dlsym(h, "cuDeviceGet"));
    auto getres = reinterpret_cast<CUresult (*)(CUdevice, CUdevResource*, CUdevResourceType)>(
        dlsym(h, "cuDeviceGetDevResource"));
    auto split = reinterpret_cast<CUresult (*)(CUdevResource*, unsigned*, const CUdevResource*, CUdevResource*,
                                               unsigned, unsigned)>(dlsym(h, "cuDevSmResourceSplitByCount"));
    auto gen = reinterpret_cast<CUresult (*)(CUdevResourceDesc*, CUdevResource*, unsigned)>(
        dlsym(h, "cuDevResourceGenerateDesc"));
    auto create = reinterpret_cast<CUresult (*)(CUgreenCtx*, CUdevResourceDesc, CUdevice, unsigned)>(
        dlsym(h, "cuGreenCtxCreate"));
    auto screate = reinterpret_cast<CUresult (*)(CUstream*, CUgreenCtx, unsigned, int)>(
        dlsym(h, "cuGreenCtxStreamCreate"));
    if (!devget || !getres || !split || !gen || !create || !screate) return nullptr;
    CUdevice dev;
    CUdevResource all, part, rest;
    unsigned groups = 1;
    CUdevResourceDesc desc;
    CUgreenCtx g;
    CUstream s;
    if (devget(&dev, device) != CUDA_SUCCESS || getres(dev, &all, CU_DEV_RESOURCE_TYPE_SM) != CUDA_SUCCESS ||
        split(&part, &groups, &all, &rest, 0, (unsigned)sms) != CUDA_SUCCESS || groups < 1 ||
        gen(&desc, &part, 1) != CUDA_SUCCESS || create(&g, desc, dev, CU_GREEN_CTX_DEFAULT_STREAM) != CUDA_SUCCESS ||
        screate(&s, g, CU_STREAM_NON_BLOCKING, priority) != CUDA_SUCCESS)
        return nullptr;
    return reinterpret_cast<cudaStream_t>(s);
}
}  // namespace

void Stream::ingest_async(const void* data, int dtype, int location, int order, const std::int64_t* dims) {
    if (shard_world != 1) throw ConfigError("octen: a sharded stream ingests through begin/merge/finish");
    if (!initialized || cfg.strict) {
        ingest(data, dtype, location, order, dims);
        return;
    }
    if (!mst) {
        int least = 0, greatest = 0;
        OCTEN_CUDA(cudaDeviceGetStreamPriorityRange(&least, &greatest));
        // the merge has slack (it is shorter than compression + CP-ALS): the
        // main stream's kernels go first when both are ready
        static const int merge_sms = [] {
            const char* e = std::getenv("OCTEN_MERGE_SMS");
            return e ? std::atoi(e) : 0;
        }();
        if (merge_sms > 0) mst = green_merge_stream(cfg.device, merge_sms, least);
        if (!mst) OCTEN_CUDA(cudaStreamCreateWithPriority(&mst, cudaStreamNonBlocking, least));
    }
    if (!ast) OCTEN_CUDA(cudaStreamCreateWithPriority(&ast, cudaStreamNonBlocking, critical_stream_priority()));
    // Two batches in flight: the previous batch's sweeps (CP-ALS worker) and
    // the merge before them (merge worker) run while this batch is
    // compressed and its CP-ALS start (GEVD attempts) runs on the other
    // engine; then this batch's sweeps and the previous batch's merge are
    // posted.  Errors of batch b surface in the call of batch b+1 (CP-ALS) or
    // b+2 (merge), with the later batches rolled back.
    BatchCtx& bc = actx[aslot];
    bc.st = mst;
    // models per context slot: batch b-1's merge may still read its models
    // while batch b+1's sweeps (same engine) write theirs
    DevBuf<double>& mbuf = aslot == 0 ? xmodels : aslot == 1 ? xmodels2 : xmodels3;
    double* models = mbuf.reserve(models_count());
    AlsEngine& eng = apar ? als_b : als;
    bc.rb_drawn = batches_drawn;
    bc.rb_seen = batches_seen;
    bc.rb_tgram = tgram;
    std::exception_ptr begin_err;
    // GEMM1 on half the SMs while the previous batch's sweeps run beside it:
    // its persistent CTAs would otherwise hold every SM for ~1.2 ms and
    // stall the sweeps, the pipeline's critical chain.  Measured at c3 (ms
    // per step, grid 148 / 128 / 100 / 74 / 48 / 32 CTAs): 11.70 / 11.64 /
    // 11.60 / 11.55 / 11.67 / 11.95.  OCTEN_G1_SMS overrides (0: every SM).
    static const int g1_env = [] {
        const char* e = std::getenv("OCTEN_G1_SMS");
        return e ? std::atoi(e) : -1;
    }();
    if (a_prev) {
        int nsm = 0;
        OCTEN_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, cfg.device));
        comp.g1_ctas = g1_env >= 0 ? g1_env : nsm / 2;
    }
    try {
        begin(bc, data, dtype, location, order, dims, models, true, false);
        try {
            als_init_phase(bc, Ynext.p, eng, st);
        } catch (...) {
            bc.init_failed = true;
            fail_pending(bc);
        }
    } catch (...) {
        begin_err = std::current_exception();
    }
    comp.g1_ctas = 0;
    // the previous batch's sweeps, then the merge posted before them
    std::exception_ptr a_err = aworker.wait();
    BatchCtx* pa = a_prev;
    a_prev = nullptr;
    // This batch's sweeps are the pipeline's critical chain: when nothing
    // has failed so far they are posted before waiting for the merge posted
    // before them (which may still run; waiting for it first put its tail,
    // ~1.2 ms at c3, between two batches' sweeps).  If that merge fails,
    // the sweeps are drained and discarded with the rollback.
    bc.models = models;
    AlsEngine* e = &eng;
    const bool early = !a_err && !begin_err;
    if (early) {
        aworker.post(cfg.device, [this, &bc, e, models] {
            try {
                als_sweep_phase(bc, models, *e, ast, 2);
            } catch (...) {
                fail_pending(bc);
            }
        });
        a_prev = &bc;
    }
    std::exception_ptr m_err = worker.wait();
    m_prev = nullptr;
    if (m_err) {
        if (early) {
            (void)aworker.wait();  // this batch is rolled back: its sweeps' outcome is moot
            a_prev = nullptr;
        }
        // the batch before pa failed in its merge (the reference throws from
        // its ingest_batch): pa and this batch were never ingested; the
        // summaries are the failed batch's (Yhold)
        if (pa) {
            rollback_to(*pa);
            Y.swap(Yhold);
            pa->pending = false;
        } else {
            rollback_to(bc);
        }
        bc.pending = false;
        std::rethrow_exception(m_err);
    }
    if (a_err) {
        // pa failed in its CP-ALS: its summaries stay (as the reference's);
        // this batch was never ingested
        rollback_to(bc);
        bc.pending = false;
        std::rethrow_exception(a_err);
    }
    // the previous batch's merge (its models and summaries are final)
    if (pa) {
        pa->Yb = Y.p;
        post_merge(*pa, pa->models);
        m_prev = pa;
    }
    if (begin_err) {
        // this batch's compression or CP-ALS start failed: the earlier
        // batch's merge completes first (its error comes first)
        std::exception_ptr e2 = worker.wait();
        m_prev = nullptr;
        if (e2) {
            rollback_to(bc);
            bc.pending = false;
            std::rethrow_exception(e2);
        }
        if (bc.init_failed) Y.swap(Ynext);  // a CP-ALS failure keeps the updated summaries
        std::rethrow_exception(begin_err);
    }
    // summaries: Yhold <- the previous batch's (its merge reads them), Y <-
    // this batch's, Ynext <- the buffer the merge before released
    Yhold.swap(Y);
    Y.swap(Ynext);
    aslot = (aslot + 1) % 3;
    apar ^= 1;
}

namespace {
// fitness support (eval.cpp:10-20 without materialising the reconstruction)
template <typename T>
struct FitXA {  // A(0, i, n) = X[i + I n]   (X_(1), n = j + J k)
    const T* X;
    long long I;
    __device__ double operator()(int, int i, int n) const { return (double)X[(size_t)i + (size_t)I * n]; }
};
struct FitKrB {  // B(0, n, r) = B(j, r) C(k0 + k, r),  n = j + J k
    const double* B;
    const double* C;
    long long J, ldc, k0;
    __device__ double operator()(int, int n, int r) const {
        const long long k = n / J, j = n - k * J;
        return B[j + J * r] * C[(k0 + k) + ldc * r];
    }
};
struct FitWC {  // W(i, r)
    double* W;
    long long I;
    __device__ void operator()(int, int i, int r, double v) const { W[(size_t)i + (size_t)I * r] = v; }
};
template <typename T>
__global__ void sumsq_kernel(const T* __restrict__ x, size_t n, double* out) {
    double acc = 0.0;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        const double v = (double)x[i];
        acc += v * v;
    }
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    __shared__ double part[32];
    if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double sacc = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) sacc += part[w];
        out[blockIdx.x] = sacc;  // per-block partials, summed in block order on the host
    }
}
}  // namespace

// Fitness of the current model on t slices X (I x J x t, first index fastest)
// that are the model's temporal rows [k0, k0 + t): eval.cpp:10-20,
//   100 (1 - |X - Xhat| / |X|),  |X - Xhat|^2 = |X|^2 - 2 <X, Xhat> + |Xhat|^2,
// with <X, Xhat> = sum_r lambda_r a_r^T X_(1) (c_r (x) b_r) as one GEMM
// (X_(1) against the Khatri-Rao rows, formed on the fly) and |Xhat|^2 from
// the R x R Grams.  The reconstruction is never materialised.
double Stream::batch_fitness(const void* data, int dtype, int location, int order, const std::int64_t* dims,
                             std::int64_t k0) {
    if (!initialized) throw ConfigError("octen: stream is not initialised");
    const int tm = cfg.temporal_mode;
    if (order != 3 || dims[tm == 0 ? 1 : 0] != I || dims[tm == 2 ? 1 : 2] != J)
        throw ConfigError("fitness: extent mismatch");
    const std::int64_t t = dims[tm];
    if (t < 1 || k0 < 0 || k0 + t > K) throw ConfigError("fitness: slice range outside the model");
    const int R = cfg.rank;
    const size_t n = (size_t)I * J * t;
    const void* dX = tm == 2 ? stage_input(data, dtype, location, n) : temporal_last(data, dtype, location, dims);
    check_finite(dX, dtype, n);  // the reference builds a DenseTensor from the batch first
    const int nb = (int)std::min<size_t>(148 * 4, (n + 255) / 256);
    DevBuf<double> part, W;
    part.reserve((size_t)nb);
    W.reserve((size_t)I * R);
    const long long Jt = (long long)J * t;
    const int ks = pick_ksplit(1, (int)I, R, (int)std::min<long long>(Jt, 1 << 30));
    DevBuf<double> wsp;
    if (ks > 1) wsp.reserve((size_t)ks * I * R);
    if (dtype == 1) {
        sumsq_kernel<float><<<nb, 256, 0, st>>>((const float*)dX, n, part.p);
        gemm_f64<false, false>(1, (int)I, R, (int)Jt, FitXA<float>{(const float*)dX, I},
                               FitKrB{B.p, C.p, J, capC, k0}, FitWC{W.p, I}, st, ks, ks > 1 ? wsp.p : nullptr);
    } else {
        sumsq_kernel<double><<<nb, 256, 0, st>>>((const double*)dX, n, part.p);
        gemm_f64<false, false>(1, (int)I, R, (int)Jt, FitXA<double>{(const double*)dX, I},
                               FitKrB{B.p, C.p, J, capC, k0}, FitWC{W.p, I}, st, ks, ks > 1 ? wsp.p : nullptr);
    }
    OCTEN_LAUNCHED(1);
    OCTEN_CUDA(cudaGetLastError());
    std::vector<double> hp = part.to_host((size_t)nb, st);
    std::vector<double> hW = W.to_host((size_t)I * R, st);
    std::vector<double> hA = A.to_host((size_t)I * R, st), hB = B.to_host((size_t)J * R, st);
    std::vector<double> hC((size_t)t * R), hl = lam.to_host((size_t)R, st);
    OCTEN_CUDA(cudaMemcpy2DAsync(hC.data(), t * sizeof(double), C.p + k0, capC * sizeof(double), t * sizeof(double), R,
                                 cudaMemcpyDeviceToHost, st));
    OCTEN_CUDA(cudaStreamSynchronize(st));
    double nx2 = 0.0;
    for (double v : hp) nx2 += v;
    double inner = 0.0;
    for (int r = 0; r < R; ++r) {
        double sacc = 0.0;
        for (std::int64_t i = 0; i < I; ++i) sacc += hA[(size_t)i + (size_t)I * r] * hW[(size_t)i + (size_t)I * r];
        inner += hl[(size_t)r] * sacc;
    }
    auto gram = [&](const std::vector<double>& f, std::int64_t rows, int a, int b) {
        double g = 0.0;
        for (std::int64_t i = 0; i < rows; ++i) g += f[(size_t)i + (size_t)rows * a] * f[(size_t)i + (size_t)rows * b];
        return g;
    };
    double nh2 = 0.0;
    for (int a = 0; a < R; ++a)
        for (int b = 0; b < R; ++b)
            nh2 += hl[(size_t)a] * hl[(size_t)b] * gram(hA, I, a, b) * gram(hB, J, a, b) * gram(hC, t, a, b);
    if (!(nx2 > 0.0)) throw NumericError("fitness: zero-norm reference tensor");  // eval.cpp:13
    const double res2 = std::max(0.0, nx2 - 2.0 * inner + nh2);
    return 100.0 * (1.0 - std::sqrt(res2) / std::sqrt(nx2));
}

void Stream::get_factor(int mode, double* out) {
    const int R = cfg.rank;
    if (mode < 0 || mode > 2) throw ConfigError("octen_stream_get_factor: mode out of range");
    mode = factor_slot(mode);
    if (mode == 0)
        OCTEN_CUDA(cudaMemcpyAsync(out, A.p, sizeof(double) * I * R, cudaMemcpyDeviceToHost, st));
    else if (mode == 1)
        OCTEN_CUDA(cudaMemcpyAsync(out, B.p, sizeof(double) * J * R, cudaMemcpyDeviceToHost, st));
    else if (mode == 2)
        OCTEN_CUDA(cudaMemcpy2DAsync(out, K * sizeof(double), C.p, capC * sizeof(double), K * sizeof(double), R,
                                     cudaMemcpyDeviceToHost, st));
    else
        throw ConfigError("octen_stream_get_factor: mode out of range");
    OCTEN_CUDA(cudaStreamSynchronize(st));
}

}  // namespace octen
