// C-ABI (include/octen_b200.h): exceptions -> status codes + thread-local
// message carrying the reference's error text.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "../../include/octen_b200.h"
#include "engine.hpp"
#include "errors.hpp"
#include "stream.hpp"
#include "synth.hpp"

struct octen_stream {
    std::unique_ptr<octen::Stream> s;
};

struct octen_synth {
    std::unique_ptr<octen::SynthStream> g;
};

struct octen_coo_summaries {
    int device = 0;
    cudaStream_t st = nullptr;
    cudaEvent_t ev[2] = {};
    octen::CooEngine eng;
    octen::AlsEngine als;
    octen::DevBuf<double> Y, W;
    octen::DevBuf<int> hi, hj, hk;
    octen::DevBuf<float> hv;
    double als_ms = 0;
    long long als_runs = 0;
    ~octen_coo_summaries() {
        if (st) cudaStreamSynchronize(st);
        for (auto e : ev)
            if (e) cudaEventDestroy(e);
        if (st) cudaStreamDestroy(st);
    }
};

namespace {

thread_local std::string g_err;

template <class F>
int guard(F&& f) {
    g_err.clear();
    try {
        f();
        return OCTEN_OK;
    } catch (const octen::ConfigError& e) {
        g_err = e.what();
        return OCTEN_ERR_CONFIG;
    } catch (const octen::NumericError& e) {
        g_err = e.what();
        return OCTEN_ERR_NUMERIC;
    } catch (const octen::IoError& e) {
        g_err = e.what();
        return OCTEN_ERR_IO;
    } catch (const octen::CudaError& e) {
        g_err = e.what();
        return OCTEN_ERR_CUDA;
    } catch (const std::exception& e) {
        g_err = e.what();
        return OCTEN_ERR_INTERNAL;
    } catch (...) {
        g_err = "unknown error";
        return OCTEN_ERR_INTERNAL;
    }
}

// Every stream entry point runs on the handle's device and restores the
// caller's current device afterwards.
struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        int cur = 0;
        OCTEN_CUDA(cudaGetDevice(&cur));
        if (cur != dev) {
            OCTEN_CUDA(cudaSetDevice(dev));
            prev = cur;
        }
    }
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

template <class F>
int sguard(const octen_stream* s, F&& f) {
    return guard([&] {
        if (!s || !s->s) throw octen::ConfigError("octen: null stream handle");
        DeviceGuard dg(s->s->cfg.device);
        f();
    });
}

octen::StreamCfg to_cfg(const octen_stream_config* c) {
    octen::StreamCfg s;
    s.rank = c->rank;
    s.p = c->p;
    s.q = c->q;
    s.shared = c->shared;
    s.temporal_mode = c->temporal_mode;
    s.als_max_iters = c->als.max_iters;
    s.als_n_restarts = c->als.n_restarts;
    s.als_rel_tol = c->als.rel_tol;
    s.als_seed = c->als.seed;
    s.seed = c->seed;
    s.enforce_bounds = c->enforce_bounds != 0;
    s.strict = c->strict != 0;
    s.workers = c->workers;
    s.residual_warning = c->residual_warning;
    s.device = c->device;
    return s;
}

void check_dtype(int dtype, int location) {
    if (dtype != OCTEN_F64 && dtype != OCTEN_F32) throw octen::ConfigError("octen: unknown dtype");
    if (location != OCTEN_HOST && location != OCTEN_DEVICE) throw octen::ConfigError("octen: unknown location");
}

// history: stacked (pQ x R) <-> per replica (p x Q x R)
void hist_to_blocks(const std::vector<double>& stk, int P, int Q, int R, double* out) {
    const size_t PQ = (size_t)P * Q;
    for (int p = 0; p < P; ++p)
        for (int r = 0; r < R; ++r)
            for (int a = 0; a < Q; ++a) out[(size_t)p * Q * R + a + (size_t)Q * r] = stk[(size_t)p * Q + a + PQ * r];
}
std::vector<double> blocks_to_hist(const double* in, int P, int Q, int R) {
    const size_t PQ = (size_t)P * Q;
    std::vector<double> stk(PQ * R);
    for (int p = 0; p < P; ++p)
        for (int r = 0; r < R; ++r)
            for (int a = 0; a < Q; ++a) stk[(size_t)p * Q + a + PQ * r] = in[(size_t)p * Q * R + a + (size_t)Q * r];
    return stk;
}

struct ScopedStream {
    cudaStream_t st = nullptr;
    ScopedStream() { OCTEN_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking)); }
    ~ScopedStream() {
        // drain before the stream's temporaries return to the block cache
        // (matters on error paths, where the body did not synchronize)
        if (st) {
            cudaStreamSynchronize(st);
            cudaStreamDestroy(st);
        }
    }
};

}  // namespace

extern "C" {

const char* octen_last_error(void) { return g_err.c_str(); }

const char* octen_version(void) { return "octen_b200 0.1 (sm_100a)"; }

int64_t octen_launch_count(void) { return (int64_t)octen::launch_counter().load(); }

void octen_kernel_counts(int64_t* out) {
    out[0] = (int64_t)octen::launch_counter().load();
    for (int i = 0; i < octen::kNumPathCounters; ++i) out[1 + i] = (int64_t)octen::path_counter(i).load();
}

int octen_stream_get_stage_times(const octen_stream* s, double* out) {
    return sguard(s, [&] {
        s->s->sync();
        const auto& x = *s->s;
        for (int i = 0; i < 4; ++i) out[i] = x.dev_ms[i];
        out[4] = x.gemm1_flops;
        out[5] = (double)x.gemm1_launches;
    });
}

int octen_stream_init(const octen_stream_config* cfg, const void* data, int dtype, int location, int order,
                      const int64_t* dims, octen_stream** out) {
    return guard([&] {
        if (!cfg || !data || !dims || !out) throw octen::ConfigError("octen_stream_init: null argument");
        check_dtype(dtype, location);
        DeviceGuard dg(cfg->device);
        auto h = std::make_unique<octen_stream>();
        h->s = std::make_unique<octen::Stream>(to_cfg(cfg));
        h->s->init(data, dtype, location, order, dims);
        *out = h.release();
    });
}

int octen_stream_ingest(octen_stream* s, const void* data, int dtype, int location, int order,
                        const int64_t* dims) {
    return sguard(s, [&] {
        if (!s || !data || !dims) throw octen::ConfigError("octen_stream_ingest: null argument");
        check_dtype(dtype, location);
        s->s->ingest(data, dtype, location, order, dims);
    });
}

int octen_stream_ingest_async(octen_stream* s, const void* data, int dtype, int location, int order,
                              const int64_t* dims) {
    return sguard(s, [&] {
        if (!data || !dims) throw octen::ConfigError("octen_stream_ingest_async: null argument");
        check_dtype(dtype, location);
        s->s->ingest_async(data, dtype, location, order, dims);
    });
}

int octen_stream_sync(octen_stream* s) {
    return sguard(s, [&] { s->s->sync(); });
}

int octen_stream_set_publish(octen_stream* s, int on) {
    return sguard(s, [&] {
        s->s->sync();
        s->s->publish = on != 0;
    });
}

int octen_stream_last_model(octen_stream* s, int64_t* info, double* a, double* b, double* c, int64_t c_rows_cap,
                            double* lambda) {
    return sguard(s, [&] {
        auto& x = *s->s;
        std::lock_guard<std::mutex> lk(x.pub_mu);
        info[0] = x.pub_K;
        info[1] = x.pub_batches;
        if (x.pub_batches == 0) return;
        if (!a || !b || !c || !lambda) throw octen::ConfigError("octen_stream_last_model: null argument");
        if (c_rows_cap < x.pub_K) throw octen::ConfigError("octen_stream_last_model: c buffer too small");
        const int R = x.cfg.rank;
        std::memcpy(a, x.pubA.data(), x.pubA.size() * sizeof(double));
        std::memcpy(b, x.pubB.data(), x.pubB.size() * sizeof(double));
        for (int r = 0; r < R; ++r)
            std::memcpy(c + (size_t)c_rows_cap * r, x.pubC.data() + (size_t)x.pub_K * r, x.pub_K * sizeof(double));
        std::memcpy(lambda, x.pubLam.data(), R * sizeof(double));
    });
}

int octen_synth_create(int order, const int64_t* dims, int rank, uint64_t seed, double noise_mu,
                       double noise_sigma, int device, octen_synth** out) {
    return guard([&] {
        if (!dims || !out || order < 0) throw octen::ConfigError("octen_synth_create: null argument");
        DeviceGuard dg(device);
        auto h = std::make_unique<octen_synth>();
        h->g = std::make_unique<octen::SynthStream>(std::vector<std::int64_t>(dims, dims + order), rank, seed,
                                                    noise_mu, noise_sigma, device);
        *out = h.release();
    });
}

int octen_synth_next(octen_synth* h, int64_t t, void* out_device, int dtype) {
    return guard([&] {
        if (!h || !out_device) throw octen::ConfigError("octen_synth_next: null argument");
        if (dtype != OCTEN_F64 && dtype != OCTEN_F32) throw octen::ConfigError("octen: unknown dtype");
        DeviceGuard dg(h->g->device);
        h->g->next(t, out_device, dtype);
    });
}

int octen_synth_truth(const octen_synth* h, double* const* factors, double* lambda) {
    return guard([&] {
        if (!h || !factors || !lambda) throw octen::ConfigError("octen_synth_truth: null argument");
        h->g->truth(factors, lambda);
    });
}

void octen_synth_destroy(octen_synth* h) {
    if (!h) return;
    int cur = 0;
    cudaGetDevice(&cur);
    if (h->g) cudaSetDevice(h->g->device);
    delete h;
    cudaSetDevice(cur);
}

int octen_stream_checkpoint_save(octen_stream* s, uint8_t* buf, int64_t cap, int64_t* size) {
    return sguard(s, [&] {
        if (!size) throw octen::ConfigError("octen_stream_checkpoint_save: null argument");
        std::vector<std::uint8_t> b = s->s->checkpoint_save();
        *size = (int64_t)b.size();
        if (buf) {
            if (cap < (int64_t)b.size()) throw octen::ConfigError("octen_stream_checkpoint_save: buffer too small");
            std::memcpy(buf, b.data(), b.size());
        }
    });
}

int octen_stream_checkpoint_load(const uint8_t* bytes, int64_t n, int device, octen_stream** out) {
    return guard([&] {
        if (!bytes || !out || n < 0) throw octen::ConfigError("octen_stream_checkpoint_load: null argument");
        DeviceGuard dg(device);
        auto h = std::make_unique<octen_stream>();
        h->s = octen::Stream::checkpoint_load(bytes, (size_t)n, device);
        *out = h.release();
    });
}

int octen_congruence(int order, int rank, const int64_t* dims, const double* ground, const double* est,
                     double* scores) {
    // eval.cpp:22-46: per-component product over modes of |cos| between the
    // normalised columns, matched exhaustively (rank <= 6) or greedily
    // (recovery.cpp:42-104).  Host-side evaluation (no device work).
    return guard([&] {
        if (order < 1 || rank < 1 || !dims || !ground || !est || !scores)
            throw octen::ConfigError("congruence: bad arguments");
        const int r = rank;
        std::vector<double> sim((size_t)r * r, 1.0);
        size_t off = 0;
        for (int n = 0; n < order; ++n) {
            const int64_t d = dims[n];
            const double* g = ground + off;
            const double* e = est + off;
            off += (size_t)d * r;
            std::vector<double> gn(r, 0.0), en(r, 0.0);
            for (int c = 0; c < r; ++c) {
                for (int64_t i = 0; i < d; ++i) {
                    gn[c] += g[i + d * c] * g[i + d * c];
                    en[c] += e[i + d * c] * e[i + d * c];
                }
                gn[c] = std::sqrt(gn[c]);
                en[c] = std::sqrt(en[c]);
            }
            for (int a = 0; a < r; ++a)
                for (int b = 0; b < r; ++b) {
                    double sacc = 0.0;
                    for (int64_t i = 0; i < d; ++i)
                        sacc += (gn[a] > 0.0 ? g[i + d * a] / gn[a] : g[i + d * a]) *
                                (en[b] > 0.0 ? e[i + d * b] / en[b] : e[i + d * b]);
                    sim[(size_t)a + (size_t)r * b] *= std::fabs(sacc);
                }
        }
        std::vector<int> perm(r);
        for (int i = 0; i < r; ++i) perm[i] = i;  // exhaustive_match starts from the identity
        if (r <= 6) {
            std::vector<int> cand(r);
            for (int i = 0; i < r; ++i) cand[i] = i;
            double best = -INFINITY;
            do {
                double tot = 0.0;
                for (int i = 0; i < r; ++i) tot += sim[(size_t)i + (size_t)r * cand[i]];
                if (tot > best) {
                    best = tot;
                    perm = cand;
                }
            } while (std::next_permutation(cand.begin(), cand.end()));
        } else {
            std::vector<unsigned char> ua(r), ub(r);
            octen::greedy_match(r, sim.data(), r, 1e-9, perm.data(), ua.data(), ub.data());
        }
        for (int i = 0; i < r; ++i) scores[i] = sim[(size_t)i + (size_t)r * perm[i]];
    });
}

int octen_stream_batch_fitness(octen_stream* s, const void* data, int dtype, int location, int order,
                               const int64_t* dims, int64_t k0, double* fitness) {
    return sguard(s, [&] {
        s->s->sync();
        if (!s || !data || !dims || !fitness) throw octen::ConfigError("octen_stream_batch_fitness: null argument");
        check_dtype(dtype, location);
        *fitness = s->s->batch_fitness(data, dtype, location, order, dims, k0);
    });
}

int octen_stream_partial_block_size(const octen_stream* s, int64_t* n) {
    return sguard(s, [&] {
        if (!s || !n) throw octen::ConfigError("octen_stream_partial_block_size: null argument");
        *n = (int64_t)s->s->partial_block_count();
    });
}

int octen_stream_begin_temporal(octen_stream* s, const void* data, int dtype, int location, int order,
                                const int64_t* dims_local, int64_t k_off, int64_t t_total, double* partial_out) {
    return sguard(s, [&] {
        s->s->sync();
        if (!s || !dims_local || !partial_out || (!data && dims_local[2] > 0))
            throw octen::ConfigError("octen_stream_begin_temporal: null argument");
        check_dtype(dtype, location);
        s->s->begin_temporal(data, dtype, location, order, dims_local, k_off, t_total, partial_out);
    });
}

int octen_stream_begin_reduced(octen_stream* s, const double* owned_block, double* models_out) {
    return sguard(s, [&] {
        if (!s || !owned_block || !models_out) throw octen::ConfigError("octen_stream_begin_reduced: null argument");
        s->s->begin_reduced(owned_block, models_out);
    });
}

int octen_stream_prefetch(octen_stream* s, const void* data, int dtype, int order, const int64_t* dims) {
    return sguard(s, [&] {
        // no sync: the prefetch touches only the main thread's staging state
        if (!s || !data || !dims) throw octen::ConfigError("octen_stream_prefetch: null argument");
        check_dtype(dtype, OCTEN_HOST);
        s->s->prefetch(data, dtype, order, dims);
    });
}

void octen_stream_destroy(octen_stream* s) {
    if (!s) return;
    int cur = 0;
    cudaGetDevice(&cur);
    if (s->s) cudaSetDevice(s->s->cfg.device);
    delete s;
    cudaSetDevice(cur);
}

int octen_stream_create(const octen_stream_config* cfg, int shard_rank, int shard_world, octen_stream** out) {
    return guard([&] {
        if (!cfg || !out) throw octen::ConfigError("octen_stream_create: null argument");
        DeviceGuard dg(cfg->device);
        auto h = std::make_unique<octen_stream>();
        h->s = std::make_unique<octen::Stream>(to_cfg(cfg), shard_rank, shard_world);
        *out = h.release();
    });
}

int octen_nccl_get_unique_id(uint8_t* out128) {
    return guard([&] {
        if (!out128) throw octen::ConfigError("octen_nccl_get_unique_id: null argument");
        octen::nccl_unique_id(out128);
    });
}

int octen_stream_create_nccl(const octen_stream_config* cfg, int shard_rank, int shard_world, const uint8_t* uid128,
                             void* nccl_comm, octen_stream** out) {
    return guard([&] {
        if (!cfg || !out || (!uid128 && !nccl_comm))
            throw octen::ConfigError("octen_stream_create_nccl: null argument");
        DeviceGuard dg(cfg->device);
        auto h = std::make_unique<octen_stream>();
        h->s = std::make_unique<octen::Stream>(to_cfg(cfg), shard_rank, shard_world);
        h->s->attach_nccl(uid128, nccl_comm);
        *out = h.release();
    });
}

int octen_stream_ingest_sharded(octen_stream* s, const void* data, int dtype, int location, int order,
                                const int64_t* dims) {
    return sguard(s, [&] {
        if (!data || !dims) throw octen::ConfigError("octen_stream_ingest_sharded: null argument");
        check_dtype(dtype, location);
        s->s->ingest_sharded(data, dtype, location, order, dims);
    });
}

int octen_stream_ingest_temporal(octen_stream* s, const void* data, int dtype, int location, int order,
                                 const int64_t* dims_local, int64_t k_off, int64_t t_total) {
    return sguard(s, [&] {
        if (!dims_local || (!data && dims_local[2] > 0))
            throw octen::ConfigError("octen_stream_ingest_temporal: null argument");
        check_dtype(dtype, location);
        s->s->ingest_temporal_nccl(data, dtype, location, order, dims_local, k_off, t_total);
    });
}

int octen_stream_exchange_sizes(const octen_stream* s, int64_t* sizes) {
    return sguard(s, [&] {
        if (!s || !sizes) throw octen::ConfigError("octen_stream_exchange_sizes: null argument");
        const auto& x = *s->s;
        sizes[0] = (int64_t)x.models_count();
        sizes[1] = (int64_t)x.rows_count();
        sizes[2] = x.p0;
        sizes[3] = x.pl;
        sizes[4] = x.shard_rank;
        sizes[5] = x.shard_world;
    });
}

int octen_stream_begin(octen_stream* s, const void* data, int dtype, int location, int order, const int64_t* dims,
                       double* models_out) {
    return sguard(s, [&] {
        s->s->sync();
        if (!s || !data || !dims || !models_out) throw octen::ConfigError("octen_stream_begin: null argument");
        check_dtype(dtype, location);
        s->s->begin(data, dtype, location, order, dims, models_out);
    });
}

int octen_stream_merge(octen_stream* s, const double* models_all, double* rows_out) {
    return sguard(s, [&] {
        if (!s || !models_all || !rows_out) throw octen::ConfigError("octen_stream_merge: null argument");
        s->s->merge_phase(models_all, rows_out);
    });
}

int octen_stream_finish(octen_stream* s, const double* rows_all) {
    return sguard(s, [&] {
        if (!s || !rows_all) throw octen::ConfigError("octen_stream_finish: null argument");
        s->s->finish(rows_all);
    });
}

int octen_stream_info(const octen_stream* s, int64_t* info) {
    return sguard(s, [&] {
        s->s->sync();
        const auto& x = *s->s;
        info[0] = 3;
        // extents in the stream's mode order (the temporal mode holds K)
        const int64_t ext[3] = {x.I, x.J, x.K};
        for (int n = 0; n < 3; ++n) info[1 + n] = x.initialized ? ext[x.factor_slot(n)] : 0;
        info[4] = x.cfg.rank;
        info[5] = x.cfg.p;
        info[6] = x.cfg.q;
        info[7] = x.batches_seen;
    });
}

int octen_stream_footprint(const octen_stream* s, int64_t* out) {
    // measure_footprint (eval.cpp:48-60) of the device-resident state: 8 bytes
    // per double held for the stream's logical state (U_p/V_p projections,
    // owned summaries, model, history accumulators); the temporal window is
    // empty between batches, as in the reference.
    return sguard(s, [&] {
        s->s->sync();
        const auto& x = *s->s;
        const int64_t P = x.cfg.p, Q = x.cfg.q, R = x.cfg.rank;
        out[0] = 8 * P * Q * (x.I + x.J);
        out[1] = 8 * (int64_t)x.pl * Q * Q * Q;
        out[2] = 8 * ((x.I + x.J + x.K) * R + R);
        out[3] = 8 * P * Q * R;
    });
}

int octen_stream_get_factor(const octen_stream* s, int mode, double* out) {
    return sguard(s, [&] {
        s->s->sync();
        s->s->get_factor(mode, out);
    });
}

int octen_stream_get_model(const octen_stream* s, double* a, double* b, double* c, double* lambda) {
    return sguard(s, [&] {
        s->s->sync();
        auto& x = *s->s;
        const int R = x.cfg.rank;
        // a, b, c: the factors of modes 0, 1, 2 (the stream's mode order)
        double* out[3] = {a, b, c};
        double* slot_out[3] = {nullptr, nullptr, nullptr};
        for (int n = 0; n < 3; ++n) slot_out[x.factor_slot(n)] = out[n];
        OCTEN_CUDA(cudaMemcpyAsync(slot_out[0], x.A.p, sizeof(double) * x.I * R, cudaMemcpyDeviceToHost, x.st));
        OCTEN_CUDA(cudaMemcpyAsync(slot_out[1], x.B.p, sizeof(double) * x.J * R, cudaMemcpyDeviceToHost, x.st));
        OCTEN_CUDA(cudaMemcpy2DAsync(slot_out[2], x.K * sizeof(double), x.C.p, x.capC * sizeof(double),
                                     x.K * sizeof(double), R, cudaMemcpyDeviceToHost, x.st));
        x.lam.download(lambda, R, x.st);
        OCTEN_CUDA(cudaStreamSynchronize(x.st));
    });
}

int octen_stream_get_lambda(const octen_stream* s, double* out) {
    return sguard(s, [&] {
        s->s->sync();
        auto& x = *s->s;
        x.lam.download(out, x.cfg.rank, x.st);
        OCTEN_CUDA(cudaStreamSynchronize(x.st));
    });
}

int octen_stream_get_kernel_stats(const octen_stream* s, double* out) {
    return sguard(s, [&] {
        s->s->sync();
        const auto& k = s->s->als.kstats;
        out[0] = k.gemm_ms;
        out[1] = (double)k.gemm_launches;
        out[2] = k.gemm_flops;
        out[3] = k.mttkrp_ms;
        out[4] = (double)k.mttkrp_launches;
        out[5] = k.mttkrp_bytes;
        out[6] = (double)k.sweeps;
        out[7] = 0.0;
    });
}

int octen_stream_log_size(const octen_stream* s, int64_t* n) {
    return sguard(s, [&] {
        s->s->sync();
        *n = (int64_t)s->s->log.size();
    });
}

int octen_stream_get_record(const octen_stream* s, int64_t index, octen_batch_record* out) {
    return sguard(s, [&] {
        s->s->sync();
        const auto& x = *s->s;
        if (index < 0 || index >= (int64_t)x.log.size()) throw octen::ConfigError("octen_stream_get_record: index");
        const auto& r = x.log[(size_t)index];
        out->batch_index = r.batch_index;
        out->t_new = r.t_new;
        out->temporal_residual = r.temporal_residual;
        out->min_match_similarity = r.min_match_similarity;
        out->max_offdiag_similarity = r.max_offdiag_similarity;
        out->warned = r.warned;
        out->compress_seconds = r.compress_seconds;
        out->als_seconds = r.als_seconds;
        out->recover_seconds = r.recover_seconds;
        out->total_seconds = r.total_seconds;
    });
}

int octen_stream_get_summaries(const octen_stream* s, double* y) {
    return sguard(s, [&] {
        s->s->sync();
        auto& x = *s->s;
        const size_t n = (size_t)x.pl * x.cfg.q * x.cfg.q * x.cfg.q;
        x.Y.download(y, n, x.st);
        OCTEN_CUDA(cudaStreamSynchronize(x.st));
    });
}

int octen_stream_get_history(const octen_stream* s, double* h) {
    return sguard(s, [&] {
        s->s->sync();
        auto& x = *s->s;
        const int P = x.cfg.p, Q = x.cfg.q, R = x.cfg.rank;
        std::vector<double> stk = x.hist.to_host((size_t)P * Q * R, x.st);
        hist_to_blocks(stk, P, Q, R, h);
    });
}

int octen_stream_get_replica_models(const octen_stream* s, double* factors, double* lambda) {
    return sguard(s, [&] {
        s->s->sync();
        auto& x = *s->s;
        const int P = x.cfg.p, Q = x.cfg.q, R = x.cfg.rank;
        const size_t qr = (size_t)Q * R;
        std::vector<double> f = x.MfAll.to_host((size_t)P * 3 * qr, x.st);
        x.MlamAll.download(lambda, (size_t)P * R, x.st);
        OCTEN_CUDA(cudaStreamSynchronize(x.st));
        // the merge keeps them in slot order; return the stream's mode order
        for (int p = 0; p < P; ++p)
            for (int n = 0; n < 3; ++n)
                std::memcpy(factors + ((size_t)p * 3 + n) * qr, f.data() + ((size_t)p * 3 + x.factor_slot(n)) * qr,
                            qr * sizeof(double));
    });
}

int octen_compress(int p, int q, int shared, int64_t I, int64_t J, int64_t t, const double* u, const double* v,
                   const double* w, const void* x, int dtype, double* z) {
    return guard([&] {
        check_dtype(dtype, OCTEN_HOST);
        if (p < 1 || q < 1 || shared < 0 || shared > q || I < 1 || J < 1 || t < 1)
            throw octen::ConfigError("octen_compress: bad shape");
        ScopedStream ss;
        octen::CompressEngine e;
        e.set_projections(p, q, shared, I, J, u, v, ss.st);
        octen::DevBuf<double> dW, dY;
        dW.upload(w, (size_t)p * t * q, ss.st);
        const size_t q3 = (size_t)q * q * q;
        dY.reserve((size_t)p * q3);
        dY.zero((size_t)p * q3, ss.st);
        const size_t n = (size_t)I * J * t;
        if (dtype == OCTEN_F32) {
            octen::DevBuf<float> dX;
            dX.upload((const float*)x, n, ss.st);
            e.compress_f32(dX.p, t, dW.p, dY.p, ss.st);
            dY.download(z, (size_t)p * q3, ss.st);
            OCTEN_CUDA(cudaStreamSynchronize(ss.st));
        } else {
            octen::DevBuf<double> dX;
            dX.upload((const double*)x, n, ss.st);
            e.compress_f64(dX.p, t, dW.p, dY.p, ss.st);
            dY.download(z, (size_t)p * q3, ss.st);
            OCTEN_CUDA(cudaStreamSynchronize(ss.st));
        }
    });
}

int octen_cp_als_batched(int p, int q, const double* y, const octen_als_config* cfg, const uint64_t* seeds,
                         double* factors, double* lambda, double* fit, int32_t* iterations) {
    return guard([&] {
        ScopedStream ss;
        octen::DevBuf<double> dY;
        dY.upload(y, (size_t)p * q * q * q, ss.st);
        octen::AlsEngine als;
        std::vector<std::uint64_t> sd(seeds, seeds + p);
        als.run(p, cfg->n_restarts, q, cfg->rank, cfg->max_iters, cfg->rel_tol, dY.p, sd, ss.st);
        als.Mf.download(factors, (size_t)p * 3 * q * cfg->rank, ss.st);
        als.Mlam.download(lambda, (size_t)p * cfg->rank, ss.st);
        OCTEN_CUDA(cudaStreamSynchronize(ss.st));
        for (int r = 0; r < p; ++r) {
            if (fit) fit[r] = als.results[r].fit;
            if (iterations) iterations[r] = als.results[r].iterations;
        }
    });
}

int octen_als_tgemm(int p, int q, int s, int r, int mode, const double* y, const double* factors, double* t,
                    int engine) {
    return guard([&] {
        ScopedStream ss;
        const size_t q2 = (size_t)q * q;
        octen::DevBuf<double> dY, dF, dT;
        dY.upload(y, (size_t)p * q2 * q, ss.st);
        dF.upload(factors, (size_t)p * s * 3 * q * r, ss.st);
        dT.reserve((size_t)p * q2 * s * r);
        octen::als_tgemm(p, q, s, r, mode, dY.p, dF.p, dT.p, engine, ss.st);
        dT.download(t, (size_t)p * q2 * s * r, ss.st);
        OCTEN_CUDA(cudaStreamSynchronize(ss.st));
    });
}

int octen_align_replicas(int p, int q, int shared, int rank, int64_t I, int64_t J, const double* u,
                         const double* v, const double* tgram, const double* factors, const double* lambda,
                         double* stacks, int32_t* perms, double* scales, double* sims) {
    return guard([&] {
        ScopedStream ss;
        octen::MergeEngine m;
        m.set_projections(p, q, shared, rank, I, J, u, v, ss.st);
        octen::DevBuf<double> dF, dL;
        dF.upload(factors, (size_t)p * 3 * q * rank, ss.st);
        dL.upload(lambda, (size_t)p * rank, ss.st);
        std::vector<double> tg(tgram, tgram + (size_t)shared * shared);
        octen::AlignResultHost ar;
        m.align(dF.p, dL.p, tg, ss.st, &ar);
        m.stacks.download(stacks, (size_t)3 * p * q * rank, ss.st);
        OCTEN_CUDA(cudaStreamSynchronize(ss.st));
        for (size_t i = 0; i < ar.perms.size(); ++i) perms[i] = ar.perms[i];
        for (size_t i = 0; i < ar.scales.size(); ++i) scales[i] = ar.scales[i];
        sims[0] = ar.min_match;
        sims[1] = ar.max_offdiag;
    });
}

int octen_recover_nontemporal(int p, int q, int64_t d, int rank, int mode, const double* proj_blocks,
                              const double* stack, double* out) {
    return guard([&] {
        if (mode != 0 && mode != 1) throw octen::ConfigError("octen_recover_nontemporal: mode must be 0 or 1");
        ScopedStream ss;
        octen::MergeEngine m;
        // the other mode is a 1-row placeholder projection
        std::vector<double> other((size_t)p * q, 1.0);
        if (mode == 0)
            m.set_projections(p, q, 0, rank, d, 1, proj_blocks, other.data(), ss.st);
        else
            m.set_projections(p, q, 0, rank, 1, d, other.data(), proj_blocks, ss.st);
        octen::DevBuf<double> dS, dO;
        dS.upload(stack, (size_t)p * q * rank, ss.st);
        dO.reserve((size_t)d * rank);
        m.solve_nontemporal(mode, dS.p, dO.p, ss.st);
        dO.download(out, (size_t)d * rank, ss.st);
        OCTEN_CUDA(cudaStreamSynchronize(ss.st));
    });
}

int octen_temporal_stack_from_summaries(int p, int q, int rank, int64_t I, int64_t J, const double* y,
                                        const double* u, const double* v, const double* a, const double* b,
                                        double* out) {
    return guard([&] {
        ScopedStream ss;
        octen::MergeEngine m;
        m.set_projections(p, q, 0, rank, I, J, u, v, ss.st);
        octen::DevBuf<double> dY, dA, dB, dO;
        dY.upload(y, (size_t)p * q * q * q, ss.st);
        dA.upload(a, (size_t)I * rank, ss.st);
        dB.upload(b, (size_t)J * rank, ss.st);
        dO.reserve((size_t)p * q * rank);
        m.temporal_stack(dY.p, 0, p, dA.p, dB.p, dO.p, false, ss.st);
        dO.download(out, (size_t)p * q * rank, ss.st);
        OCTEN_CUDA(cudaStreamSynchronize(ss.st));
    });
}

int octen_recover_temporal_append(int p, int q, int rank, int64_t t, const double* temporal_stack,
                                  const double* w, double* history, double* new_rows, double* residual) {
    return guard([&] {
        ScopedStream ss;
        octen::MergeEngine m;
        m.P = p;
        m.Q = q;
        m.R = rank;
        octen::DevBuf<double> dT, dW, dH, dR;
        dT.upload(temporal_stack, (size_t)p * q * rank, ss.st);
        dW.upload(w, (size_t)p * t * q, ss.st);
        std::vector<double> stk = blocks_to_hist(history, p, q, rank);
        dH.upload(stk.data(), stk.size(), ss.st);
        dR.reserve((size_t)t * rank);
        m.temporal_append(dT.p, dW.p, t, dH.p, dR.p, residual, ss.st);
        dR.download(new_rows, (size_t)t * rank, ss.st);
        std::vector<double> h2 = dH.to_host(stk.size(), ss.st);
        hist_to_blocks(h2, p, q, rank, history);
    });
}


int octen_coo_create(int p, int q, int64_t I, int64_t J, const double* u, const double* v, int device,
                     octen_coo_summaries** out) {
    return guard([&] {
        *out = nullptr;
        if (p < 1 || q < 1 || I < 1 || J < 1) throw octen::ConfigError("octen_coo_create: bad shape");
        OCTEN_CUDA(cudaSetDevice(device));
        auto h = std::make_unique<octen_coo_summaries>();
        h->device = device;
        OCTEN_CUDA(cudaStreamCreateWithFlags(&h->st, cudaStreamNonBlocking));
        for (auto& e : h->ev) OCTEN_CUDA(cudaEventCreate(&e));
        h->eng.set_projections(p, q, I, J, u, v, h->st);
        const size_t n = (size_t)p * q * q * q;
        h->Y.reserve(n);
        h->Y.zero(n, h->st);
        OCTEN_CUDA(cudaStreamSynchronize(h->st));
        *out = h.release();
    });
}

int octen_coo_compress(octen_coo_summaries* h, int64_t t, const double* w, int64_t nnz, const int32_t* i,
                       const int32_t* j, const int32_t* k, const float* values, int location) {
    return guard([&] {
        check_dtype(OCTEN_F32, location);
        OCTEN_CUDA(cudaSetDevice(h->device));
        auto& e = h->eng;
        if (t < 1) throw octen::ConfigError("compress: temporal extent must be >= 1");
        const double* dW = w;
        const int *di = i, *dj = j, *dk = k;
        const float* dv = values;
        if (location == OCTEN_HOST) {
            h->W.upload(w, (size_t)e.P * t * e.Q, h->st);
            dW = h->W.p;
            if (nnz > 0) {
                h->hi.upload(i, (size_t)nnz, h->st);
                h->hj.upload(j, (size_t)nnz, h->st);
                h->hk.upload(k, (size_t)nnz, h->st);
                h->hv.upload(values, (size_t)nnz, h->st);
                di = h->hi.p, dj = h->hj.p, dk = h->hk.p, dv = h->hv.p;
            }
        }
        e.compress(t, nnz, di, dj, dk, dv, dW, h->Y.p, h->st);
        e.collect(h->st);
    });
}

int octen_coo_get_summaries(const octen_coo_summaries* h, double* y) {
    return guard([&] {
        OCTEN_CUDA(cudaSetDevice(h->device));
        const auto& e = h->eng;
        h->Y.download(y, (size_t)e.P * e.Q * e.Q * e.Q, h->st);
        OCTEN_CUDA(cudaStreamSynchronize(h->st));
    });
}

int octen_coo_reset(octen_coo_summaries* h) {
    return guard([&] {
        OCTEN_CUDA(cudaSetDevice(h->device));
        const auto& e = h->eng;
        h->Y.zero((size_t)e.P * e.Q * e.Q * e.Q, h->st);
        OCTEN_CUDA(cudaStreamSynchronize(h->st));
    });
}

int octen_coo_cp_als(octen_coo_summaries* h, const octen_als_config* cfg, const uint64_t* seeds, double* factors,
                     double* lambda, double* fit, int32_t* iterations) {
    return guard([&] {
        OCTEN_CUDA(cudaSetDevice(h->device));
        const int p = h->eng.P, q = h->eng.Q;
        std::vector<std::uint64_t> sd(seeds, seeds + p);
        OCTEN_CUDA(cudaEventRecord(h->ev[0], h->st));
        h->als.run(p, cfg->n_restarts, q, cfg->rank, cfg->max_iters, cfg->rel_tol, h->Y.p, sd, h->st);
        OCTEN_CUDA(cudaEventRecord(h->ev[1], h->st));
        if (factors) h->als.Mf.download(factors, (size_t)p * 3 * q * cfg->rank, h->st);
        if (lambda) h->als.Mlam.download(lambda, (size_t)p * cfg->rank, h->st);
        OCTEN_CUDA(cudaStreamSynchronize(h->st));
        float ms = 0.f;
        OCTEN_CUDA(cudaEventElapsedTime(&ms, h->ev[0], h->ev[1]));
        h->als_ms += ms;
        ++h->als_runs;
        for (int r = 0; r < p; ++r) {
            if (fit) fit[r] = h->als.results[r].fit;
            if (iterations) iterations[r] = h->als.results[r].iterations;
        }
    });
}

int octen_coo_stage_times(const octen_coo_summaries* h, double* out) {
    return guard([&] {
        const auto& e = h->eng;
        out[0] = e.ms_prep;
        out[1] = e.ms_slice;
        out[2] = e.ms_accum;
        out[3] = e.groups_total;
        out[4] = e.nnz_total;
        out[5] = (double)e.batches;
        out[6] = h->als_ms;
        out[7] = (double)h->als_runs;
    });
}

void* octen_coo_cuda_stream(const octen_coo_summaries* h) { return h ? (void*)h->st : nullptr; }

void octen_coo_destroy(octen_coo_summaries* h) { delete h; }

int octen_compress_coo(int p, int q, int64_t I, int64_t J, int64_t t, const double* u, const double* v,
                       const double* w, int64_t nnz, const int32_t* i, const int32_t* j, const int32_t* k,
                       const float* values, double* z) {
    octen_coo_summaries* h = nullptr;
    int rc = octen_coo_create(p, q, I, J, u, v, 0, &h);
    if (rc != OCTEN_OK) return rc;
    rc = octen_coo_compress(h, t, w, nnz, i, j, k, values, OCTEN_HOST);
    if (rc == OCTEN_OK) rc = octen_coo_get_summaries(h, z);
    std::string msg = g_err;
    octen_coo_destroy(h);
    g_err = msg;
    return rc;
}

}  // extern "C"

// ---- COO text files (read_tensor_coo, proj/src/io.cpp:49-84) ----
// Parsed on the host (file I/O), validated per entry for arity, bounds and
// finiteness with the reference's messages prefixed by the path (io.cpp:79-83
// wraps the SparseTensor constructor's errors in IoError).  Duplicate
// indices are left to the device COO compression (octen_coo_compress), which
// raises the constructor's "SparseTensor: duplicate index".
#include <cerrno>
#include <cstdio>
#include <fstream>
#include <sstream>

struct octen_coo_file {
    std::vector<int64_t> dims;
    std::vector<int64_t> idx;  // nnz x order, 0-based
    std::vector<double> val;
};

extern "C" {

int octen_read_coo(const char* path, octen_coo_file** out) {
    return guard([&] {
        if (!path || !out) throw octen::ConfigError("octen_read_coo: null argument");
        const std::string p(path);
        std::ifstream in(p);
        if (!in) throw octen::IoError("cannot open '" + p + "' for reading");
        std::string line;
        if (!std::getline(in, line)) throw octen::IoError("'" + p + "': empty file");
        std::istringstream header(line);
        int order = 0;
        if (!(header >> order) || order < 2) throw octen::IoError("'" + p + "': bad header");
        auto f = std::make_unique<octen_coo_file>();
        f->dims.resize((size_t)order);
        for (int n = 0; n < order; ++n)
            if (!(header >> f->dims[(size_t)n]))
                throw octen::IoError("'" + p + "': header lists fewer extents than the order");
        for (int64_t d : f->dims)
            if (d < 1) throw octen::IoError("'" + p + "': Shape: dimensions must be positive");
        size_t line_no = 1;
        std::vector<int64_t> e((size_t)order);
        while (std::getline(in, line)) {
            ++line_no;
            if (line.empty()) continue;
            std::istringstream row(line);
            for (int n = 0; n < order; ++n) {
                if (!(row >> e[(size_t)n]))
                    throw octen::IoError("'" + p + "': malformed entry at line " + std::to_string(line_no));
                e[(size_t)n] -= 1;  // the file is 1-based
            }
            double v = 0.0;
            if (!(row >> v)) throw octen::IoError("'" + p + "': missing value at line " + std::to_string(line_no));
            // the SparseTensor constructor's checks, in its order (tensor.cpp:87-102)
            for (int n = 0; n < order; ++n)
                if (e[(size_t)n] < 0 || e[(size_t)n] >= f->dims[(size_t)n])
                    throw octen::IoError("'" + p + "': SparseTensor: index out of bounds");
            if (!std::isfinite(v)) throw octen::IoError("'" + p + "': SparseTensor: non-finite value");
            f->idx.insert(f->idx.end(), e.begin(), e.end());
            f->val.push_back(v);
        }
        *out = f.release();
    });
}

int octen_coo_file_info(const octen_coo_file* f, int64_t* order, int64_t* dims, int64_t* nnz) {
    return guard([&] {
        if (!f || !order || !nnz) throw octen::ConfigError("octen_coo_file_info: null argument");
        *order = (int64_t)f->dims.size();
        if (dims)
            for (size_t n = 0; n < f->dims.size(); ++n) dims[n] = f->dims[n];
        *nnz = (int64_t)f->val.size();
    });
}

int octen_coo_file_entries(const octen_coo_file* f, int64_t* indices, double* values) {
    return guard([&] {
        if (!f || !indices || !values) throw octen::ConfigError("octen_coo_file_entries: null argument");
        std::memcpy(indices, f->idx.data(), f->idx.size() * sizeof(int64_t));
        std::memcpy(values, f->val.data(), f->val.size() * sizeof(double));
    });
}

void octen_coo_file_destroy(octen_coo_file* f) { delete f; }

}  // extern "C"
