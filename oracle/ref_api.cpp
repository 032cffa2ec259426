// TEST INFRASTRUCTURE ONLY (oracle/).  C entry points over the reference
// library compiled from its own sources (see Makefile), for the parity tests
// (tests/test_ref_pin.py, tests/golden/make_ref_golden.py) and the CPU
// reference arm of bench.py.  Plain pointers and sizes; every call returns
// 0 or an error class (1 ConfigError, 2 NumericError, 3 IoError, 4 other)
// whose message ref_last_error() returns.  Tensors are first-index-fastest,
// matrices column-major, factors concatenated in mode order.
#include <cstdint>
#include <cstring>
#include <exception>
#include <limits>
#include <memory>
#include <fstream>
#include <string>
#include <vector>

#include "cpstream/commands.hpp"
#include "cpstream/cp_als.hpp"
#include "cpstream/errors.hpp"
#include "cpstream/eval.hpp"
#include "cpstream/streaming.hpp"
#include "cpstream/tensor.hpp"

extern "C" void scipy_openblas_set_num_threads(int);

using namespace cpstream;

namespace {

thread_local std::string g_err;

template <class F>
int guard(F&& f) {
    try {
        f();
        g_err.clear();
        return 0;
    } catch (const ConfigError& e) {
        g_err = e.what();
        return 1;
    } catch (const NumericError& e) {
        g_err = e.what();
        return 2;
    } catch (const IoError& e) {
        g_err = e.what();
        return 3;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 4;
    }
}

DenseTensor make_tensor(int order, const std::int64_t* dims, const double* values) {
    Shape s;
    std::int64_t n = 1;
    for (int i = 0; i < order; ++i) {
        s.dims.push_back(dims[i]);
        n *= dims[i];
    }
    return DenseTensor(s, std::vector<double>(values, values + n));
}

KruskalModel make_model(int order, const std::int64_t* dims, int rank, const double* factors, const double* lambda) {
    KruskalModel m;
    std::size_t off = 0;
    for (int n = 0; n < order; ++n) {
        Matrix f(dims[n], rank);
        std::memcpy(f.data(), factors + off, sizeof(double) * static_cast<std::size_t>(dims[n] * rank));
        off += static_cast<std::size_t>(dims[n] * rank);
        m.factors.push_back(f);
    }
    m.lambda = Vector(rank);
    for (int r = 0; r < rank; ++r) m.lambda(r) = lambda ? lambda[r] : 1.0;
    return m;
}

void put_model(const KruskalModel& m, double* factors_out, double* lambda_out) {
    std::size_t off = 0;
    for (const Matrix& f : m.factors) {
        if (factors_out) std::memcpy(factors_out + off, f.data(), sizeof(double) * static_cast<std::size_t>(f.size()));
        off += static_cast<std::size_t>(f.size());
    }
    if (lambda_out)
        for (Eigen::Index r = 0; r < m.lambda.size(); ++r) lambda_out[r] = m.lambda(r);
}

struct Handle {
    StreamState st;
};

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// The reference's Eigen is single-threaded per call; so is the stand-in's
// OpenBLAS.  Replica-level parallelism is the reference's own
// (StreamConfig::workers, std::thread fan-out).
void ref_set_blas_threads(int n) { scipy_openblas_set_num_threads(n); }

// generate_synthetic (proj/src/commands.cpp:110-134)
int ref_generate_synthetic(int order, const std::int64_t* dims, int rank, double mu, double sigma, std::uint64_t seed,
                           double* tensor_out, double* factors_out, double* lambda_out) {
    return guard([&] {
        SynthSpec spec;
        spec.dims.assign(dims, dims + order);
        spec.rank = rank;
        spec.noise_mu = mu;
        spec.noise_sigma = sigma;
        spec.seed = seed;
        const SynthData d = generate_synthetic(spec);
        if (tensor_out)
            std::memcpy(tensor_out, d.tensor.values().data(), sizeof(double) * d.tensor.values().size());
        put_model(d.truth, factors_out, lambda_out);
    });
}

// cp_als (proj/src/cp_als.cpp:240-359).  fit_hist_out holds max_iters
// entries (the winning restart's history, NaN past its iterations).
int ref_cp_als(int order, const std::int64_t* dims, const double* values, int rank, int max_iters, double rel_tol,
               int n_restarts, std::uint64_t seed, double* factors_out, double* lambda_out, double* fit_out,
               int* iters_out, double* fit_hist_out, int* rescued_out) {
    return guard([&] {
        AlsConfig cfg;
        cfg.rank = rank;
        cfg.max_iters = max_iters;
        cfg.rel_tol = rel_tol;
        cfg.n_restarts = n_restarts;
        cfg.seed = seed;
        const AlsResult r = cp_als(make_tensor(order, dims, values), cfg);
        put_model(r.model, factors_out, lambda_out);
        if (fit_out) *fit_out = r.fit;
        if (iters_out) *iters_out = r.iterations;
        if (rescued_out) *rescued_out = r.rescued_degenerate ? 1 : 0;
        if (fit_hist_out)
            for (int i = 0; i < max_iters; ++i)
                fit_hist_out[i] = i < static_cast<int>(r.fit_history.size()) ? r.fit_history[static_cast<std::size_t>(i)]
                                                                              : std::numeric_limits<double>::quiet_NaN();
    });
}

// init_stream (proj/src/streaming.cpp:180-260)
int ref_stream_init(int order, const std::int64_t* dims, const double* values, int rank, int p, int q, int shared,
                    int temporal_mode, int als_max_iters, double als_rel_tol, int als_restarts, std::uint64_t seed,
                    int enforce_bounds, int workers, int strict, double residual_warning, void** out) {
    *out = nullptr;
    return guard([&] {
        StreamConfig cfg;
        cfg.rank = rank;
        cfg.p = p;
        cfg.q = q;
        cfg.shared = shared;
        cfg.temporal_mode = temporal_mode;
        cfg.als.max_iters = als_max_iters;
        cfg.als.rel_tol = als_rel_tol;
        cfg.als.n_restarts = als_restarts;
        cfg.seed = seed;
        cfg.enforce_bounds = enforce_bounds != 0;
        cfg.workers = workers;
        cfg.strict = strict != 0;
        cfg.residual_warning = residual_warning;
        auto h = std::make_unique<Handle>();
        h->st = init_stream(make_tensor(order, dims, values), cfg);
        *out = h.release();
    });
}

// ingest_batch (proj/src/streaming.cpp:262-348)
int ref_stream_ingest(void* h, int order, const std::int64_t* dims, const double* values) {
    return guard([&] { ingest_batch(static_cast<Handle*>(h)->st, make_tensor(order, dims, values)); });
}

void ref_stream_free(void* h) { delete static_cast<Handle*>(h); }

// [order, rank, p, q, shared, temporal_mode, slices_seen, batches_seen,
//  log size, model dims (order)]
int ref_stream_info(void* h, std::int64_t* out) {
    return guard([&] {
        const StreamState& st = static_cast<Handle*>(h)->st;
        out[0] = st.order();
        out[1] = st.config.rank;
        out[2] = st.config.p;
        out[3] = st.config.q;
        out[4] = st.config.shared;
        out[5] = st.config.temporal_mode;
        out[6] = st.slices_seen;
        out[7] = st.summaries.batches_seen;
        out[8] = static_cast<std::int64_t>(st.log.size());
        for (int n = 0; n < st.order(); ++n) out[9 + n] = st.model.factors[static_cast<std::size_t>(n)].rows();
    });
}

int ref_stream_model(void* h, double* factors_out, double* lambda_out) {
    return guard([&] { put_model(static_cast<Handle*>(h)->st.model, factors_out, lambda_out); });
}

// summaries y_p (p x Q^N, first index fastest) and history accumulators
// (p x Q x R) when sized
int ref_stream_summaries(void* h, double* y_out, double* hist_out) {
    return guard([&] {
        const StreamState& st = static_cast<Handle*>(h)->st;
        std::size_t off = 0;
        for (const DenseTensor& y : st.summaries.y) {
            if (y_out) std::memcpy(y_out + off, y.values().data(), sizeof(double) * y.values().size());
            off += y.values().size();
        }
        off = 0;
        for (const Matrix& m : st.summaries.history) {
            if (hist_out) std::memcpy(hist_out + off, m.data(), sizeof(double) * static_cast<std::size_t>(m.size()));
            off += static_cast<std::size_t>(m.size());
        }
    });
}

// per batch: batch_index, t_new, temporal_residual, min_match_similarity,
// max_offdiag_similarity, warned
int ref_stream_log(void* h, double* out) {
    return guard([&] {
        std::size_t i = 0;
        for (const BatchRecord& r : static_cast<Handle*>(h)->st.log) {
            out[i++] = static_cast<double>(r.batch_index);
            out[i++] = static_cast<double>(r.t_new);
            out[i++] = r.temporal_residual;
            out[i++] = r.min_match_similarity;
            out[i++] = r.max_offdiag_similarity;
            out[i++] = r.warned ? 1.0 : 0.0;
        }
    });
}

// per batch stage timers (compress, als, recover, total seconds)
int ref_stream_timers(void* h, double* out) {
    return guard([&] {
        std::size_t i = 0;
        for (const BatchRecord& r : static_cast<Handle*>(h)->st.log) {
            out[i++] = r.compress_seconds;
            out[i++] = r.als_seconds;
            out[i++] = r.recover_seconds;
            out[i++] = r.total_seconds;
        }
    });
}

// checkpoint_save / checkpoint_load (proj/src/checkpoint.cpp:125-295)
int ref_stream_checkpoint_size(void* h, std::int64_t* size) {
    return guard([&] { *size = static_cast<std::int64_t>(checkpoint_save(static_cast<Handle*>(h)->st).size()); });
}
int ref_stream_checkpoint(void* h, std::uint8_t* out, std::int64_t cap) {
    return guard([&] {
        const std::vector<std::uint8_t> b = checkpoint_save(static_cast<Handle*>(h)->st);
        if (static_cast<std::int64_t>(b.size()) > cap) throw IoError("ref_stream_checkpoint: buffer too small");
        std::memcpy(out, b.data(), b.size());
    });
}
int ref_stream_load(const std::uint8_t* bytes, std::int64_t n, void** out) {
    *out = nullptr;
    return guard([&] {
        auto h = std::make_unique<Handle>();
        h->st = checkpoint_load(std::vector<std::uint8_t>(bytes, bytes + n));
        *out = h.release();
    });
}

// fitness / congruence (proj/src/eval.cpp)
int ref_fitness(std::int64_t n, const double* x, const double* x_hat, double* out) {
    return guard([&] {
        const std::int64_t dims[2] = {n, 1};
        *out = fitness(make_tensor(2, dims, x), make_tensor(2, dims, x_hat));
    });
}
int ref_congruence(int order, const std::int64_t* dims, int rank, const double* ground_f, const double* ground_l,
                   const double* est_f, const double* est_l, double* out) {
    return guard([&] {
        const std::vector<double> c =
            congruence(make_model(order, dims, rank, ground_f, ground_l), make_model(order, dims, rank, est_f, est_l));
        for (std::size_t i = 0; i < c.size(); ++i) out[i] = c[i];
    });
}
int ref_reconstruct(int order, const std::int64_t* dims, int rank, const double* factors, const double* lambda,
                    double* out) {
    return guard([&] {
        const DenseTensor t = reconstruct(make_model(order, dims, rank, factors, lambda));
        std::memcpy(out, t.values().data(), sizeof(double) * t.values().size());
    });
}

// run_stream over a synthetic tensor (proj/src/commands.cpp:190-300, the
// acceptance-criterion-3 driver): [stream_fitness_pct, oracle_fitness_pct]
int ref_run_stream_synth(int order, const std::int64_t* dims, int rank, double mu, double sigma, std::uint64_t synth_seed,
                         int p, int q, int shared, std::uint64_t seed, int enforce_bounds, int als_max_iters,
                         double als_rel_tol, int als_restarts, std::int64_t batch_size, int with_oracle,
                         double* out) {
    return guard([&] {
        RunSpec spec;
        spec.use_synth = true;
        spec.synth.dims.assign(dims, dims + order);
        spec.synth.rank = rank;
        spec.synth.noise_mu = mu;
        spec.synth.noise_sigma = sigma;
        spec.synth.seed = synth_seed;
        spec.config.rank = rank;
        spec.config.p = p;
        spec.config.q = q;
        spec.config.shared = shared;
        spec.config.seed = seed;
        spec.config.enforce_bounds = enforce_bounds != 0;
        spec.config.als.max_iters = als_max_iters;
        spec.config.als.rel_tol = als_rel_tol;
        spec.config.als.n_restarts = als_restarts;
        spec.batch_size = batch_size;
        spec.with_oracle = with_oracle != 0;
        spec.zero_timings = true;
        const RunOutput r = run_stream(spec);
        out[0] = r.stream_fitness_pct;
        out[1] = r.oracle_fitness_pct;
    });
}

}  // extern "C"
