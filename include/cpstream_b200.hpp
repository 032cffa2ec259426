// cpstream_b200.hpp -- C++ host mirror of the reference's streaming API over
// the C-ABI in octen_b200.h.
//
// The reference library `cpstream` (/root/reference/proj) is C++20 + Eigen;
// its boundary is the C++ API of proj/include/cpstream/streaming.hpp.  This
// header keeps those names, argument meanings and error behaviour --
// init_stream / ingest_batch take a DenseTensor (first index fastest) and a
// StreamConfig, mutate a StreamState whose KruskalModel is in normal form,
// append a BatchRecord per batch, and throw ConfigError / NumericError /
// IoError (proj/include/cpstream/errors.hpp:9-26) carrying the reference's
// message text -- while every computation runs on the B200 through
// libocten_b200.so.  Header-only; link with -locten_b200.
//
// Eigen is not part of the boundary: Matrix is a plain column-major fp64
// block (the Eigen::MatrixXd default layout), so a reference build can map
// it onto Eigen::Map without copies.
#pragma once

#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "octen_b200.h"

namespace cpstream_b200 {

// ---- errors (proj/include/cpstream/errors.hpp:9-26) ----
struct Error : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct ConfigError : Error {
    using Error::Error;
};
struct NumericError : Error {
    using Error::Error;
};
struct IoError : Error {
    using Error::Error;
};
// device failures have no reference counterpart
struct DeviceError : Error {
    using Error::Error;
};

inline void check(int status) {
    if (status == OCTEN_OK) return;
    const char* m = octen_last_error();
    const std::string msg = m ? m : "";
    switch (status) {
        case OCTEN_ERR_CONFIG: throw ConfigError(msg);
        case OCTEN_ERR_NUMERIC: throw NumericError(msg);
        case OCTEN_ERR_IO: throw IoError(msg);
        case OCTEN_ERR_CUDA: throw DeviceError(msg);
        default: throw Error(msg);
    }
}

// ---- data types (proj/include/cpstream/tensor.hpp:21-64) ----
struct Matrix {
    std::int64_t r = 0, c = 0;
    std::vector<double> v;  // column-major
    Matrix() = default;
    Matrix(std::int64_t rows, std::int64_t cols) : r(rows), c(cols), v((size_t)(rows * cols), 0.0) {}
    std::int64_t rows() const { return r; }
    std::int64_t cols() const { return c; }
    double& operator()(std::int64_t i, std::int64_t j) { return v[(size_t)(i + r * j)]; }
    double operator()(std::int64_t i, std::int64_t j) const { return v[(size_t)(i + r * j)]; }
    double* data() { return v.data(); }
    const double* data() const { return v.data(); }
};

struct DenseTensor {
    std::vector<std::int64_t> dims;
    std::vector<double> data;  // first index fastest
    DenseTensor() = default;
    DenseTensor(std::vector<std::int64_t> d, std::vector<double> x) : dims(std::move(d)), data(std::move(x)) {
        std::int64_t n = 1;
        for (std::int64_t e : dims) n *= e;
        if (n != (std::int64_t)data.size()) throw ConfigError("DenseTensor: data size does not match dims");
    }
    static DenseTensor zeros(std::vector<std::int64_t> d) {
        std::int64_t n = 1;
        for (std::int64_t e : d) n *= e;
        return DenseTensor(std::move(d), std::vector<double>((size_t)n, 0.0));
    }
    int order() const { return (int)dims.size(); }
    std::int64_t numel() const { return (std::int64_t)data.size(); }
};

// proj/include/cpstream/tensor.hpp KruskalModel: factors (dim x rank, unit
// columns in normal form) and lambda
struct KruskalModel {
    std::vector<Matrix> factors;
    std::vector<double> lambda;
    int order() const { return (int)factors.size(); }
    int rank() const { return (int)lambda.size(); }
};

// proj/include/cpstream/cp_als.hpp:25-31
struct AlsConfig {
    int rank = 1;
    int max_iters = 100;
    double rel_tol = 1e-8;
    int n_restarts = 3;
    std::uint64_t seed = 0;
};

// proj/include/cpstream/streaming.hpp:15-27
struct StreamConfig {
    int rank = 1;
    int p = 1;
    int q = 1;
    int shared = 0;
    int temporal_mode = -1;  // -1: last mode
    AlsConfig als;
    std::uint64_t seed = 0;
    bool enforce_bounds = false;
    int workers = 0;  // accepted; the device path has no worker pool
    bool strict = false;
    double residual_warning = 1e-3;
    int device = 0;  // CUDA ordinal (B200-specific)
};

// proj/include/cpstream/streaming.hpp:31-42
struct BatchRecord {
    std::int64_t batch_index = 0;
    std::int64_t t_new = 0;
    double temporal_residual = 0.0;
    double min_match_similarity = 1.0;
    double max_offdiag_similarity = 0.0;
    bool warned = false;
    double compress_seconds = 0.0;
    double als_seconds = 0.0;
    double recover_seconds = 0.0;
    double total_seconds = 0.0;
};

// proj/include/cpstream/streaming.hpp:48-59.  The replicas and summaries live
// on the device inside `handle`; `model`, `slices_seen` and `log` are host
// copies refreshed after every call, as the reference exposes them.
struct StreamState {
    StreamConfig config;
    KruskalModel model;
    std::int64_t slices_seen = 0;
    std::vector<BatchRecord> log;
    std::shared_ptr<octen_stream> handle;

    int order() const { return model.order(); }
    int temporal_mode() const { return 2; }
    // SummaryState (compression.hpp:56-60): y p x Q^3, history p x Q x rank
    std::vector<double> summaries() const {
        std::vector<double> y((size_t)config.p * config.q * config.q * config.q);
        check(octen_stream_get_summaries(handle.get(), y.data()));
        return y;
    }
    std::vector<double> history() const {
        std::vector<double> h((size_t)config.p * config.q * config.rank);
        check(octen_stream_get_history(handle.get(), h.data()));
        return h;
    }
};

namespace detail {
inline octen_stream_config to_c(const StreamConfig& c) {
    octen_stream_config o{};
    o.rank = c.rank;
    o.p = c.p;
    o.q = c.q;
    o.shared = c.shared;
    o.temporal_mode = c.temporal_mode;
    o.als.rank = c.als.rank;
    o.als.max_iters = c.als.max_iters;
    o.als.rel_tol = c.als.rel_tol;
    o.als.n_restarts = c.als.n_restarts;
    o.als.seed = c.als.seed;
    o.seed = c.seed;
    o.enforce_bounds = c.enforce_bounds ? 1 : 0;
    o.workers = c.workers;
    o.strict = c.strict ? 1 : 0;
    o.residual_warning = c.residual_warning;
    o.device = c.device;
    return o;
}

inline void refresh(StreamState& st) {
    std::int64_t info[8];
    check(octen_stream_info(st.handle.get(), info));
    const int order = (int)info[0], rank = (int)info[4];
    st.slices_seen = info[3];
    st.model.factors.assign((size_t)order, Matrix());
    for (int m = 0; m < order; ++m) {
        st.model.factors[(size_t)m] = Matrix(info[1 + m], rank);
        check(octen_stream_get_factor(st.handle.get(), m, st.model.factors[(size_t)m].data()));
    }
    st.model.lambda.assign((size_t)rank, 0.0);
    check(octen_stream_get_lambda(st.handle.get(), st.model.lambda.data()));
    const std::int64_t nlog = info[7];
    st.log.resize((size_t)nlog);
    for (std::int64_t i = 0; i < nlog; ++i) {
        octen_batch_record r{};
        check(octen_stream_get_record(st.handle.get(), i, &r));
        BatchRecord& b = st.log[(size_t)i];
        b.batch_index = r.batch_index;
        b.t_new = r.t_new;
        b.temporal_residual = r.temporal_residual;
        b.min_match_similarity = r.min_match_similarity;
        b.max_offdiag_similarity = r.max_offdiag_similarity;
        b.warned = r.warned != 0;
        b.compress_seconds = r.compress_seconds;
        b.als_seconds = r.als_seconds;
        b.recover_seconds = r.recover_seconds;
        b.total_seconds = r.total_seconds;
    }
}
}  // namespace detail

// init_stream (proj/include/cpstream/streaming.hpp:64; src/streaming.cpp:181-256)
inline StreamState init_stream(const DenseTensor& first_batch, const StreamConfig& cfg) {
    const octen_stream_config c = detail::to_c(cfg);
    octen_stream* raw = nullptr;
    check(octen_stream_init(&c, first_batch.data.data(), OCTEN_F64, OCTEN_HOST, first_batch.order(),
                            first_batch.dims.data(), &raw));
    StreamState st;
    st.config = cfg;
    st.handle = std::shared_ptr<octen_stream>(raw, octen_stream_destroy);
    detail::refresh(st);
    return st;
}

// ingest_batch (proj/include/cpstream/streaming.hpp:70; src/streaming.cpp:258-346).
// Strict mode rolls the device state back on error, as the reference does.
inline void ingest_batch(StreamState& st, const DenseTensor& batch) {
    if (!st.handle) throw ConfigError("ingest_batch: stream is not initialised");
    check(octen_stream_ingest(st.handle.get(), batch.data.data(), OCTEN_F64, OCTEN_HOST, batch.order(),
                              batch.dims.data()));
    detail::refresh(st);
}

// fp32 batches (the BASELINE fp32 configs) go through the same entry points
inline void ingest_batch_f32(StreamState& st, const std::vector<std::int64_t>& dims, const float* data) {
    if (!st.handle) throw ConfigError("ingest_batch: stream is not initialised");
    check(octen_stream_ingest(st.handle.get(), data, OCTEN_F32, OCTEN_HOST, (int)dims.size(), dims.data()));
    detail::refresh(st);
}

}  // namespace cpstream_b200
