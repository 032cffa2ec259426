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

#include <climits>
#include <cstdint>
#include <cstring>
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
    std::int64_t nlog = 0;  // one record per successful batch (a failed one still counts in batches_seen)
    check(octen_stream_log_size(st.handle.get(), &nlog));
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

// Pipelined ingest (no reference counterpart; same results as ingest_batch),
// two batches in flight: the CP-ALS sweeps and the merges run on library
// worker threads beside the next batch's compression and CP-ALS start.  The
// host model/log copies are refreshed by sync(); a CP-ALS error of batch b is
// thrown by the call of batch b+1, a merge error by the call of batch b+2 or
// sync (the later batches are then not ingested).
inline void ingest_batch_async(StreamState& st, const DenseTensor& batch) {
    if (!st.handle) throw ConfigError("ingest_batch: stream is not initialised");
    check(octen_stream_ingest_async(st.handle.get(), batch.data.data(), OCTEN_F64, OCTEN_HOST, batch.order(),
                                    batch.dims.data()));
}
inline void sync(StreamState& st) {
    check(octen_stream_sync(st.handle.get()));
    detail::refresh(st);
}

// checkpoint_save / checkpoint_load (proj/include/cpstream/streaming.hpp:78-79):
// the OCTS bytes of the device-resident stream, byte-compatible with the
// reference's container.
inline std::vector<std::uint8_t> checkpoint_save(const StreamState& st) {
    std::int64_t n = 0;
    check(octen_stream_checkpoint_save(st.handle.get(), nullptr, 0, &n));
    std::vector<std::uint8_t> b((size_t)n);
    check(octen_stream_checkpoint_save(st.handle.get(), b.data(), n, &n));
    return b;
}
inline StreamState checkpoint_load(const std::vector<std::uint8_t>& bytes, int device = 0) {
    octen_stream* raw = nullptr;
    check(octen_stream_checkpoint_load(bytes.data(), (std::int64_t)bytes.size(), device, &raw));
    StreamState st;
    st.handle = std::shared_ptr<octen_stream>(raw, octen_stream_destroy);
    // the config the container holds (checkpoint.cpp:125-143)
    auto u32 = [&](size_t off) {
        std::uint32_t v;
        std::memcpy(&v, bytes.data() + off, 4);
        return (int)v;
    };
    st.config.rank = u32(24);
    st.config.p = u32(28);
    st.config.q = u32(32);
    st.config.shared = u32(36);
    st.config.temporal_mode = u32(40);
    std::memcpy(&st.config.seed, bytes.data() + 44, 8);
    st.config.device = device;
    detail::refresh(st);
    return st;
}

// One rank of a replica-sharded stream with library-owned NCCL collectives
// (octen_stream_create_nccl): the caller distributes the unique id of rank 0
// and every rank ingests the same sequence of batches.  The reference's
// parallel_replicas (src/streaming.cpp:45-69) across GPUs.
class ShardedStream {
public:
    static std::vector<std::uint8_t> nccl_unique_id() {
        std::vector<std::uint8_t> id(128);
        check(octen_nccl_get_unique_id(id.data()));
        return id;
    }
    ShardedStream(const StreamConfig& cfg, int rank, int world, const std::vector<std::uint8_t>& uid) {
        const octen_stream_config c = detail::to_c(cfg);
        octen_stream* raw = nullptr;
        check(octen_stream_create_nccl(&c, rank, world, uid.data(), nullptr, &raw));
        st_.config = cfg;
        st_.handle = std::shared_ptr<octen_stream>(raw, octen_stream_destroy);
    }
    // init_stream on the first call, ingest_batch afterwards
    void ingest(const DenseTensor& batch) {
        check(octen_stream_ingest_sharded(st_.handle.get(), batch.data.data(), OCTEN_F64, OCTEN_HOST, batch.order(),
                                          batch.dims.data()));
        detail::refresh(st_);
    }
    // this rank's slices [k_off, k_off + local t) of a batch of t_total
    void ingest_temporal(const DenseTensor& local, std::int64_t k_off, std::int64_t t_total) {
        check(octen_stream_ingest_temporal(st_.handle.get(), local.data.data(), OCTEN_F64, OCTEN_HOST, local.order(),
                                           local.dims.data(), k_off, t_total));
        detail::refresh(st_);
    }
    const StreamState& state() const { return st_; }

private:
    StreamState st_;
};

// ---- sparse (COO) batches: proj/include/cpstream/tensor.hpp:66-90 ----
// The reference validates entries in the SparseTensor constructor and
// densifies before compress; here the entries go to the device as they are
// (octen_coo_*), validated there with the same errors and messages.
struct SparseTensor {
    struct Entry {
        std::vector<std::int64_t> index;
        double value = 0.0;
    };
    std::vector<std::int64_t> dims;
    std::vector<Entry> entries;
    SparseTensor() = default;
    SparseTensor(std::vector<std::int64_t> d, std::vector<Entry> e) : dims(std::move(d)), entries(std::move(e)) {}
    std::int64_t nnz() const { return (std::int64_t)entries.size(); }
};

// Device-resident SummaryState fed by COO batches (compression.hpp:56-60):
// compress() is update_summaries(compress(batch.to_dense())) for every replica.
class CooSummaries {
public:
    // u[r]: I x Q, v[r]: J x Q (column-major) per replica
    CooSummaries(const std::vector<Matrix>& u, const std::vector<Matrix>& v, int device = 0)
        : p_((int)u.size()), q_(u.empty() ? 0 : (int)u[0].cols()) {
        if (u.empty() || u.size() != v.size()) throw ConfigError("CooSummaries: replica count mismatch");
        i_ = u[0].rows();
        j_ = v[0].rows();
        std::vector<double> U, V;
        for (const Matrix& m : u) U.insert(U.end(), m.v.begin(), m.v.end());
        for (const Matrix& m : v) V.insert(V.end(), m.v.begin(), m.v.end());
        octen_coo_summaries* raw = nullptr;
        check(octen_coo_create(p_, q_, i_, j_, U.data(), V.data(), device, &raw));
        h_ = std::shared_ptr<octen_coo_summaries>(raw, octen_coo_destroy);
    }
    // w[r]: t x Q temporal rows of this batch per replica
    void compress(const SparseTensor& batch, const std::vector<Matrix>& w) {
        if (batch.dims.size() != 3) throw ConfigError("compress: tensor order mismatch");
        if (batch.dims[0] != i_ || batch.dims[1] != j_) throw ConfigError("compress: extent mismatch on mode 1");
        const std::int64_t t = batch.dims[2], n = batch.nnz();
        std::vector<std::int32_t> ii((size_t)n), jj((size_t)n), kk((size_t)n);
        std::vector<float> vals((size_t)n);
        for (std::int64_t e = 0; e < n; ++e) {
            const auto& en = batch.entries[(size_t)e];
            if (en.index.size() != 3) throw ConfigError("SparseTensor: index arity mismatch");
            auto narrow = [](std::int64_t x) {  // out-of-range values stay out of range
                return (std::int32_t)(x < INT32_MIN ? INT32_MIN : x > INT32_MAX ? INT32_MAX : x);
            };
            ii[(size_t)e] = narrow(en.index[0]);
            jj[(size_t)e] = narrow(en.index[1]);
            kk[(size_t)e] = narrow(en.index[2]);
            vals[(size_t)e] = (float)en.value;
        }
        std::vector<double> W;
        for (const Matrix& m : w) W.insert(W.end(), m.v.begin(), m.v.end());
        if ((std::int64_t)W.size() != (std::int64_t)p_ * t * q_) throw ConfigError("compress: temporal rows mismatch");
        check(octen_coo_compress(h_.get(), t, W.data(), n, ii.data(), jj.data(), kk.data(), vals.data(), OCTEN_HOST));
    }
    // summaries: p tensors Q x Q x Q
    std::vector<DenseTensor> summaries() const {
        const size_t q3 = (size_t)q_ * q_ * q_;
        std::vector<double> y((size_t)p_ * q3);
        check(octen_coo_get_summaries(h_.get(), y.data()));
        std::vector<DenseTensor> out;
        for (int r = 0; r < p_; ++r)
            out.emplace_back(std::vector<std::int64_t>{q_, q_, q_},
                             std::vector<double>(y.begin() + (std::ptrdiff_t)(r * q3), y.begin() + (std::ptrdiff_t)((r + 1) * q3)));
        return out;
    }

private:
    int p_ = 0, q_ = 0;
    std::int64_t i_ = 0, j_ = 0;
    std::shared_ptr<octen_coo_summaries> h_;
};

}  // namespace cpstream_b200
