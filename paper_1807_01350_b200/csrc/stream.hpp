// One OCTen stream: configuration, host RNG state and device-resident state
// (summaries, history accumulators, model).  Mirrors cpstream::StreamState
// (proj/include/cpstream/streaming.hpp:48-59).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "devbuf.hpp"
#include "engine.hpp"

namespace octen {

struct StreamCfg {
    int rank = 1, p = 1, q = 1, shared = 0, temporal_mode = -1;
    int als_max_iters = 100, als_n_restarts = 3;
    double als_rel_tol = 1e-8;
    std::uint64_t seed = 0;
    bool enforce_bounds = false, strict = false;
    int workers = 0;
    double residual_warning = 1e-3;
    int device = 0;
};

struct BatchRecordC {
    std::int64_t batch_index, t_new;
    double temporal_residual, min_match_similarity, max_offdiag_similarity;
    int warned;
    double compress_seconds, als_seconds, recover_seconds, total_seconds;
};

class Stream {
public:
    explicit Stream(const StreamCfg& c);
    ~Stream();
    Stream(const Stream&) = delete;
    Stream& operator=(const Stream&) = delete;

    void init(const void* data, int dtype, int location, int order, const std::int64_t* dims);
    void ingest(const void* data, int dtype, int location, int order, const std::int64_t* dims);
    void get_factor(int mode, double* out);

    StreamCfg cfg;
    cudaStream_t st = nullptr;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    std::int64_t I = 0, J = 0, K = 0, capC = 0;
    std::int64_t batches_seen = 0, batches_drawn = 0;
    bool initialized = false;
    std::vector<double> hU, hV, hW, tgram;
    CompressEngine comp;
    AlsEngine als;
    MergeEngine merge;
    DevBuf<double> Y, hist, A, B, C, lam, dW, Anew, Bnew, rows, X64;
    DevBuf<float> X32;
    DevBuf<int> flag;
    std::vector<BatchRecordC> log;
    // cumulative device milliseconds: compress, als, recover, gemm1 (mode-1 contraction)
    double dev_ms[4] = {0, 0, 0, 0};
    double gemm1_flops = 0.0;
    long long gemm1_launches = 0;
    cudaEvent_t evs[6] = {};

private:
    struct Snapshot {
        DevBuf<double> Y, hist, A, B, C, lam;
        std::int64_t capC = 0, K = 0, batches_seen = 0, batches_drawn = 0;
        std::vector<double> tgram;
        size_t log_len = 0;
    };
    void validate(int order);
    void gen_replicas();
    void extend_temporal(std::int64_t t_new);
    const void* stage_input(const void* data, int dtype, int location, size_t n);
    void check_finite(const void* dX, int dtype, size_t n);
    void compress_stage(const void* dX, int dtype, std::int64_t t);
    void als_stage(std::int64_t batch_index);
    void recover_stage(std::int64_t t_new, bool first, BatchRecordC& rec);
    void ensure_c_capacity(std::int64_t rows);
    void accumulate_stage_times();
    void snapshot(Snapshot& s);
    void restore(Snapshot& s);
};

}  // namespace octen
