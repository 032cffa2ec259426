// One OCTen stream: configuration, host RNG state and device-resident state
// (summaries, history accumulators, model).  Mirrors cpstream::StreamState
// (proj/include/cpstream/streaming.hpp:48-59).
#pragma once

#include <cuda_runtime.h>

#include <chrono>
#include <cstdint>
#include <string>
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

// One stream handle.  Unsharded (world == 1) it owns every replica.  As rank
// g of a replica-sharded stream (one process per GPU) it owns replicas
// [p0, p0 + pl), pl <= chunk = ceil(P / world): it compresses the batch into
// and runs CP-ALS on those replicas only, and runs the alignment/merge
// redundantly after two all-gathers the caller performs between the phases:
//   begin  -> models_out  (models_count() doubles: status header, chunk x 3 x Q x R
//                          factors, chunk x R lambdas)
//   merge  <- models_all  (world blocks, rank order) -> rows_out (rows_count():
//                          chunk x Q x R temporal-stack rows of the owned replicas)
//   finish <- rows_all    (world blocks)
// init_stream / ingest_batch (streaming.cpp:181-346) are the three phases
// back to back with internal exchange buffers.
class Stream {
public:
    Stream(const StreamCfg& c, int shard_rank = 0, int shard_world = 1);
    ~Stream();
    Stream(const Stream&) = delete;
    Stream& operator=(const Stream&) = delete;

    void init(const void* data, int dtype, int location, int order, const std::int64_t* dims);
    void ingest(const void* data, int dtype, int location, int order, const std::int64_t* dims);
    void get_factor(int mode, double* out);
    // eval.cpp:10-20 fitness of the model on slices [k0, k0 + t) given as a batch
    double batch_fitness(const void* data, int dtype, int location, int order, const std::int64_t* dims,
                         std::int64_t k0);
    // Start the host->device copy of a later batch (host, pinned for overlap)
    // on a copy stream, so it overlaps the device work of the batches before
    // it.  A later begin/ingest whose data pointer, dtype and extents match
    // the oldest pending prefetch consumes it.  At most two prefetches are
    // pending; the host buffer must not change until the batch is ingested.
    void prefetch(const void* data, int dtype, int order, const std::int64_t* dims);

    void begin(const void* data, int dtype, int location, int order, const std::int64_t* dims, double* models_out);
    void merge_phase(const double* models_all, double* rows_out);
    // temporal sharding of the compression (octen_stream_begin_temporal /
    // octen_stream_begin_reduced): partial summaries of every replica from
    // this rank's slices, reduce-scattered by the caller, then CP-ALS.
    void begin_temporal(const void* data, int dtype, int location, int order, const std::int64_t* dims_local,
                        std::int64_t k_off, std::int64_t t_total, double* partial_out);
    void begin_reduced(const double* owned_block, double* models_out);
    size_t partial_block_count() const { return (size_t)chunk * cfg.q * cfg.q * cfg.q + 1; }
    void finish(const double* rows_all);
    size_t models_count() const { return 4 + (size_t)chunk * (3 * (size_t)cfg.q * cfg.rank + cfg.rank); }
    size_t rows_count() const { return (size_t)chunk * cfg.q * cfg.rank; }

    StreamCfg cfg;
    int shard_rank = 0, shard_world = 1, p0 = 0, pl = 0, chunk = 0;
    cudaStream_t st = nullptr;
    cudaStream_t cp = nullptr;           // host->device batch copies (chunked)
    std::vector<cudaEvent_t> copy_ev;    // one per copied chunk
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    std::int64_t I = 0, J = 0, K = 0, capC = 0;
    std::int64_t batches_seen = 0, batches_drawn = 0;
    bool initialized = false;
    std::vector<double> hU, hV, hW, tgram;
    CompressEngine comp;
    CompressEngine comp_all;  // every replica (temporal sharding)
    bool comp_all_ready = false;
    AlsEngine als;
    MergeEngine merge;
    // Y: pl x Q^3 (owned replicas); hist: P*Q x R (all replicas, kept redundantly)
    DevBuf<double> Y, hist, A, B, C, lam, dW, Anew, Bnew, rows, X64;
    DevBuf<double> xmodels, xrows, MfAll, MlamAll, tstackAll;
    DevBuf<float> X32;
    DevBuf<int> flag;
    DevBuf<double> Zpart;                 // temporal sharding: partial summaries, world x chunk x Q^3
    std::int64_t tshard_drawn = 0;        // temporal state before begin_temporal (rollback)
    std::vector<double> tshard_tgram;
    struct Prefetch {
        const void* host = nullptr;
        int dtype = 0, slot = 0;
        std::int64_t dims[3] = {0, 0, 0};
        std::int64_t sub = 1, nch = 0;
    };
    std::vector<Prefetch> pf;            // pending, oldest first (<= 2)
    DevBuf<float> PX32[2];
    DevBuf<double> PX64[2];
    std::vector<cudaEvent_t> pf_ev[2];   // per copied chunk
    cudaEvent_t slot_free[2] = {};       // recorded on st once a slot's batch is read
    cudaStream_t pcp = nullptr;          // prefetch copy stream
    double* pin_buf = nullptr;           // pinned, mapped staging of small per-batch uploads
    size_t pin_cap = 0;
    cudaEvent_t pin_ev = nullptr;
    std::vector<BatchRecordC> log;
    // cumulative device milliseconds: compress, als, recover, gemm1 (mode-1 contraction)
    double dev_ms[4] = {0, 0, 0, 0};
    double gemm1_flops = 0.0;
    long long gemm1_launches = 0;
    cudaEvent_t evs[6] = {};

private:
    using Clock = std::chrono::steady_clock;
    struct Snapshot {
        DevBuf<double> Y, hist, A, B, C, lam;
        std::int64_t capC = 0, K = 0, batches_seen = 0, batches_drawn = 0;
        std::vector<double> tgram;
        size_t log_len = 0;
    };
    void validate(int order);
    void prepare(int order, const std::int64_t* dims);
    void gen_replicas();
    void extend_temporal(std::int64_t t_new);
    void upload_mapped(DevBuf<double>& dst, const double* h, size_t n);
    const void* stage_input(const void* data, int dtype, int location, size_t n);
    void check_finite(const void* dX, int dtype, size_t n);
    void ensure_c_capacity(std::int64_t rows);
    void accumulate_stage_times();
    void als_phase(double* models_out);
    void snapshot(Snapshot& s);
    void restore(Snapshot& s);
    [[noreturn]] void fail_pending();

    // the batch between begin and finish
    bool pending = false, pending_first = false;
    std::int64_t pending_t = 0;
    BatchRecordC prec{};
    Clock::time_point t_start, t_recover;
    Snapshot backup;
    std::string context;
};

}  // namespace octen
