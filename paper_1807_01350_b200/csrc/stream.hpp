// One OCTen stream: configuration, host RNG state and device-resident state
// (summaries, history accumulators, model).  Mirrors cpstream::StreamState
// (proj/include/cpstream/streaming.hpp:48-59).
#pragma once

#include <cuda_runtime.h>

#include <chrono>
#include <condition_variable>
#include <cstdint>
#include <exception>
#include <functional>
#include <future>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "devbuf.hpp"
#include "engine.hpp"

namespace octen {

struct StreamCfg {
    int rank = 1, p = 1, q = 1, shared = 0, temporal_mode = -1;
    int als_max_iters = 100, als_n_restarts = 3;
    double als_rel_tol = 1e-8;
    std::uint64_t als_seed = 0;  // AlsConfig.seed (checkpointed; per-replica seeds derive from `seed`)
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

// The state of one batch between begin and finish.  The synchronous paths use
// one (Stream::cur); the pipelined ingest keeps two, since batch b's merge
// runs on the worker thread while batch b+1 is compressed and decomposed.
struct BatchCtx {
    bool pending = false, first = false, compressed = false;
    std::int64_t t = 0;
    BatchRecordC rec{};
    std::string context;
    std::chrono::steady_clock::time_point t_start, t_recover;
    cudaStream_t st = nullptr;         // stream of the merge phases
    cudaEvent_t ev[3] = {};            // merge start / end (device timing), inputs ready on the main stream
    std::vector<double> tgram;         // shared temporal Gram including this batch's rows (align)
    const double* dW = nullptr;        // this batch's temporal rows (P x t x Q)
    // pipelined ingest: the summaries after this batch (read by its merge),
    // its models block, and the stream counters before it (rollback)
    const double* Yb = nullptr;
    double* models = nullptr;
    std::int64_t rb_drawn = 0, rb_seen = 0;
    std::vector<double> rb_tgram;
    bool init_failed = false;          // its CP-ALS start raised
    float als_init_ms = 0.f;           // CP-ALS start: device ms, wall s
    double als_init_s = 0.0;
    ~BatchCtx();
};

// One persistent host thread that runs posted tasks in order (the merge of
// the pipelined ingest).  A persistent thread keeps its per-thread device
// block cache (devbuf.hpp) warm across batches.
class Worker {
public:
    ~Worker();
    void post(int device, std::function<void()> f);
    // Wait for the posted task; returns its exception (null if it succeeded
    // or nothing was posted).
    std::exception_ptr wait();
    bool busy() const { return posted; }

private:
    void loop(int device);
    std::thread th;
    std::mutex mu;
    std::condition_variable cv;
    std::function<void()> task;
    std::exception_ptr err;
    bool posted = false, running = false, done = false, quit = false;
};

// One batch's temporal projection rows (all replicas, P x t x Q) and the
// shared columns' Gram contribution, drawn on the host (extend_temporal).
struct TemporalDraw {
    std::uint64_t key = 0;
    std::int64_t t = 0;
    std::vector<double> w, gram;
};
TemporalDraw draw_temporal(std::uint64_t seed, int P, int Q, int sh, std::uint64_t key, std::int64_t t_new);

// A sharded stream's NCCL communicator (nccl_exchange.cu).
struct NcclExchange {
    void* comm = nullptr;  // ncclComm_t
    bool owned = false;
    ~NcclExchange();
};
void nccl_unique_id(unsigned char* out128);

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
    // Pipelined ingest_batch, two batches in flight: this batch is compressed
    // and its CP-ALS started (GEVD attempts, on the other of two engines)
    // while the previous batch's sweeps (CP-ALS worker thread) and the merge
    // before them (merge worker thread) run; then this batch's sweeps and
    // the previous batch's merge are posted.  The results are the same bits
    // as ingest(): every stage reads the same inputs (three summaries
    // buffers, per-batch temporal rows and Gram).  A CP-ALS error of batch b
    // surfaces at the call of batch b+1, a merge error at the call of batch
    // b+2 or sync (with the batch prefix); the later batches are rolled back.
    // Strict streams and the first batch run synchronously.
    void ingest_async(const void* data, int dtype, int location, int order, const std::int64_t* dims);
    // Wait for the pending merge; rethrows its error.
    void sync();
    // OCTS checkpoint (checkpoint.cpp:125-295) of the stream between batches,
    // and a stream rebuilt from one (checkpoint.cu).
    std::vector<std::uint8_t> checkpoint_save();
    static std::unique_ptr<Stream> checkpoint_load(const std::uint8_t* bytes, size_t n, int device);
    // Library-owned collectives (nccl_exchange.cu): a communicator from a
    // unique id (or a borrowed ncclComm_t), then whole batches with the
    // all-gathers / reduce-scatter on the stream's own CUDA stream.
    void attach_nccl(const unsigned char* uid128, void* borrowed_comm);
    void ingest_sharded(const void* data, int dtype, int location, int order, const std::int64_t* dims);
    void ingest_temporal_nccl(const void* data, int dtype, int location, int order, const std::int64_t* dims_local,
                              std::int64_t k_off, std::int64_t t_total);
    std::unique_ptr<NcclExchange> nccl_x;
    // Model publication for pipelined callers: with `publish` on, every
    // finished batch copies its model (A, B, C, lambda) to host memory; the
    // copy is read without waiting for the merge in flight.
    bool publish = false;
    std::mutex pub_mu;
    std::vector<double> pubA, pubB, pubC, pubLam;
    std::int64_t pub_K = 0, pub_batches = 0;
    double* pub_pin = nullptr;
    size_t pub_cap = 0;
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

    void begin(const void* data, int dtype, int location, int order, const std::int64_t* dims, double* models_out) {
        begin(cur, data, dtype, location, order, dims, models_out, false);
    }
    void merge_phase(const double* models_all, double* rows_out) { merge_phase(cur, models_all, rows_out); }
    // temporal sharding of the compression (octen_stream_begin_temporal /
    // octen_stream_begin_reduced): partial summaries of every replica from
    // this rank's slices, reduce-scattered by the caller, then CP-ALS.
    void begin_temporal(const void* data, int dtype, int location, int order, const std::int64_t* dims_local,
                        std::int64_t k_off, std::int64_t t_total, double* partial_out);
    void begin_reduced(const double* owned_block, double* models_out);
    size_t partial_block_count() const { return (size_t)chunk * cfg.q * cfg.q * cfg.q + 1; }
    void finish(const double* rows_all) { finish(cur, rows_all); }
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
    AlsEngine als_b;  // pipelined ingest: batches alternate engines (one starts while the other sweeps)
    MergeEngine merge;
    // Y: pl x Q^3 (owned replicas); hist: P*Q x R (all replicas, kept redundantly)
    // Ynext: the pipelined ingest's summaries after the batch in flight
    // (Y + its compression, out of place: the merge of the previous batch
    // still reads Y); dWb: temporal rows of the last two batches
    DevBuf<double> Y, Ynext, hist, A, B, C, lam, Anew, Bnew, rows, X64;
    DevBuf<double> dWb[3];  // temporal rows of the last three batches (pipelined ingest)
    int wslot = 0;
    double* dW = nullptr;
    DevBuf<double> xmodels, xrows, MfAll, MlamAll, tstackAll;
    DevBuf<double> xmodels2;     // pipelined ingest: models of the batch in flight (NCCL: all-gathered models)
    DevBuf<double> xmodels3;     // pipelined ingest: one models buffer per context slot (three batches overlap)
    DevBuf<double> rows_all_buf, part_buf, owned_buf;  // NCCL exchange buffers
    DevBuf<float> X32, XT32;     // staged batch; its temporal-last reorder (temporal mode not last)
    DevBuf<double> XT64, MfSlot;
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

    BatchCtx cur;                 // synchronous / sharded phases
    BatchCtx actx[3];             // pipelined ingest: rotating per batch
    int aslot = 0, apar = 0;      // context slot (mod 3); engine / models parity
    Worker worker;                // pipelined ingest: the merges
    Worker aworker;               // pipelined ingest: the CP-ALS runs
    cudaStream_t mst = nullptr;   // merge stream of the pipelined ingest (lower priority)
    cudaStream_t ast = nullptr;   // CP-ALS stream of the pipelined ingest
    // pipelined ingest: the batch whose CP-ALS sweeps are posted (aworker),
    // and the batch whose merge is posted (worker) and not yet waited for
    BatchCtx* a_prev = nullptr;
    BatchCtx* m_prev = nullptr;
    DevBuf<double> Yhold;         // the summaries m_prev's merge reads
    cudaEvent_t aevs[2] = {};     // CP-ALS sweeps device timing (the CP-ALS worker's events)
    cudaEvent_t ievs[2] = {};     // CP-ALS start device timing (the caller's events)

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
    std::future<TemporalDraw> next_draw;  // the next batch's temporal rows, drawn ahead
    void upload_mapped(DevBuf<double>& dst, const double* h, size_t n);
    const void* stage_input(const void* data, int dtype, int location, size_t n);
    void check_finite(const void* dX, int dtype, size_t n);
    void ensure_c_capacity(std::int64_t rows, cudaStream_t st);
    void begin(BatchCtx& b, const void* data, int dtype, int location, int order, const std::int64_t* dims,
               double* models_out, bool out_of_place, bool run_als = true);
    void merge_phase(BatchCtx& b, const double* models_all, double* rows_out);
    void finish(BatchCtx& b, const double* rows_all);
    void als_phase(BatchCtx& b, const double* dY, double* models_out, cudaStream_t as);
    void als_init_phase(BatchCtx& b, const double* dY, AlsEngine& e, cudaStream_t st);
    void als_sweep_phase(BatchCtx& b, double* models_out, AlsEngine& e, cudaStream_t st, int ahead);
    void post_merge(BatchCtx& b, double* models);
    void rollback_to(const BatchCtx& b);
    void snapshot(Snapshot& s);
    void restore(Snapshot& s);
    [[noreturn]] void fail_pending(BatchCtx& b);
    void begin_ctx(BatchCtx& b, bool first, std::int64_t t);
    void next_w_slot();
    void check_extents(const std::int64_t* dims);
    const void* temporal_last(const void* data, int dtype, int location, const std::int64_t* dims);
    void set_mode_strides();

public:
    int factor_slot(int mode) const;

private:
    void exchange_allgather(const double* send, double* recv, size_t count);

    Snapshot backup;
};

}  // namespace octen
