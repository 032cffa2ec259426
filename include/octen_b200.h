/* octen_b200.h -- C-ABI of the B200-native OCTen per-batch pipeline.
 *
 * Drop-in boundary for the reference library `cpstream`
 * (/root/reference/proj, C++20 + Eigen).  The reference exposes no FFI; its
 * boundary is the C++ API of the static library (proj/src/CMakeLists.txt:1-13).
 * Each entry point below replaces the reference function cited beside it and
 * takes plain pointers in the reference's own layouts:
 *   - matrices: column-major fp64 (Eigen::MatrixXd default);
 *   - tensors:  first index fastest (proj/include/cpstream/tensor.hpp:32-34);
 *   - per-replica blocks are stacked replica-major.
 * No torch types cross this boundary.
 *
 * Errors follow proj/include/cpstream/errors.hpp: every call returns
 * OCTEN_OK or the status of the exception the reference would throw; the
 * message (the reference's text) is available from octen_last_error() in the
 * calling thread.  A stream handle is not thread-safe (one ingest at a time,
 * SPEC.md:453); distinct handles are independent.
 */
#ifndef OCTEN_B200_H
#define OCTEN_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define OCTEN_OK 0
#define OCTEN_ERR_CONFIG 2   /* cpstream::ConfigError  */
#define OCTEN_ERR_NUMERIC 3  /* cpstream::NumericError */
#define OCTEN_ERR_IO 4       /* cpstream::IoError      */
#define OCTEN_ERR_CUDA 5     /* device failure          */
#define OCTEN_ERR_INTERNAL 6

#define OCTEN_F64 0 /* batch element type */
#define OCTEN_F32 1
#define OCTEN_HOST 0 /* batch location */
#define OCTEN_DEVICE 1

/* cpstream::AlsConfig (proj/include/cpstream/cp_als.hpp:25-31) */
typedef struct octen_als_config {
    int32_t rank;
    int32_t max_iters;
    double rel_tol;
    int32_t n_restarts;
    uint64_t seed;
} octen_als_config;

/* cpstream::StreamConfig (proj/include/cpstream/streaming.hpp:15-27) */
typedef struct octen_stream_config {
    int32_t rank;
    int32_t p;
    int32_t q;
    int32_t shared;
    int32_t temporal_mode; /* -1: last mode */
    octen_als_config als;
    uint64_t seed;
    int32_t enforce_bounds;
    int32_t workers; /* accepted for API parity; the device path is schedule-free */
    int32_t strict;
    double residual_warning;
    int32_t device; /* CUDA ordinal */
} octen_stream_config;

/* cpstream::BatchRecord (proj/include/cpstream/streaming.hpp:31-42) */
typedef struct octen_batch_record {
    int64_t batch_index;
    int64_t t_new;
    double temporal_residual;
    double min_match_similarity;
    double max_offdiag_similarity;
    int32_t warned;
    double compress_seconds;
    double als_seconds;
    double recover_seconds;
    double total_seconds;
} octen_batch_record;

typedef struct octen_stream octen_stream;

/* Message of the last failed call in this thread (empty if none). */
const char* octen_last_error(void);
/* Library version string. */
const char* octen_version(void);
/* Number of kernels this library has launched in this process. */
int64_t octen_launch_count(void);
/* Kernel path counters of this process (no reference counterpart; the
 * evidence that the tensor-core path ran):
 * out[0] all launches (= octen_launch_count), out[1] tcgen05 launches of
 * the fp32 dense compression (GEMM1 + mode-2), out[2] fp32 compression
 * chunks that ran on the SIMT GEMM because their shape is outside the
 * tcgen05 kernels' limits, out[3] DMMA launches of the fp64 compression,
 * out[4] tcgen05 (kind::i8 digit-split fp64) launches of the CP-ALS T-GEMM.
 * out must hold 5 values. */
void octen_kernel_counts(int64_t* out);

/* init_stream (proj/include/cpstream/streaming.hpp:64; src/streaming.cpp:181-256).
 * data: I x J x t0 batch, first index fastest, dtype OCTEN_F64/F32 at
 * location OCTEN_HOST/DEVICE; dims[order].  On success *out owns the stream. */
int octen_stream_init(const octen_stream_config* cfg, const void* data, int dtype, int location, int order,
                      const int64_t* dims, octen_stream** out);

/* ingest_batch (streaming.hpp:70; src/streaming.cpp:258-346). */
int octen_stream_ingest(octen_stream* s, const void* data, int dtype, int location, int order,
                        const int64_t* dims);

/* Start the host->device copy of a LATER batch (host memory; pinned for
 * the copy to overlap) on a copy stream of the handle, so it runs while the
 * device works on the batches before it.  The next octen_stream_ingest /
 * octen_stream_begin whose data pointer, dtype and dims match the oldest
 * pending prefetch consumes the copy instead of transferring the batch again.
 * At most two prefetches may be pending; the host buffer must stay unchanged
 * until its batch is ingested.  (An extension: the reference's ingest_batch
 * is synchronous and has no prefetch, streaming.hpp:70.) */
int octen_stream_prefetch(octen_stream* s, const void* data, int dtype, int order, const int64_t* dims);

/* Fitness (proj/src/eval.cpp:10-20, 100 (1 - |X - Xhat| / |X|)) of the
 * stream's current model on slices [k0, k0 + t) of the stream, given as a
 * batch I x J x t (dtype/location as octen_stream_ingest); computed on the
 * device without materialising the reconstruction. */
/* Pipelined ingest_batch (no reference counterpart; same results as
 * octen_stream_ingest, bit for bit), two batches in flight: the batch is
 * compressed and its CP-ALS started (GEVD attempts) before the call returns,
 * beside the previous batch's CP-ALS sweeps (library worker thread) and the
 * merge before them (another worker); then the batch's sweeps and the
 * previous batch's merge are posted.  A CP-ALS error of batch b is returned
 * by the call of batch b+1, a merge error by the call of batch b+2 or
 * octen_stream_sync (or any getter), with the reference's "batch N: "
 * prefix; the later batches are rolled back (not ingested), so the state is
 * the reference's after its failed ingest_batch.  The batch buffer may be
 * reused when the call returns.  Strict streams and the first batch run
 * synchronously. */
int octen_stream_ingest_async(octen_stream* s, const void* data, int dtype, int location, int order,
                              const int64_t* dims);
/* Finish the batches in flight of octen_stream_ingest_async (the sweeps and
 * merges); returns the first error. */
int octen_stream_sync(octen_stream* s);
/* Model publication for pipelined callers: with on != 0 every finished batch
 * copies its model to host memory, readable with octen_stream_last_model
 * without waiting for the merge in flight. */
int octen_stream_set_publish(octen_stream* s, int on);
/* The last published model: info[0] = rows of the temporal factor (slices),
 * info[1] = batches finished (0: nothing published yet, nothing copied);
 * a, b: the two non-temporal factors in mode order (I x R, J x R), c: the
 * temporal factor (c_rows_cap x R, first info[0] rows written), lambda (R);
 * col-major. */
int octen_stream_last_model(octen_stream* s, int64_t* info, double* a, double* b, double* c, int64_t c_rows_cap,
                            double* lambda);

/* Library-owned collectives of a sharded stream (parallel_replicas,
 * proj/src/streaming.cpp:45-69, across GPUs over NCCL on the stream's own
 * CUDA stream; no reference counterpart).  octen_nccl_get_unique_id fills a
 * 128-byte ncclUniqueId on one rank, which the caller distributes;
 * octen_stream_create_nccl creates rank shard_rank of shard_world with a
 * communicator from that id (uid128) or borrows the caller's ncclComm_t
 * (nccl_comm, uid128 NULL).  octen_stream_ingest_sharded runs one batch
 * (init on the first) with the replicas sharded: compress + CP-ALS of the
 * owned replicas, ncclAllGather of the replica models, the merge,
 * ncclAllGather of the temporal-stack rows, the temporal append.
 * octen_stream_ingest_temporal runs one batch whose slices
 * [k_off, k_off + local t) of t_total are this rank's: partial summaries of
 * every replica, ncclReduceScatter to the owners, then the same.  Every rank
 * calls with the same sequence of batches. */
int octen_nccl_get_unique_id(uint8_t* out128);
int octen_stream_create_nccl(const octen_stream_config* cfg, int shard_rank, int shard_world, const uint8_t* uid128,
                             void* nccl_comm, octen_stream** out);
int octen_stream_ingest_sharded(octen_stream* s, const void* data, int dtype, int location, int order,
                                const int64_t* dims);
int octen_stream_ingest_temporal(octen_stream* s, const void* data, int dtype, int location, int order,
                                 const int64_t* dims_local, int64_t k_off, int64_t t_total);

/* checkpoint_save / checkpoint_load (proj/include/cpstream/streaming.hpp:78-79;
 * src/checkpoint.cpp:125-295): the OCTS container of an unsharded stream
 * between batches, byte-compatible with the reference's.  save with
 * buf == NULL returns the size only; errors of a bad container are
 * OCTEN_ERR_IO with the reference's messages. */
int octen_stream_checkpoint_save(octen_stream* s, uint8_t* buf, int64_t cap, int64_t* size);
int octen_stream_checkpoint_load(const uint8_t* bytes, int64_t n, int device, octen_stream** out);

/* read_tensor_coo (proj/include/cpstream/io.hpp; src/io.cpp:49-84): the
 * 1-based COO text format ("order d1 .. dN" header, one "i1 .. iN value" line
 * per entry), parsed on the host with the reference's IoError messages and
 * the SparseTensor constructor's per-entry checks (bounds, finiteness) in
 * IoError("'path': ...") form; duplicates are reported by the device COO
 * compression.  Entries come back 0-based, nnz x order row-major. */
typedef struct octen_coo_file octen_coo_file;
int octen_read_coo(const char* path, octen_coo_file** out);
int octen_coo_file_info(const octen_coo_file* f, int64_t* order, int64_t* dims, int64_t* nnz);
int octen_coo_file_entries(const octen_coo_file* f, int64_t* indices, double* values);
void octen_coo_file_destroy(octen_coo_file* f);

/* On-device generate_synthetic (proj/src/commands.cpp:110-134; SynthSpec,
 * proj/include/cpstream/commands.hpp): U(0,1) factors from derive(seed,
 * {9, n}), X = reconstruct(model) + N(mu, sigma) in flat order from one
 * mt19937_64 stream derive(seed, {10}) with the reference's Box-Muller.
 * octen_synth_next writes the next t slices along the last mode (I x J x t,
 * first index fastest) to device memory as fp64 or fp32; batches come in
 * stream order.  Values equal the reference's up to the last ulp of
 * log/sin/cos.  Order-3 tensors. */
typedef struct octen_synth octen_synth;
int octen_synth_create(int order, const int64_t* dims, int rank, uint64_t seed, double noise_mu,
                       double noise_sigma, int device, octen_synth** out);
int octen_synth_next(octen_synth* h, int64_t t, void* out_device, int dtype);
/* The normalized truth model (model.normalize()): factors[n] dims[n] x rank. */
int octen_synth_truth(const octen_synth* h, double* const* factors, double* lambda);
void octen_synth_destroy(octen_synth* h);

/* congruence (proj/src/eval.cpp:22-46): per-component factor match score
 * (product over modes of |cos|) after exhaustive (rank <= 6) or greedy
 * matching.  ground/est: factors of every mode stacked, dims[n] x rank
 * col-major each; scores: rank.  Host computation. */
int octen_congruence(int order, int rank, const int64_t* dims, const double* ground, const double* est,
                     double* scores);
int octen_stream_batch_fitness(octen_stream* s, const void* data, int dtype, int location, int order,
                               const int64_t* dims, int64_t k0, double* fitness);

void octen_stream_destroy(octen_stream* s);

/* Stream state accessors (StreamState, streaming.hpp:48-59).
 * info[0..7] = order, I, J, K(slices_seen), rank, p, q, batches_seen. */
int octen_stream_info(const octen_stream* s, int64_t* info);
/* measure_footprint (proj/include/cpstream/eval.hpp; src/eval.cpp:48-60) of
 * the stream's device-resident state: out[0] replica bytes, out[1] summary
 * bytes (owned replicas), out[2] factor bytes, out[3] accumulator bytes. */
int octen_stream_footprint(const octen_stream* s, int64_t* out);

/* KruskalModel factor `mode` (dim x rank, col-major; the stream's mode
 * order) and lambda (rank).  octen_stream_get_model: the factors of modes
 * 0, 1, 2 into a, b, c. */
int octen_stream_get_factor(const octen_stream* s, int mode, double* out);
int octen_stream_get_lambda(const octen_stream* s, double* out);
/* The whole model in one call (one synchronisation): a I x R, b J x R,
 * c K x R (col-major), lambda R. */
int octen_stream_get_model(const octen_stream* s, double* a, double* b, double* c, double* lambda);
/* Live kernel timing of the CP-ALS stage, cumulative over the stream (CUDA
 * events on the launching streams; no reference counterpart): out[0] T-GEMM
 * milliseconds, out[1] T-GEMM launches, out[2] their algorithmic flops,
 * out[3] MTTKRP (+ fused update) milliseconds, out[4] launches, out[5] bytes
 * of the partial contractions they read, out[6] sweeps, out[7] reserved. */
int octen_stream_get_kernel_stats(const octen_stream* s, double* out);
/* Number of BatchRecords in the stream's log (streaming.hpp:57: one per
 * successful init/ingest; a failed batch still counts in batches_seen). */
int octen_stream_log_size(const octen_stream* s, int64_t* n);
/* BatchRecord of log entry `index` (0 = init). */
int octen_stream_get_record(const octen_stream* s, int64_t index, octen_batch_record* out);
/* SummaryState: y (p x Q^3; a sharded handle returns its p_local owned
 * replicas) and history (p x Q x rank). */
int octen_stream_get_summaries(const octen_stream* s, double* y);
int octen_stream_get_history(const octen_stream* s, double* h);
/* The per-replica CP-ALS models of the last batch: factors p x 3 x Q x rank,
 * lambda p x rank. */
int octen_stream_get_replica_models(const octen_stream* s, double* factors, double* lambda);
/* Cumulative device time (CUDA events on the stream's own CUDA stream), ms:
 * out[0] compress stage, out[1] CP-ALS stage, out[2] merge stage,
 * out[3] mode-1 contraction kernels; out[4] their algorithmic flops,
 * out[5] their launch count. */
int octen_stream_get_stage_times(const octen_stream* s, double* out);

/* ---- replica-sharded streams (multi-GPU, one process per GPU) ----
 * The reference fans replicas out over worker threads (streaming.cpp:36-69,
 * parallel_replicas); here rank g of `shard_world` owns replicas
 * [p0, p0 + p_local), chunk = ceil(p / shard_world): it compresses every
 * batch into, and runs CP-ALS on, its own replicas, then runs the alignment
 * and merge redundantly (bit-identical on every rank) after two all-gathers
 * that the CALLER performs between the phases over any transport (NCCL via
 * torch.distributed in bench.py):
 *   octen_stream_begin  -> models_out : sizes[0] doubles  (device pointer)
 *   all-gather          -> models_all : shard_world * sizes[0], rank order
 *   octen_stream_merge  -> rows_out   : sizes[1] doubles  (device pointer)
 *   all-gather          -> rows_all   : shard_world * sizes[1], rank order
 *   octen_stream_finish
 * The first begin on a new handle performs init_stream; later ones
 * ingest_batch.  A CP-ALS failure on one rank travels in the exchanged block
 * so every rank raises the same NumericError in merge (no rank is left
 * waiting in a collective).  octen_stream_init/ingest are the three phases
 * back to back with shard_world == 1. */
int octen_stream_create(const octen_stream_config* cfg, int shard_rank, int shard_world, octen_stream** out);
/* sizes[0..5] = models doubles per rank, rows doubles per rank, p0, p_local,
 * shard_rank, shard_world. */
int octen_stream_exchange_sizes(const octen_stream* s, int64_t* sizes);
int octen_stream_begin(octen_stream* s, const void* data, int dtype, int location, int order, const int64_t* dims,
                       double* models_out);
int octen_stream_merge(octen_stream* s, const double* models_all, double* rows_out);
int octen_stream_finish(octen_stream* s, const double* rows_all);

/* ---- temporal sharding of the compression (the largest tensors) ----
 * Instead of octen_stream_begin, rank g compresses only its share of the
 * batch's slices, [k_off, k_off + dims_local[2]) of t_total, into partial
 * summaries of EVERY replica (the compression is additive over slices,
 * compression.cpp:141-153), and the caller reduce-scatters them by owner:
 *   octen_stream_begin_temporal -> partial_out : shard_world * B doubles (device)
 *                                   block g = replicas of rank g (chunk x Q^3)
 *                                   + 1 status double (non-finite flag)
 *   reduce-scatter (sum)         -> owned      : B doubles (this rank's block)
 *   octen_stream_begin_reduced   -> models_out (as octen_stream_begin)
 * then the all-gathers / merge / finish as in the replica-sharded protocol.
 * B = octen_stream_partial_block_size().  A non-finite value on any rank
 * makes every rank raise the same NumericError in begin_reduced.  Results
 * equal the unsharded stream up to the summation order of the partials. */
int octen_stream_partial_block_size(const octen_stream* s, int64_t* n);
int octen_stream_begin_temporal(octen_stream* s, const void* data, int dtype, int location, int order,
                                const int64_t* dims_local, int64_t k_off, int64_t t_total, double* partial_out);
int octen_stream_begin_reduced(octen_stream* s, const double* owned_block, double* models_out);

/* ---- stage-level entry points (the reference's L2 API, batched over replicas) ---- */

/* compress (proj/include/cpstream/compression.hpp:82-83; src/compression.cpp:108-130)
 * for all replicas: z[r] = x x1 U_r^T x2 V_r^T x3 W_r^T.
 * u: p x I x Q, v: p x J x Q, w: p x t x Q (col-major per replica), x: I x J x t
 * (dtype OCTEN_F64 or OCTEN_F32, host); z: p x Q^3 (host, overwritten). */
int octen_compress(int p, int q, int shared, int64_t I, int64_t J, int64_t t, const double* u, const double* v,
                   const double* w, const void* x, int dtype, double* z);

/* cp_als (proj/include/cpstream/cp_als.hpp:48; src/cp_als.cpp:240-359) on p
 * cubic Q^3 tensors (host, p x Q^3) with seeds[p]; cfg->seed is ignored.
 * factors: p x 3 x Q x rank, lambda: p x rank, fit: p, iterations: p. */
int octen_cp_als_batched(int p, int q, const double* y, const octen_als_config* cfg, const uint64_t* seeds,
                         double* factors, double* lambda, double* fit, int32_t* iterations);

/* One partial MTTKRP contraction of the device CP-ALS (the fp64 GEMM of
 * cp_als.cpp:296-303 as the dimension tree forms it): T = Y x_mode F for all
 * s restarts.  y: p x Q^3 (first index fastest); factors: p x s x 3 x Q x r
 * (restart-major, the mode's Q x r block column-major); t: p x Q^2 x (s r),
 * t[p][m + Q^2 (s_ r + c)] with m the two remaining indices, first fastest.
 * engine 1: int8 tcgen05 with exact digit splitting (the sweeps' path),
 * engine 0: the FP64 DMMA GEMM. */
int octen_als_tgemm(int p, int q, int s, int r, int mode, const double* y, const double* factors, double* t,
                    int engine);

/* align_replicas (proj/include/cpstream/recovery.hpp:43; src/recovery.cpp:106-291).
 * models: factors p x 3 x Q x R, lambda p x R; u/v: p x I x Q / p x J x Q;
 * tgram: shared x shared temporal_shared_gram.  stacks: 3 x (pQ x R),
 * perms: p x R, scales: p x 3 x R, sims[2] = {min_match, max_offdiag}. */
int octen_align_replicas(int p, int q, int shared, int rank, int64_t I, int64_t J, const double* u,
                         const double* v, const double* tgram, const double* factors, const double* lambda,
                         double* stacks, int32_t* perms, double* scales, double* sims);

/* recover_nontemporal (recovery.hpp:54; src/recovery.cpp:315-319) for mode
 * 0 (proj = stacked U^T) or 1 (stacked V^T): out = argmin |P~ out - stack|.
 * proj_blocks: p x d x Q, stack: pQ x R, out: d x R. */
int octen_recover_nontemporal(int p, int q, int64_t d, int rank, int mode, const double* proj_blocks,
                              const double* stack, double* out);

/* temporal_stack_from_summaries (recovery.hpp:98-99; src/recovery.cpp:429-462).
 * y: p x Q^3; u, v as above; a: I x R, b: J x R; out: pQ x R. */
int octen_temporal_stack_from_summaries(int p, int q, int rank, int64_t I, int64_t J, const double* y,
                                        const double* u, const double* v, const double* a, const double* b,
                                        double* out);

/* recover_temporal_append (recovery.hpp:85-88; src/recovery.cpp:341-427),
 * without column weights.  w: p x t x Q; history: p x Q x R (in/out, zero on
 * the first batch); new_rows: t x R; residual: relative solve residual. */
int octen_recover_temporal_append(int p, int q, int rank, int64_t t, const double* temporal_stack,
                                  const double* w, double* history, double* new_rows, double* residual);

/* ---- sparse (COO) temporal batches ----
 * The reference ingests coordinate data as SparseTensor
 * (proj/include/cpstream/tensor.hpp:66-90; read_tensor_coo, src/io.cpp:49-84),
 * whose constructor validates it (src/tensor.cpp:87-102), and densifies it
 * before compress/update_summaries (read_tensor_any, src/io.cpp:124-132;
 * src/compression.cpp:108-153).  These entry points compress the COO batch
 * directly, with the same result (to fp32 accumulation of the slice products)
 * and the same errors, checked before the summaries change:
 *   index out of bounds -> OCTEN_ERR_CONFIG "SparseTensor: index out of bounds"
 *   non-finite value    -> OCTEN_ERR_NUMERIC "SparseTensor: non-finite value"
 *   duplicate index     -> OCTEN_ERR_CONFIG "SparseTensor: duplicate index"
 * (the first offending entry in input order wins, as in the reference).
 * Entries are SoA: i[nnz], j[nnz], k[nnz] (0-based int32, k is the slice
 * within this batch, 0 <= k < t) and values[nnz] (fp32).  Q <= 128. */
typedef struct octen_coo_summaries octen_coo_summaries;

/* Device-resident SummaryState for a COO stream (compression.hpp:56-60,
 * init_summaries compression.cpp:132-139) over replicas u: p x I x Q,
 * v: p x J x Q (host, col-major per replica). */
int octen_coo_create(int p, int q, int64_t I, int64_t J, const double* u, const double* v, int device,
                     octen_coo_summaries** out);
/* update_summaries(S, compress(to_dense(batch))) for every replica.
 * w: p x t x Q temporal rows of this batch (col-major per replica).  With
 * location OCTEN_DEVICE, w/i/j/k/values are device pointers. */
int octen_coo_compress(octen_coo_summaries* h, int64_t t, const double* w, int64_t nnz, const int32_t* i,
                       const int32_t* j, const int32_t* k, const float* values, int location);
/* y: p x Q^3 (host). */
int octen_coo_get_summaries(const octen_coo_summaries* h, double* y);
/* Zero the summaries. */
int octen_coo_reset(octen_coo_summaries* h);
/* cp_als (cp_als.hpp:48) on every resident summary, seeds[p]; outputs as
 * octen_cp_als_batched (any output pointer may be NULL). */
int octen_coo_cp_als(octen_coo_summaries* h, const octen_als_config* cfg, const uint64_t* seeds, double* factors,
                     double* lambda, double* fit, int32_t* iterations);
/* Cumulative device times (CUDA events on the handle's stream):
 * out[0] validate + sort ms, out[1] slice-kernel ms, out[2] mode-3
 * accumulate ms, out[3] distinct (k, i) groups, out[4] nnz, out[5] batches,
 * out[6] CP-ALS ms, out[7] CP-ALS runs. */
int octen_coo_stage_times(const octen_coo_summaries* h, double* out);
/* Raw CUDA stream of the handle (cudaStream_t), for callers that order
 * their own device work against it. */
void* octen_coo_cuda_stream(const octen_coo_summaries* h);
void octen_coo_destroy(octen_coo_summaries* h);

/* One-shot compress of a COO batch (host arrays): z = p x Q^3 (host,
 * overwritten) = compress(to_dense(batch)) per replica. */
int octen_compress_coo(int p, int q, int64_t I, int64_t J, int64_t t, const double* u, const double* v,
                       const double* w, int64_t nnz, const int32_t* i, const int32_t* j, const int32_t* k,
                       const float* values, double* z);

#ifdef __cplusplus
}
#endif

#endif /* OCTEN_B200_H */
