// Device engines for the three stages of the per-batch OCTen pipeline.
// All matrices are column-major fp64 unless noted (Eigen's default, as in the
// reference); tensors are first-index-fastest (tensor.hpp:32-34).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <future>
#include <memory>
#include <vector>

#include "devbuf.hpp"
#include "errors.hpp"
#include "octen_common.cuh"
#include "small_linalg.cuh"

namespace octen {

// ---------------------------------------------------------------------------
// Stage 2: batched CP-ALS over the P replica summaries (cp_als.cpp:240-359),
// all n_restarts restarts of every replica run concurrently.
// ---------------------------------------------------------------------------
struct AlsReplicaResult {
    double fit = 0.0;
    int iterations = 0;
    int restart = 0;
    int gevd_attempt = -1;  // -1: random init
    bool rescued = false;
    std::vector<double> fit_history, residual_history;
};

struct AlsState {  // per (replica, restart) problem, device resident
    double prev_fit;
    int active;
    int iterations;
    int rescued;
    int rng_init;
    int failed;
    int pad;
};

// NumericError text of a failed CP-ALS (kind 1 zero input, 2 non-finite
// factor at sweep a / mode b, 3 non-finite fit at sweep a).
std::string als_failure_message(int kind, int a, int b);

struct AlsFailure {
    int kind = 0, a = 0, b = 0;
};

// The host-RNG draws of one CP-ALS batch (restart seeds, GEVD slice
// mixtures, rescue seeds; cp_als.cpp:265-283, 110-121), a pure function of
// the per-replica seeds: prefetch_host_draws() computes the next batch's on a
// helper thread so they are off its critical path.
struct AlsHostDraws {
    int S = 0, Q = 0;
    std::vector<std::uint64_t> seeds, restart_seed, hres;
    std::vector<double> hw;
};
AlsHostDraws als_host_draws(const std::vector<std::uint64_t>& seeds, int S, int Q);

// One dimension-tree T-GEMM, T = Y x_mode F (als.cu; engine 1: tcgen05
// digit split, engine 0: DMMA), for kernel-level tests.
void als_tgemm(int P, int Q, int S, int R, int mode, const double* Y, const double* F, double* T, int engine,
               cudaStream_t st);

class AlsEngine {
public:
    // Y: P x Q^3 device summaries.  seeds: per replica AlsConfig.seed.
    void run(int P, int S, int Q, int R, int max_iters, double rel_tol, const double* dY,
             const std::vector<std::uint64_t>& seeds, cudaStream_t st);
    // run() in two parts: the start (norms, GEVD attempts, initial factors;
    // host syncs on `st`) and the sweeps with the results (on a stream
    // ordered after the start).  The pipelined ingest runs the next batch's
    // start on another engine while this one sweeps.
    void run_init(int P, int S, int Q, int R, int max_iters, double rel_tol, const double* dY,
                  const std::vector<std::uint64_t>& seeds, cudaStream_t st);
    void run_sweeps(cudaStream_t st);
    // Draw the host RNG of a later run() with these seeds now (helper thread).
    void prefetch_host_draws(const std::vector<std::uint64_t>& seeds, int S, int Q);

    // Results: factors P x 3 x Q x R, lambda P x R (device).
    DevBuf<double> Mf, Mlam;
    std::vector<AlsReplicaResult> results;
    int last_sweeps = 0;
    int host_syncs = 0;
    AlsFailure failure;  // set when run() throws a NumericError
    // Live kernel timing (CUDA events on the launching lane stream, summed
    // after each run; sampled: lane 0, every fifth sweep): the T-GEMMs and
    // the MTTKRP (+ fused update) launches, with their algorithmic flops /
    // bytes.  `sweeps` counts every sweep.
    struct KernelStats {
        double gemm_ms = 0, gemm_flops = 0, mttkrp_ms = 0, mttkrp_bytes = 0;
        long long gemm_launches = 0, mttkrp_launches = 0, sweeps = 0;
    } kstats;
    ~AlsEngine();

private:
    void alloc(int P, int S, int Q, int R, int max_iters);
    int P_ = 0, S_ = 0, Q_ = 0, R_ = 0, I_ = 0;
    DevBuf<double> normx2, F, G, lam, T, KR, Mb, Vinv, fit_hist, res_hist, ws, tscbuf;
    static constexpr int kMaxLanes = 8;
    int* hact = nullptr;  // host-mapped per-sweep activity flags
    size_t hact_n = 0;
    cudaStream_t lane_st[kMaxLanes] = {};   // sweep lanes 1..L-1 (lane 0 runs on the caller's stream)
    cudaStream_t lane_hp[kMaxLanes] = {};   // OCTEN_ALS_GEMM_STREAM=1: high-priority lanes
    cudaStream_t gemm_st = nullptr;         //   and the lanes' T-GEMMs (low priority)
    cudaStream_t lane_gemm[kMaxLanes] = {}; // OCTEN_ALS_GEMM_STREAM=2: one low-priority GEMM stream per lane
    // lane_ev: [0] fork/join, [kGin + l] lane -> GEMM stream, [kGout + l]
    // GEMM stream -> lane, [kSweepEv + kMaxLanes (sweep & 3) + l] end of a sweep
    static constexpr int kGin = 1, kGout = 1 + kMaxLanes, kSweepEv = 1 + 2 * kMaxLanes;
    cudaEvent_t lane_ev[1 + 6 * kMaxLanes] = {};
    std::vector<cudaEvent_t> kev;   // timing event pool: pairs (start, end)
    struct KevRec {
        int ev;        // index of the start event (end = ev + 1)
        bool gemm;     // T-GEMM (else MTTKRP)
        double work;   // flops (GEMM) or bytes (MTTKRP)
    };
    std::vector<KevRec> krec;
    DevBuf<double> Gev, EV, Ur, Wmix, Smix, Tmp6, Pm, Hh, gscr;
    DevBuf<std::uint8_t> oz_a;  // digit slices of the summaries, 3 orientations (ozaki.hpp)
    DevBuf<int> oz_e;           // their row exponents
    DevBuf<std::uint8_t> oz_fd; // digits of the factors (written by the mode updates)
    DevBuf<double> oz_fcs;      // their column scales
    DevBuf<int> usable, att_start, att_used, todo, peel_fail, eigdbg, mcount;
    DevBuf<AlsState> state;
    DevBuf<DevStatus> err;
    DevBuf<Mt64> rngs;
    DevBuf<std::uint64_t> rescue_seed;
    std::future<AlsHostDraws> next_draws;
    std::shared_ptr<void> pend;  // run_init -> run_sweeps (als.cu)
    unsigned char* res_pin = nullptr;  // pinned landing area of run()'s results (one read)
    size_t res_cap = 0;
};

// ---------------------------------------------------------------------------
// Stage 1: compression of one temporal batch into the P summaries,
// Y_p += X x1 U_p^T x2 V_p^T x3 W_p^T (compression.cpp:108-153).
// ---------------------------------------------------------------------------
class CompressEngine {
public:
    // Projections (host, column-major per replica: U_p I x Q, V_p J x Q).
    void set_projections(int P, int Q, int shared, std::int64_t I, std::int64_t J, const double* hU,
                         const double* hV, cudaStream_t st);
    // Accumulate the compression of batch X (I x J x t, first index fastest,
    // device) with temporal rows W (P x t x Q col-major per replica, device)
    // into Y (P x Q^3, device).  X is fp32 or fp64.
    void compress_f32(const float* dX, std::int64_t t, const double* dW, double* dY, cudaStream_t st);
    void compress_f64(const double* dX, std::int64_t t, const double* dW, double* dY, cudaStream_t st);
    // The same in two phases.  project: modes 1-2 of the whole batch into
    // Z2 (P x Q^2 x t), chunk by chunk; chunk c waits for ready[c] when given
    // (ready_slices slices per chunk) and is scanned for non-finite values
    // into *flag when flag != null.  accumulate: Y = Yin + Z2 x3 W (fp64; in
    // place when Yin == Y).
    void project(const void* dX, int dtype, std::int64_t t, cudaStream_t st, const cudaEvent_t* ready,
                 std::int64_t ready_slices, int* flag);
    void accumulate(int dtype, std::int64_t t, const double* dW, const double* dYin, double* dY, cudaStream_t st);
    // The same for t slices whose temporal rows are rows [k0, k0 + t) of a
    // W with t_total rows per replica (temporal sharding).
    void accumulate_rows(int dtype, std::int64_t t, const double* dW, std::int64_t t_total, std::int64_t k0,
                         double* dY, cudaStream_t st);

    int P = 0, Q = 0, shared = 0;
    std::int64_t I = 0, J = 0, Meff = 0;
    // element strides in Y_p of (non-temporal slot 0, slot 1, temporal): the
    // summaries keep the stream's mode order (set_temporal_mode)
    int ys[3] = {1, 0, 0};
    void set_temporal_mode(int tm) {
        const int q2 = Q * Q;
        if (tm == 2) { ys[0] = 1; ys[1] = Q; ys[2] = q2; }
        else if (tm == 1) { ys[0] = 1; ys[1] = q2; ys[2] = Q; }
        else { ys[0] = Q; ys[1] = q2; ys[2] = 1; }
    }
    DevBuf<float> A32;   // Meff x I row-major (deduplicated shared columns)
    DevBuf<float> Ahi, Alo;  // TF32 split of the fp64 projections (tcgen05 path)
    int lda_tc = 0;
    DevBuf<float> Vhi, Vlo;  // TF32 split of V: P*Q x ldv_tc, row p Q + b = V_p[:, b]
    int ldv_tc = 0;
    DevBuf<int> rowmap_id;   // identity row map (replica-contiguous Z1 of the tc path)
    bool used_tc = false;
    // cap on GEMM1's persistent grid (0: one CTA per SM); the pipelined
    // ingest sets it while the previous batch's CP-ALS sweeps run beside
    int g1_ctas = 0;
    DevBuf<double> A64;  // Meff x I row-major
    DevBuf<float> V32;   // P x J x Q
    DevBuf<double> V64;  // P x J x Q
    DevBuf<int> rowmap;  // P x Q -> row of A
    DevBuf<float> Z1f, Z2f;
    DevBuf<double> Z1d, Z2d;
    std::int64_t chunk_slices = 0;
    // device time of the mode-1 contraction (the dominant compression kernel)
    std::vector<cudaEvent_t> g1_events;  // pairs, reused
    int g1_used = 0;
    long long gemm1_launches = 0;
    double gemm1_flops = 0.0;  // algorithmic, accumulated
    double collect_gemm1_ms();  // call after the stream is synchronized
    cudaEvent_t event(int i);
    ~CompressEngine();
};

// Y_p += Z2_p (Q^2 x t) W_p (t x Q) for every replica (fp64 DMMA), Z2 fp32
// P x Q^2 x t (the mode-1/2 output layout of the dense path).
void accumulate_z2_f32(int P, int Q, std::int64_t t, const float* Z2, const double* dW, double* dY, cudaStream_t st);

// ---------------------------------------------------------------------------
// Stage 1, sparse input: compression of one COO temporal batch
// (SparseTensor, tensor.hpp:66-90, validated as tensor.cpp:87-102) into the
// P summaries without densifying it (coo.cu).
// ---------------------------------------------------------------------------
struct CooStatus {
    int bounds, nonfinite, dup, pad;  // first offending entry (input order), INT_MAX if none
    unsigned long long groups;        // distinct (k, i) pairs of the batch
};

class CooEngine {
public:
    CooEngine();
    ~CooEngine();
    // Projections (host, column-major per replica: U_p I x Q, V_p J x Q).
    void set_projections(int P, int Q, std::int64_t I, std::int64_t J, const double* hU, const double* hV,
                         cudaStream_t st);
    // Validate a COO batch (device arrays i, j, k int32 with k < t, values
    // fp32) and accumulate its compression with temporal rows W (P x t x Q,
    // device) into Y (P x Q^3, device).  Throws the reference's SparseTensor
    // errors before Y changes.
    void compress(std::int64_t t, std::int64_t nnz, const int* di, const int* dj, const int* dk, const float* dv,
                  const double* dW, double* dY, cudaStream_t st);
    // Fold the last compress's event times into the counters (synchronizes).
    void collect(cudaStream_t st);

    int P = 0, Q = 0, QP = 0, ldp = 0;
    std::int64_t I = 0, J = 0;
    DevBuf<float> U32, V32;  // I x (P QP), J x (P QP) row-major, zero-padded
    DevBuf<unsigned long long> keys, keys2;
    DevBuf<int> idx, idx2, off;
    DevBuf<int4> ent;
    DevBuf<char> sort_tmp;
    DevBuf<CooStatus> err;
    DevBuf<float> Z2;
    cudaEvent_t evs[4] = {};
    bool pending = false;
    double ms_prep = 0, ms_slice = 0, ms_accum = 0, groups_total = 0, nnz_total = 0;
    long long batches = 0;
};

// ---------------------------------------------------------------------------
// Stage 3: alignment and merge (recovery.cpp / streaming.cpp:89-177).
// ---------------------------------------------------------------------------
struct AlignResultHost {
    std::vector<int> perms;       // P x R
    std::vector<double> scales;   // P x 3 x R
    double min_match = 1.0, max_offdiag = 0.0;
    int ambiguous = 0;
};

class MergeEngine {
public:
    // Fixed-for-the-stream projections (host col-major, per replica).
    void set_projections(int P, int Q, int shared, int R, std::int64_t I, std::int64_t J, const double* hU,
                         const double* hV, cudaStream_t st);

    // Align replica models (device: factors P x 3 x Q x R, lambda P x R).
    // tgram: shared x shared temporal_shared_gram (host).
    void align(const double* dMf, const double* dMlam, const std::vector<double>& tgram, cudaStream_t st,
               AlignResultHost* out);
    // Full recover_batch: solves, refinement, gauge match, temporal append.
    // Y: P x Q^3; dW: P x t x Q; hist: PQ x R stacked (updated);
    // stored (device) nontemporal factors or null on the first batch.
    // Outputs A_fin (I x R), B_fin (J x R), new_rows (t x R), residual.
    void recover(const double* dY, const double* dW, std::int64_t t, double* dHist, const double* dStoredA,
                 const double* dStoredB, double* dAfin, double* dBfin, double* dRows, double* residual,
                 cudaStream_t st);
    // The non-temporal part of recover: solves, two refinement passes and the
    // gauge match (streaming.cpp:89-131) -> dAfin, dBfin.
    void recover_ab(const double* dStoredA, const double* dStoredB, double* dAfin, double* dBfin, cudaStream_t st);

    // Stage-level helpers (also exposed through the C-ABI for parity tests).
    void solve_nontemporal(int n, const double* dStack, double* dOut, cudaStream_t st);
    // temporal_stack_from_summaries for replicas [p0, p0 + pl), dY holding
    // those pl summaries; output stacked (P*Q x R) or replica-major (pl x Q x R).
    void temporal_stack(const double* dY, int p0, int pl, const double* dA, const double* dB, double* dOut,
                        bool replica_major, cudaStream_t st);
    void temporal_append(const double* dTstack, const double* dW, std::int64_t t, double* dHist, double* dRows,
                         double* residual, cudaStream_t st);

    int P = 0, Q = 0, shared = 0, R = 0;
    std::int64_t dims[2] = {0, 0};
    DevBuf<double> stacks;   // 3 x (PQ x R)
    DevBuf<double> Ud[2];    // P x d x Q
    DevBuf<double> Gp[2];    // P x d x d
    DevBuf<double> Lsum[2];  // d x d (Cholesky of sum_p G_p)
    DevBuf<double> Lsum_inv[2], Gw_inv;  // diagonal-block inverses of the factors
    DevBuf<double> Ginv[2];  // (sum_p G_p)^-1, full d x d
    int sum_rank[2] = {0, 0};
    // strides of (slot 0, slot 1, temporal) in the summaries (temporal_stack)
    int ys[3] = {1, 0, 0};
    void set_ystrides(const int* s) { ys[0] = s[0]; ys[1] = s[1]; ys[2] = s[2]; }
    bool sum_qr[2] = {false, false};  // full rank only by the QR rule: solve by QR each batch
    int qr_rank_check(int n, const double* w, int r, const double* rhs, double* x, cudaStream_t st);
    DevBuf<double> Lw[2];    // shared x shared whitener (non-temporal modes)
    int white_ok[2] = {0, 0};
    DevBuf<double> Lp[2];    // P x Q x Q chol(U_p^T U_p)
    DevBuf<int> lp_ok[2];    // P
    bool pair_solve = false;
    DevBuf<double> solved[2], Gw, rhs, tmp, tg, red, sw, sw2, maxdiag, RF, SC, sims, tscr;
    DevBuf<double> kws;  // split-K partials
    DevBuf<int> ranks, perms, iscr;
    DevBuf<DevStatus> err;
    std::vector<int> last_perm;
};

}  // namespace octen
