// Batched semi-definite Cholesky (right-looking, 64-wide panels) and the
// matching triangular solves, fp64.  These carry the least-squares systems of
// the merge stage in normal-equation form:
//   recover_nontemporal / recover_nontemporal_weighted  (recovery.cpp:315-339)
//   recover_temporal_append                            (recovery.cpp:341-427)
// The reference solves them with ColPivHouseholderQR at threshold 1e-10 and
// raises NumericError on rank deficiency (recovery.cpp:26-38).  Here a pivot
// <= tol * max(diag) of the Gram matrix marks a deficient column (zeroed,
// counted), and rank = n - #deficient is reported to the host, which raises
// the reference's message.  See DESIGN.md §Numerics for the threshold.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <string>
#include <vector>

#include "devbuf.hpp"
#include "evprof.hpp"
#include "gemm_dmma.cuh"
#include "octen_common.cuh"
#include "small_linalg.cuh"

namespace octen {

constexpr int kCholNB = 64;

__global__ void chol_maxdiag_kernel(const double* A, int n, int lda, long long sA, double* maxdiag,
                                    int* rank) {
    const double* a = A + (size_t)blockIdx.x * sA;
    __shared__ double red[256];
    double m = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) m = fmax(m, a[i + (size_t)lda * i]);
    red[threadIdx.x] = m;
    __syncthreads();
    for (int s = blockDim.x / 2; s > 0; s >>= 1) {
        if ((int)threadIdx.x < s) red[threadIdx.x] = fmax(red[threadIdx.x], red[threadIdx.x + s]);
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        maxdiag[blockIdx.x] = red[0];
        rank[blockIdx.x] = n;
    }
}

// Factor the nb x nb diagonal block at offset k0 of every matrix and invert
// it (for the panel GEMM and the blocked solves) as a 2 x 2 block of 32 x 32
// halves:
//   L11 = chol(A11), X11 = L11^-1            (block_chol_inv_t, registers)
//   L21 = A21 X11^T;  A22 -= L21 L21^T        (shared-memory products)
//   L22 = chol(A22), X22 = L22^-1
//   X21 = -X22 L21 X11
// The fused register factorizations cost two barriers per column and touch
// only 528 elements (one or two per thread), so the 64 sequential steps are
// cheap; the coupling products are fully parallel.  A pivot <= tol * maxdiag
// is dead: its column of L and row of L^-1 become zero and the rank drops.
constexpr int kDiagThreads = 256;
constexpr int kHalf = kCholNB / 2;
constexpr int kDiagPer = (kHalf * (kHalf + 1) / 2 + kDiagThreads - 1) / kDiagThreads;  // packed elements per thread
constexpr int kDLD = kCholNB + 1;  // shared leading dimension
constexpr size_t kDiagSmem = (size_t)(2 * kCholNB * kDLD + kHalf * (kHalf + 1) + 160) * sizeof(double);
__device__ long long g_diag_tsc[16];  // OCTEN_PROFILE: phase clocks of block 0 at k0 == 0
#define DIAG_TSC(i) \
    if (blockIdx.x == 0 && k0 == 0 && threadIdx.x == 0) g_diag_tsc[(i)] = clock64();

__global__ void __launch_bounds__(kDiagThreads) chol_diag_kernel(double* A, int n, int lda, long long sA, int k0,
                                                                 double tol, const double* maxdiag, int* rank,
                                                                 double* Linv, int nblk) {
    extern __shared__ double diag_smem[];
    double* S = diag_smem;                  // A -> L (lower), column-major, ld kDLD
    double* X = S + kCholNB * kDLD;         // L^-1 (lower)
    double* T = X + kCholNB * kDLD;         // kHalf x (kHalf + 1)
    double* scr = T + kHalf * (kHalf + 1);  // 160
    double* a = A + (size_t)blockIdx.x * sA;
    const int nb = min(kCholNB, n - k0);
    const int tid = threadIdx.x;
    DIAG_TSC(0)
#pragma unroll
    for (int h = 0; h < kCholNB * kCholNB / (8 * kDiagThreads); ++h) {
        double v[8];
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            const int e = tid + kDiagThreads * (8 * h + r);
            const int i = e & (kCholNB - 1), j = e >> 6;
            v[r] = (i < nb && j < nb && i >= j) ? a[(k0 + i) + (size_t)lda * (k0 + j)] : 0.0;
        }
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            const int e = tid + kDiagThreads * (8 * h + r);
            const int i = e & (kCholNB - 1), j = e >> 6;
            S[i + kDLD * j] = v[r];
            X[i + kDLD * j] = 0.0;
        }
    }
    const double md = maxdiag[blockIdx.x];
    const double thr = (md > 0.0) ? tol * md : INFINITY;
    __syncthreads();
    DIAG_TSC(1)
    const int n1 = min(kHalf, nb);
    const int rk1 = block_chol_inv_t<kDiagPer, kDiagThreads>(S, kDLD, n1, thr, S, kDLD, X, kDLD, scr);
    DIAG_TSC(2)
    int dead = n1 - rk1;
    const int n2 = nb - n1;
    if (n2 > 0) {
        double* A21 = S + kHalf;                 // rows 32.., cols 0..31
        double* A22 = S + kHalf + kDLD * kHalf;  // rows 32.., cols 32..
        double* X21 = X + kHalf;
        double* X22 = X + kHalf + kDLD * kHalf;
        // T = A21 X11^T   (T(i, j) = sum_{k <= j} A21(i, k) X11(j, k))
        for (int e = tid; e < kHalf * kHalf; e += kDiagThreads) {
            const int i = e % kHalf, j = e / kHalf;
            double s0 = 0.0, s1 = 0.0;
            int k = 0;
            for (; k + 1 <= j; k += 2) {
                s0 += A21[i + kDLD * k] * X[j + kDLD * k];
                s1 += A21[i + kDLD * (k + 1)] * X[j + kDLD * (k + 1)];
            }
            if (k <= j) s0 += A21[i + kDLD * k] * X[j + kDLD * k];
            T[i + (kHalf + 1) * j] = (i < n2) ? s0 + s1 : 0.0;
        }
        __syncthreads();
        for (int e = tid; e < kHalf * kHalf; e += kDiagThreads) {
            const int i = e % kHalf, j = e / kHalf;
            A21[i + kDLD * j] = T[i + (kHalf + 1) * j];  // L21
        }
        __syncthreads();
        // A22 -= L21 L21^T (lower)
        for (int e = tid; e < kHalf * kHalf; e += kDiagThreads) {
            const int i = e % kHalf, j = e / kHalf;
            if (i < j) continue;
            double s0 = 0.0, s1 = 0.0;
            for (int k = 0; k < kHalf; k += 2) {
                s0 += A21[i + kDLD * k] * A21[j + kDLD * k];
                s1 += A21[i + kDLD * (k + 1)] * A21[j + kDLD * (k + 1)];
            }
            A22[i + kDLD * j] -= s0 + s1;
        }
        __syncthreads();
        DIAG_TSC(3)
        const int rk2 = block_chol_inv_t<kDiagPer, kDiagThreads>(A22, kDLD, n2, thr, A22, kDLD, X22, kDLD, scr);
        DIAG_TSC(4)
        dead += n2 - rk2;
        // X21 = -X22 (L21 X11): T = L21 X11, then X21 = -X22 T
        for (int e = tid; e < kHalf * kHalf; e += kDiagThreads) {
            const int i = e % kHalf, j = e / kHalf;
            double s0 = 0.0, s1 = 0.0;
            int k = j;
            for (; k + 1 < kHalf; k += 2) {
                s0 += A21[i + kDLD * k] * X[k + kDLD * j];
                s1 += A21[i + kDLD * (k + 1)] * X[k + 1 + kDLD * j];
            }
            if (k < kHalf) s0 += A21[i + kDLD * k] * X[k + kDLD * j];
            T[i + (kHalf + 1) * j] = s0 + s1;
        }
        __syncthreads();
        for (int e = tid; e < kHalf * kHalf; e += kDiagThreads) {
            const int i = e % kHalf, j = e / kHalf;
            double s0 = 0.0, s1 = 0.0;
            int k = 0;
            for (; k + 1 <= i; k += 2) {
                s0 += X22[i + kDLD * k] * T[k + (kHalf + 1) * j];
                s1 += X22[i + kDLD * (k + 1)] * T[k + 1 + (kHalf + 1) * j];
            }
            if (k <= i) s0 += X22[i + kDLD * k] * T[k + (kHalf + 1) * j];
            X21[i + kDLD * j] = -(s0 + s1);
        }
        __syncthreads();
    }
    DIAG_TSC(5)
    if (tid == 0 && dead) atomicSub(&rank[blockIdx.x], dead);
    // write back: L (lower of the nb x nb block, upper zeroed) and L^-1
    double* inv = Linv + ((size_t)blockIdx.x * nblk + k0 / kCholNB) * kCholNB * kCholNB;
    for (int e = tid; e < kCholNB * kCholNB; e += kDiagThreads) {
        const int i = e & (kCholNB - 1), j = e >> 6;
        const bool in = i < nb && j < nb;
        inv[e] = (in && i >= j) ? X[i + kDLD * j] : 0.0;
        if (in) a[(k0 + i) + (size_t)lda * (k0 + j)] = (i >= j) ? S[i + kDLD * j] : 0.0;
    }
    DIAG_TSC(6)
}

// Rows below the diagonal block: L21 = A21 * L11^-T as an in-place GEMM
// (one block owns whole rows: N = nb <= BN), dead columns come out zero.
struct PanelA {
    double* A;
    int lda;
    long long sA;
    int r0, k0;
    __device__ double operator()(int b, int m, int k) const {
        return A[(size_t)b * sA + (r0 + m) + (size_t)lda * (k0 + k)];
    }
};
struct PanelB {  // B(k, j) = Linv(j, k) of diagonal block kb of matrix b
    const double* Linv;
    int nblk, kb;
    __device__ double operator()(int b, int k, int j) const {
        return Linv[((size_t)b * nblk + kb) * kCholNB * kCholNB + j + kCholNB * k];
    }
};
struct PanelC {
    double* A;
    int lda;
    long long sA;
    int r0, k0;
    __device__ void operator()(int b, int m, int j, double v) const {
        A[(size_t)b * sA + (r0 + m) + (size_t)lda * (k0 + j)] = v;
    }
};

// Trailing update of the right-looking step: for the lower triangle of the
// trailing block (rows/columns r0..n-1)
//   A(i, j) -= sum_k L21(i, k) L21(j, k),   L21 = A[r0:, k0:k0+nb]
// One CTA per 64 x 64 lower tile (tile (ti, tj), ti >= tj) and matrix: both
// panel slices are staged whole in shared memory (K = nb <= 64), the product
// runs on the FP64 tensor cores (DMMA m8n8k4, 8 warps x 32 x 16), and the
// result goes back through shared memory so the read-modify-write of A is
// column-coalesced.
constexpr int kTrailLD = kCholNB + 4;

// With k0b >= 0 the update carries a second (earlier, delayed) panel of 64
// columns at k0b as well: A(i, j) -= sum_k L(i, k0b + k) L(j, k0b + k) + ...,
// one read-modify-write of A for both (rank-128 update).
__global__ void __launch_bounds__(256, 3) chol_trail_kernel(double* A, int n, int lda, long long sA, int r0, int k0,
                                                         int nb, int part, int ntiles, int ntasks, int k0b) {
    extern __shared__ double trail_smem[];
    double* Pi = trail_smem;                       // [64 k][kTrailLD m]
    double* Pj = trail_smem + kCholNB * kTrailLD;  // [64 k][kTrailLD m]
    // part 0: every lower tile; 1: tile column tj = 0 only (the next panel
    // column, on the critical path); 2: tile columns tj >= 1 (lookahead).
    // Tasks (tile, matrix) are strided over the grid, so a capped grid
    // leaves room on the SMs for the critical chain's kernels.
    for (int task = blockIdx.x; task < ntasks; task += gridDim.x) {
    const int t = task % ntiles, mat = task / ntiles;
    int ti, tj;
    if (part == 1) {
        ti = t;
        tj = 0;
    } else {
        ti = (int)((sqrtf(8.0f * (float)t + 1.0f) - 1.0f) * 0.5f);
        while ((ti + 1) * (ti + 2) / 2 <= t) ++ti;
        while (ti * (ti + 1) / 2 > t) --ti;
        tj = t - ti * (ti + 1) / 2;
        if (part == 2) {
            ++ti;
            ++tj;
        }
    }
    double* a = A + (size_t)mat * sA;
    const int i0 = r0 + kCholNB * ti, j0 = r0 + kCholNB * tj;
    const int tid = threadIdx.x;
    const int lane = tid & 31, warp = tid >> 5;
    const int g = lane >> 2, t4 = lane & 3;
    const int wm = (warp & 1) * 32, wn = (warp >> 1) * 16;
    double acc[4][2][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    for (int pnl = k0b >= 0 ? 0 : 1; pnl < 2; ++pnl) {
    const int kc = pnl == 0 ? k0b : k0;  // the delayed panel first, then this step's
    const int nbp = pnl == 0 ? kCholNB : nb;
    // panels: batches of loads into registers, then shared stores
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        double pi[8], pj[8];
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            const int e = tid + 256 * (8 * h + r);
            const int m = e & (kCholNB - 1), kk = e >> 6;
            const bool kin = kk < nbp;
            pi[r] = (kin && i0 + m < n) ? a[(i0 + m) + (size_t)lda * (kc + kk)] : 0.0;
            pj[r] = (kin && j0 + m < n) ? a[(j0 + m) + (size_t)lda * (kc + kk)] : 0.0;
        }
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            const int e = tid + 256 * (8 * h + r);
            const int m = e & (kCholNB - 1), kk = e >> 6;
            Pi[kk * kTrailLD + m] = pi[r];
            Pj[kk * kTrailLD + m] = pj[r];
        }
    }
    __syncthreads();
    const int kend = (nbp + 3) & ~3;
    for (int kk = 0; kk < kend; kk += 4) {
        double fa[4], fb[2];
#pragma unroll
        for (int i = 0; i < 4; ++i) fa[i] = Pi[(kk + t4) * kTrailLD + wm + i * 8 + g];
#pragma unroll
        for (int j = 0; j < 2; ++j) fb[j] = Pj[(kk + t4) * kTrailLD + wn + j * 8 + g];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 2; ++j) dmma_m8n8k4(acc[i][j][0], acc[i][j][1], fa[i], fb[j]);
    }
    __syncthreads();
    }  // panels
    // stage the 64 x 64 product column-major (ld 65) over the panel buffers
    double* Cs = trail_smem;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
            for (int v = 0; v < 2; ++v) {
                const int m = wm + i * 8 + g, nn = wn + j * 8 + 2 * t4 + v;
                Cs[m + (kCholNB + 1) * nn] = acc[i][j][v];
            }
    __syncthreads();
    // read-modify-write of the C tile (lower part), 8 loads in flight per thread
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        double cv[8];
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            const int e = tid + 256 * (8 * h + r);
            const int m = e & (kCholNB - 1), nn = e >> 6;
            const int gi = i0 + m, gj = j0 + nn;
            cv[r] = (gi < n && gj < n && gi >= gj) ? a[gi + (size_t)lda * gj] : 0.0;
        }
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            const int e = tid + 256 * (8 * h + r);
            const int m = e & (kCholNB - 1), nn = e >> 6;
            const int gi = i0 + m, gj = j0 + nn;
            if (gi < n && gj < n && gi >= gj) a[gi + (size_t)lda * gj] = cv[r] - Cs[m + (kCholNB + 1) * nn];
        }
    }
    __syncthreads();  // Cs aliases the panel buffers of the next task
    }
}

// In-place batched semi-definite Cholesky.  Lower triangle holds L on return;
// the strict upper triangle outside the diagonal blocks is left as it was
// (the solves below read only the lower triangle).  rank[b] (device) = n - #deficient pivots.
// linv receives the inverses of the diagonal blocks (batch x nblk x 64 x 64),
// used by the panel GEMM here and by the blocked solves below.
inline void chol_batched(double* A, int n, int lda, long long sA, int batch, double tol, double* maxdiag,
                         int* rank, DevBuf<double>& linv, cudaStream_t st) {
    if (batch <= 0 || n <= 0) return;
    constexpr size_t kTrailSmem = 2 * kCholNB * kTrailLD * sizeof(double);
    static PerDevice attr;
    attr.once([&] {
        OCTEN_CUDA(cudaFuncSetAttribute(chol_trail_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)kTrailSmem));
        OCTEN_CUDA(cudaFuncSetAttribute(chol_diag_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)kDiagSmem));
    });
    const int nblk = (n + kCholNB - 1) / kCholNB;
    linv.reserve((size_t)batch * nblk * kCholNB * kCholNB);
    chol_maxdiag_kernel<<<batch, 256, 0, st>>>(A, n, lda, sA, maxdiag, rank); OCTEN_LAUNCHED(1);
    // Lookahead (depth 1): the trailing update of step k is split into the
    // next block column (part 1) and the rest (part 2).  The critical chain
    // diag -> panel -> part 1 runs on a high-priority stream, part 2 on the
    // caller's stream, so part 2 of step k overlaps the diagonal
    // factorization and panel of step k+1 (the scheduler hands freed SMs to
    // the high-priority CTAs first).  Part 1 of step k+1 waits for part 2 of
    // step k: both update block column k+2.
    // The chain's stream priority: chain_priority_over (octen_common.cuh).
    static thread_local cudaStream_t crit_by_level[8] = {};
    static thread_local std::vector<cudaEvent_t> ev_panel, ev_rest;
    static thread_local cudaEvent_t ev_start = nullptr, ev_end = nullptr;
    const int cprio = chain_priority_over(st);
    cudaStream_t& crit = crit_by_level[(cprio < 0 ? -cprio : cprio) & 7];
    if (!crit) OCTEN_CUDA(cudaStreamCreateWithPriority(&crit, cudaStreamNonBlocking, cprio));
    if (!ev_start) {
        OCTEN_CUDA(cudaEventCreateWithFlags(&ev_start, cudaEventDisableTiming));
        OCTEN_CUDA(cudaEventCreateWithFlags(&ev_end, cudaEventDisableTiming));
    }
    while ((int)ev_panel.size() < nblk) {
        cudaEvent_t a, b;
        OCTEN_CUDA(cudaEventCreateWithFlags(&a, cudaEventDisableTiming));
        OCTEN_CUDA(cudaEventCreateWithFlags(&b, cudaEventDisableTiming));
        ev_panel.push_back(a);
        ev_rest.push_back(b);
    }
    OCTEN_CUDA(cudaEventRecord(ev_start, st));
    OCTEN_CUDA(cudaStreamWaitEvent(crit, ev_start, 0));
    int pending_rest = -1;  // step whose part 2 is in flight on `st`
    // Delayed updates: every other step's part 2 is skipped and applied with
    // the next step's panel in one rank-128 update (one read-modify-write of
    // the trailing matrix for two panels); the next step's part 1 then
    // carries both panels too.  OCTEN_CHOL_DELAY=0 turns it off.
    static const bool delay_ok = [] {
        const char* e = std::getenv("OCTEN_CHOL_DELAY");
        return !(e && e[0] == '0');
    }();
    int delayed = -1;  // column offset of the panel whose trailing update is pending
    static thread_local EvProf cp;
    const bool prof = EvProf::enabled() && n >= 512;
    if (prof) cp.mark("begin", crit);
    for (int kb = 0; kb < nblk; ++kb) {
        const int k0 = kb * kCholNB;
        chol_diag_kernel<<<batch, kDiagThreads, kDiagSmem, crit>>>(A, n, lda, sA, k0, tol, maxdiag, rank, linv.p,
                                                                    nblk);
        OCTEN_LAUNCHED(1);
        if (prof) cp.mark("diag", crit);
        const int nb = min(kCholNB, n - k0);
        const int rows = n - k0 - nb;
        if (rows <= 0) break;
        const int r0 = k0 + nb;
        gemm_f64<false, true>(batch, rows, nb, nb, PanelA{A, lda, sA, r0, k0}, PanelB{linv.p, nblk, k0 / kCholNB},
                                               PanelC{A, lda, sA, r0, k0}, crit);
        if (prof) cp.mark("panel", crit);
        const int tiles = (rows + kCholNB - 1) / kCholNB;
        if (tiles > 1) {
            OCTEN_CUDA(cudaEventRecord(ev_panel[kb], crit));
            OCTEN_CUDA(cudaStreamWaitEvent(st, ev_panel[kb], 0));
        }
        if (pending_rest >= 0) {
            OCTEN_CUDA(cudaStreamWaitEvent(crit, ev_rest[pending_rest], 0));
            pending_rest = -1;
        }
        if (prof) cp.mark("wait", crit);
        chol_trail_kernel<<<tiles * batch, 256, kTrailSmem, crit>>>(A, n, lda, sA, r0, k0, nb, 1, tiles,
                                                                    tiles * batch, delayed);
        OCTEN_LAUNCHED(1);
        if (prof) cp.mark("part1", crit);
        if (tiles > 1 && delay_ok && delayed < 0 && nb == kCholNB) {
            delayed = k0;  // this step's part 2 goes with the next step's
        } else if (tiles > 1) {
            // OCTEN_TRAIL_CAP: cap the grid (tasks are strided over it) to
            // leave SM room for the critical chain (diagnostics)
            const int t2 = (tiles - 1) * tiles / 2;
            static const int cap_env = [] {
                const char* e = std::getenv("OCTEN_TRAIL_CAP");
                return e ? std::atoi(e) : 0;
            }();
            const int cap = cap_env > 0 ? cap_env : 1 << 30;
            chol_trail_kernel<<<std::min(t2 * batch, cap), 256, kTrailSmem, st>>>(A, n, lda, sA, r0, k0, nb, 2, t2,
                                                                                  t2 * batch, delayed);
            OCTEN_LAUNCHED(1);
            OCTEN_CUDA(cudaEventRecord(ev_rest[kb], st));
            pending_rest = kb;
            delayed = -1;
        } else {
            delayed = -1;  // (no tile column beyond the next one: nothing was delayed)
        }
    }
    // join: everything on `st` after this waits for the critical chain
    OCTEN_CUDA(cudaEventRecord(ev_end, crit));
    OCTEN_CUDA(cudaStreamWaitEvent(st, ev_end, 0));
    if (prof) {
        cp.mark("join", st);
        cp.report("chol_batched crit chain");
        long long t[16];
        OCTEN_CUDA(cudaMemcpyFromSymbol(t, g_diag_tsc, sizeof t));
        std::fprintf(stderr, "octen chol_diag phases (cycles, block 0, k0 = 0):");
        for (int i = 1; i < 12; ++i)
            if (t[i]) std::fprintf(stderr, " [%d] %lld", i, t[i] - t[0]);
        std::fprintf(stderr, "\n");
    }
}

// Blocked solves with the stored diagonal-block inverses.  Step k of the
// forward pass forms y_k = Linv_k x_k and updates every later row
//   x_i -= sum_j L(i, k0 + j) y_k(j)
// in parallel across many blocks (the kernel boundary is the only
// synchronization); the backward pass forms x_k = Linv_k^T y_k and updates
// every earlier row  y_i -= sum_j L(k0 + j, i) x_k(j)  reading the block row
// of the lower triangle directly (no mirrored copy).  Each block recomputes
// the 64 x 64 mat-vec from L2-resident Linv_k (all 256 threads, 16 columns
// each); rows are split four ways so every thread keeps 16 independent loads
// in flight.  2 * nblk launches.
constexpr int kStepRows = 64;  // rows per block (4 threads each)

__device__ __forceinline__ void chol_block_matvec(const double* iv, const double* v, double* out, bool transposed,
                                                  int nb, double* part) {
    // out(t) = sum_j M(t, j) v(j), M = Linv (lower) or Linv^T; thread (t, q)
    // covers columns j in [16q, 16q + 16)
    const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
    const int t = lane + 32 * (w & 1), q = w >> 1;
    double acc = 0.0;
#pragma unroll
    for (int jj = 0; jj < 16; ++jj) {
        const int j = 16 * q + jj;
        const double m = transposed ? iv[j + kCholNB * t] : iv[t + kCholNB * j];  // zero outside the triangle
        acc += m * v[j];
    }
    part[q * kCholNB + t] = acc;
    __syncthreads();
    if (tid < kCholNB) out[tid] = (tid < nb) ? (part[tid] + part[kCholNB + tid]) + (part[2 * kCholNB + tid] + part[3 * kCholNB + tid]) : 0.0;
    __syncthreads();
}

__global__ void __launch_bounds__(256) chol_fwd_step_kernel(const double* L, int n, int ldl, long long sL,
                                                            const double* linv, int nblk, double* X, int ldx,
                                                            long long sX, double* Y, int kb) {
    __shared__ double xv[kCholNB], yk[kCholNB], part[4 * kCholNB];
    const int b = blockIdx.z, r = blockIdx.y;
    const double* Lb = L + (size_t)b * sL;
    const double* iv = linv + ((size_t)b * nblk + kb) * kCholNB * kCholNB;
    double* x = X + (size_t)b * sX + (size_t)r * ldx;
    double* y = Y + (size_t)b * sX + (size_t)r * ldx;
    const int k0 = kb * kCholNB, nb = min(kCholNB, n - k0);
    const int tid = threadIdx.x;
    if (tid < kCholNB) xv[tid] = (tid < nb) ? x[k0 + tid] : 0.0;
    __syncthreads();
    chol_block_matvec(iv, xv, yk, false, nb, part);
    if (blockIdx.x == 0 && tid < nb) y[k0 + tid] = yk[tid];
    // rows: warp w covers rows base + 32 (w & 1) + lane, columns [16q, 16q+16)
    const int w = tid >> 5, lane = tid & 31, q = w >> 1;
    const int rl = lane + 32 * (w & 1);
    const int i = k0 + nb + blockIdx.x * kStepRows + rl;
    double acc = 0.0;
    if (i < n) {
        const double* col = Lb + i + (size_t)ldl * (k0 + 16 * q);
#pragma unroll
        for (int jj = 0; jj < 16; ++jj)
            if (16 * q + jj < nb) acc += col[(size_t)ldl * jj] * yk[16 * q + jj];
    }
    part[q * kCholNB + rl] = acc;  // part reuse is ordered by the matvec's trailing barrier
    __syncthreads();
    if (tid < kStepRows) {
        const int ii = k0 + nb + blockIdx.x * kStepRows + tid;
        if (ii < n)
            x[ii] -= (part[tid] + part[kCholNB + tid]) + (part[2 * kCholNB + tid] + part[3 * kCholNB + tid]);
    }
}

__global__ void __launch_bounds__(256) chol_bwd_step_kernel(const double* L, int n, int ldl, long long sL,
                                                            const double* linv, int nblk, double* X, int ldx,
                                                            long long sX, double* Y, int kb) {
    __shared__ double yv[kCholNB], xk[kCholNB], part[4 * kCholNB];
    const int b = blockIdx.z, r = blockIdx.y;
    const double* Lb = L + (size_t)b * sL;
    const double* iv = linv + ((size_t)b * nblk + kb) * kCholNB * kCholNB;
    double* x = X + (size_t)b * sX + (size_t)r * ldx;
    double* y = Y + (size_t)b * sX + (size_t)r * ldx;
    const int k0 = kb * kCholNB, nb = min(kCholNB, n - k0);
    const int tid = threadIdx.x;
    if (tid < kCholNB) yv[tid] = (tid < nb) ? y[k0 + tid] : 0.0;
    __syncthreads();
    chol_block_matvec(iv, yv, xk, true, nb, part);
    if (blockIdx.x == 0 && tid < nb) x[k0 + tid] = xk[tid];
    // rows i < k0: y_i -= sum_j L(k0 + j, i) xk(j); the 64 entries of the
    // block row are contiguous, so a warp reads 8 rows x 64 columns as
    // 8 coalesced segments: lane = 8 * jq + ri  (ri: row in group, jq: 8 columns)
    const int w = tid >> 5, lane = tid & 31;
    const int ri = lane & 7, jq = lane >> 3;  // jq in 0..3, 16 columns each
    const int i = blockIdx.x * kStepRows + w * 8 + ri;
    double acc = 0.0;
    if (i < k0) {
        const double* row = Lb + k0 + (size_t)ldl * i;
#pragma unroll
        for (int jj = 0; jj < 16; ++jj) {
            const int j = 16 * jq + jj;
            if (j < nb) acc += row[j] * xk[j];
        }
    }
    acc += __shfl_xor_sync(0xffffffffu, acc, 8);
    acc += __shfl_xor_sync(0xffffffffu, acc, 16);
    if (jq == 0 && i < k0) y[i] -= acc;
}

// Whole solve L L^T x = b in ONE CTA per (right-hand side, matrix): the
// vector lives in shared memory and the 2 * nblk block steps are separated
// by barriers instead of kernel launches.  Forward step k: x_k <- Linv_k x_k,
// then every later row i: x_i -= L(i, k-block) x_k (threads along rows,
// coalesced column reads).  Backward step k: x_k <- Linv_k^T x_k, then every
// earlier row i: x_i -= L(k-block, i) . x_k (one warp per row, lanes along
// the contiguous block row, shuffle reduction).  All right-hand sides and
// matrices run concurrently, one SM each, each streaming its factor once per
// direction.
constexpr int kSolveThreads = 1024;

__global__ void __launch_bounds__(kSolveThreads) chol_solve_cta_kernel(const double* L, int n, int ldl, long long sL,
                                                                    const double* linv, int nblk, double* X, int ldx,
                                                                    long long sX, int backward_only, int nblk_f) {
    extern __shared__ double xs[];  // n (+ 64 padding) + 16 * 64 partials
    double* part = xs + n + kCholNB;
    const int b = blockIdx.y, r = blockIdx.x;
    const double* Lb = L + (size_t)b * sL;
    const double* ivb = linv + (size_t)b * nblk_f * kCholNB * kCholNB;  // the factor's block count
    double* x = X + (size_t)b * sX + (size_t)r * ldx;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int i = tid; i < n + kCholNB; i += kSolveThreads) xs[i] = i < n ? x[i] : 0.0;
    __syncthreads();
    // 64 x 64 (transposed) block mat-vec in place on xs[k0 .. k0+64):
    // thread (row t, group q of 4 columns); 16 partials per row
    auto block_matvec = [&](const double* iv, int k0, int nb, bool transposed) {
        const int t = tid & 63, q = tid >> 6;  // q in 0..15
        double acc = 0.0;
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) {
            const int j = 4 * q + jj;
            const double m = transposed ? iv[j + kCholNB * t] : iv[t + kCholNB * j];
            acc += m * xs[k0 + j];
        }
        part[q * kCholNB + t] = acc;
        __syncthreads();
        if (tid < kCholNB) {
            double sacc = 0.0;
#pragma unroll
            for (int qq = 0; qq < 16; ++qq) sacc += part[qq * kCholNB + tid];
            if (tid < nb) xs[k0 + tid] = sacc;
        }
        __syncthreads();
    };
    for (int kb = 0; kb < (backward_only ? 0 : nblk); ++kb) {
        const int k0 = kb * kCholNB, nb = min(kCholNB, n - k0);
        block_matvec(ivb + (size_t)kb * kCholNB * kCholNB, k0, nb, false);
        for (int i = k0 + nb + tid; i < n; i += kSolveThreads) {
            // 16 independent loads in flight per batch (memory-level
            // parallelism is what bounds a single-SM stream)
            const double* col = Lb + i + (size_t)ldl * k0;
            double sacc = 0.0;
            for (int j0 = 0; j0 < nb; j0 += 16) {
                double v[16];
#pragma unroll
                for (int jj = 0; jj < 16; ++jj) v[jj] = (j0 + jj < nb) ? __ldg(col + (size_t)ldl * (j0 + jj)) : 0.0;
                double s0 = 0.0, s1 = 0.0;
#pragma unroll
                for (int jj = 0; jj < 16; jj += 2) {
                    s0 += v[jj] * xs[k0 + j0 + jj];
                    s1 += v[jj + 1] * xs[k0 + j0 + jj + 1];
                }
                sacc += s0 + s1;
            }
            xs[i] -= sacc;
        }
        __syncthreads();
    }
    for (int kb = nblk - 1; kb >= 0; --kb) {
        const int k0 = kb * kCholNB, nb = min(kCholNB, n - k0);
        block_matvec(ivb + (size_t)kb * kCholNB * kCholNB, k0, nb, true);
        const double x0 = xs[k0 + lane], x1 = xs[k0 + 32 + lane];  // zero past nb (Linv padding)
        // 8 rows per warp pass: 16 independent loads per lane in flight
        constexpr int RW = 8;
        for (int i0 = warp * RW; i0 < k0; i0 += (kSolveThreads / 32) * RW) {
            double acc[RW];
#pragma unroll
            for (int rr = 0; rr < RW; ++rr) {
                const int i = i0 + rr;
                const double* row = Lb + k0 + (size_t)ldl * i;  // L(k0 + j, i), j contiguous
                const double a0 = (i < k0 && lane < nb) ? __ldg(row + lane) : 0.0;
                const double a1 = (i < k0 && lane + 32 < nb) ? __ldg(row + lane + 32) : 0.0;
                acc[rr] = a0 * x0 + a1 * x1;
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1)
#pragma unroll
                for (int rr = 0; rr < RW; ++rr) acc[rr] += __shfl_xor_sync(0xffffffffu, acc[rr], o);
            if (lane < RW && i0 + lane < k0) {
                double v = acc[0];
#pragma unroll
                for (int rr = 1; rr < RW; ++rr)
                    if (lane == rr) v = acc[rr];
                xs[i0 + lane] -= v;
            }
        }
        __syncthreads();
    }
    for (int i = tid; i < n; i += kSolveThreads) x[i] = xs[i];
}

// Solve L L^T x = b in place (X) using the diagonal-block inverses from
// chol_batched; Y is scratch of the same layout.
inline void chol_solve_blocked_impl(const double* L, int n, int ldl, long long sL, const DevBuf<double>& linv, double* X,
                               int ldx, long long sX, int nrhs, int batch, cudaStream_t st) {
    if (n <= 0 || nrhs <= 0 || batch <= 0) return;
    static thread_local DevBuf<double> Y;
    const size_t need = (size_t)(batch - 1) * sX + (size_t)(nrhs - 1) * ldx + n;
    Y.reserve(need);
    const int nblk = (n + kCholNB - 1) / kCholNB;
    for (int kb = 0; kb < nblk; ++kb) {
        const int rows = n - std::min(n, (kb + 1) * kCholNB);
        const int chunks = std::max(1, (rows + kStepRows - 1) / kStepRows);
        chol_fwd_step_kernel<<<dim3(chunks, nrhs, batch), 256, 0, st>>>(L, n, ldl, sL, linv.p, nblk, X, ldx, sX, Y.p,
                                                                         kb);
        OCTEN_LAUNCHED(1);
    }
    for (int kb = nblk - 1; kb >= 0; --kb) {
        const int rows = kb * kCholNB;
        const int chunks = std::max(1, (rows + kStepRows - 1) / kStepRows);
        chol_bwd_step_kernel<<<dim3(chunks, nrhs, batch), 256, 0, st>>>(L, n, ldl, sL, linv.p, nblk, X, ldx, sX, Y.p,
                                                                         kb);
        OCTEN_LAUNCHED(1);
    }
}

// backward_only: X already holds L^-1 b (e.g. the border row of an augmented
// factorization); only L^-T is applied.  The factor may carry more rows than
// n (ldl >= n): its diagonal-block inverses are indexed by ceil(ldl / 64)
// blocks.
inline void chol_solve_cta(const double* L, int n, int ldl, long long sL, const DevBuf<double>& linv, double* X,
                           int ldx, long long sX, int nrhs, int batch, cudaStream_t st, bool backward_only = false) {
    if (n <= 0 || nrhs <= 0 || batch <= 0) return;
    const int nblk = (n + kCholNB - 1) / kCholNB;
    static const bool blocked = [] {  // diagnostics: OCTEN_SOLVE_MODE=blocked (one launch per block step)
        const char* e = std::getenv("OCTEN_SOLVE_MODE");
        return e && std::string(e) == "blocked";
    }();
    if (blocked && !backward_only && ldl == n) {
        chol_solve_blocked_impl(L, n, ldl, sL, linv, X, ldx, sX, nrhs, batch, st);
        return;
    }
    const int nblk_f = (ldl + kCholNB - 1) / kCholNB;  // blocks of the stored factor (Linv indexing)
    const size_t smem = (size_t)(n + kCholNB + 16 * kCholNB) * sizeof(double);
    if (smem > 48 * 1024)
        OCTEN_CUDA(cudaFuncSetAttribute(chol_solve_cta_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    chol_solve_cta_kernel<<<dim3(nrhs, batch), kSolveThreads, smem, st>>>(L, n, ldl, sL, linv.p, nblk, X, ldx, sX,
                                                                          backward_only ? 1 : 0, nblk_f);
    OCTEN_LAUNCHED(1);
}

}  // namespace octen
