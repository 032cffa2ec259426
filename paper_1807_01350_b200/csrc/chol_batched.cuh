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

#include "devbuf.hpp"
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
// it (for the panel GEMM and the blocked solves), fused in one right-looking
// sweep.  Every thread keeps a fixed share of the packed lower triangle of
// both the block (A -> L) and of B (I -> L^-1) in registers; step k publishes
// column k of L and row k of L^-1 through shared memory and every thread
// applies the rank-1 updates to its own elements:
//   A(i,j) -= L(i,k) L(j,k)      (j > k)        -- Cholesky trailing update
//   B(i,j) -= L(i,k) X(k,j)      (j <= k < i)   -- forward substitution
// so one step costs two barriers and ~9 FMAs per thread.  A pivot
// <= tol * maxdiag is dead: its column of L and row of L^-1 become zero and
// the rank is decremented.
constexpr int kDiagThreads = 1024;
constexpr int kDiagPer = (kCholNB * (kCholNB + 1) / 2 + kDiagThreads - 1) / kDiagThreads;  // 3

// Branch-free form of the updates: colk[i] is zero for i <= k and rowk[j] is
// zero for j > k (both start zeroed; step k zeroes colk[k] and writes rowk
// only up to k), so every owned element applies
//   A(i,j) -= colk[i] colk[j];  B(i,j) -= colk[i] rowk[j]
// unconditionally and the products vanish outside the trailing / forward
// ranges.  Unused slots point at row/column 64 (zero entries).
__global__ void __launch_bounds__(kDiagThreads) chol_diag_kernel(double* A, int n, int lda, long long sA, int k0,
                                                                 double tol, const double* maxdiag, int* rank,
                                                                 double* Linv, int nblk) {
    __shared__ double colk[kCholNB + 1], rowk[kCholNB + 1];
    __shared__ double shv_rp[2];
    __shared__ int sh_dead;
    double* a = A + (size_t)blockIdx.x * sA;
    const int nb = min(kCholNB, n - k0);
    const int tid = threadIdx.x;
    double av[kDiagPer], bv[kDiagPer];
    int iv[kDiagPer], jv[kDiagPer];
    if (tid <= kCholNB) {
        colk[tid] = 0.0;
        rowk[tid] = 0.0;
    }
    if (tid == 0) sh_dead = 0;
#pragma unroll
    for (int s = 0; s < kDiagPer; ++s) {
        // packed lower-triangle index e -> (i, j), j <= i (row-major packing)
        const int e = tid + kDiagThreads * s;
        int i = (int)((sqrtf(8.0f * (float)e + 1.0f) - 1.0f) * 0.5f);
        while ((i + 1) * (i + 2) / 2 <= e) ++i;
        while (i * (i + 1) / 2 > e) --i;
        const int j = e - i * (i + 1) / 2;
        const bool ok = e < kCholNB * (kCholNB + 1) / 2 && i < nb;
        iv[s] = ok ? i : kCholNB;
        jv[s] = ok ? j : kCholNB;
        av[s] = ok ? a[(k0 + i) + (size_t)lda * (k0 + j)] : 0.0;
        bv[s] = (ok && i == j) ? 1.0 : 0.0;
    }
    const double md = maxdiag[blockIdx.x];
    const double thr = (md > 0.0) ? tol * md : INFINITY;
    // The owner of diagonal element (k, k) (packed index k(k+3)/2) turns it
    // into the pivot as soon as its own update of step k-1 is done, so the
    // pivot's rsqrt overlaps the other threads' updates: two barriers a step.
    auto pivot = [&](int k) {
        const int ed = k * (k + 3) / 2;
        if (tid == ed % kDiagThreads) {
            const int sd = ed / kDiagThreads;
#pragma unroll
            for (int s = 0; s < kDiagPer; ++s)
                if (s == sd) {
                    const double d = av[s];
                    const bool dead = !(d > thr);
                    const double rp = dead ? 0.0 : rsqrt(d);
                    av[s] = dead ? 0.0 : d * rp;
                    shv_rp[k & 1] = rp;
                    if (dead) ++sh_dead;
                }
        }
    };
    __syncthreads();
    pivot(0);
    __syncthreads();
    for (int k = 0; k < nb; ++k) {
        const double rp = shv_rp[k & 1];
#pragma unroll
        for (int s = 0; s < kDiagPer; ++s) {
            const int i = iv[s], j = jv[s];
            if (j == k && i > k) {  // column k of L (i < 64 for used slots)
                av[s] *= rp;
                colk[i] = av[s];
            }
            if (i == k) {  // row k of L^-1
                bv[s] *= rp;
                rowk[j] = bv[s];
            }
        }
        if (tid == 0) colk[k] = 0.0;
        __syncthreads();
#pragma unroll
        for (int s = 0; s < kDiagPer; ++s) {
            const double ci = colk[iv[s]];
            av[s] -= ci * colk[jv[s]];
            bv[s] -= ci * rowk[jv[s]];
        }
        if (k + 1 < nb) pivot(k + 1);
        __syncthreads();
    }
    if (tid == 0 && sh_dead) atomicSub(&rank[blockIdx.x], sh_dead);
    double* inv = Linv + ((size_t)blockIdx.x * nblk + k0 / kCholNB) * kCholNB * kCholNB;
    for (int e = tid; e < kCholNB * kCholNB; e += kDiagThreads) {
        const int i = e % kCholNB, j = e / kCholNB;
        if (i < j) {
            inv[e] = 0.0;
            if (i < nb && j < nb) a[(k0 + i) + (size_t)lda * (k0 + j)] = 0.0;
        } else if (i >= nb) {
            inv[e] = 0.0;
        }
    }
#pragma unroll
    for (int s = 0; s < kDiagPer; ++s) {
        const int i = iv[s], j = jv[s];
        if (i < kCholNB) {
            a[(k0 + i) + (size_t)lda * (k0 + j)] = av[s];
            inv[i + kCholNB * j] = bv[s];
        }
    }
}

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

__global__ void __launch_bounds__(256, 2) chol_trail_kernel(double* A, int n, int lda, long long sA, int r0, int k0,
                                                         int nb) {
    extern __shared__ double trail_smem[];
    double* Pi = trail_smem;                       // [64 k][kTrailLD m]
    double* Pj = trail_smem + kCholNB * kTrailLD;  // [64 k][kTrailLD m]
    const int t = blockIdx.x;
    int ti = (int)((sqrtf(8.0f * (float)t + 1.0f) - 1.0f) * 0.5f);
    while ((ti + 1) * (ti + 2) / 2 <= t) ++ti;
    while (ti * (ti + 1) / 2 > t) --ti;
    const int tj = t - ti * (ti + 1) / 2;
    double* a = A + (size_t)blockIdx.z * sA;
    const int i0 = r0 + kCholNB * ti, j0 = r0 + kCholNB * tj;
    const int tid = threadIdx.x;
    // C tile prefetch (lower part) into registers: its latency overlaps the
    // panel staging and the DMMAs
    double cv[16];
#pragma unroll
    for (int r = 0; r < 16; ++r) {
        const int e = tid + 256 * r;
        const int m = e & (kCholNB - 1), nn = e >> 6;
        const int gi = i0 + m, gj = j0 + nn;
        cv[r] = (gi < n && gj < n && gi >= gj) ? a[gi + (size_t)lda * gj] : 0.0;
    }
    // panels: batches of loads into registers, then shared stores
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        double pi[8], pj[8];
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            const int e = tid + 256 * (8 * h + r);
            const int m = e & (kCholNB - 1), kk = e >> 6;
            const bool kin = kk < nb;
            pi[r] = (kin && i0 + m < n) ? a[(i0 + m) + (size_t)lda * (k0 + kk)] : 0.0;
            pj[r] = (kin && j0 + m < n) ? a[(j0 + m) + (size_t)lda * (k0 + kk)] : 0.0;
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
    const int lane = tid & 31, warp = tid >> 5;
    const int g = lane >> 2, t4 = lane & 3;
    const int wm = (warp & 1) * 32, wn = (warp >> 1) * 16;
    double acc[4][2][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    const int kend = (nb + 3) & ~3;
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
#pragma unroll
    for (int r = 0; r < 16; ++r) {
        const int e = tid + 256 * r;
        const int m = e & (kCholNB - 1), nn = e >> 6;
        const int gi = i0 + m, gj = j0 + nn;
        if (gi < n && gj < n && gi >= gj) a[gi + (size_t)lda * gj] = cv[r] - Cs[m + (kCholNB + 1) * nn];
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
    static bool attr = false;
    if (!attr) {
        OCTEN_CUDA(cudaFuncSetAttribute(chol_trail_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)kTrailSmem));
        attr = true;
    }
    const int nblk = (n + kCholNB - 1) / kCholNB;
    linv.reserve((size_t)batch * nblk * kCholNB * kCholNB);
    chol_maxdiag_kernel<<<batch, 256, 0, st>>>(A, n, lda, sA, maxdiag, rank); OCTEN_LAUNCHED(1);
    for (int k0 = 0; k0 < n; k0 += kCholNB) {
        chol_diag_kernel<<<batch, kDiagThreads, 0, st>>>(A, n, lda, sA, k0, tol, maxdiag, rank, linv.p, nblk);
        OCTEN_LAUNCHED(1);
        const int nb = min(kCholNB, n - k0);
        const int rows = n - k0 - nb;
        if (rows <= 0) break;
        const int r0 = k0 + nb;
        gemm_f64<false, true>(batch, rows, nb, nb, PanelA{A, lda, sA, r0, k0}, PanelB{linv.p, nblk, k0 / kCholNB},
                                               PanelC{A, lda, sA, r0, k0}, st);
        const int tiles = (rows + kCholNB - 1) / kCholNB;
        chol_trail_kernel<<<dim3(tiles * (tiles + 1) / 2, 1, batch), 256, kTrailSmem, st>>>(A, n, lda, sA, r0, k0,
                                                                                              nb);
        OCTEN_LAUNCHED(1);
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

// Solve L L^T x = b in place (X) using the diagonal-block inverses from
// chol_batched; Y is scratch of the same layout.
inline void chol_solve_blocked(const double* L, int n, int ldl, long long sL, const DevBuf<double>& linv, double* X,
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

}  // namespace octen
