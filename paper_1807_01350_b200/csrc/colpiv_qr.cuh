// Column-pivoted Householder QR least-squares solve on the device, one CTA
// per system: the reference's rank-revealing solve (Eigen
// ColPivHouseholderQR with setThreshold, proj/src/recovery.cpp:26-38, 396)
// for the systems whose normal-equation Cholesky cannot decide the rank.
//
// The merge factors Gram matrices (csrc/chol_batched.cuh).  A Gram pivot
// below kGramRankTol (1e-11 of the largest diagonal) means |r_ii| / |r_00|
// < 3.2e-6 for the R factor of the tall matrix, but the reference only calls
// a system rank-deficient below 1e-10.  Such systems are re-solved here on
// the tall matrix itself with the reference's rule: rank = #{i : |r_ii| >
// thr * max_j |r_jj|}, and when the rank is full x = P R^-1 (Q^T b).
//
// Pivoting follows Eigen: the remaining column of largest norm, lowest index
// on ties; the Householder vectors are Eigen's makeHouseholder (beta takes the
// sign opposite to the leading entry).  Column norms are recomputed exactly at
// every step rather than downdated.  The path is rare (only systems the Gram
// test flagged), so it favours simplicity over speed: 1024 threads, A and B
// in global memory (L2-resident), the Householder vector in shared memory.
#pragma once

#include <cuda_runtime.h>

#include "octen_common.cuh"

namespace octen {

constexpr int kQrThreads = 1024;

// A: m x n (lda, batch stride sA), overwritten by R and the reflectors;
// B: m x nrhs (ldb, sB), overwritten by Q^T B; X: n x nrhs (ldx, sX) gets the
// solution when the rank is full (untouched otherwise); rank_out[sys].
// Scratch: norms n doubles and piv n ints per system.  Dynamic shared memory:
// m doubles (Householder vector).
__global__ void __launch_bounds__(kQrThreads) colpiv_qr_solve_kernel(int m, int n, double* A, long long lda,
                                                                     long long sA, double* B, long long ldb,
                                                                     long long sB, int nrhs, double thr, double* X,
                                                                     long long ldx, long long sX, int* rank_out,
                                                                     double* norms_ws, int* piv_ws) {
    extern __shared__ double qr_v[];
    __shared__ double red_v[32];
    __shared__ int red_i[32];
    __shared__ double s_beta, s_tau, s_maxpiv;
    __shared__ int s_piv;
    const int sys = blockIdx.x;
    A += (size_t)sys * sA;
    B += (size_t)sys * sB;
    X += (size_t)sys * sX;
    double* norms = norms_ws + (size_t)sys * n;
    int* piv = piv_ws + (size_t)sys * n;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;

    // initial column norms (one warp per column)
    for (int j = warp; j < n; j += nw) {
        double s = 0.0;
        const double* a = A + (size_t)lda * j;
        for (int i = lane; i < m; i += 32) s += a[i] * a[i];
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) norms[j] = s;
    }
    for (int j = tid; j < n; j += blockDim.x) piv[j] = j;
    if (tid == 0) s_maxpiv = 0.0;
    __syncthreads();
    const int steps = m < n ? m : n;
    for (int k = 0; k < steps; ++k) {
        // pivot: largest remaining norm, lowest index on ties
        double bv = -1.0;
        int bi = n;
        for (int j = k + tid; j < n; j += blockDim.x) {
            const double v = norms[j];
            if (v > bv) {
                bv = v;
                bi = j;
            }
        }
        for (int o = 16; o > 0; o >>= 1) {
            const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
            const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
            if (ov > bv || (ov == bv && oi < bi)) {
                bv = ov;
                bi = oi;
            }
        }
        if (lane == 0) {
            red_v[warp] = bv;
            red_i[warp] = bi;
        }
        __syncthreads();
        if (tid == 0) {
            double v = red_v[0];
            int ix = red_i[0];
            for (int w = 1; w < nw; ++w)
                if (red_v[w] > v || (red_v[w] == v && red_i[w] < ix)) {
                    v = red_v[w];
                    ix = red_i[w];
                }
            s_piv = ix;
        }
        __syncthreads();
        const int p = s_piv;
        if (p != k) {
            double* ak = A + (size_t)lda * k;
            double* ap = A + (size_t)lda * p;
            for (int i = tid; i < m; i += blockDim.x) {
                const double t = ak[i];
                ak[i] = ap[i];
                ap[i] = t;
            }
            if (tid == 0) {
                const double t = norms[k];
                norms[k] = norms[p];
                norms[p] = t;
                const int ti = piv[k];
                piv[k] = piv[p];
                piv[p] = ti;
            }
        }
        __syncthreads();
        // Householder of A(k:m, k): tail norm, beta, tau, v = [1; tail / (c0 - beta)]
        double* ak = A + (size_t)lda * k;
        double s = 0.0;
        for (int i = k + 1 + tid; i < m; i += blockDim.x) s += ak[i] * ak[i];
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) red_v[warp] = s;
        __syncthreads();
        if (tid == 0) {
            double tail = 0.0;
            for (int w = 0; w < nw; ++w) tail += red_v[w];
            const double c0 = ak[k];
            double beta, tau;
            if (tail <= 2.2250738585072014e-308) {
                beta = c0;
                tau = 0.0;
            } else {
                beta = sqrt(c0 * c0 + tail);
                if (c0 >= 0.0) beta = -beta;
                tau = (beta - c0) / beta;
            }
            s_beta = beta;
            s_tau = tau;
            red_v[0] = c0 - beta;  // divisor of the essential part
            s_maxpiv = fmax(s_maxpiv, fabs(beta));
        }
        __syncthreads();
        const double tau = s_tau, div = red_v[0];
        for (int i = k + tid; i < m; i += blockDim.x) qr_v[i] = i == k ? 1.0 : (tau == 0.0 ? 0.0 : ak[i] / div);
        __syncthreads();
        if (tid == 0) ak[k] = s_beta;
        for (int i = k + 1 + tid; i < m; i += blockDim.x) ak[i] = qr_v[i];  // reflector kept below the diagonal
        // apply H = I - tau v v^T to the trailing columns and to B (one warp
        // per column), then the exact tail norms of the trailing columns
        const int ncols = (n - k - 1) + nrhs;
        for (int c = warp; c < ncols; c += nw) {
            double* col = c < n - k - 1 ? A + (size_t)lda * (k + 1 + c) : B + (size_t)ldb * (c - (n - k - 1));
            double w = 0.0;
            for (int i = k + lane; i < m; i += 32) w += qr_v[i] * col[i];
            for (int o = 16; o > 0; o >>= 1) w += __shfl_xor_sync(0xffffffffu, w, o);
            w *= tau;
            double nt = 0.0;
            for (int i = k + lane; i < m; i += 32) {
                const double x = col[i] - w * qr_v[i];
                col[i] = x;
                if (i > k) nt += x * x;
            }
            if (c < n - k - 1) {
                for (int o = 16; o > 0; o >>= 1) nt += __shfl_xor_sync(0xffffffffu, nt, o);
                if (lane == 0) norms[k + 1 + c] = nt;
            }
        }
        __syncthreads();
    }
    // rank by the reference's rule, then the back substitution R z = (Q^T b)(0:n)
    __shared__ int s_rank;
    if (tid == 0) {
        int r = 0;
        const double cut = s_maxpiv * thr;
        for (int i = 0; i < steps; ++i)
            if (fabs(A[i + (size_t)lda * i]) > cut) ++r;
        s_rank = r;
        rank_out[sys] = r;
    }
    __syncthreads();
    if (s_rank < n) return;
    for (int c = warp; c < nrhs; c += nw) {
        double* b = B + (size_t)ldb * c;
        for (int i = n - 1; i >= 0; --i) {
            double acc = 0.0;
            for (int j = i + 1 + lane; j < n; j += 32) acc += A[i + (size_t)lda * j] * b[j];
            for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
            if (lane == 0) b[i] = (b[i] - acc) / A[i + (size_t)lda * i];
            __syncwarp();
        }
        for (int i = lane; i < n; i += 32) X[piv[i] + (size_t)ldx * c] = b[i];
    }
}

// Launch over `batch` systems.  Shared memory m doubles (m <= 27000).
inline void colpiv_qr_solve(int m, int n, double* A, long long lda, long long sA, double* B, long long ldb,
                            long long sB, int nrhs, double thr, double* X, long long ldx, long long sX, int* rank_out,
                            double* norms_ws, int* piv_ws, int batch, cudaStream_t st) {
    const size_t smem = (size_t)m * sizeof(double);
    if (smem > 48 * 1024)
        OCTEN_CUDA(cudaFuncSetAttribute(colpiv_qr_solve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)smem));
    colpiv_qr_solve_kernel<<<batch, kQrThreads, smem, st>>>(m, n, A, lda, sA, B, ldb, sB, nrhs, thr, X, ldx, sX,
                                                            rank_out, norms_ws, piv_ws);
    OCTEN_LAUNCHED(1);
    OCTEN_CUDA(cudaGetLastError());
}

}  // namespace octen
