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
// it (for the panel GEMM).  Right-looking with the whole block: one thread
// forms the pivot, the column scaling and the rank-1 trailing update are
// spread over all threads (fixed row/column-group mapping, no index
// division); the inverse is built in 8-row blocks (parallel dot products,
// then a short substitution per column).  Shared tiles column-major, ld 65.
__global__ void __launch_bounds__(256) chol_diag_kernel(double* A, int n, int lda, long long sA, int k0, double tol,
                                                        const double* maxdiag, int* rank, double* Linv,
                                                        int nblk) {
    extern __shared__ double chol_smem[];
    constexpr int LD = kCholNB + 1;
    double* S = chol_smem;                   // L (lower), column-major
    double* X = chol_smem + LD * kCholNB;    // L^-1
    __shared__ double rinv[kCholNB];
    __shared__ double sh_piv, sh_rp;
    double* a = A + (size_t)blockIdx.x * sA;
    const int nb = min(kCholNB, n - k0);
    const int tid = threadIdx.x;
    for (int e = tid; e < nb * nb; e += blockDim.x) {
        const int i = e % nb, j = e / nb;
        S[i + LD * j] = (i >= j) ? a[(k0 + i) + (size_t)lda * (k0 + j)] : 0.0;
    }
    __syncthreads();
    const double md = maxdiag[blockIdx.x];
    const double thr = (md > 0.0) ? tol * md : INFINITY;
    const int my_i = tid & 63, my_jg = tid >> 6;  // trailing-update mapping: row, column group (4)
    for (int k = 0; k < nb; ++k) {
        if (tid == 0) {
            const double d = S[k + LD * k];
            const bool dead = !(d > thr);
            const double piv = dead ? 0.0 : sqrt(d);
            sh_piv = piv;
            sh_rp = dead ? 0.0 : 1.0 / piv;
            rinv[k] = sh_rp;
            if (dead) atomicSub(&rank[blockIdx.x], 1);
        }
        __syncthreads();
        const double rp = sh_rp;
        if (tid == 0) S[k + LD * k] = sh_piv;
        {
            const int i = k + 1 + tid;
            if (i < nb) S[i + LD * k] *= rp;
        }
        __syncthreads();
        if (my_i > k && my_i < nb) {
            const double lik = S[my_i + LD * k];
            for (int j = k + 1 + my_jg; j <= my_i; j += 4) S[my_i + LD * j] -= lik * S[j + LD * k];
        }
        __syncthreads();
    }
    // inverse in 8-row blocks
    for (int I0 = 0; I0 < nb; I0 += 8) {
        const int ib = min(8, nb - I0);
        for (int e = tid; e < 8 * nb; e += blockDim.x) {
            const int ii = e & 7, j = e >> 3;
            if (ii >= ib) continue;
            const int i = I0 + ii;
            double v0 = (i == j) ? 1.0 : 0.0, v1 = 0.0, v2 = 0.0, v3 = 0.0;
            int p = j;
            for (; p + 3 < I0; p += 4) {
                v0 -= S[i + LD * p] * X[p + LD * j];
                v1 -= S[i + LD * (p + 1)] * X[p + 1 + LD * j];
                v2 -= S[i + LD * (p + 2)] * X[p + 2 + LD * j];
                v3 -= S[i + LD * (p + 3)] * X[p + 3 + LD * j];
            }
            for (; p < I0; ++p) v0 -= S[i + LD * p] * X[p + LD * j];
            X[i + LD * j] = (v0 + v1) + (v2 + v3);
        }
        __syncthreads();
        for (int j = tid; j < nb; j += blockDim.x) {
            for (int ii = 0; ii < ib; ++ii) {
                const int i = I0 + ii;
                double v = X[i + LD * j];
                for (int pp = (j > I0 ? j : I0); pp < i; ++pp) v -= S[i + LD * pp] * X[pp + LD * j];
                X[i + LD * j] = (i < j) ? 0.0 : v * rinv[i];
            }
        }
        __syncthreads();
    }
    for (int e = tid; e < nb * nb; e += blockDim.x) {
        const int i = e % nb, j = e / nb;
        a[(k0 + i) + (size_t)lda * (k0 + j)] = (i >= j) ? S[i + LD * j] : 0.0;
    }
    double* inv = Linv + ((size_t)blockIdx.x * nblk + k0 / kCholNB) * kCholNB * kCholNB;
    for (int e = tid; e < kCholNB * kCholNB; e += blockDim.x) {
        const int i = e % kCholNB, j = e / kCholNB;
        inv[e] = (i < nb && j < nb) ? X[i + LD * j] : 0.0;
    }
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

struct CholTrailA {
    double* A;
    int lda;
    long long sA;
    int r0, k0;
    __device__ double operator()(int b, int m, int k) const {
        return A[(size_t)b * sA + (r0 + m) + (size_t)lda * (k0 + k)];
    }
};
struct CholTrailB {
    double* A;
    int lda;
    long long sA;
    int r0, k0;
    __device__ double operator()(int b, int k, int nn) const {
        return A[(size_t)b * sA + (r0 + nn) + (size_t)lda * (k0 + k)];
    }
};
struct CholTrailC {
    double* A;
    int lda;
    long long sA;
    int r0;
    __device__ void operator()(int b, int m, int nn, double v) const {
        if (m >= nn) A[(size_t)b * sA + (r0 + m) + (size_t)lda * (r0 + nn)] -= v;
    }
};

// Copy the strictly lower triangle into the upper one (L^T columns become
// contiguous for the backward substitution).
__global__ void chol_mirror_kernel(double* A, int n, int lda, long long sA, int batch) {
    const size_t per = (size_t)n * n, total = per * batch;
    for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < total; e += (size_t)gridDim.x * blockDim.x) {
        const int b = (int)(e / per);
        const size_t r = e % per;
        const int i = (int)(r % n), j = (int)(r / n);
        if (i > j) A[(size_t)b * sA + j + (size_t)lda * i] = A[(size_t)b * sA + i + (size_t)lda * j];
    }
}

// In-place batched semi-definite Cholesky.  Lower triangle holds L on return,
// upper triangle is zeroed.  rank[b] (device) = n - #deficient pivots.
// linv receives the inverses of the diagonal blocks (batch x nblk x 64 x 64),
// used by the panel GEMM here and by the blocked solves below.
inline void chol_batched(double* A, int n, int lda, long long sA, int batch, double tol, double* maxdiag,
                         int* rank, DevBuf<double>& linv, cudaStream_t st) {
    if (batch <= 0 || n <= 0) return;
    constexpr size_t kDiagSmem = 2 * kCholNB * (kCholNB + 1) * sizeof(double);
    static bool attr = false;
    if (!attr) {
        OCTEN_CUDA(cudaFuncSetAttribute(chol_diag_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kDiagSmem));
        attr = true;
    }
    const int nblk = (n + kCholNB - 1) / kCholNB;
    linv.reserve((size_t)batch * nblk * kCholNB * kCholNB);
    chol_maxdiag_kernel<<<batch, 256, 0, st>>>(A, n, lda, sA, maxdiag, rank); OCTEN_LAUNCHED(1);
    for (int k0 = 0; k0 < n; k0 += kCholNB) {
        chol_diag_kernel<<<batch, 256, kDiagSmem, st>>>(A, n, lda, sA, k0, tol, maxdiag, rank, linv.p, nblk);
        OCTEN_LAUNCHED(1);
        const int nb = min(kCholNB, n - k0);
        const int rows = n - k0 - nb;
        if (rows <= 0) break;
        const int r0 = k0 + nb;
        gemm_f64<false, true>(batch, rows, nb, nb, PanelA{A, lda, sA, r0, k0}, PanelB{linv.p, nblk, k0 / kCholNB},
                                               PanelC{A, lda, sA, r0, k0}, st);
        gemm_f64<false, false>(batch, rows, rows, nb, CholTrailA{A, lda, sA, r0, k0},
                                                CholTrailB{A, lda, sA, r0, k0}, CholTrailC{A, lda, sA, r0},
                                                st, 1, nullptr, 1);
    }
    {
        const size_t total = (size_t)n * n * batch;
        int blocks = (int)((total + 255) / 256);
        if (blocks > 148 * 16) blocks = 148 * 16;
        chol_mirror_kernel<<<blocks, 256, 0, st>>>(A, n, lda, sA, batch);
        OCTEN_LAUNCHED(1);
    }
}

// Blocked solves with the stored diagonal-block inverses: step k of the
// forward pass forms y_k = Linv_k x_k and updates every later row in
// parallel across many blocks (the kernel boundary is the only
// synchronization); the backward pass does the same with Linv_k^T and the
// mirrored upper triangle.  2 * nblk launches, all SMs busy.
__global__ void __launch_bounds__(256) chol_fwd_step_kernel(const double* L, int n, int ldl, long long sL,
                                                            const double* linv, int nblk, double* X, int ldx,
                                                            long long sX, double* Y, int kb) {
    __shared__ double ivs[kCholNB][kCholNB + 1];
    __shared__ double xv[kCholNB], yk[kCholNB];
    const int b = blockIdx.z, r = blockIdx.y;
    const double* Lb = L + (size_t)b * sL;
    const double* iv = linv + ((size_t)b * nblk + kb) * kCholNB * kCholNB;
    double* x = X + (size_t)b * sX + (size_t)r * ldx;
    double* y = Y + (size_t)b * sX + (size_t)r * ldx;
    const int k0 = kb * kCholNB, nb = min(kCholNB, n - k0);
    const int t = threadIdx.x;
    for (int e = t; e < kCholNB * kCholNB; e += blockDim.x) ivs[e % kCholNB][e / kCholNB] = iv[e];
    if (t < nb) xv[t] = x[k0 + t];
    __syncthreads();
    if (t < nb) {
        double v0 = 0.0, v1 = 0.0, v2 = 0.0, v3 = 0.0;
        int j = 0;
        for (; j + 3 <= t; j += 4) {
            v0 += ivs[t][j] * xv[j];
            v1 += ivs[t][j + 1] * xv[j + 1];
            v2 += ivs[t][j + 2] * xv[j + 2];
            v3 += ivs[t][j + 3] * xv[j + 3];
        }
        for (; j <= t; ++j) v0 += ivs[t][j] * xv[j];
        yk[t] = (v0 + v1) + (v2 + v3);
    }
    __syncthreads();
    if (blockIdx.x == 0 && t < nb) y[k0 + t] = yk[t];
    const int i = k0 + nb + blockIdx.x * blockDim.x + t;
    if (i < n) {
        const double* col = Lb + i + (size_t)ldl * k0;
        double s0 = x[i], s1 = 0.0, s2 = 0.0, s3 = 0.0;
        int j = 0;
#pragma unroll 4
        for (; j + 3 < nb; j += 4) {
            s0 -= col[(size_t)ldl * j] * yk[j];
            s1 -= col[(size_t)ldl * (j + 1)] * yk[j + 1];
            s2 -= col[(size_t)ldl * (j + 2)] * yk[j + 2];
            s3 -= col[(size_t)ldl * (j + 3)] * yk[j + 3];
        }
        for (; j < nb; ++j) s0 -= col[(size_t)ldl * j] * yk[j];
        x[i] = (s0 + s1) + (s2 + s3);
    }
}

__global__ void __launch_bounds__(256) chol_bwd_step_kernel(const double* L, int n, int ldl, long long sL,
                                                            const double* linv, int nblk, double* X, int ldx,
                                                            long long sX, double* Y, int kb) {
    __shared__ double ivs[kCholNB][kCholNB + 1];
    __shared__ double yv[kCholNB], xk[kCholNB];
    const int b = blockIdx.z, r = blockIdx.y;
    const double* Lb = L + (size_t)b * sL;
    const double* iv = linv + ((size_t)b * nblk + kb) * kCholNB * kCholNB;
    double* x = X + (size_t)b * sX + (size_t)r * ldx;
    double* y = Y + (size_t)b * sX + (size_t)r * ldx;
    const int k0 = kb * kCholNB, nb = min(kCholNB, n - k0);
    const int t = threadIdx.x;
    for (int e = t; e < kCholNB * kCholNB; e += blockDim.x) ivs[e % kCholNB][e / kCholNB] = iv[e];
    if (t < nb) yv[t] = y[k0 + t];
    __syncthreads();
    if (t < nb) {
        double v0 = 0.0, v1 = 0.0, v2 = 0.0, v3 = 0.0;
        int j = t;
        for (; j + 3 < nb; j += 4) {  // (Linv^T)(t, j) = Linv(j, t)
            v0 += ivs[j][t] * yv[j];
            v1 += ivs[j + 1][t] * yv[j + 1];
            v2 += ivs[j + 2][t] * yv[j + 2];
            v3 += ivs[j + 3][t] * yv[j + 3];
        }
        for (; j < nb; ++j) v0 += ivs[j][t] * yv[j];
        xk[t] = (v0 + v1) + (v2 + v3);
    }
    __syncthreads();
    if (blockIdx.x == 0 && t < nb) x[k0 + t] = xk[t];
    const int i = blockIdx.x * blockDim.x + t;
    if (i < k0) {
        const double* col = Lb + i + (size_t)ldl * k0;  // L^T(i, k0 + j) = L(k0 + j, i), mirrored upper
        double s0 = y[i], s1 = 0.0, s2 = 0.0, s3 = 0.0;
        int j = 0;
#pragma unroll 4
        for (; j + 3 < nb; j += 4) {
            s0 -= col[(size_t)ldl * j] * xk[j];
            s1 -= col[(size_t)ldl * (j + 1)] * xk[j + 1];
            s2 -= col[(size_t)ldl * (j + 2)] * xk[j + 2];
            s3 -= col[(size_t)ldl * (j + 3)] * xk[j + 3];
        }
        for (; j < nb; ++j) s0 -= col[(size_t)ldl * j] * xk[j];
        y[i] = (s0 + s1) + (s2 + s3);
    }
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
        const int chunks = std::max(1, (rows + 255) / 256);
        chol_fwd_step_kernel<<<dim3(chunks, nrhs, batch), 256, 0, st>>>(L, n, ldl, sL, linv.p, nblk, X, ldx, sX, Y.p,
                                                                         kb);
        OCTEN_LAUNCHED(1);
    }
    for (int kb = nblk - 1; kb >= 0; --kb) {
        const int rows = kb * kCholNB;
        const int chunks = std::max(1, (rows + 255) / 256);
        chol_bwd_step_kernel<<<dim3(chunks, nrhs, batch), 256, 0, st>>>(L, n, ldl, sL, linv.p, nblk, X, ldx, sX, Y.p,
                                                                         kb);
        OCTEN_LAUNCHED(1);
    }
}

// Solve L L^T x = b for nrhs right-hand sides per matrix.  Matrix b uses
// factor L[b * sL]; rhs r of matrix b lives at X + b*sX + r*ldx.  Dead
// pivots (L_ii == 0) produce x_i = 0 (callers reject rank-deficient systems
// before solving).  One block per (rhs, matrix).
__global__ void chol_solve_kernel(const double* Lbase, int n, int ldl, long long sL, double* Xbase, int ldx,
                                  long long sX) {
    extern __shared__ double xs[];
    double* rd = xs + n;  // reciprocal diagonal (0 for dead pivots)
    __shared__ double D[32][33];
    const double* L = Lbase + (size_t)blockIdx.y * sL;
    double* X = Xbase + (size_t)blockIdx.y * sX + (size_t)blockIdx.x * ldx;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        xs[i] = X[i];
        const double d = L[i + (size_t)ldl * i];
        rd[i] = (d != 0.0) ? 1.0 / d : 0.0;
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // forward: L y = b
    for (int b0 = 0; b0 < n; b0 += 32) {
        const int nb = min(32, n - b0);
        for (int e = threadIdx.x; e < nb * nb; e += blockDim.x) D[e % nb][e / nb] = L[(b0 + e % nb) + (size_t)ldl * (b0 + e / nb)];
        __syncthreads();
        if (warp == 0) {
            const int i = b0 + lane;
            double xi = (lane < nb) ? xs[i] : 0.0;
            for (int j = 0; j < nb; ++j) {
                if (lane == j) xi *= rd[i];
                const double xj = __shfl_sync(0xffffffffu, xi, j);
                if (lane > j && lane < nb) xi -= D[lane][j] * xj;
            }
            if (lane < nb) xs[i] = xi;
        }
        __syncthreads();
        for (int i = b0 + nb + threadIdx.x; i < n; i += blockDim.x) {
            double s = xs[i];
            for (int j = 0; j < nb; ++j) s -= L[i + (size_t)ldl * (b0 + j)] * xs[b0 + j];
            xs[i] = s;
        }
        __syncthreads();
    }
    // backward: L^T x = y
    const int last0 = ((n - 1) / 32) * 32;
    for (int b0 = last0; b0 >= 0; b0 -= 32) {
        const int nb = min(32, n - b0);
        for (int e = threadIdx.x; e < nb * nb; e += blockDim.x) D[e % nb][e / nb] = L[(b0 + e % nb) + (size_t)ldl * (b0 + e / nb)];
        __syncthreads();
        if (warp == 0) {
            const int i = b0 + lane;
            double xi = (lane < nb) ? xs[i] : 0.0;
            for (int jj = nb - 1; jj >= 0; --jj) {
                if (lane == jj) xi *= rd[i];
                const double xj = __shfl_sync(0xffffffffu, xi, jj);
                if (lane < jj) xi -= D[jj][lane] * xj;
            }
            if (lane < nb) xs[i] = xi;
        }
        __syncthreads();
        for (int i = threadIdx.x; i < b0; i += blockDim.x) {
            double s = xs[i];
            // L^T(i, b0 + j) = L(b0 + j, i), mirrored into the upper triangle
            for (int j = 0; j < nb; ++j) s -= L[i + (size_t)ldl * (b0 + j)] * xs[b0 + j];
            xs[i] = s;
        }
        __syncthreads();
    }
    for (int i = threadIdx.x; i < n; i += blockDim.x) X[i] = xs[i];
}

inline void chol_solve_batched(const double* L, int n, int ldl, long long sL, double* X, int ldx, long long sX,
                               int nrhs, int batch, cudaStream_t st) {
    if (n <= 0 || nrhs <= 0 || batch <= 0) return;
    dim3 g(nrhs, batch);
    const size_t smem = (size_t)2 * n * sizeof(double);
    if (smem > 48 * 1024) cudaFuncSetAttribute(chol_solve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    chol_solve_kernel<<<g, 1024, smem, st>>>(L, n, ldl, sL, X, ldx, sX); OCTEN_LAUNCHED(1);
}

}  // namespace octen
