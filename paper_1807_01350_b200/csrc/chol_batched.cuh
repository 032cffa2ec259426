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
// it (for the panel GEMM), as a 2 x 2 blocked factorization of 32-wide
// halves: warp-level Cholesky / triangular inverse of each half, block-wide
// products for the coupling terms.  Shared tiles are column-major (ld 65).
__global__ void chol_diag_kernel(double* A, int n, int lda, long long sA, int k0, double tol,
                                 const double* maxdiag, int* rank, double* Linv) {
    extern __shared__ double chol_smem[];
    constexpr int LD = kCholNB + 1;
    double* S = chol_smem;               // L (lower), column-major
    double* X = chol_smem + LD * kCholNB;  // L^-1
    double* a = A + (size_t)blockIdx.x * sA;
    const int nb = min(kCholNB, n - k0);
    const int n1 = min(32, nb), n2 = nb - n1;
    for (int e = threadIdx.x; e < nb * nb; e += blockDim.x) {
        const int i = e % nb, j = e / nb;
        S[i + LD * j] = (i >= j) ? a[(k0 + i) + (size_t)lda * (k0 + j)] : 0.0;
        X[i + LD * j] = 0.0;
    }
    __syncthreads();
    const double md = maxdiag[blockIdx.x];
    const double thr = (md > 0.0) ? tol * md : INFINITY;
    if (threadIdx.x < 32) {
        const int rk = warp_chol_inv32(S, LD, n1, thr, X, LD);
        if (threadIdx.x == 0 && rk < n1) atomicSub(&rank[blockIdx.x], n1 - rk);
    }
    __syncthreads();
    if (n2 > 0) {
        // L21 = A21 X11^T
        double tmp[8];
        int cnt = 0;
        for (int e = threadIdx.x; e < n2 * n1; e += blockDim.x, ++cnt) {
            const int i = n1 + e % n2, j = e / n2;
            double v = 0.0;
            for (int k = 0; k <= j; ++k) v += S[i + LD * k] * X[j + LD * k];
            tmp[cnt] = v;
        }
        __syncthreads();
        cnt = 0;
        for (int e = threadIdx.x; e < n2 * n1; e += blockDim.x, ++cnt) {
            const int i = n1 + e % n2, j = e / n2;
            S[i + LD * j] = tmp[cnt];
        }
        __syncthreads();
        // A22 -= L21 L21^T (lower)
        for (int e = threadIdx.x; e < n2 * n2; e += blockDim.x) {
            const int i = n1 + e % n2, j = n1 + e / n2;
            if (i < j) continue;
            double v = S[i + LD * j];
            for (int k = 0; k < n1; ++k) v -= S[i + LD * k] * S[j + LD * k];
            S[i + LD * j] = v;
        }
        __syncthreads();
        if (threadIdx.x < 32) {
            double* S22 = S + n1 + LD * n1;
            const int rk = warp_chol_inv32(S22, LD, n2, thr, X + n1 + LD * n1, LD);
            if (threadIdx.x == 0 && rk < n2) atomicSub(&rank[blockIdx.x], n2 - rk);
        }
        __syncthreads();
        // X21 = -X22 (L21 X11): first T = L21 X11 into registers, then X21
        cnt = 0;
        for (int e = threadIdx.x; e < n2 * n1; e += blockDim.x, ++cnt) {
            const int i = n1 + e % n2, j = e / n2;
            double v = 0.0;
            for (int k = j; k < n1; ++k) v += S[i + LD * k] * X[k + LD * j];
            tmp[cnt] = v;
        }
        __syncthreads();
        cnt = 0;
        for (int e = threadIdx.x; e < n2 * n1; e += blockDim.x, ++cnt) {
            const int i = n1 + e % n2, j = e / n2;
            X[i + LD * j] = tmp[cnt];  // T stored in the X21 slot temporarily
        }
        __syncthreads();
        for (int e = threadIdx.x; e < n2 * n1; e += blockDim.x) {
            const int i = n1 + e % n2, j = e / n2;
            double v = 0.0;
            for (int k = n1; k <= i; ++k) v += X[i + LD * k] * X[k + LD * j];
            tmp[e / blockDim.x] = -v;
        }
        __syncthreads();
        for (int e = threadIdx.x; e < n2 * n1; e += blockDim.x) {
            const int i = n1 + e % n2, j = e / n2;
            X[i + LD * j] = tmp[e / blockDim.x];
        }
        __syncthreads();
    }
    for (int e = threadIdx.x; e < nb * nb; e += blockDim.x) {
        const int i = e % nb, j = e / nb;
        a[(k0 + i) + (size_t)lda * (k0 + j)] = (i >= j) ? S[i + LD * j] : 0.0;
    }
    double* inv = Linv + (size_t)blockIdx.x * kCholNB * kCholNB;
    for (int e = threadIdx.x; e < nb * nb; e += blockDim.x) inv[(e % nb) + kCholNB * (e / nb)] = X[(e % nb) + LD * (e / nb)];
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
struct PanelB {  // B(k, j) = Linv(j, k)
    const double* Linv;
    __device__ double operator()(int b, int k, int j) const {
        return Linv[(size_t)b * kCholNB * kCholNB + j + kCholNB * k];
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

// In-place batched semi-definite Cholesky.  Lower triangle holds L on return,
// upper triangle is zeroed.  rank[b] (device) = n - #deficient pivots.
inline void chol_batched(double* A, int n, int lda, long long sA, int batch, double tol, double* maxdiag,
                         int* rank, cudaStream_t st) {
    if (batch <= 0 || n <= 0) return;
    constexpr size_t kDiagSmem = 2 * kCholNB * (kCholNB + 1) * sizeof(double);
    static bool attr = false;
    if (!attr) {
        OCTEN_CUDA(cudaFuncSetAttribute(chol_diag_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kDiagSmem));
        attr = true;
    }
    static thread_local DevBuf<double> linv;
    linv.reserve((size_t)batch * kCholNB * kCholNB);
    chol_maxdiag_kernel<<<batch, 256, 0, st>>>(A, n, lda, sA, maxdiag, rank); OCTEN_LAUNCHED(1);
    for (int k0 = 0; k0 < n; k0 += kCholNB) {
        chol_diag_kernel<<<batch, 256, kDiagSmem, st>>>(A, n, lda, sA, k0, tol, maxdiag, rank, linv.p); OCTEN_LAUNCHED(1);
        const int nb = min(kCholNB, n - k0);
        const int rows = n - k0 - nb;
        if (rows <= 0) break;
        const int r0 = k0 + nb;
        gemm_f64<false, true>(batch, rows, nb, nb, PanelA{A, lda, sA, r0, k0}, PanelB{linv.p},
                                               PanelC{A, lda, sA, r0, k0}, st);
        gemm_f64<false, false>(batch, rows, rows, nb, CholTrailA{A, lda, sA, r0, k0},
                                                CholTrailB{A, lda, sA, r0, k0}, CholTrailC{A, lda, sA, r0},
                                                st, 1, nullptr, 1);
    }
}

// Solve L L^T x = b for nrhs right-hand sides per matrix.  Matrix b uses
// factor L[b * sL]; rhs r of matrix b lives at X + b*sX + r*ldx.  Dead
// pivots (L_ii == 0) produce x_i = 0 (callers reject rank-deficient systems
// before solving).  One block per (rhs, matrix).
__global__ void chol_solve_kernel(const double* Lbase, int n, int ldl, long long sL, double* Xbase, int ldx,
                                  long long sX) {
    extern __shared__ double xs[];
    __shared__ double D[32][33];
    const double* L = Lbase + (size_t)blockIdx.y * sL;
    double* X = Xbase + (size_t)blockIdx.y * sX + (size_t)blockIdx.x * ldx;
    for (int i = threadIdx.x; i < n; i += blockDim.x) xs[i] = X[i];
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
                if (lane == j) {
                    const double d = D[lane][lane];
                    xi = (d != 0.0) ? xi / d : 0.0;
                }
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
                if (lane == jj) {
                    const double d = D[lane][lane];
                    xi = (d != 0.0) ? xi / d : 0.0;
                }
                const double xj = __shfl_sync(0xffffffffu, xi, jj);
                if (lane < jj) xi -= D[jj][lane] * xj;
            }
            if (lane < nb) xs[i] = xi;
        }
        __syncthreads();
        for (int i = threadIdx.x; i < b0; i += blockDim.x) {
            double s = xs[i];
            const double* lrow = L + (size_t)ldl * i;  // column i of L = row i of L^T
            for (int j = 0; j < nb; ++j) s -= lrow[b0 + j] * xs[b0 + j];
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
    const size_t smem = (size_t)n * sizeof(double);
    if (smem > 48 * 1024) cudaFuncSetAttribute(chol_solve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    chol_solve_kernel<<<g, 1024, smem, st>>>(L, n, ldl, sL, X, ldx, sX); OCTEN_LAUNCHED(1);
}

}  // namespace octen
