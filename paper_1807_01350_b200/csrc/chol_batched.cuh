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

#include "gemm_simt.cuh"
#include "octen_common.cuh"

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

// Factor the nb x nb diagonal block at offset k0 of every matrix.
__global__ void chol_diag_kernel(double* A, int n, int lda, long long sA, int k0, double tol,
                                 const double* maxdiag, int* rank) {
    __shared__ double S[kCholNB][kCholNB + 1];
    __shared__ double piv;
    __shared__ int dead;
    double* a = A + (size_t)blockIdx.x * sA;
    const int nb = min(kCholNB, n - k0);
    for (int e = threadIdx.x; e < nb * nb; e += blockDim.x) {
        const int i = e % nb, j = e / nb;
        S[i][j] = a[(k0 + i) + (size_t)lda * (k0 + j)];
    }
    __syncthreads();
    const double thr = tol * maxdiag[blockIdx.x];
    for (int k = 0; k < nb; ++k) {
        if (threadIdx.x == 0) {
            const double d = S[k][k];
            if (!(d > thr) || !(maxdiag[blockIdx.x] > 0.0)) {
                dead = 1;
                piv = 0.0;
                atomicSub(&rank[blockIdx.x], 1);
            } else {
                dead = 0;
                piv = sqrt(d);
            }
        }
        __syncthreads();
        for (int i = k + threadIdx.x; i < nb; i += blockDim.x) S[i][k] = dead ? 0.0 : (i == k ? piv : S[i][k] / piv);
        __syncthreads();
        for (int e = threadIdx.x; e < (nb - k - 1) * (nb - k - 1); e += blockDim.x) {
            const int i = k + 1 + e % (nb - k - 1), j = k + 1 + e / (nb - k - 1);
            if (i >= j) S[i][j] -= S[i][k] * S[j][k];
        }
        __syncthreads();
    }
    for (int e = threadIdx.x; e < nb * nb; e += blockDim.x) {
        const int i = e % nb, j = e / nb;
        a[(k0 + i) + (size_t)lda * (k0 + j)] = (i >= j) ? S[i][j] : 0.0;
    }
}

// Rows below the diagonal block: L21 = A21 * L11^-T (zero for dead columns).
__global__ void chol_panel_kernel(double* A, int n, int lda, long long sA, int k0) {
    __shared__ double L[kCholNB][kCholNB + 1];
    double* a = A + (size_t)blockIdx.y * sA;
    const int nb = min(kCholNB, n - k0);
    for (int e = threadIdx.x; e < nb * nb; e += blockDim.x) {
        const int i = e % nb, j = e / nb;
        L[i][j] = a[(k0 + i) + (size_t)lda * (k0 + j)];
    }
    __syncthreads();
    const int i = k0 + nb + blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double x[kCholNB];
#pragma unroll 4
    for (int j = 0; j < nb; ++j) x[j] = a[i + (size_t)lda * (k0 + j)];
    for (int j = 0; j < nb; ++j) {
        double s = x[j];
        for (int p = 0; p < j; ++p) s -= x[p] * L[j][p];
        x[j] = (L[j][j] != 0.0) ? s / L[j][j] : 0.0;
    }
#pragma unroll 4
    for (int j = 0; j < nb; ++j) a[i + (size_t)lda * (k0 + j)] = x[j];
}

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
    chol_maxdiag_kernel<<<batch, 256, 0, st>>>(A, n, lda, sA, maxdiag, rank); OCTEN_LAUNCHED(1);
    for (int k0 = 0; k0 < n; k0 += kCholNB) {
        chol_diag_kernel<<<batch, 256, 0, st>>>(A, n, lda, sA, k0, tol, maxdiag, rank); OCTEN_LAUNCHED(1);
        const int nb = min(kCholNB, n - k0);
        const int rows = n - k0 - nb;
        if (rows <= 0) break;
        dim3 g((rows + 127) / 128, batch);
        chol_panel_kernel<<<g, 128, 0, st>>>(A, n, lda, sA, k0); OCTEN_LAUNCHED(1);
        const int r0 = k0 + nb;
        gemm_simt<double, double, false, false>(batch, rows, rows, nb, CholTrailA{A, lda, sA, r0, k0},
                                                CholTrailB{A, lda, sA, r0, k0}, CholTrailC{A, lda, sA, r0},
                                                st);
    }
}

// Solve L L^T x = b for nrhs right-hand sides per matrix.  Matrix b uses
// factor L[b * sL]; rhs r of matrix b lives at X + b*sX + r*ldx.  Dead
// pivots (L_ii == 0) produce x_i = 0 (callers reject rank-deficient systems
// before solving).  One block per (rhs, matrix).
__global__ void chol_solve_kernel(const double* Lbase, int n, int ldl, long long sL, double* Xbase, int ldx,
                                  long long sX) {
    extern __shared__ double xs[];
    const double* L = Lbase + (size_t)blockIdx.y * sL;
    double* X = Xbase + (size_t)blockIdx.y * sX + (size_t)blockIdx.x * ldx;
    for (int i = threadIdx.x; i < n; i += blockDim.x) xs[i] = X[i];
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // forward: L y = b
    for (int b0 = 0; b0 < n; b0 += 32) {
        const int nb = min(32, n - b0);
        if (warp == 0) {
            const int i = b0 + lane;
            double xi = (lane < nb) ? xs[i] : 0.0;
            for (int j = 0; j < nb; ++j) {
                if (lane == j) {
                    const double d = L[i + (size_t)ldl * i];
                    xi = (d != 0.0) ? xi / d : 0.0;
                }
                const double xj = __shfl_sync(0xffffffffu, xi, j);
                if (lane > j && lane < nb) xi -= L[i + (size_t)ldl * (b0 + j)] * xj;
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
        if (warp == 0) {
            const int i = b0 + lane;
            double xi = (lane < nb) ? xs[i] : 0.0;
            for (int jj = nb - 1; jj >= 0; --jj) {
                if (lane == jj) {
                    const double d = L[i + (size_t)ldl * i];
                    xi = (d != 0.0) ? xi / d : 0.0;
                }
                const double xj = __shfl_sync(0xffffffffu, xi, jj);
                if (lane < jj) xi -= L[(b0 + jj) + (size_t)ldl * i] * xj;
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
    chol_solve_kernel<<<g, 256, smem, st>>>(L, n, ldl, sL, X, ldx, sX); OCTEN_LAUNCHED(1);
}

}  // namespace octen
