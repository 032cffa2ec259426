#pragma once
namespace octen {
template <int kPer, int kThreads>
__device__ inline int block_chol_inv_old(const double* a, int lda, int n, double thr, double* l, int ldl, double* x,
                                       int ldx, double* scratch) {
    // kThreads == blockDim.x (compile time: the owner arithmetic below divides by it)
    // branch-free updates: colk[i] = 0 for i <= k, rowk[j] = 0 for j > k;
    // unused slots point at the zero entries colk[64] / rowk[64]
    double* colk = scratch;        // 65
    double* rowk = scratch + 65;   // 65
    double* shv = scratch + 130;   // [0..1] reciprocal pivots (double-buffered), [2] dead count
    const int tid = threadIdx.x;
    double av[kPer], bv[kPer];
    int iv[kPer], jv[kPer];
    if (tid <= 64) {
        colk[tid] = 0.0;
        rowk[tid] = 0.0;
    }
    if (tid == 0) shv[2] = 0.0;
#pragma unroll
    for (int s = 0; s < kPer; ++s) {
        const int e = tid + kThreads * s;
        int i = (int)((sqrtf(8.0f * (float)e + 1.0f) - 1.0f) * 0.5f);
        while ((i + 1) * (i + 2) / 2 <= e) ++i;
        while (i * (i + 1) / 2 > e) --i;
        const int j = e - i * (i + 1) / 2;
        const bool ok = i < n;
        iv[s] = ok ? i : 64;
        jv[s] = ok ? j : 64;
        av[s] = ok ? a[i + (size_t)lda * j] : 0.0;
        bv[s] = (ok && i == j) ? 1.0 : 0.0;
    }
    auto pivot = [&](int k) {
        const int ed = k * (k + 3) / 2;
        if (tid == ed % kThreads) {
            const int sd = ed / kThreads;
#pragma unroll
            for (int s = 0; s < kPer; ++s)
                if (s == sd) {
                    const double d = av[s];
                    const bool dead = !(d > thr);
                    const double rp = dead ? 0.0 : rsqrt(d);
                    av[s] = dead ? 0.0 : d * rp;
                    shv[k & 1] = rp;
                    if (dead) shv[2] += 1.0;
                }
        }
    };
    __syncthreads();
    if (n > 0) pivot(0);
    __syncthreads();
    for (int k = 0; k < n; ++k) {
        const double rp = shv[k & 1];
#pragma unroll
        for (int s = 0; s < kPer; ++s) {
            const int i = iv[s], j = jv[s];
            if (j == k && i > k) {
                av[s] *= rp;
                colk[i] = av[s];
            }
            if (i == k) {
                bv[s] *= rp;
                rowk[j] = bv[s];
            }
        }
        if (tid == 0) colk[k] = 0.0;
        __syncthreads();
#pragma unroll
        for (int s = 0; s < kPer; ++s) {
            const double ci = colk[iv[s]];
            av[s] -= ci * colk[jv[s]];
            bv[s] -= ci * rowk[jv[s]];
        }
        if (k + 1 < n) pivot(k + 1);
        __syncthreads();
    }
    for (int e = tid; e < n * n; e += kThreads) {
        const int i = e % n, j = e / n;
        if (i < j) {
            l[i + (size_t)ldl * j] = 0.0;
            x[i + (size_t)ldx * j] = 0.0;
        }
    }
#pragma unroll
    for (int s = 0; s < kPer; ++s)
        if (iv[s] < 64) {
            l[iv[s] + (size_t)ldl * jv[s]] = av[s];
            x[iv[s] + (size_t)ldx * jv[s]] = bv[s];
        }
    __syncthreads();
    return n - (int)shv[2];
}

}
