// Small dense linear algebra used inside the OCTen kernels: one problem per
// thread block ("team"), matrices resident in shared memory.  Every routine
// is OCTEN_HD so tests/cpu_harness can run the exact same code on the host
// (one-thread team) against numpy.
//
// These replace the Eigen decompositions the reference calls on small
// matrices (reference paths relative to /root/reference/proj):
//   * jacobi_eig_sym      -- BDCSVD thin-U of the unfoldings (cp_als.cpp:96-100)
//                            via the Gram eigenbasis; also the pseudo-inverse
//                            fallback for rank-deficient COD solves
//   * eig_real (orthes+hqr2) -- Eigen::EigenSolver on the R x R GEVD pencil
//                            (cp_als.cpp:126-140)
//   * lu_fullpiv_*        -- Eigen::FullPivLU isInvertible/inverse (cp_als.cpp:122-124)
//   * chol_semidef        -- LLT / rank-revealing solves (recovery.cpp:26-38,151-173,486)
//   * greedy_match        -- recovery.cpp:42-85
//   * top_singular_pair   -- JacobiSVD rank-1 peel (cp_als.cpp:24-36)
//   * Mt64                -- std::mt19937_64 for the ALS column rescue stream
//                            (cp_als.cpp:293,311-316; rng.hpp:51-85)
#pragma once

#include "octen_common.cuh"
#if defined(__CUDACC__)
#include "gemm_dmma.cuh"  // block_dmma_small (device paths of the team routines)
#endif

namespace octen {

// ---------------------------------------------------------------------------
// std::mt19937_64 (published definition), 53-bit uniforms as rng.hpp:56.
// ---------------------------------------------------------------------------
struct Mt64 {
    uint64_t mt[312];
    int idx;

    OCTEN_HD void seed(uint64_t s) {
        mt[0] = s;
        for (int i = 1; i < 312; ++i)
            mt[i] = 6364136223846793005ULL * (mt[i - 1] ^ (mt[i - 1] >> 62)) + (uint64_t)i;
        idx = 312;
    }
    OCTEN_HD void twist() {
        const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL, A = 0xB5026F5AA96619E9ULL;
        for (int i = 0; i < 312; ++i) {
            uint64_t x = (mt[i] & UM) | (mt[(i + 1) % 312] & LM);
            uint64_t xa = x >> 1;
            if (x & 1ULL) xa ^= A;
            mt[i] = mt[(i + 156) % 312] ^ xa;
        }
        idx = 0;
    }
    OCTEN_HD uint64_t next() {
        if (idx >= 312) twist();
        uint64_t y = mt[idx++];
        y ^= (y >> 29) & 0x5555555555555555ULL;
        y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
        y ^= (y << 37) & 0xFFF7EEE000000000ULL;
        y ^= y >> 43;
        return y;
    }
    OCTEN_HD double uniform01() { return (double)(next() >> 11) * 0x1.0p-53; }
};

OCTEN_HD inline uint64_t splitmix(uint64_t z) {
    z += 0x9e3779b97f4a7c15ULL;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

// ---------------------------------------------------------------------------
// Greedy column matching (recovery.cpp:42-85).  sim is r x r column-major
// with leading dimension ld; perm[ref] = cand.  Returns the number of steps
// that saw more than one candidate within tie_tol (the reference logs these).
// Single thread.
// ---------------------------------------------------------------------------
OCTEN_HD inline int greedy_match(int r, const double* sim, int ld, double tie_tol, int* perm,
                                 unsigned char* ref_used, unsigned char* cand_used) {
    int ambiguous = 0;
    for (int i = 0; i < r; ++i) {
        perm[i] = -1;
        ref_used[i] = 0;
        cand_used[i] = 0;
    }
    for (int step = 0; step < r; ++step) {
        double best = -INFINITY;
        for (int i = 0; i < r; ++i) {
            if (ref_used[i]) continue;
            for (int j = 0; j < r; ++j) {
                if (cand_used[j]) continue;
                const double v = sim[i + (size_t)ld * j];
                best = v > best ? v : best;
            }
        }
        int bi = -1, bj = -1, ties = 0;
        for (int i = 0; i < r && bi < 0; ++i) {
            if (ref_used[i]) continue;
            for (int j = 0; j < r; ++j) {
                if (cand_used[j]) continue;
                if (sim[i + (size_t)ld * j] >= best - tie_tol) {
                    bi = i;
                    bj = j;
                    break;
                }
            }
        }
        for (int i = 0; i < r; ++i) {
            if (ref_used[i]) continue;
            for (int j = 0; j < r; ++j)
                if (!cand_used[j] && sim[i + (size_t)ld * j] >= best - tie_tol) ++ties;
        }
        if (ties > 1) ++ambiguous;
        if (bi < 0) {  // NaN similarities: take the first free pair
            for (int i = 0; i < r && bi < 0; ++i)
                if (!ref_used[i])
                    for (int j = 0; j < r; ++j)
                        if (!cand_used[j]) {
                            bi = i;
                            bj = j;
                            break;
                        }
        }
        perm[bi] = bj;
        ref_used[bi] = 1;
        cand_used[bj] = 1;
    }
    return ambiguous;
}

// ---------------------------------------------------------------------------
// Semi-definite Cholesky, in place, lower triangle of a column-major n x n
// matrix.  A pivot <= tol * max_diag(A) marks the column deficient: it is
// zeroed and skipped (exact for PSD input, whose Schur complement then has a
// zero row/column).  Returns the numerical rank.  Single thread.
// ---------------------------------------------------------------------------
OCTEN_HD inline int chol_semidef(int n, double* a, int lda, double tol) {
    double maxd = 0.0;
    for (int i = 0; i < n; ++i) {
        const double v = a[i + (size_t)lda * i];
        maxd = v > maxd ? v : maxd;
    }
    const double thr = tol * maxd;
    int rank = 0;
    for (int k = 0; k < n; ++k) {
        double d = a[k + (size_t)lda * k];
        for (int p = 0; p < k; ++p) d -= dsq(a[k + (size_t)lda * p]);
        if (!(d > thr) || maxd <= 0.0) {
            for (int i = k; i < n; ++i) a[i + (size_t)lda * k] = 0.0;
            continue;
        }
        ++rank;
        const double lkk = sqrt(d);
        a[k + (size_t)lda * k] = lkk;
        for (int i = k + 1; i < n; ++i) {
            double s = a[i + (size_t)lda * k];
            for (int p = 0; p < k; ++p) s -= a[i + (size_t)lda * p] * a[k + (size_t)lda * p];
            a[i + (size_t)lda * k] = s / lkk;
        }
    }
    return rank;
}

// Team-parallel version of chol_semidef (right-looking, rows over the team).
// sc: 1 double + 2 ints of shared scratch.  Returns the rank to every thread.
// thr_abs >= 0 replaces tol * max(diag) as the absolute pivot threshold.
template <class Team>
OCTEN_HD int team_chol_semidef(const Team& team, int n, double* a, int lda, double tol, double* sc, int* irank,
                               double thr_abs = -1.0) {
    if (team.tid() == 0) {
        double maxd = 0.0;
        for (int i = 0; i < n; ++i) maxd = fmax(maxd, a[i + (size_t)lda * i]);
        sc[0] = thr_abs >= 0.0 ? 1.0 : maxd;
        *irank = 0;
    }
    team.sync();
    const double maxd = sc[0];
    const double thr = thr_abs >= 0.0 ? thr_abs : tol * maxd;
    for (int k = 0; k < n; ++k) {
        const double d = a[k + (size_t)lda * k];
        const bool dead = !(d > thr) || !(maxd > 0.0);
        const double piv = dead ? 0.0 : sqrt(d);
        team.sync();
        for (int i = k + team.tid(); i < n; i += team.size())
            a[i + (size_t)lda * k] = dead ? 0.0 : (i == k ? piv : a[i + (size_t)lda * k] / piv);
        team.sync();
        if (!dead) {
            for (int i = k + 1 + team.tid(); i < n; i += team.size()) {
                const double lik = a[i + (size_t)lda * k];
                for (int j = k + 1; j <= i; ++j) a[i + (size_t)lda * j] -= lik * a[j + (size_t)lda * k];
            }
        }
        if (team.tid() == 0 && !dead) ++*irank;
        team.sync();
    }
    const int r = *irank;
    team.sync();
    return r;
}

// Inverse of a lower-triangular n x n matrix (column j per team thread);
// zero pivots give zero rows/columns.  x: n x n (ld ldx), may alias nothing.
template <class Team>
OCTEN_HD void team_tri_inv_lower(const Team& team, int n, const double* l, int ldl, double* x, int ldx) {
    for (int j = team.tid(); j < n; j += team.size())
        for (int i = 0; i < n; ++i) {
            double v = (i == j) ? 1.0 : 0.0;
            for (int p = j; p < i; ++p) v -= l[i + (size_t)ldl * p] * x[p + (size_t)ldx * j];
            const double d = l[i + (size_t)ldl * i];
            x[i + (size_t)ldx * j] = (i < j || d == 0.0) ? 0.0 : v / d;
        }
    team.sync();
}

#if defined(__CUDACC__)
// Warp Cholesky + triangular inverse of an n x n (n <= 32) symmetric block in
// shared memory (column-major, ld lds; lower part read).  Left-looking: for
// column j, lane i > j forms L_ij from independent loads of rows i and j (no
// load/store chains), one reciprocal per column.  Loops are kept rolled: an
// unrolled version overflows the instruction cache (executed once per
// launch).  s is overwritten with L (upper zeroed), x (ld ldx) receives L^-1.
// A pivot <= thr marks a deficient column (zeroed, as chol_semidef).  Returns
// the rank; must be called by all 32 lanes of one warp.
__device__ inline int warp_chol_inv32(double* s, int lds, int n, double thr, double* x, int ldx) {
    const int lane = threadIdx.x & 31;
    int rank = 0;
#pragma unroll 1
    for (int j = 0; j < n; ++j) {
        // diagonal: L_jj^2 = a_jj - sum_{p<j} L_jp^2 (every lane computes it);
        // four independent partial sums break the FMA dependency chain
        double d0 = 0.0, d1 = 0.0, d2 = 0.0, d3 = 0.0;
        int p = 0;
#pragma unroll 1
        for (; p + 3 < j; p += 4) {
            const double l0 = s[j + (size_t)lds * p], l1 = s[j + (size_t)lds * (p + 1)];
            const double l2 = s[j + (size_t)lds * (p + 2)], l3 = s[j + (size_t)lds * (p + 3)];
            d0 += l0 * l0;
            d1 += l1 * l1;
            d2 += l2 * l2;
            d3 += l3 * l3;
        }
        for (; p < j; ++p) {
            const double l = s[j + (size_t)lds * p];
            d0 += l * l;
        }
        const double d = s[j + (size_t)lds * j] - ((d0 + d1) + (d2 + d3));
        const bool dead = !(d > thr);
        const double piv = dead ? 0.0 : sqrt(d);
        const double rp = dead ? 0.0 : 1.0 / piv;
        double lij = 0.0;
        const int i = lane;
        if (i > j && i < n) {
            double v0 = 0.0, v1 = 0.0, v2 = 0.0, v3 = 0.0;
            int q = 0;
#pragma unroll 1
            for (; q + 3 < j; q += 4) {
                v0 += s[i + (size_t)lds * q] * s[j + (size_t)lds * q];
                v1 += s[i + (size_t)lds * (q + 1)] * s[j + (size_t)lds * (q + 1)];
                v2 += s[i + (size_t)lds * (q + 2)] * s[j + (size_t)lds * (q + 2)];
                v3 += s[i + (size_t)lds * (q + 3)] * s[j + (size_t)lds * (q + 3)];
            }
            for (; q < j; ++q) v0 += s[i + (size_t)lds * q] * s[j + (size_t)lds * q];
            lij = (s[i + (size_t)lds * j] - ((v0 + v1) + (v2 + v3))) * rp;
        }
        __syncwarp();
        if (i > j && i < n) s[i + (size_t)lds * j] = lij;
        if (i == j) s[j + (size_t)lds * j] = piv;
        if (i < j && i < n) s[i + (size_t)lds * j] = 0.0;
        rank += dead ? 0 : 1;
        __syncwarp();
    }
    // inverse: lane j owns column j of L^-1
    if (lane < n) {
        const int j = lane;
#pragma unroll 1
        for (int i = 0; i < n; ++i) {
            double v0 = (i == j) ? 1.0 : 0.0, v1 = 0.0, v2 = 0.0, v3 = 0.0;
            if (i > j) {
                int p = j;
#pragma unroll 1
                for (; p + 3 < i; p += 4) {
                    v0 -= s[i + (size_t)lds * p] * x[p + (size_t)ldx * j];
                    v1 -= s[i + (size_t)lds * (p + 1)] * x[p + 1 + (size_t)ldx * j];
                    v2 -= s[i + (size_t)lds * (p + 2)] * x[p + 2 + (size_t)ldx * j];
                    v3 -= s[i + (size_t)lds * (p + 3)] * x[p + 3 + (size_t)ldx * j];
                }
                for (; p < i; ++p) v0 -= s[i + (size_t)lds * p] * x[p + (size_t)ldx * j];
            }
            const double lii = s[i + (size_t)lds * i];
            x[i + (size_t)ldx * j] = (i < j || lii == 0.0) ? 0.0 : ((v0 + v1) + (v2 + v3)) / lii;
        }
    }
    __syncwarp();
    return rank;
}
#endif

#if defined(__CUDACC__)
// ---------------------------------------------------------------------------
// greedy_match (above) with the whole block: per step one max-reduction for
// the best free similarity, then one combined reduction for the
// lexicographically first free pair within tie_tol of it (lowest ref, then
// lowest candidate) and the number of such pairs.  Same result as the serial
// routine, R steps of O(R^2 / blockDim) work.  blockDim.x % 32 == 0, r <= 64.
// scratch: 3 * 32 doubles.  Returns the ambiguity count (all threads).
// ---------------------------------------------------------------------------
__device__ inline int block_greedy_match(int r, const double* sim, int ld, double tie_tol, int* perm,
                                         unsigned char* ref_used, unsigned char* cand_used, double* scratch) {
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = blockDim.x >> 5;
    double* rmax = scratch;        // per-warp max
    double* rkey = scratch + 32;   // per-warp min key
    double* rcnt = scratch + 64;   // per-warp tie count
    for (int i = tid; i < r; i += blockDim.x) {
        perm[i] = -1;
        ref_used[i] = 0;
        cand_used[i] = 0;
    }
    __syncthreads();
    int ambiguous = 0;
    const int rr = r * r;
    for (int step = 0; step < r; ++step) {
        double best = -INFINITY;
        int firstfree = 0x7fffffff;
        for (int e = tid; e < rr; e += blockDim.x) {
            const int i = e / r, j = e % r;  // key order: ref-major
            if (ref_used[i] || cand_used[j]) continue;
            const double v = sim[i + (size_t)ld * j];
            best = v > best ? v : best;
            firstfree = min(firstfree, e);
        }
        for (int o = 16; o > 0; o >>= 1) {
            best = fmax(best, __shfl_xor_sync(0xffffffffu, best, o));
            firstfree = min(firstfree, __shfl_xor_sync(0xffffffffu, firstfree, o));
        }
        if (lane == 0) {
            rmax[wid] = best;
            rkey[wid] = (double)firstfree;
        }
        __syncthreads();
        best = -INFINITY;
        double ff = 2147483647.0;
        for (int w = 0; w < nw; ++w) {
            best = fmax(best, rmax[w]);
            ff = fmin(ff, rkey[w]);
        }
        __syncthreads();
        int key = 0x7fffffff, cnt = 0;
        for (int e = tid; e < rr; e += blockDim.x) {
            const int i = e / r, j = e % r;
            if (ref_used[i] || cand_used[j]) continue;
            if (sim[i + (size_t)ld * j] >= best - tie_tol) {
                key = min(key, e);
                ++cnt;
            }
        }
        for (int o = 16; o > 0; o >>= 1) {
            key = min(key, __shfl_xor_sync(0xffffffffu, key, o));
            cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
        }
        if (lane == 0) {
            rkey[wid] = (double)key;
            rcnt[wid] = (double)cnt;
        }
        __syncthreads();
        double kk = 2147483647.0, cc = 0.0;
        for (int w = 0; w < nw; ++w) {
            kk = fmin(kk, rkey[w]);
            cc += rcnt[w];
        }
        if (cc > 1.0) ++ambiguous;
        // NaN similarities: no pair qualifies -> the first free pair
        const int pick = (kk < 2147483647.0) ? (int)kk : (int)ff;
        __syncthreads();
        if (tid == 0) {
            const int bi = pick / r, bj = pick % r;
            perm[bi] = bj;
            ref_used[bi] = 1;
            cand_used[bj] = 1;
        }
        __syncthreads();
    }
    return ambiguous;
}
#endif

#if defined(__CUDACC__)
// ---------------------------------------------------------------------------
// Block-cooperative semi-definite Cholesky with the inverse of the factor,
// n <= 64, blockDim.x == 256.  Every thread keeps a fixed share of the packed
// lower triangle of A (-> L) and of B (I -> L^-1) in registers; step k
// publishes column k of L and row k of L^-1 through shared memory and all
// threads apply the rank-1 updates to their own elements (two barriers per
// step, no serial warp).  A pivot <= thr is dead: column k of L and row k of
// L^-1 become zero.  a (ld lda) is read only; l (ld ldl, lower; upper zeroed)
// and x (ld ldx, lower; upper zeroed) are written.  Returns the rank (all
// threads).
// ---------------------------------------------------------------------------
template <int kPer, int kThreads>
__device__ inline int block_chol_inv_t(const double* a, int lda, int n, double thr, double* l, int ldl, double* x,
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

// Block-cooperative semi-definite Cholesky with the inverse of the factor,
// n <= 64, blockDim.x == 256 (see block_chol_inv_t): every thread keeps
// ceil(n(n+1)/2 / 256) elements of the packed lower triangles of A (-> L) and I
// (-> L^-1) in registers; the pivot of step k+1 is formed by its owner
// during step k.  scratch: 133 doubles of shared memory.
__device__ inline int block_chol_inv64(const double* a, int lda, int n, double thr, double* l, int ldl, double* x,
                                       int ldx, double* scratch) {
    // blockDim.x == 256 (the ALS update kernel)
    const int per = (n * (n + 1) / 2 + 255) / 256;
    if (per <= 1) return block_chol_inv_t<1, 256>(a, lda, n, thr, l, ldl, x, ldx, scratch);
    if (per <= 3) return block_chol_inv_t<3, 256>(a, lda, n, thr, l, ldl, x, ldx, scratch);
    if (per <= 5) return block_chol_inv_t<5, 256>(a, lda, n, thr, l, ldl, x, ldx, scratch);
    return block_chol_inv_t<9, 256>(a, lda, n, thr, l, ldl, x, ldx, scratch);
}
#endif

#if defined(__CUDACC__)
// max of the diagonal of an n x n matrix, reduced over one warp (all lanes get it)
__device__ inline double warp_max_diag(const double* a, int lda, int n) {
    double m = 0.0;
    for (int i = threadIdx.x & 31; i < n; i += 32) m = fmax(m, a[i + (size_t)lda * i]);
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    return m;
}
#endif

// Solve L L^T x = b in place for one vector (full-rank factor from chol_semidef).
OCTEN_HD inline void chol_solve_vec(int n, const double* l, int ldl, double* x, int incx) {
    for (int i = 0; i < n; ++i) {
        double s = x[(size_t)incx * i];
        for (int p = 0; p < i; ++p) s -= l[i + (size_t)ldl * p] * x[(size_t)incx * p];
        x[(size_t)incx * i] = s / l[i + (size_t)ldl * i];
    }
    for (int i = n - 1; i >= 0; --i) {
        double s = x[(size_t)incx * i];
        for (int p = i + 1; p < n; ++p) s -= l[p + (size_t)ldl * i] * x[(size_t)incx * p];
        x[(size_t)incx * i] = s / l[i + (size_t)ldl * i];
    }
}

// Forward substitution L y = b (lower, non-unit).  Single thread.
OCTEN_HD inline void trsv_lower(int n, const double* l, int ldl, double* x, int incx) {
    for (int i = 0; i < n; ++i) {
        double s = x[(size_t)incx * i];
        for (int p = 0; p < i; ++p) s -= l[i + (size_t)ldl * p] * x[(size_t)incx * p];
        x[(size_t)incx * i] = s / l[i + (size_t)ldl * i];
    }
}

// ---------------------------------------------------------------------------
// Full-pivot LU (Eigen::FullPivLU semantics): rank counts pivots
// > epsilon * n * |maxpivot|.  On return `inv` holds the inverse when the
// matrix is invertible.  a is destroyed.  Single thread.  perm scratch: 2n ints.
// ---------------------------------------------------------------------------
OCTEN_HD inline bool lu_fullpiv_inverse(int n, double* a, int lda, double* inv, int ldi, int* rowp,
                                        int* colp) {
    double maxpiv = 0.0;
    double piv_abs[64];
    for (int k = 0; k < n; ++k) {
        int bi = k, bj = k;
        double best = -1.0;
        for (int j = k; j < n; ++j)
            for (int i = k; i < n; ++i) {
                const double v = fabs(a[i + (size_t)lda * j]);
                if (v > best) {
                    best = v;
                    bi = i;
                    bj = j;
                }
            }
        rowp[k] = bi;
        colp[k] = bj;
        if (bi != k)
            for (int j = 0; j < n; ++j) {
                const double t = a[k + (size_t)lda * j];
                a[k + (size_t)lda * j] = a[bi + (size_t)lda * j];
                a[bi + (size_t)lda * j] = t;
            }
        if (bj != k)
            for (int i = 0; i < n; ++i) {
                const double t = a[i + (size_t)lda * k];
                a[i + (size_t)lda * k] = a[i + (size_t)lda * bj];
                a[i + (size_t)lda * bj] = t;
            }
        const double p = a[k + (size_t)lda * k];
        piv_abs[k] = fabs(p);
        if (fabs(p) > maxpiv) maxpiv = fabs(p);
        if (p != 0.0) {
            for (int i = k + 1; i < n; ++i) a[i + (size_t)lda * k] /= p;
            for (int j = k + 1; j < n; ++j) {
                const double u = a[k + (size_t)lda * j];
                for (int i = k + 1; i < n; ++i) a[i + (size_t)lda * j] -= a[i + (size_t)lda * k] * u;
            }
        }
    }
    const double thr = 2.220446049250313e-16 * (double)n * maxpiv;
    int rank = 0;
    for (int k = 0; k < n; ++k)
        if (piv_abs[k] > thr) ++rank;
    if (rank < n) return false;
    // inverse: solve (P A Q) = L U  ->  A^-1 = Q U^-1 L^-1 P
    for (int c = 0; c < n; ++c) {
        double* x = inv + (size_t)ldi * c;
        for (int i = 0; i < n; ++i) x[i] = (i == c) ? 1.0 : 0.0;
        for (int k = 0; k < n; ++k)  // apply row swaps P
            if (rowp[k] != k) {
                const double t = x[k];
                x[k] = x[rowp[k]];
                x[rowp[k]] = t;
            }
        for (int i = 0; i < n; ++i)  // L y = Pb (unit lower)
            for (int p = 0; p < i; ++p) x[i] -= a[i + (size_t)lda * p] * x[p];
        for (int i = n - 1; i >= 0; --i) {  // U z = y
            for (int p = i + 1; p < n; ++p) x[i] -= a[i + (size_t)lda * p] * x[p];
            x[i] /= a[i + (size_t)lda * i];
        }
        for (int k = n - 1; k >= 0; --k)  // undo column swaps Q
            if (colp[k] != k) {
                const double t = x[k];
                x[k] = x[colp[k]];
                x[colp[k]] = t;
            }
    }
    return true;
}

// ---------------------------------------------------------------------------
// Real nonsymmetric eigen-decomposition: Householder reduction to Hessenberg
// form (EISPACK orthes) followed by the shifted double-step QR iteration with
// eigenvector back-substitution (EISPACK hqr2), as in Eigen's EigenSolver
// (RealSchur + complex back-substitution).  Eigenvalues come back as (wr, wi);
// complex pairs are adjacent with the positive imaginary part first and their
// eigenvector stored as [Re | Im] in columns (c, c+1) -- the layout the
// reference turns into a_sub (cp_als.cpp:128-140).  Eigenvectors are not
// normalized (the reference normalizes each a1 column afterwards, which makes
// the scale irrelevant).  h and v are n x n column-major (ld n), ort is n
// scratch.  Returns false if the QR iteration does not converge within 40n
// steps (Eigen's maxIterations).  Single thread.
// ---------------------------------------------------------------------------
namespace detail {
OCTEN_HD inline void cdiv(double xr, double xi, double yr, double yi, double& cr, double& ci) {
    double r, d;
    if (fabs(yr) > fabs(yi)) {
        r = yi / yr;
        d = yr + r * yi;
        cr = (xr + r * xi) / d;
        ci = (xi - r * xr) / d;
    } else {
        r = yr / yi;
        d = yi + r * yr;
        cr = (r * xr + xi) / d;
        ci = (r * xi - xr) / d;
    }
}
}  // namespace detail

OCTEN_HD inline bool eig_real(int nn, double* hm, double* vm, double* wr, double* wi, double* ort) {
#define H_(i, j) hm[(i) + (size_t)nn * (j)]
#define V_(i, j) vm[(i) + (size_t)nn * (j)]
    const int low = 0, high = nn - 1;
    // --- orthes ---
    for (int m = low + 1; m <= high - 1; ++m) {
        double scale = 0.0;
        for (int i = m; i <= high; ++i) scale += fabs(H_(i, m - 1));
        if (scale != 0.0) {
            double h = 0.0;
            for (int i = high; i >= m; --i) {
                ort[i] = H_(i, m - 1) / scale;
                h += ort[i] * ort[i];
            }
            double g = sqrt(h);
            if (ort[m] > 0) g = -g;
            h = h - ort[m] * g;
            ort[m] = ort[m] - g;
            for (int j = m; j < nn; ++j) {
                double f = 0.0;
                for (int i = high; i >= m; --i) f += ort[i] * H_(i, j);
                f = f / h;
                for (int i = m; i <= high; ++i) H_(i, j) -= f * ort[i];
            }
            for (int i = 0; i <= high; ++i) {
                double f = 0.0;
                for (int j = high; j >= m; --j) f += ort[j] * H_(i, j);
                f = f / h;
                for (int j = m; j <= high; ++j) H_(i, j) -= f * ort[j];
            }
            ort[m] = scale * ort[m];
            H_(m, m - 1) = scale * g;
        }
    }
    for (int i = 0; i < nn; ++i)
        for (int j = 0; j < nn; ++j) V_(i, j) = (i == j) ? 1.0 : 0.0;
    for (int m = high - 1; m >= low + 1; --m) {
        if (H_(m, m - 1) != 0.0) {
            for (int i = m + 1; i <= high; ++i) ort[i] = H_(i, m - 1);
            for (int j = m; j <= high; ++j) {
                double g = 0.0;
                for (int i = m; i <= high; ++i) g += ort[i] * V_(i, j);
                g = (g / ort[m]) / H_(m, m - 1);
                for (int i = m; i <= high; ++i) V_(i, j) += g * ort[i];
            }
        }
    }
    // --- hqr2 ---
    int n = nn - 1;
    const double eps = 2.220446049250313e-16;
    double exshift = 0.0, p = 0, q = 0, r = 0, s = 0, z = 0, t, w, x, y;
    double norm = 0.0;
    for (int i = 0; i < nn; ++i) {
        if (i < low || i > high) {
            wr[i] = H_(i, i);
            wi[i] = 0.0;
        }
        for (int j = (i - 1 > 0 ? i - 1 : 0); j < nn; ++j) norm += fabs(H_(i, j));
    }
    int iter = 0, total_iter = 0;
    const int max_total = 40 * nn;
    while (n >= low) {
        int l = n;
        while (l > low) {
            s = fabs(H_(l - 1, l - 1)) + fabs(H_(l, l));
            if (s == 0.0) s = norm;
            if (fabs(H_(l, l - 1)) < eps * s) break;
            l--;
        }
        if (l == n) {
            H_(n, n) = H_(n, n) + exshift;
            wr[n] = H_(n, n);
            wi[n] = 0.0;
            n--;
            iter = 0;
        } else if (l == n - 1) {
            w = H_(n, n - 1) * H_(n - 1, n);
            p = (H_(n - 1, n - 1) - H_(n, n)) / 2.0;
            q = p * p + w;
            z = sqrt(fabs(q));
            H_(n, n) = H_(n, n) + exshift;
            H_(n - 1, n - 1) = H_(n - 1, n - 1) + exshift;
            x = H_(n, n);
            if (q >= 0) {
                z = (p >= 0) ? p + z : p - z;
                wr[n - 1] = x + z;
                wr[n] = wr[n - 1];
                if (z != 0.0) wr[n] = x - w / z;
                wi[n - 1] = 0.0;
                wi[n] = 0.0;
                x = H_(n, n - 1);
                s = fabs(x) + fabs(z);
                p = x / s;
                q = z / s;
                r = sqrt(p * p + q * q);
                p = p / r;
                q = q / r;
                for (int j = n - 1; j < nn; ++j) {
                    z = H_(n - 1, j);
                    H_(n - 1, j) = q * z + p * H_(n, j);
                    H_(n, j) = q * H_(n, j) - p * z;
                }
                for (int i = 0; i <= n; ++i) {
                    z = H_(i, n - 1);
                    H_(i, n - 1) = q * z + p * H_(i, n);
                    H_(i, n) = q * H_(i, n) - p * z;
                }
                for (int i = low; i <= high; ++i) {
                    z = V_(i, n - 1);
                    V_(i, n - 1) = q * z + p * V_(i, n);
                    V_(i, n) = q * V_(i, n) - p * z;
                }
            } else {
                wr[n - 1] = x + p;
                wr[n] = x + p;
                wi[n - 1] = z;
                wi[n] = -z;
            }
            n = n - 2;
            iter = 0;
        } else {
            x = H_(n, n);
            y = 0.0;
            w = 0.0;
            if (l < n) {
                y = H_(n - 1, n - 1);
                w = H_(n, n - 1) * H_(n - 1, n);
            }
            if (iter == 10) {
                exshift += x;
                for (int i = low; i <= n; ++i) H_(i, i) -= x;
                s = fabs(H_(n, n - 1)) + fabs(H_(n - 1, n - 2));
                x = y = 0.75 * s;
                w = -0.4375 * s * s;
            }
            if (iter == 30) {
                s = (y - x) / 2.0;
                s = s * s + w;
                if (s > 0) {
                    s = sqrt(s);
                    if (y < x) s = -s;
                    s = x - w / ((y - x) / 2.0 + s);
                    for (int i = low; i <= n; ++i) H_(i, i) -= s;
                    exshift += s;
                    x = y = w = 0.964;
                }
            }
            iter = iter + 1;
            if (++total_iter > max_total) return false;
            int m = n - 2;
            while (m >= l) {
                z = H_(m, m);
                r = x - z;
                s = y - z;
                p = (r * s - w) / H_(m + 1, m) + H_(m, m + 1);
                q = H_(m + 1, m + 1) - z - r - s;
                r = H_(m + 2, m + 1);
                s = fabs(p) + fabs(q) + fabs(r);
                p = p / s;
                q = q / s;
                r = r / s;
                if (m == l) break;
                if (fabs(H_(m, m - 1)) * (fabs(q) + fabs(r)) <
                    eps * (fabs(p) * (fabs(H_(m - 1, m - 1)) + fabs(z) + fabs(H_(m + 1, m + 1)))))
                    break;
                m--;
            }
            for (int i = m + 2; i <= n; ++i) {
                H_(i, i - 2) = 0.0;
                if (i > m + 2) H_(i, i - 3) = 0.0;
            }
            for (int k = m; k <= n - 1; ++k) {
                const bool notlast = (k != n - 1);
                if (k != m) {
                    p = H_(k, k - 1);
                    q = H_(k + 1, k - 1);
                    r = notlast ? H_(k + 2, k - 1) : 0.0;
                    x = fabs(p) + fabs(q) + fabs(r);
                    if (x == 0.0) continue;
                    p = p / x;
                    q = q / x;
                    r = r / x;
                }
                s = sqrt(p * p + q * q + r * r);
                if (p < 0) s = -s;
                if (s != 0) {
                    if (k != m)
                        H_(k, k - 1) = -s * x;
                    else if (l != m)
                        H_(k, k - 1) = -H_(k, k - 1);
                    p = p + s;
                    x = p / s;
                    y = q / s;
                    z = r / s;
                    q = q / p;
                    r = r / p;
                    for (int j = k; j < nn; ++j) {
                        p = H_(k, j) + q * H_(k + 1, j);
                        if (notlast) {
                            p = p + r * H_(k + 2, j);
                            H_(k + 2, j) = H_(k + 2, j) - p * z;
                        }
                        H_(k, j) = H_(k, j) - p * x;
                        H_(k + 1, j) = H_(k + 1, j) - p * y;
                    }
                    const int imax = (n < k + 3) ? n : k + 3;
                    for (int i = 0; i <= imax; ++i) {
                        p = x * H_(i, k) + y * H_(i, k + 1);
                        if (notlast) {
                            p = p + z * H_(i, k + 2);
                            H_(i, k + 2) = H_(i, k + 2) - p * r;
                        }
                        H_(i, k) = H_(i, k) - p;
                        H_(i, k + 1) = H_(i, k + 1) - p * q;
                    }
                    for (int i = low; i <= high; ++i) {
                        p = x * V_(i, k) + y * V_(i, k + 1);
                        if (notlast) {
                            p = p + z * V_(i, k + 2);
                            V_(i, k + 2) = V_(i, k + 2) - p * r;
                        }
                        V_(i, k) = V_(i, k) - p;
                        V_(i, k + 1) = V_(i, k + 1) - p * q;
                    }
                }
            }
        }
    }
    // back-substitution
    if (norm == 0.0) return true;
    for (n = nn - 1; n >= 0; n--) {
        p = wr[n];
        q = wi[n];
        if (q == 0) {
            int l = n;
            H_(n, n) = 1.0;
            for (int i = n - 1; i >= 0; i--) {
                w = H_(i, i) - p;
                r = 0.0;
                for (int j = l; j <= n; j++) r = r + H_(i, j) * H_(j, n);
                if (wi[i] < 0.0) {
                    z = w;
                    s = r;
                } else {
                    l = i;
                    if (wi[i] == 0.0) {
                        if (w != 0.0)
                            H_(i, n) = -r / w;
                        else
                            H_(i, n) = -r / (eps * norm);
                    } else {
                        x = H_(i, i + 1);
                        y = H_(i + 1, i);
                        q = (wr[i] - p) * (wr[i] - p) + wi[i] * wi[i];
                        t = (x * s - z * r) / q;
                        H_(i, n) = t;
                        if (fabs(x) > fabs(z))
                            H_(i + 1, n) = (-r - w * t) / x;
                        else
                            H_(i + 1, n) = (-s - y * t) / z;
                    }
                    t = fabs(H_(i, n));
                    if ((eps * t) * t > 1)
                        for (int j = i; j <= n; j++) H_(j, n) = H_(j, n) / t;
                }
            }
        } else if (q < 0) {
            int l = n - 1;
            double cr, ci;
            if (fabs(H_(n, n - 1)) > fabs(H_(n - 1, n))) {
                H_(n - 1, n - 1) = q / H_(n, n - 1);
                H_(n - 1, n) = -(H_(n, n) - p) / H_(n, n - 1);
            } else {
                detail::cdiv(0.0, -H_(n - 1, n), H_(n - 1, n - 1) - p, q, cr, ci);
                H_(n - 1, n - 1) = cr;
                H_(n - 1, n) = ci;
            }
            H_(n, n - 1) = 0.0;
            H_(n, n) = 1.0;
            for (int i = n - 2; i >= 0; i--) {
                double ra = 0.0, sa = 0.0, vr, vi;
                for (int j = l; j <= n; j++) {
                    ra = ra + H_(i, j) * H_(j, n - 1);
                    sa = sa + H_(i, j) * H_(j, n);
                }
                w = H_(i, i) - p;
                if (wi[i] < 0.0) {
                    z = w;
                    r = ra;
                    s = sa;
                } else {
                    l = i;
                    if (wi[i] == 0) {
                        detail::cdiv(-ra, -sa, w, q, cr, ci);
                        H_(i, n - 1) = cr;
                        H_(i, n) = ci;
                    } else {
                        x = H_(i, i + 1);
                        y = H_(i + 1, i);
                        vr = (wr[i] - p) * (wr[i] - p) + wi[i] * wi[i] - q * q;
                        vi = (wr[i] - p) * 2.0 * q;
                        if (vr == 0.0 && vi == 0.0)
                            vr = eps * norm * (fabs(w) + fabs(q) + fabs(x) + fabs(y) + fabs(z));
                        detail::cdiv(x * r - z * ra + q * sa, x * s - z * sa - q * ra, vr, vi, cr, ci);
                        H_(i, n - 1) = cr;
                        H_(i, n) = ci;
                        if (fabs(x) > (fabs(z) + fabs(q))) {
                            H_(i + 1, n - 1) = (-ra - w * H_(i, n - 1) + q * H_(i, n)) / x;
                            H_(i + 1, n) = (-sa - w * H_(i, n) - q * H_(i, n - 1)) / x;
                        } else {
                            detail::cdiv(-r - y * H_(i, n - 1), -s - y * H_(i, n), z, q, cr, ci);
                            H_(i + 1, n - 1) = cr;
                            H_(i + 1, n) = ci;
                        }
                    }
                    t = fmax(fabs(H_(i, n - 1)), fabs(H_(i, n)));
                    if ((eps * t) * t > 1)
                        for (int j = i; j <= n; j++) {
                            H_(j, n - 1) = H_(j, n - 1) / t;
                            H_(j, n) = H_(j, n) / t;
                        }
                }
            }
        }
    }
    for (int j = nn - 1; j >= low; j--)
        for (int i = low; i <= high; i++) {
            z = 0.0;
            const int kmax = j < high ? j : high;
            for (int k = low; k <= kmax; k++) z = z + V_(i, k) * H_(k, j);
            V_(i, j) = z;
        }
    return true;
#undef H_
#undef V_
}

// ---------------------------------------------------------------------------
// Team-parallel twins of lu_fullpiv_inverse and eig_real (same arithmetic per
// element, same pivot/shift/deflation decisions): the O(n) inner loops of
// every O(n) step -- pivot search, row/column swaps and eliminations, the
// Householder applications of orthes, the row/column/vector updates of each
// Francis double-shift step, the eigenvector back-transformation -- are split
// over the team; the scalar control flow runs redundantly in every thread
// from shared values and every scalar store is done by thread 0 between
// barriers.  Used by one warp per GEVD problem (TeamWarp); the host harness
// instantiates them with TeamHost.  scratch: 2 * team.size() doubles.
// ---------------------------------------------------------------------------
template <class Team>
OCTEN_HD void team_argmax_first(const Team& team, double& v, int& key, double* scratch) {
    // max v; ties -> smallest key.  All threads receive the winner.
#if defined(__CUDA_ARCH__)
    if (team.size() == 32) {
        for (int o = 16; o > 0; o >>= 1) {
            const double ov = __shfl_xor_sync(0xffffffffu, v, o);
            const int ok = __shfl_xor_sync(0xffffffffu, key, o);
            if (ov > v || (ov == v && ok < key)) {
                v = ov;
                key = ok;
            }
        }
        return;
    }
#endif
    scratch[2 * team.tid()] = v;
    scratch[2 * team.tid() + 1] = (double)key;
    team.sync();
    double bv = scratch[0];
    int bk = (int)scratch[1];
    for (int t = 1; t < team.size(); ++t) {
        const double ov = scratch[2 * t];
        const int ok = (int)scratch[2 * t + 1];
        if (ov > bv || (ov == bv && ok < bk)) {
            bv = ov;
            bk = ok;
        }
    }
    team.sync();
    v = bv;
    key = bk;
}

template <class Team>
OCTEN_HD bool lu_fullpiv_inverse_team(const Team& team, int n, double* a, int lda, double* inv, int ldi,
                                      int* rowp, int* colp, double* piv_abs, double* scratch) {
    const int T = team.tid(), NT = team.size();
    double maxpiv = 0.0;
    for (int k = 0; k < n; ++k) {
        // first maximum in column-major scan order (as the serial routine)
        const int m = n - k;
        double best = -1.0;
        int bkey = 0x7fffffff;
        for (int e = T; e < m * m; e += NT) {
            const int i = k + e % m, j = k + e / m;
            const double v = fabs(a[i + (size_t)lda * j]);
            if (v > best) {
                best = v;
                bkey = e;
            }
        }
        team_argmax_first(team, best, bkey, scratch);
        const int bi = k + bkey % m, bj = k + bkey / m;
        if (T == 0) {
            rowp[k] = bi;
            colp[k] = bj;
        }
        if (bi != k)
            for (int j = T; j < n; j += NT) {
                const double t = a[k + (size_t)lda * j];
                a[k + (size_t)lda * j] = a[bi + (size_t)lda * j];
                a[bi + (size_t)lda * j] = t;
            }
        team.sync();
        if (bj != k)
            for (int i = T; i < n; i += NT) {
                const double t = a[i + (size_t)lda * k];
                a[i + (size_t)lda * k] = a[i + (size_t)lda * bj];
                a[i + (size_t)lda * bj] = t;
            }
        team.sync();
        const double p = a[k + (size_t)lda * k];
        if (T == 0) piv_abs[k] = fabs(p);
        if (fabs(p) > maxpiv) maxpiv = fabs(p);
        if (p != 0.0) {
            for (int i = k + 1 + T; i < n; i += NT) a[i + (size_t)lda * k] /= p;
            team.sync();
            const int mm = n - k - 1;
            for (int e = T; e < mm * mm; e += NT) {
                const int i = k + 1 + e % mm, j = k + 1 + e / mm;
                a[i + (size_t)lda * j] -= a[i + (size_t)lda * k] * a[k + (size_t)lda * j];
            }
        }
        team.sync();
    }
    const double thr = 2.220446049250313e-16 * (double)n * maxpiv;
    int rank = 0;
    for (int k = 0; k < n; ++k)
        if (piv_abs[k] > thr) ++rank;
    if (rank < n) return false;
    for (int c = T; c < n; c += NT) {
        double* x = inv + (size_t)ldi * c;
        for (int i = 0; i < n; ++i) x[i] = (i == c) ? 1.0 : 0.0;
        for (int k = 0; k < n; ++k)
            if (rowp[k] != k) {
                const double t = x[k];
                x[k] = x[rowp[k]];
                x[rowp[k]] = t;
            }
        for (int i = 0; i < n; ++i)
            for (int p = 0; p < i; ++p) x[i] -= a[i + (size_t)lda * p] * x[p];
        for (int i = n - 1; i >= 0; --i) {
            for (int p = i + 1; p < n; ++p) x[i] -= a[i + (size_t)lda * p] * x[p];
            x[i] /= a[i + (size_t)lda * i];
        }
        for (int k = n - 1; k >= 0; --k)
            if (colp[k] != k) {
                const double t = x[k];
                x[k] = x[colp[k]];
                x[colp[k]] = t;
            }
    }
    team.sync();
    return true;
}

template <class Team>
OCTEN_HD bool eig_real_team(const Team& team, int nn, double* hm, double* vm, double* wr, double* wi, double* ort) {
#define H_(i, j) hm[(i) + (size_t)nn * (j)]
#define V_(i, j) vm[(i) + (size_t)nn * (j)]
    const int T = team.tid(), NT = team.size();
    const bool lead = (T == 0);
    const int low = 0, high = nn - 1;
    // --- orthes ---
    for (int m = low + 1; m <= high - 1; ++m) {
        double scale = 0.0;
        for (int i = m; i <= high; ++i) scale += fabs(H_(i, m - 1));
        if (scale != 0.0) {
            double h = 0.0;
            for (int i = high; i >= m; --i) {
                const double o = H_(i, m - 1) / scale;
                h += o * o;
            }
            double g = sqrt(h);
            const double om = H_(m, m - 1) / scale;
            if (om > 0) g = -g;
            h = h - om * g;
            for (int i = m + T; i <= high; i += NT) ort[i] = (i == m) ? om - g : H_(i, m - 1) / scale;
            team.sync();
            for (int j = m + T; j < nn; j += NT) {
                double f = 0.0;
                for (int i = high; i >= m; --i) f += ort[i] * H_(i, j);
                f = f / h;
                for (int i = m; i <= high; ++i) H_(i, j) -= f * ort[i];
            }
            team.sync();
            for (int i = T; i <= high; i += NT) {
                double f = 0.0;
                for (int j = high; j >= m; --j) f += ort[j] * H_(i, j);
                f = f / h;
                for (int j = m; j <= high; ++j) H_(i, j) -= f * ort[j];
            }
            team.sync();
            if (lead) {
                ort[m] = scale * ort[m];
                H_(m, m - 1) = scale * g;
            }
            team.sync();
        }
    }
    for (int e = T; e < nn * nn; e += NT) vm[e] = ((e % nn) == (e / nn)) ? 1.0 : 0.0;
    team.sync();
    for (int m = high - 1; m >= low + 1; --m) {
        if (H_(m, m - 1) != 0.0) {
            for (int i = m + 1 + T; i <= high; i += NT) ort[i] = H_(i, m - 1);
            team.sync();
            for (int j = m + T; j <= high; j += NT) {
                double g = 0.0;
                for (int i = m; i <= high; ++i) g += ort[i] * V_(i, j);
                g = (g / ort[m]) / H_(m, m - 1);
                for (int i = m; i <= high; ++i) V_(i, j) += g * ort[i];
            }
            team.sync();
        }
    }
    // --- hqr2 ---
    int n = nn - 1;
    const double eps = 2.220446049250313e-16;
    double exshift = 0.0, p = 0, q = 0, r = 0, s = 0, z = 0, t, w, x, y;
    double norm = 0.0;
    for (int i = 0; i < nn; ++i)
        for (int j = (i - 1 > 0 ? i - 1 : 0); j < nn; ++j) norm += fabs(H_(i, j));
    int iter = 0, total_iter = 0;
    const int max_total = 40 * nn;
    while (n >= low) {
        int l = n;
        while (l > low) {
            s = fabs(H_(l - 1, l - 1)) + fabs(H_(l, l));
            if (s == 0.0) s = norm;
            if (fabs(H_(l, l - 1)) < eps * s) break;
            l--;
        }
        if (l == n) {
            const double hv = H_(n, n) + exshift;
            team.sync();
            if (lead) {
                H_(n, n) = hv;
                wr[n] = hv;
                wi[n] = 0.0;
            }
            team.sync();
            n--;
            iter = 0;
        } else if (l == n - 1) {
            w = H_(n, n - 1) * H_(n - 1, n);
            p = (H_(n - 1, n - 1) - H_(n, n)) / 2.0;
            q = p * p + w;
            z = sqrt(fabs(q));
            const double hnn = H_(n, n) + exshift, hmm = H_(n - 1, n - 1) + exshift;
            const double hsub = H_(n, n - 1);
            x = hnn;
            team.sync();
            if (lead) {
                H_(n, n) = hnn;
                H_(n - 1, n - 1) = hmm;
            }
            if (q >= 0) {
                z = (p >= 0) ? p + z : p - z;
                const double wa = x + z;
                const double wb = (z != 0.0) ? x - w / z : wa;
                if (lead) {
                    wr[n - 1] = wa;
                    wr[n] = wb;
                    wi[n - 1] = 0.0;
                    wi[n] = 0.0;
                }
                x = hsub;
                s = fabs(x) + fabs(z);
                p = x / s;
                q = z / s;
                r = sqrt(p * p + q * q);
                p = p / r;
                q = q / r;
                team.sync();
                for (int j = n - 1 + T; j < nn; j += NT) {
                    const double zz = H_(n - 1, j);
                    H_(n - 1, j) = q * zz + p * H_(n, j);
                    H_(n, j) = q * H_(n, j) - p * zz;
                }
                team.sync();
                for (int i = T; i <= n; i += NT) {
                    const double zz = H_(i, n - 1);
                    H_(i, n - 1) = q * zz + p * H_(i, n);
                    H_(i, n) = q * H_(i, n) - p * zz;
                }
                for (int i = low + T; i <= high; i += NT) {
                    const double zz = V_(i, n - 1);
                    V_(i, n - 1) = q * zz + p * V_(i, n);
                    V_(i, n) = q * V_(i, n) - p * zz;
                }
            } else {
                if (lead) {
                    wr[n - 1] = x + p;
                    wr[n] = x + p;
                    wi[n - 1] = z;
                    wi[n] = -z;
                }
            }
            team.sync();
            n = n - 2;
            iter = 0;
        } else {
            x = H_(n, n);
            y = 0.0;
            w = 0.0;
            if (l < n) {
                y = H_(n - 1, n - 1);
                w = H_(n, n - 1) * H_(n - 1, n);
            }
            if (iter == 10) {
                exshift += x;
                team.sync();
                for (int i = low + T; i <= n; i += NT) H_(i, i) -= x;
                team.sync();
                s = fabs(H_(n, n - 1)) + fabs(H_(n - 1, n - 2));
                x = y = 0.75 * s;
                w = -0.4375 * s * s;
            }
            if (iter == 30) {
                s = (y - x) / 2.0;
                s = s * s + w;
                if (s > 0) {
                    s = sqrt(s);
                    if (y < x) s = -s;
                    s = x - w / ((y - x) / 2.0 + s);
                    team.sync();
                    for (int i = low + T; i <= n; i += NT) H_(i, i) -= s;
                    team.sync();
                    exshift += s;
                    x = y = w = 0.964;
                }
            }
            iter = iter + 1;
            if (++total_iter > max_total) return false;
            int m = n - 2;
            while (m >= l) {
                z = H_(m, m);
                r = x - z;
                s = y - z;
                p = (r * s - w) / H_(m + 1, m) + H_(m, m + 1);
                q = H_(m + 1, m + 1) - z - r - s;
                r = H_(m + 2, m + 1);
                s = fabs(p) + fabs(q) + fabs(r);
                {
                    const double is = 1.0 / s;  // one division, three products
                    p = p * is;
                    q = q * is;
                    r = r * is;
                }
                if (m == l) break;
                if (fabs(H_(m, m - 1)) * (fabs(q) + fabs(r)) <
                    eps * (fabs(p) * (fabs(H_(m - 1, m - 1)) + fabs(z) + fabs(H_(m + 1, m + 1)))))
                    break;
                m--;
            }
            team.sync();
            for (int i = m + 2 + T; i <= n; i += NT) {
                H_(i, i - 2) = 0.0;
                if (i > m + 2) H_(i, i - 3) = 0.0;
            }
            team.sync();
            for (int k = m; k <= n - 1; ++k) {
                const bool notlast = (k != n - 1);
                if (k != m) {
                    p = H_(k, k - 1);
                    q = H_(k + 1, k - 1);
                    r = notlast ? H_(k + 2, k - 1) : 0.0;
                    x = fabs(p) + fabs(q) + fabs(r);
                    if (x == 0.0) continue;
                    const double ix = 1.0 / x;
                    p = p * ix;
                    q = q * ix;
                    r = r * ix;
                }
                s = sqrt(p * p + q * q + r * r);
                if (p < 0) s = -s;
                if (s != 0) {
                    double hk = 0.0;
                    bool store = false;
                    if (k != m) {
                        hk = -s * x;
                        store = true;
                    } else if (l != m) {
                        hk = -H_(k, k - 1);
                        store = true;
                    }
                    team.sync();
                    if (lead && store) H_(k, k - 1) = hk;
                    p = p + s;
                    const double is = 1.0 / s, ip = 1.0 / p;
                    x = p * is;
                    y = q * is;
                    z = r * is;
                    q = q * ip;
                    r = r * ip;
                    for (int j = k + T; j < nn; j += NT) {
                        double pp = H_(k, j) + q * H_(k + 1, j);
                        if (notlast) {
                            pp = pp + r * H_(k + 2, j);
                            H_(k + 2, j) = H_(k + 2, j) - pp * z;
                        }
                        H_(k, j) = H_(k, j) - pp * x;
                        H_(k + 1, j) = H_(k + 1, j) - pp * y;
                    }
                    team.sync();
                    const int imax = (n < k + 3) ? n : k + 3;
                    for (int i = T; i <= imax; i += NT) {
                        double pp = x * H_(i, k) + y * H_(i, k + 1);
                        if (notlast) {
                            pp = pp + z * H_(i, k + 2);
                            H_(i, k + 2) = H_(i, k + 2) - pp * r;
                        }
                        H_(i, k) = H_(i, k) - pp;
                        H_(i, k + 1) = H_(i, k + 1) - pp * q;
                    }
                    for (int i = low + T; i <= high; i += NT) {
                        double pp = x * V_(i, k) + y * V_(i, k + 1);
                        if (notlast) {
                            pp = pp + z * V_(i, k + 2);
                            V_(i, k + 2) = V_(i, k + 2) - pp * r;
                        }
                        V_(i, k) = V_(i, k) - pp;
                        V_(i, k + 1) = V_(i, k + 1) - pp * q;
                    }
                    team.sync();
                }
            }
        }
    }
    // back-substitution (O(n^2) per vector, redundant in every thread; the
    // stores are thread 0's)
    if (norm == 0.0) return true;
    for (n = nn - 1; n >= 0; n--) {
        p = wr[n];
        q = wi[n];
        if (q == 0) {
            int l = n;
            team.sync();
            if (lead) H_(n, n) = 1.0;
            team.sync();
            for (int i = n - 1; i >= 0; i--) {
                w = H_(i, i) - p;
                r = 0.0;
                for (int j = l; j <= n; j++) r = r + H_(i, j) * H_(j, n);
                if (wi[i] < 0.0) {
                    z = w;
                    s = r;
                } else {
                    l = i;
                    double a0, a1 = 0.0;
                    bool two = false;
                    if (wi[i] == 0.0) {
                        a0 = (w != 0.0) ? -r / w : -r / (eps * norm);
                    } else {
                        x = H_(i, i + 1);
                        y = H_(i + 1, i);
                        q = (wr[i] - p) * (wr[i] - p) + wi[i] * wi[i];
                        t = (x * s - z * r) / q;
                        a0 = t;
                        a1 = (fabs(x) > fabs(z)) ? (-r - w * t) / x : (-s - y * t) / z;
                        two = true;
                    }
                    team.sync();
                    if (lead) {
                        H_(i, n) = a0;
                        if (two) H_(i + 1, n) = a1;
                    }
                    team.sync();
                    t = fabs(a0);
                    if ((eps * t) * t > 1) {
                        for (int j = i + T; j <= n; j += NT) H_(j, n) = H_(j, n) / t;
                        team.sync();
                    }
                }
            }
        } else if (q < 0) {
            int l = n - 1;
            double cr, ci;
            double h00, h01;
            if (fabs(H_(n, n - 1)) > fabs(H_(n - 1, n))) {
                h00 = q / H_(n, n - 1);
                h01 = -(H_(n, n) - p) / H_(n, n - 1);
            } else {
                detail::cdiv(0.0, -H_(n - 1, n), H_(n - 1, n - 1) - p, q, cr, ci);
                h00 = cr;
                h01 = ci;
            }
            team.sync();
            if (lead) {
                H_(n - 1, n - 1) = h00;
                H_(n - 1, n) = h01;
                H_(n, n - 1) = 0.0;
                H_(n, n) = 1.0;
            }
            team.sync();
            for (int i = n - 2; i >= 0; i--) {
                double ra = 0.0, sa = 0.0, vr, vi;
                for (int j = l; j <= n; j++) {
                    ra = ra + H_(i, j) * H_(j, n - 1);
                    sa = sa + H_(i, j) * H_(j, n);
                }
                w = H_(i, i) - p;
                if (wi[i] < 0.0) {
                    z = w;
                    r = ra;
                    s = sa;
                } else {
                    l = i;
                    double b0, b1, b2 = 0.0, b3 = 0.0;
                    bool two = false;
                    if (wi[i] == 0) {
                        detail::cdiv(-ra, -sa, w, q, cr, ci);
                        b0 = cr;
                        b1 = ci;
                    } else {
                        x = H_(i, i + 1);
                        y = H_(i + 1, i);
                        vr = (wr[i] - p) * (wr[i] - p) + wi[i] * wi[i] - q * q;
                        vi = (wr[i] - p) * 2.0 * q;
                        if (vr == 0.0 && vi == 0.0)
                            vr = eps * norm * (fabs(w) + fabs(q) + fabs(x) + fabs(y) + fabs(z));
                        detail::cdiv(x * r - z * ra + q * sa, x * s - z * sa - q * ra, vr, vi, cr, ci);
                        b0 = cr;
                        b1 = ci;
                        if (fabs(x) > (fabs(z) + fabs(q))) {
                            b2 = (-ra - w * b0 + q * b1) / x;
                            b3 = (-sa - w * b1 - q * b0) / x;
                        } else {
                            detail::cdiv(-r - y * b0, -s - y * b1, z, q, cr, ci);
                            b2 = cr;
                            b3 = ci;
                        }
                        two = true;
                    }
                    team.sync();
                    if (lead) {
                        H_(i, n - 1) = b0;
                        H_(i, n) = b1;
                        if (two) {
                            H_(i + 1, n - 1) = b2;
                            H_(i + 1, n) = b3;
                        }
                    }
                    team.sync();
                    t = fmax(fabs(b0), fabs(b1));
                    if ((eps * t) * t > 1) {
                        for (int j = i + T; j <= n; j += NT) {
                            H_(j, n - 1) = H_(j, n - 1) / t;
                            H_(j, n) = H_(j, n) / t;
                        }
                        team.sync();
                    }
                }
            }
        }
    }
    team.sync();
    // back-transformation: each thread owns whole rows of V
    for (int i = low + T; i <= high; i += NT)
        for (int j = nn - 1; j >= low; j--) {
            double zz = 0.0;
            const int kmax = j < high ? j : high;
            for (int k = low; k <= kmax; k++) zz = zz + V_(i, k) * H_(k, j);
            V_(i, j) = zz;
        }
    team.sync();
    return true;
#undef H_
#undef V_
}

// ---------------------------------------------------------------------------
// Team-parallel cyclic Jacobi eigen-decomposition of a symmetric n x n matrix
// held column-major (ld n) in `a` (shared memory on the device).  Rotations
// of one round-robin round act on disjoint index pairs, so every 2x2 block of
// A' = G^T A G and every row pair of V' = V G updates independently.  On
// return the diagonal of `a` holds the eigenvalues and the columns of `v`
// (ld n) the eigenvectors.  Scratch (shared): cs = 2*(n+2) doubles,
// iw = n + 4 ints (iw[0] is the sweep flag, iw[2..] the round's pair table).
// ---------------------------------------------------------------------------
template <class Team>
OCTEN_HD void jacobi_eig_sym(const Team& team, int n, double* a, double* v, double* cs, int* iw,
                             int max_sweeps = 40) {
    const int m = (n % 2) ? n + 1 : n;  // padded player count (index n is a dummy)
    const int half = m / 2;
    int* flag = iw;
    int* pp = iw + 2;         // half entries
    int* qq = iw + 2 + half;  // half entries
    for (int idx = team.tid(); idx < n * n; idx += team.size())
        v[idx] = ((idx % n) == (idx / n)) ? 1.0 : 0.0;
    team.sync();
    double* cc = cs;
    double* ss = cs + half;
    for (int sweep = 0; sweep < max_sweeps; ++sweep) {
        if (team.tid() == 0) {
            *flag = 0;
            double dm = 0.0;
            for (int i = 0; i < n; ++i) dm = fmax(dm, fabs(a[i + n * i]));
            cs[2 * half] = dm;
        }
        team.sync();
        // rotate only pairs whose coupling exceeds 1e-15 of the largest
        // diagonal (dominant-subspace accuracy; tiny eigenpairs are not refined)
        const double skip = 1e-15 * cs[2 * half];
        for (int round = 0; round < m - 1; ++round) {
            // circle method: k==0 -> (round, m-1); else ((round+k) % (m-1), (round-k+m-1) % (m-1))
            for (int k = team.tid(); k < half; k += team.size()) {
                int p, q;
                if (k == 0) {
                    p = round;
                    q = m - 1;
                } else {
                    p = (round + k) % (m - 1);
                    q = (round - k + m - 1) % (m - 1);
                }
                if (p > q) {
                    const int tt = p;
                    p = q;
                    q = tt;
                }
                double c = 1.0, s = 0.0;
                if (q < n) {
                    const double apq = a[p + n * q];
                    const double app = a[p + n * p], aqq = a[q + n * q];
                    if (fabs(apq) > 1e-300 && fabs(apq) > skip && fabs(apq) > 1e-15 * sqrt(fabs(app) * fabs(aqq))) {
                        const double theta = (aqq - app) / (2.0 * apq);
                        double t = 1.0 / (fabs(theta) + sqrt(theta * theta + 1.0));
                        if (theta < 0.0) t = -t;
                        c = 1.0 / sqrt(t * t + 1.0);
                        s = t * c;
                        *flag = 1;
                    }
                }
                cc[k] = c;
                ss[k] = s;
                pp[k] = p;
                qq[k] = q;
            }
            team.sync();
            // A' = G^T A G on 2x2 blocks (pair k1 rows, pair k2 cols)
            for (int blk = team.tid(); blk < half * half; blk += team.size()) {
                const int k1 = blk % half, k2 = blk / half;
                const int p1 = pp[k1], q1 = qq[k1], p2 = pp[k2], q2 = qq[k2];
                const double c1 = cc[k1], s1 = ss[k1], c2 = cc[k2], s2 = ss[k2];
                if (q1 < n && q2 < n) {
                    const double b00 = a[p1 + n * p2], b01 = a[p1 + n * q2];
                    const double b10 = a[q1 + n * p2], b11 = a[q1 + n * q2];
                    // rows: r_p = c1 b_p - s1 b_q ; r_q = s1 b_p + c1 b_q
                    const double r00 = c1 * b00 - s1 * b10, r01 = c1 * b01 - s1 * b11;
                    const double r10 = s1 * b00 + c1 * b10, r11 = s1 * b01 + c1 * b11;
                    // cols: c_p = c2 r_p - s2 r_q ; c_q = s2 r_p + c2 r_q
                    double n00 = c2 * r00 - s2 * r01, n01 = s2 * r00 + c2 * r01;
                    double n10 = c2 * r10 - s2 * r11, n11 = s2 * r10 + c2 * r11;
                    if (k1 == k2 && s1 != 0.0) {
                        // diagonal block: exact annihilation, NR-style diagonal update
                        const double t = s1 / c1;
                        n00 = b00 - t * b01;
                        n11 = b11 + t * b01;
                        n01 = 0.0;
                        n10 = 0.0;
                    }
                    a[p1 + n * p2] = n00;
                    a[p1 + n * q2] = n01;
                    a[q1 + n * p2] = n10;
                    a[q1 + n * q2] = n11;
                } else if (q1 < n) {  // column pair is the dummy: rows only on real column p2
                    const double b0 = a[p1 + n * p2], b1 = a[q1 + n * p2];
                    a[p1 + n * p2] = c1 * b0 - s1 * b1;
                    a[q1 + n * p2] = s1 * b0 + c1 * b1;
                } else if (q2 < n) {  // row pair is the dummy: columns only on real row p1
                    const double b0 = a[p1 + n * p2], b1 = a[p1 + n * q2];
                    a[p1 + n * p2] = c2 * b0 - s2 * b1;
                    a[p1 + n * q2] = s2 * b0 + c2 * b1;
                }
            }
            // V' = V G : columns (p,q) of every row
            for (int e = team.tid(); e < n * half; e += team.size()) {
                const int row = e % n, k = e / n;
                const int p = pp[k], q = qq[k];
                if (q >= n) continue;
                const double c = cc[k], s = ss[k];
                const double vp = v[row + n * p], vq = v[row + n * q];
                v[row + n * p] = c * vp - s * vq;
                v[row + n * q] = s * vp + c * vq;
            }
            team.sync();
        }
        const int any = *flag;
        team.sync();
        if (!any) break;
    }
}

// ---------------------------------------------------------------------------
// Top singular triplet of an m x n matrix (column-major, ld m) by power
// iteration on A^T A: returns sigma, u (m), v (n) with A v = sigma u.  Stops
// when the right vector moves by <= 1e-14 or after max_iter.
// Replaces the rank-1 JacobiSVD peel (cp_als.cpp:24-36).  Team-parallel;
// scratch `red` (shared): team.size() + 2 + n doubles.
// ---------------------------------------------------------------------------
template <class Team>
OCTEN_HD double team_reduce_sum(const Team& team, double v, double* red) {
#if defined(__CUDA_ARCH__)
    // device: warp shuffle tree, then warp partials summed in warp order
    // (fixed order, deterministic); requires blockDim.x % 32 == 0
    if (team.size() > 1) {
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        const int nw = team.size() >> 5;
        if ((team.tid() & 31) == 0) red[team.tid() >> 5] = v;
        team.sync();
        double s = 0.0;
        for (int i = 0; i < nw; ++i) s += red[i];
        team.sync();
        return s;
    }
#endif
    // deterministic: every thread writes, thread 0 sums in index order
    red[team.tid()] = v;
    team.sync();
    if (team.tid() == 0) {
        double s = 0.0;
        for (int i = 0; i < team.size(); ++i) s += red[i];
        red[team.size()] = s;
    }
    team.sync();
    const double out = red[team.size()];
    team.sync();
    return out;
}

template <class Team>
OCTEN_HD double top_singular_pair(const Team& team, int m, int n, const double* a, double* u, double* v,
                                  double* red, int max_iter = 500) {
    // start: the row of A with the largest norm (transposed); first row
    // wins ties.  Row norms in parallel, then a (max, lowest index) reduction.
    {
        double bn = -1.0;
        int best = 0x7fffffff;
        for (int i = team.tid(); i < m; i += team.size()) {
            double s = 0.0;
            for (int j = 0; j < n; ++j) s += dsq(a[i + (size_t)m * j]);
            if (s > bn) {
                bn = s;
                best = i;
            }
        }
#if defined(__CUDA_ARCH__)
        if (team.size() > 1) {
            for (int o = 16; o > 0; o >>= 1) {
                const double ov = __shfl_xor_sync(0xffffffffu, bn, o);
                const int ob = __shfl_xor_sync(0xffffffffu, best, o);
                if (ov > bn || (ov == bn && ob < best)) {
                    bn = ov;
                    best = ob;
                }
            }
            const int nw = team.size() >> 5, w = team.tid() >> 5;
            if ((team.tid() & 31) == 0) {
                red[2 * w] = bn;
                red[2 * w + 1] = (double)best;
            }
            team.sync();
            if (team.tid() == 0) {
                double b = red[0];
                int bi = (int)red[1];
                for (int q = 1; q < nw; ++q)
                    if (red[2 * q] > b || (red[2 * q] == b && (int)red[2 * q + 1] < bi)) {
                        b = red[2 * q];
                        bi = (int)red[2 * q + 1];
                    }
                red[team.size() + 1] = (double)bi;
            }
        } else
#endif
        {
            if (team.tid() == 0) red[team.size() + 1] = (double)best;
        }
    }
    team.sync();
    const int row = (int)red[team.size() + 1];
    team.sync();
    double loc = 0.0;
    for (int j = team.tid(); j < n; j += team.size()) {
        v[j] = a[row + (size_t)m * j];
        loc += v[j] * v[j];
    }
    double vn = sqrt(team_reduce_sum(team, loc, red));
    if (vn == 0.0) {
        for (int i = team.tid(); i < m; i += team.size()) u[i] = 0.0;
        team.sync();
        return 0.0;
    }
    for (int j = team.tid(); j < n; j += team.size()) v[j] /= vn;
    team.sync();
    double sigma = 0.0;
    for (int it = 0; it < max_iter; ++it) {
        // u = A v / |A v|
        loc = 0.0;
        for (int i = team.tid(); i < m; i += team.size()) {
            double s = 0.0;
            for (int j = 0; j < n; ++j) s += a[i + (size_t)m * j] * v[j];
            u[i] = s;
            loc += s * s;
        }
        sigma = sqrt(team_reduce_sum(team, loc, red));
        if (sigma == 0.0) break;
        for (int i = team.tid(); i < m; i += team.size()) u[i] /= sigma;
        team.sync();
        // w = A^T u ; v_new = w / |w| ; diff = |v_new - v|
        double l2 = 0.0;
        for (int j = team.tid(); j < n; j += team.size()) {
            double s = 0.0;
            for (int i = 0; i < m; ++i) s += a[i + (size_t)m * j] * u[i];
            red[team.size() + 2 + j] = s;  // staged in the tail of red (size >= size+2+n)
            l2 += s * s;
        }
        const double wn = sqrt(team_reduce_sum(team, l2, red));
        loc = 0.0;
        for (int j = team.tid(); j < n; j += team.size()) {
            const double nv = red[team.size() + 2 + j] / wn;
            loc += dsq(nv - v[j]);
            v[j] = nv;
        }
        const double diff = sqrt(team_reduce_sum(team, loc, red));
        if (diff <= 1e-14) {
            sigma = wn;  // |A^T u| = sigma at convergence
            break;
        }
        sigma = wn;
    }
    // final consistent pair: u = A v / sigma
    loc = 0.0;
    for (int i = team.tid(); i < m; i += team.size()) {
        double s = 0.0;
        for (int j = 0; j < n; ++j) s += a[i + (size_t)m * j] * v[j];
        u[i] = s;
        loc += s * s;
    }
    sigma = sqrt(team_reduce_sum(team, loc, red));
    if (sigma > 0.0)
        for (int i = team.tid(); i < m; i += team.size()) u[i] /= sigma;
    team.sync();
    return sigma;
}

// ---------------------------------------------------------------------------
// Top-k eigenpairs of a symmetric positive semidefinite n x n matrix `a`
// (column-major, ld n, read only) by block subspace (orthogonal) iteration:
// a block of m >= k columns, each product W = A U re-orthonormalised by
// classical Gram-Schmidt run twice (CGS2), with a Rayleigh-Ritz projection
// H = U^T A U whose Ritz values give the convergence rate
// rho = theta_{m-1} / theta_{k-1}.  The iteration stops once rho^products
// <= 1e-18; it gives up (returns 0, the caller falls back to the full Jacobi
// solver) when that needs more than max_products, when the block collapses
// (A U has a zero column) or when theta_{k-1} <= 0.  The Gram spectrum of a
// compressed low-rank replica has a gap of ~1e-4 at k = rank, so a handful of
// products replace the O(n^3)-per-sweep Jacobi solve of the whole matrix.
// Same role as jacobi_eig_sym: the BDCSVD thin-U of the unfoldings
// (cp_als.cpp:96-100), top-k only.
// On success: u (n x m) columns 0..k-1 = eigenvectors by descending
// eigenvalue, theta[0..m) = Ritz values descending.
// Scratch: w n*m, h m*m, hv m*m, cs 2*(m+2) + team.size() + 2 doubles,
// iw 2*m + 8 ints.
// ---------------------------------------------------------------------------
template <class Team>
OCTEN_HD void team_symm_block(const Team& team, int n, const double* a, int m, const double* u,
                              double* w) {
#if defined(__CUDA_ARCH__)
    if (team.size() >= 64) {  // a whole block: FP64 tensor cores
        block_dmma_small(n, m, n, a, 1, n, u, 1, n, w, 1, n);
        team.sync();
        return;
    }
#endif
    for (int e = team.tid(); e < n * m; e += team.size()) {
        const int i = e % n, j = e / n;
        const double* uj = u + (size_t)n * j;
        double s = 0.0;
        for (int l = 0; l < n; ++l) s += a[i + (size_t)n * l] * uj[l];
        w[e] = s;
    }
    team.sync();
}

// coefficients cf[i] = <w_i, w_j>, i < j
template <class Team>
OCTEN_HD void team_cgs_coeffs(const Team& team, int n, int j, const double* w, double* cf) {
    const double* wj = w + (size_t)n * j;
#if defined(__CUDA_ARCH__)
    if (team.size() >= 64) {
        const int lane = team.tid() & 31, wid = team.tid() >> 5, nw = team.size() >> 5;
        for (int i = wid; i < j; i += nw) {
            const double* wi = w + (size_t)n * i;
            double s = 0.0;
            for (int r = lane; r < n; r += 32) s += wi[r] * wj[r];
            for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
            if (lane == 0) cf[i] = s;
        }
        team.sync();
        return;
    }
#endif
    for (int i = team.tid(); i < j; i += team.size()) {
        const double* wi = w + (size_t)n * i;
        double s = 0.0;
        for (int r = 0; r < n; ++r) s += wi[r] * wj[r];
        cf[i] = s;
    }
    team.sync();
}

// orthonormalise the m columns of w in place (CGS2); 0 if a column vanishes
template <class Team>
OCTEN_HD int team_cgs2(const Team& team, int n, int m, double* w, double* cf, double* red) {
    for (int j = 0; j < m; ++j) {
        double* wj = w + (size_t)n * j;
        if (j > 0) {
            for (int pass = 0; pass < 2; ++pass) {
                team_cgs_coeffs(team, n, j, w, cf);
                for (int r = team.tid(); r < n; r += team.size()) {
                    double s = wj[r];
                    for (int i = 0; i < j; ++i) s -= cf[i] * w[r + (size_t)n * i];
                    wj[r] = s;
                }
                team.sync();
            }
        }
        double loc = 0.0;
        for (int r = team.tid(); r < n; r += team.size()) loc += wj[r] * wj[r];
        const double nrm2 = team_reduce_sum(team, loc, red);
        if (!(nrm2 > 0.0) || !(nrm2 < 1e300)) return 0;
        const double inv = 1.0 / sqrt(nrm2);
        for (int r = team.tid(); r < n; r += team.size()) wj[r] *= inv;
        team.sync();
    }
    return 1;
}

template <class Team>
OCTEN_HD int subspace_eig_top(const Team& team, int n, const double* a, int k, int m, double* u,
                              double* w, double* h, double* hv, double* theta, double* cs, int* iw,
                              int max_products = 24) {
    double* cf = cs;                 // m (also Jacobi scratch 2*(m+2))
    double* red = cs + 2 * (m + 2);  // team.size() + 2
    int* order = iw + m + 8;         // m
    double* const u0 = u;
    // deterministic start block, entries uniform in [-1, 1)
    for (int e = team.tid(); e < n * m; e += team.size())
        u[e] = (double)(splitmix(0x5eedULL + (uint64_t)e) >> 11) * 0x1.0p-52 - 1.0;
    team.sync();
    if (!team_cgs2(team, n, m, u, cf, red)) return 0;
    // first Rayleigh-Ritz after 6 products: with a gap of ~1e-4 at k (the
    // compressed low-rank Gram) that is already converged, so one RR suffices
    int products = 0, target = 6;
    for (;;) {
        team_symm_block(team, n, a, m, u, w);  // W = A U
        ++products;
        if (products >= target) {
            // Rayleigh-Ritz: H = U^T W (symmetrised), H = Hv diag(theta) Hv^T
#if defined(__CUDA_ARCH__)
            if (team.size() >= 64) {
                block_dmma_small(m, m, n, u, n, 1, w, 1, n, hv, 1, m);  // hv: scratch here
                team.sync();
                for (int e = team.tid(); e < m * m; e += team.size()) {
                    const int i = e % m, j = e / m;
                    h[e] = 0.5 * (hv[i + (size_t)m * j] + hv[j + (size_t)m * i]);
                }
            } else
#endif
            for (int e = team.tid(); e < m * m; e += team.size()) {
                const int i = e % m, j = e / m;
                if (i > j) continue;
                double s1 = 0.0, s2 = 0.0;
                for (int r = 0; r < n; ++r) {
                    s1 += u[r + (size_t)n * i] * w[r + (size_t)n * j];
                    s2 += u[r + (size_t)n * j] * w[r + (size_t)n * i];
                }
                const double hij = 0.5 * (s1 + s2);
                h[i + (size_t)m * j] = hij;
                h[j + (size_t)m * i] = hij;
            }
            team.sync();
            // 12 sweeps: the top-k pairs converge quadratically in a few; the
            // trailing noise-level block (|h_pq| at the rounding floor) would
            // otherwise keep the cyclic sweeps going to the cap
            jacobi_eig_sym(team, m, h, hv, cs, iw, 12);
            team.sync();
            if (team.tid() == 0) {
                for (int i = 0; i < m; ++i) order[i] = i;
                for (int i = 1; i < m; ++i) {
                    const int key = order[i];
                    const double kv = h[key + (size_t)m * key];
                    int j = i - 1;
                    while (j >= 0 && h[order[j] + (size_t)m * order[j]] < kv) {
                        order[j + 1] = order[j];
                        --j;
                    }
                    order[j + 1] = key;
                }
                for (int i = 0; i < m; ++i) theta[i] = h[order[i] + (size_t)m * order[i]];
                // products needed for rho^N <= 1e-18
                const double tk = theta[k - 1], tm = fabs(theta[m - 1]);
                int need = max_products + 1;
                if (tk > 0.0 && theta[0] > 0.0) {
                    const double rho = fmax(tm / tk, 1e-300);
                    if (rho < 1.0) {
                        const double nn = ceil(log(1e-18) / log(rho));
                        need = nn < (double)(max_products + 1) ? (int)nn : max_products + 1;
                    }
                }
                iw[m + 4] = need;
            }
            team.sync();
            const int need = iw[m + 4];
            team.sync();
            if (need > max_products) return 0;
            if (products >= need) break;
            target = need;
        }
        if (!team_cgs2(team, n, m, w, cf, red)) return 0;
        double* t = u;
        u = w;
        w = t;
    }
    // Ritz vectors: column c = U hv[:, order[c]], c < k; computed into the
    // buffer not holding U, then moved to the caller's u if needed
    for (int e = team.tid(); e < n * k; e += team.size()) {
        const int r = e % n, c = e / n;
        const double* hc = hv + (size_t)m * order[c];
        double s = 0.0;
        for (int l = 0; l < m; ++l) s += u[r + (size_t)n * l] * hc[l];
        w[e] = s;
    }
    team.sync();
    if (w != u0) {
        for (int e = team.tid(); e < n * k; e += team.size()) u0[e] = w[e];
        team.sync();
    }
    return 1;
}

// ---------------------------------------------------------------------------
// Top-k eigenpairs of a symmetric n x n matrix (column-major, destroyed) by
// Householder tridiagonalisation, Sturm bisection of the k largest
// eigenvalues, inverse iteration on the tridiagonal matrix, CGS2 and the
// back-transformation -- the dense fallback of subspace_eig_top when the
// spectrum has no gap at k (e.g. summaries of unstructured sparse data),
// where the cyclic Jacobi solver took ~40x more barriers.  Same role as the
// BDCSVD thin-U of the unfoldings (cp_als.cpp:96-100): the first k columns of
// the Gram eigenbasis in descending eigenvalue order.
//   u      n x k output (eigenvectors), theta k output (descending)
//   work   3 n + 4 n kb doubles (d, e, Householder norms, inverse-iteration
//          LU and vectors for batches of kb eigenvectors), kb >= 1
//   cf, red  CGS2 / reduction scratch (k and team.size() + 2 doubles)
// Returns 0 if a vector vanishes (not expected for symmetric input).
// ---------------------------------------------------------------------------
OCTEN_HD inline int tridiag_count_below(int n, const double* d, const double* e, double x) {
    // number of eigenvalues of T strictly below x (Sturm count, LDL^T pivots)
    int cnt = 0;
    double q = d[0] - x;
    if (q < 0.0) ++cnt;
    for (int i = 1; i < n; ++i) {
        const double qq = (q == 0.0) ? 1e-300 : q;
        q = d[i] - x - e[i - 1] * e[i - 1] / qq;
        if (q < 0.0) ++cnt;
    }
    return cnt;
}

template <class Team>
OCTEN_HD int sym_eig_top_tridiag(const Team& team, int n, double* a, int k, double* u, double* theta,
                                 double* work, int kb, double* cf, double* red) {
    double* d = work;
    double* e = work + n;
    double* vn = work + 2 * n;
    double* scr = work + 3 * n;  // 4 n kb
    const int tid = team.tid(), nt = team.size();
    // ---- 1. Householder tridiagonalisation (lower): A <- H A H, v stored in
    //      column kk below the subdiagonal, |v|^2 in vn[kk]
    for (int kk = 0; kk + 2 < n; ++kk) {
        double* x = a + (size_t)n * kk + kk + 1;  // length L
        const int L = n - kk - 1;
        double loc = 0.0;
        for (int i = tid; i < L; i += nt) loc += x[i] * x[i];
        const double xn2 = team_reduce_sum(team, loc, red);
        const double alpha = x[0];
        const double tail = xn2 - alpha * alpha;
        if (!(tail > 1e-300 * (xn2 + 1e-300))) {  // already reduced
            team.sync();
            if (tid == 0) {
                e[kk] = alpha;
                vn[kk] = 0.0;
            }
            team.sync();
            continue;
        }
        const double beta = alpha > 0.0 ? -sqrt(xn2) : sqrt(xn2);
        const double v0 = alpha - beta;
        const double vv = tail + v0 * v0, c = 2.0 / vv;
        double* B = a + (size_t)n * (kk + 1) + kk + 1;  // L x L, ld n
        double* p = scr;                                 // L
        // p = c B v  (v = x with v[0] = v0)
        for (int i = tid; i < L; i += nt) {
            double sacc = B[i] * v0;
            for (int j = 1; j < L; ++j) sacc += B[i + (size_t)n * j] * x[j];
            p[i] = c * sacc;
        }
        team.sync();
        double loc2 = 0.0;
        for (int i = tid; i < L; i += nt) loc2 += (i == 0 ? v0 : x[i]) * p[i];
        const double vp = team_reduce_sum(team, loc2, red);
        const double K = 0.5 * c * vp;
        // B -= v w^T + w v^T,  w = p - K v
        for (int idx = tid; idx < L * L; idx += nt) {
            const int i = idx % L, j = idx / L;
            const double vi = i == 0 ? v0 : x[i], vj = j == 0 ? v0 : x[j];
            const double wi = p[i] - K * vi, wj = p[j] - K * vj;
            B[i + (size_t)n * j] -= vi * wj + wi * vj;
        }
        team.sync();
        if (tid == 0) {
            e[kk] = beta;
            vn[kk] = vv;
            x[0] = v0;  // column kk below the diagonal now holds v
        }
        team.sync();
    }
    if (tid == 0) {
        for (int i = 0; i < n; ++i) d[i] = a[i + (size_t)n * i];
        if (n >= 2) {
            e[n - 2] = a[(n - 1) + (size_t)n * (n - 2)];
            vn[n - 2] = 0.0;
        }
        vn[n - 1] = 0.0;
    }
    team.sync();
    // ---- 2. the k largest eigenvalues by bisection, one per thread
    double gl = 0.0, gu = 0.0, tnorm = 0.0;
    for (int i = 0; i < n; ++i) {
        const double r = (i > 0 ? fabs(e[i - 1]) : 0.0) + (i + 1 < n ? fabs(e[i]) : 0.0);
        const double lo = d[i] - r, hi = d[i] + r;
        if (i == 0 || lo < gl) gl = lo;
        if (i == 0 || hi > gu) gu = hi;
    }
    tnorm = fmax(fabs(gl), fabs(gu));
    for (int r = tid; r < k; r += nt) {
        const int m = n - 1 - r;  // ascending index of the (r+1)-th largest
        double lo = gl - 1e-300 - 2.2e-16 * tnorm, hi = gu + 2.2e-16 * tnorm + 1e-300;
        for (int it = 0; it < 200; ++it) {
            const double mid = 0.5 * (lo + hi);
            if (hi - lo <= 4.4e-16 * fmax(fabs(lo), fabs(hi)) + 1e-300 || mid == lo || mid == hi) break;
            if (tridiag_count_below(n, d, e, mid) > m)
                hi = mid;
            else
                lo = mid;
        }
        theta[r] = 0.5 * (lo + hi);
    }
    team.sync();
    // ---- 3. eigenvectors of T by inverse iteration: Gaussian elimination with
    //      partial pivoting of T - theta I (U has two superdiagonals), three
    //      solves from a fixed pseudo-random start; one thread per vector,
    //      kb vectors at a time (5 n doubles of scratch each)
    for (int r0 = 0; r0 < k; r0 += kb) {
        const int nb = (k - r0) < kb ? (k - r0) : kb;
        for (int rr = tid; rr < nb; rr += nt) {
            const int r = r0 + rr;
            double* ml = scr + (size_t)5 * n * rr;  // multipliers
            double* u0 = ml + n;                     // U diagonal
            double* u1 = u0 + n;                     // U superdiagonal
            double* u2 = u1 + n;                     // U second superdiagonal (pivoting fill)
            double* sw = u2 + n;                     // 1.0 where rows i, i+1 were swapped
            double* y = u + (size_t)n * r;
            const double tiny = 2.2e-16 * tnorm + 1e-300;
            const double sh = theta[r];
            double ci = d[0] - sh, bi = n > 1 ? e[0] : 0.0;
            for (int i = 0; i + 1 < n; ++i) {
                const double sub = e[i], cn = d[i + 1] - sh, bn = (i + 2 < n) ? e[i + 1] : 0.0;
                if (fabs(ci) >= fabs(sub)) {
                    const double piv = (ci == 0.0) ? tiny : ci;
                    const double mlt = sub / piv;
                    u0[i] = piv;
                    u1[i] = bi;
                    u2[i] = 0.0;
                    ml[i] = mlt;
                    sw[i] = 0.0;
                    ci = cn - mlt * bi;
                    bi = bn;
                } else {
                    const double mlt = ci / sub;
                    u0[i] = sub;
                    u1[i] = cn;
                    u2[i] = bn;
                    ml[i] = mlt;
                    sw[i] = 1.0;
                    ci = bi - mlt * cn;
                    bi = -mlt * bn;
                }
            }
            u0[n - 1] = (fabs(ci) < tiny) ? (ci < 0.0 ? -tiny : tiny) : ci;
            for (int i = 0; i < n; ++i)
                if (fabs(u0[i]) < tiny) u0[i] = u0[i] < 0.0 ? -tiny : tiny;
            for (int i = 0; i < n; ++i)
                y[i] = (double)(splitmix(0x7e1dULL + (uint64_t)i * 131 + (uint64_t)r) >> 11) * 0x1.0p-53 + 0.25;
            for (int it = 0; it < 3; ++it) {
                for (int i = 0; i + 1 < n; ++i) {  // b <- L^-1 P b
                    if (sw[i] != 0.0) {
                        const double t0 = y[i];
                        y[i] = y[i + 1];
                        y[i + 1] = t0;
                    }
                    y[i + 1] -= ml[i] * y[i];
                }
                double nrm = 0.0;
                for (int i = n - 1; i >= 0; --i) {  // U y = b
                    double v = y[i];
                    if (i + 1 < n) v -= u1[i] * y[i + 1];
                    if (i + 2 < n) v -= u2[i] * y[i + 2];
                    v /= u0[i];
                    y[i] = v;
                    nrm = fmax(nrm, fabs(v));
                }
                const double inv = nrm > 0.0 ? 1.0 / nrm : 1.0;
                for (int i = 0; i < n; ++i) y[i] *= inv;
            }
        }
        team.sync();
    }
    // ---- 4. orthonormalise (clusters of close eigenvalues), descending order
    if (!team_cgs2(team, n, k, u, cf, red)) return 0;
    // ---- 5. back-transformation u <- H_0 ... H_{n-3} u (one thread per vector)
    for (int r = tid; r < k; r += nt) {
        double* y = u + (size_t)n * r;
        for (int kk = n - 3; kk >= 0; --kk) {
            if (!(vn[kk] > 0.0)) continue;
            const double* v = a + (size_t)n * kk + kk + 1;
            const int L = n - kk - 1;
            double sacc = 0.0;
            for (int i = 0; i < L; ++i) sacc += v[i] * y[kk + 1 + i];
            sacc *= 2.0 / vn[kk];
            for (int i = 0; i < L; ++i) y[kk + 1 + i] -= sacc * v[i];
        }
    }
    team.sync();
    return 1;
}

}  // namespace octen
