// Stage 2: batched CP-ALS over every (replica, restart) problem.
//
// Restates cp_als (reference proj/src/cp_als.cpp:240-359) with
//   * the GEVD warm start (cp_als.cpp:46-190): thin-U of the mode-0/1
//     unfoldings from the Gram eigenbasis (Jacobi), slice mixtures w ~ U(-1,1)
//     from derive(restart_seed,{11,attempt}) (host RNG, bit-exact), R x R
//     pencil eigen-decomposition (orthes+hqr2), COD solve, rank-1 peel;
//   * cyclic mode updates with the Hadamard-of-Grams solve, per-update
//     normalization into lambda and the seeded column rescue (device
//     mt19937_64, cp_als.cpp:293,309-319);
//   * fit from the cached last-mode MTTKRP and the |dfit| < rel_tol stop
//     (cp_als.cpp:325-345); best of n_restarts with first-wins ties.
// MTTKRPs use a dimension tree: T = Y x3 C is shared by the mode-0 and mode-1
// updates (C does not change between them), mode 2 contracts Y_(2) with the
// Khatri-Rao product of the new A, B.  All restarts of a replica share every
// read of Y_p.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <stdexcept>

#include "engine.hpp"
#include "evprof.hpp"
#include "gemm_dmma.cuh"
#include "h2d_param.cuh"
#include "ozaki.hpp"
#include "ozaki_digits.cuh"
#include "rng_host.hpp"
#include "small_linalg.cuh"

namespace octen {

namespace {

constexpr double kDegenerateNorm = 1e-14;  // cp_als.cpp:17
constexpr double kEps = 2.220446049250313e-16;
constexpr int kAlsMaxLanes = 8;  // AlsEngine::kMaxLanes

struct AlsDev {
    int P, S, Q, R, NP, max_iters;
    double rel_tol;
    const double* Y;
    double* normx2;
    double* F;
    double* G;
    double* lam;
    double* T;
    double* KR;
    double* Mb;
    double* Vinv;  // per problem R x R: inverse (or pseudo-inverse) of the mode's Hadamard Gram
    int* mcount;   // per problem: finished blocks of the current fused MTTKRP + update launch
    double* fit_hist;
    double* res_hist;
    AlsState* state;
    DevStatus* err;
    Mt64* rngs;
    const std::uint64_t* rescue_seed;
    int* hact;  // host-mapped [sweep][kMaxLanes] "a problem of this lane is still active" flags
    // GEVD
    double* Gev;
    double* EV;
    double* Ur;
    double* Wmix;
    double* Smix;
    double* Tmp6;
    double* Pm;
    double* Hh;
    int* eigdbg;  // [0] subspace fallbacks to Jacobi (diagnostics)
    long long* tsc;  // per-phase clock64 stamps of the update kernel (diagnostics; null normally)
    double* gscr;
    int* usable;
    int* att_start;
    int* att_used;
    int* todo;
    int* peel_fail;
    // digits of every factor for the int8 tensor-core T-GEMM (ozaki_digits.cuh
    // layout; null: the DMMA T-GEMM, no digits written)
    std::uint8_t* Fd;
    double* Fcs;
    int oz_G;
    __device__ size_t q3() const { return (size_t)Q * Q * Q; }
    __device__ size_t q2() const { return (size_t)Q * Q; }
    __device__ double* f(int prob, int n) const { return F + ((size_t)prob * 3 + n) * Q * R; }
    __device__ double* g(int prob, int n) const { return G + ((size_t)prob * 3 + n) * R * R; }
};

__device__ double block_sum(double v, double* red) {
    // deterministic block reduction (fixed tree): butterfly within each warp,
    // then the warp sums in warp order; two barriers (blockDim a multiple of 32)
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) red[warp] = v;
    __syncthreads();
    if (warp == 0) {
        double w = lane < nw ? red[lane] : 0.0;
        for (int o = 16; o > 0; o >>= 1) w += __shfl_xor_sync(0xffffffffu, w, o);
        if (lane == 0) red[32] = w;
    }
    __syncthreads();
    const double out = red[32];
    __syncthreads();
    return out;
}

// ||Y_p||_F^2 per replica: 64 chunk partials per replica (grid P x 64), then
// a fixed-order sum (deterministic).
__global__ void als_norm_kernel(AlsDev d, double* part) {
    __shared__ double red[256];
    const int p = blockIdx.y, c = blockIdx.x, nc = gridDim.x;
    const size_t n = d.q3(), chunk = (n + nc - 1) / nc;
    const double* y = d.Y + (size_t)p * n;
    const size_t b = chunk * c, e = min(n, b + chunk);
    double s = 0.0;
    for (size_t i = b + threadIdx.x; i < e; i += blockDim.x) s += y[i] * y[i];
    s = block_sum(s, red);
    if (threadIdx.x == 0) part[(size_t)p * nc + c] = s;
}
__global__ void als_norm_finish_kernel(AlsDev d, const double* part, int nc) {
    const int p = threadIdx.x + blockIdx.x * blockDim.x;
    if (p >= d.P) return;
    double s = 0.0;
    for (int c = 0; c < nc; ++c) s += part[(size_t)p * nc + c];
    d.normx2[p] = s;
}

// ---------------- GEVD init ----------------

// Jacobi eigen-decomposition of the two Gram matrices of replica p, top-R
// eigenvectors into Ur[p][which] (descending eigenvalue), usability flag.
__global__ void __launch_bounds__(256) gevd_eig_sym_kernel(AlsDev d, int v_in_smem, int mblk) {
    extern __shared__ double sm[];
    const int p = blockIdx.x / 2, which = blockIdx.x % 2;
    const int Q = d.Q, R = d.R;
    double* A = sm;                      // Q*Q
    double* cs = A + (size_t)Q * Q;      // 2*(Q+2) (+ reduction scratch)
    double* Vs = cs + 2 * (Q + 2) + blockDim.x / 32 + 4;  // Q*Q when v_in_smem
    int* iw = (int*)(Vs + (v_in_smem ? (size_t)Q * Q : 0));  // 2Q + 16
    int* order = iw + Q + 8;             // Q
    const double* src = d.Gev + ((size_t)p * 2 + which) * Q * Q;
    double* Vg = d.EV + ((size_t)p * 2 + which) * Q * Q;
    double* V = v_in_smem ? Vs : Vg;
    double* ur = d.Ur + ((size_t)p * 2 + which) * Q * R;
    g2s_copy(A, src, Q * Q);
    __syncthreads();
    TeamDev team;
    if (mblk > 0) {
        // top-R by subspace iteration; the V region holds U, W, H, Hv, theta
        const int m = mblk;
        double* U = V;
        double* W = U + (size_t)Q * m;
        double* H = W + (size_t)Q * m;
        double* Hv = H + (size_t)m * m;
        double* th = Hv + (size_t)m * m;
        const int ok = subspace_eig_top(team, Q, A, R, m, U, W, H, Hv, th, cs, iw);
        if (ok) {
            for (int e = threadIdx.x; e < Q * R; e += blockDim.x) ur[e] = U[e];
            // nonzero singular values: top-R Ritz values above the rounding floor
            if (threadIdx.x == 0)
                atomicAnd(&d.usable[p], (th[0] > 0.0 && th[R - 1] > kEps * Q * th[0]) ? 1 : 0);
            return;
        }
        // no usable gap at R: dense top-R solve below (A is untouched)
        if (threadIdx.x == 0) atomicAdd(&d.eigdbg[0], 1);
    }
    {
        // Householder + bisection + inverse iteration for the top R (the
        // cyclic Jacobi solver needed ~40x more barriers: 2.5 ms at Q = 64);
        // V holds [u (Q R) | theta (R) | work (3 Q + 5 Q kb)]
        const int kb = (int)(((long long)Q * Q - (long long)Q * R - R - 3LL * Q) / (5LL * Q));
        if (kb >= 1) {
            double* u = V;
            double* th = u + (size_t)Q * R;
            double* work = th + R;
            const int ok = sym_eig_top_tridiag(team, Q, A, R, u, th, work, kb, cs, cs + (Q + 2));
            if (ok) {
                for (int e = threadIdx.x; e < Q * R; e += blockDim.x) ur[e] = u[e];
                if (threadIdx.x == 0)
                    atomicAnd(&d.usable[p], (th[0] > 0.0 && th[R - 1] > kEps * Q * th[0]) ? 1 : 0);
                return;
            }
            // (not expected) a vanished vector: restore A and use Jacobi
            __syncthreads();
            g2s_copy(A, src, Q * Q);
            __syncthreads();
        }
    }
    jacobi_eig_sym(team, Q, A, V, cs, iw);
    __syncthreads();
    if (threadIdx.x == 0) {
        // order by descending eigenvalue (stable: lower index first on ties)
        for (int i = 0; i < Q; ++i) order[i] = i;
        for (int i = 1; i < Q; ++i) {
            const int key = order[i];
            const double kv = A[key + (size_t)Q * key];
            int j = i - 1;
            while (j >= 0 && A[order[j] + (size_t)Q * order[j]] < kv) {
                order[j + 1] = order[j];
                --j;
            }
            order[j + 1] = key;
        }
        const double lmax = A[order[0] + (size_t)Q * order[0]];
        // nonzero singular values: eigenvalues above the rounding floor
        int nz = 0;
        for (int i = 0; i < Q; ++i)
            if (A[order[i] + (size_t)Q * order[i]] > kEps * Q * lmax && lmax > 0.0) ++nz;
        atomicAnd(&d.usable[p], nz >= R ? 1 : 0);
    }
    __syncthreads();
    for (int e = threadIdx.x; e < Q * R; e += blockDim.x) {
        const int i = e % Q, r = e / Q;
        ur[i + (size_t)Q * r] = V[i + (size_t)Q * order[r]];
    }
}

// GEVD slice mixtures for every attempt of every restart of replica p
// (cp_als.cpp:117-121): Smix[prob][j][m] = sum_c Y[p][m + Q^2 c] w[prob][j][c],
// j = 0..5 (3 attempts x 2 mixtures).  One thread per m reads Y once per
// replica (coalesced) for all S restarts; the weights sit in shared memory.
__global__ void __launch_bounds__(256) gevd_mix_kernel(AlsDev d) {
    extern __shared__ double wmix[];  // S * 6 * Q
    const int p = blockIdx.y, Q = d.Q, S = d.S;
    const int nw = S * 6;
    for (int e = threadIdx.x; e < nw * Q; e += blockDim.x) wmix[e] = d.Wmix[(size_t)p * S * 6 * Q + e];
    __syncthreads();
    const size_t q2 = d.q2();
    const size_t m = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    if (m >= q2) return;
    const double* y = d.Y + (size_t)p * d.q3() + m;
    double acc[24];
#pragma unroll
    for (int j = 0; j < 24; ++j) acc[j] = 0.0;
    for (int c = 0; c < Q; ++c) {
        const double v = __ldg(y + q2 * c);
#pragma unroll
        for (int j = 0; j < 24; ++j)
            if (j < nw) acc[j] += v * wmix[j * Q + c];
    }
#pragma unroll
    for (int j = 0; j < 24; ++j)
        if (j < nw) {
            const int prob = p * S + j / 6, jj = j % 6;
            d.Smix[((size_t)prob * 6 + jj) * q2 + m] = acc[j];
        }
}

// Round 0 of the GEVD attempts: every problem of a usable replica starts at
// attempt 0.
__global__ void gevd_round0_kernel(AlsDev d) {
    const int prob = blockIdx.x * blockDim.x + threadIdx.x;
    if (prob >= d.NP) return;
    d.att_start[prob] = 0;
    d.todo[prob] = d.usable[prob / d.S] ? 1 : 0;
}

// Per problem: pick the first GEVD attempt whose pencil is invertible, has a
// real Schur form and gives non-degenerate a1 columns (cp_als.cpp:110-150).
__global__ void gevd_pencil_kernel(AlsDev d) {
    const int prob = blockIdx.x;
    if (!d.todo[prob]) return;
    const int p = prob / d.S;
    const int Q = d.Q, R = d.R;
    extern __shared__ double sm[];
    double* asub = sm;                  // R*R
    double* nrm = asub + R * R;         // R
    __shared__ int ok, att;
    double* scr = nrm + R;  // shared: 4R^2 + 4R doubles
    double* m_inv = scr;
    double* m_pen = m_inv + R * R;
    double* m_h = m_pen + R * R;
    double* m_v = m_h + R * R;
    double* wr = m_v + R * R;
    double* wi = wr + R;
    double* ort = wi + R;
    int* rowp = (int*)(ort + R);  // 2R ints = R doubles
    int* colp = rowp + R;
    double* piv = ort + 2 * R;    // R
    double* wscr = piv + R;       // 64 (team argmax scratch)
    const double* ur = d.Ur + ((size_t)p * 2 + 0) * Q * R;
    double* a1 = d.f(prob, 0);
    if (threadIdx.x == 0) att = -1;
    __syncthreads();
    for (int a = d.att_start[prob]; a < 3; ++a) {
        const double* p1 = d.Pm + (((size_t)prob * 6) + a * 2 + 0) * R * R;
        const double* p2 = d.Pm + (((size_t)prob * 6) + a * 2 + 1) * R * R;
        if (threadIdx.x < 32) {
            // one warp: FullPivLU of p2 (cp_als.cpp:122-124), pencil p1 p2^-1,
            // real Schur form + eigenvectors (cp_als.cpp:126-140)
            TeamWarp w;
            for (int i = w.tid(); i < R * R; i += 32) m_h[i] = p2[i];
            __syncwarp();
            bool good = lu_fullpiv_inverse_team(w, R, m_h, R, m_inv, R, rowp, colp, piv, wscr);
            if (good) {
                for (int e = w.tid(); e < R * R; e += 32) {
                    const int i = e % R, j = e / R;
                    double s = 0.0;
                    for (int k = 0; k < R; ++k) s += p1[i + R * k] * m_inv[k + R * j];
                    m_pen[e] = s;
                }
                __syncwarp();
                good = eig_real_team(w, R, m_pen, m_v, wr, wi, ort);
            }
            if (good) {
                if (w.tid() == 0) {
                    int c = 0;
                    while (c < R) {
                        if (fabs(wi[c]) > 1e-9 * fabs(wr[c]) && c + 1 < R) {
                            for (int i = 0; i < R; ++i) {
                                asub[i + R * c] = m_v[i + R * c];
                                asub[i + R * (c + 1)] = m_v[i + R * (c + 1)];
                            }
                            c += 2;
                        } else {
                            const int src = (wi[c] < 0.0 && c > 0) ? c - 1 : c;
                            for (int i = 0; i < R; ++i) asub[i + R * c] = m_v[i + R * src];
                            c += 1;
                        }
                    }
                }
            }
            if (w.tid() == 0) ok = good ? 1 : 0;
        }
        __syncthreads();
        if (!ok) continue;
        // a1 = U_r a_sub, column norms
        for (int e = threadIdx.x; e < Q * R; e += blockDim.x) {
            const int i = e % Q, c = e / Q;
            double s = 0.0;
            for (int k = 0; k < R; ++k) s += ur[i + (size_t)Q * k] * asub[k + R * c];
            a1[i + (size_t)Q * c] = s;
        }
        __syncthreads();
        for (int c = threadIdx.x; c < R; c += blockDim.x) {
            double s = 0.0;
            for (int i = 0; i < Q; ++i) s += dsq(a1[i + (size_t)Q * c]);
            nrm[c] = sqrt(s);
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            for (int c = 0; c < R; ++c)
                if (nrm[c] < kDegenerateNorm) ok = 0;
        }
        __syncthreads();
        if (!ok) continue;
        for (int e = threadIdx.x; e < Q * R; e += blockDim.x) {
            const int c = e / Q;
            a1[e] /= nrm[c];
        }
        if (threadIdx.x == 0) att = a;
        __syncthreads();
        break;
    }
    if (threadIdx.x == 0) d.att_used[prob] = att;
}

// h = (a1^T a1)^-1 (a1^T Y_(0)) in place on Hh (R x Q^2), per problem.
__global__ void gevd_hsolve_kernel(AlsDev d) {
    const int prob = blockIdx.x;
    if (!d.todo[prob] || d.att_used[prob] < 0) return;
    const int Q = d.Q, R = d.R;
    extern __shared__ double sm[];
    double* Lf = sm;           // R*R
    double* Vp = Lf + R * R;   // R*R (Gram; pinv fallback / inverse)
    double* Li = Vp + R * R;   // R*R (L^-1)
    double* cs = Li + R * R;   // 2(R+2)
    int* flag = (int*)(cs + 2 * (R + 2));
    __shared__ int rank;
    const double* a1 = d.f(prob, 0);
    for (int e = threadIdx.x; e < R * R; e += blockDim.x) {
        const int i = e % R, j = e / R;
        double s = 0.0;
        for (int q = 0; q < Q; ++q) s += a1[q + (size_t)Q * i] * a1[q + (size_t)Q * j];
        Lf[e] = s;
        Vp[e] = s;
    }
    __syncthreads();
    if (threadIdx.x < 32) {
        TeamWarp w;
        int rk;
        if (R <= 32) {
            const double md = warp_max_diag(Lf, R, R);
            rk = warp_chol_inv32(Lf, R, R, md > 0.0 ? kEps * R * md : INFINITY, Li, R);
        } else {
            rk = team_chol_semidef(w, R, Lf, R, kEps * R, cs, flag);
            if (rk == R) team_tri_inv_lower(w, R, Lf, R, Li, R);
        }
        if (threadIdx.x == 0) rank = rk;
    }
    __syncthreads();
    double* h = d.Hh + (size_t)prob * R * d.q2();
    if (rank == R) {
        // Vp <- (a1^T a1)^-1 = L^-T L^-1
        for (int e = threadIdx.x; e < R * R; e += blockDim.x) {
            const int i = e % R, j = e / R;
            double sacc = 0.0;
            for (int k = (i > j ? i : j); k < R; ++k) sacc += Li[k + R * i] * Li[k + R * j];
            Vp[e] = sacc;
        }
    } else {
        // minimum-norm fallback: Vp <- pseudo-inverse from the eigen-decomposition
        double* Ev = d.gscr + (size_t)prob * (6 * R * R + 4 * R);
        TeamDev team;
        jacobi_eig_sym(team, R, Vp, Ev, cs, flag);
        __syncthreads();
        double wmax = 0.0;
        for (int i = 0; i < R; ++i) wmax = fmax(wmax, fabs(Vp[i + R * i]));
        const double thr = kEps * R * wmax;
        for (int e = threadIdx.x; e < R * R; e += blockDim.x) {
            const int i = e % R, j = e / R;
            double sacc = 0.0;
            for (int k = 0; k < R; ++k) {
                const double w = Vp[k + R * k];
                if (w > thr) sacc += Ev[i + R * k] * Ev[j + R * k] / w;
            }
            Li[e] = sacc;
        }
        __syncthreads();
        for (int e = threadIdx.x; e < R * R; e += blockDim.x) Vp[e] = Li[e];
    }
    __syncthreads();
    // Vp to global: h <- Vp h runs next as a batched GEMM (gevd_hsolve)
    double* vg = d.gscr + (size_t)prob * (6 * R * R + 4 * R) + 3 * R * R;
    for (int e = threadIdx.x; e < R * R; e += blockDim.x) vg[e] = Vp[e];
}

// Rank-1 peel of every h row (cp_als.cpp:168-173): H_r(b,c) = h(r, b + Q c).
__global__ void gevd_peel_kernel(AlsDev d) {
    const int prob = blockIdx.x / d.R, r = blockIdx.x % d.R;
    if (!d.todo[prob] || d.att_used[prob] < 0) return;
    const int Q = d.Q, R = d.R;
    extern __shared__ double sm[];
    double* H = sm;                     // Q*Q
    double* u = H + (size_t)Q * Q;      // Q
    double* v = u + Q;                  // Q
    double* red = v + Q;                // blockDim + 2 + Q
    const double* h = d.KR + (size_t)prob * R * d.q2();  // h2 = Vp h (gevd_hsolve + GEMM)
    g2s_copy(H, h + (size_t)r * d.q2(), Q * Q);
    __syncthreads();
    TeamDev team;
    const double sigma = top_singular_pair(team, Q, Q, H, u, v, red);
    double* fb = d.f(prob, 1);
    double* fc = d.f(prob, 2);
    int bad = 0;
    for (int i = threadIdx.x; i < Q; i += blockDim.x) {
        fb[i + (size_t)Q * r] = u[i];
        const double cv = sigma * v[i];
        fc[i + (size_t)Q * r] = cv;
        if (!isfinite(u[i]) || !isfinite(cv)) bad = 1;
    }
    if (bad) atomicOr(&d.peel_fail[prob], 1);
}

// Grams of the initial factors, lambda = 1, fresh sweep state.
__global__ void als_init_state_kernel(AlsDev d) {
    const int prob = blockIdx.x;
    const int Q = d.Q, R = d.R;
    for (int n = 0; n < 3; ++n) {
        const double* f = d.f(prob, n);
        double* g = d.g(prob, n);
        for (int e = threadIdx.x; e < R * R; e += blockDim.x) {
            const int i = e % R, j = e / R;
            double s = 0.0;
            for (int q = 0; q < Q; ++q) s += f[q + (size_t)Q * i] * f[q + (size_t)Q * j];
            g[e] = s;
        }
    }
    for (int c = threadIdx.x; c < R; c += blockDim.x) d.lam[(size_t)prob * R + c] = 1.0;
    if (threadIdx.x == 0) {
        AlsState s;
        s.prev_fit = 0.0;
        s.active = 1;
        s.iterations = 0;
        s.rescued = 0;
        s.rng_init = 0;
        s.failed = 0;
        s.pad = 0;
        d.state[prob] = s;
        d.err[prob].code = kOk;
    }
}

// ---------------- sweeps ----------------

// V = Hadamard product of the other two modes' Grams, then Vi = V^-1 from
// the Cholesky factor, or the eigen pseudo-inverse when V is numerically
// singular (matching COD's minimum-norm solve; cp_als.cpp:298-323).  It needs
// only the other modes' Grams, so it runs in extra blocks of the MTTKRP launch
// of the same mode, off the update's critical path.  256 threads; sm holds
// 4 R^2 + 2 (R + 2) + 256 doubles and R + 8 ints.
__device__ void als_vinv_block(const AlsDev& d, int prob, int mode, double* sm) {
    const int R = d.R;
    double* V = sm;                  // R*R
    double* Lf = V + R * R;          // R*R
    double* Ev = Lf + R * R;         // R*R  (eigenvectors / L^-1)
    double* Vi = Ev + R * R;         // R*R
    double* cs = Vi + R * R;         // 2(R+2)
    double* red = cs + 2 * (R + 2);  // blockDim
    int* iw = (int*)(red + blockDim.x);  // R + 8
    __shared__ int rank;
    for (int e = threadIdx.x; e < R * R; e += blockDim.x) {
        double v = 1.0;
        for (int k = 0; k < 3; ++k)
            if (k != mode) v *= d.g(prob, k)[e];
        V[e] = v;
        Lf[e] = v;
    }
    __syncthreads();
    {
        // Lf = chol(V), Ev = Lf^-1, block-cooperative (R <= 64).  (A fully
        // unrolled one-warp register version measured 3.5x slower: its
        // straight-line code streams through the instruction cache once.)
        double md = 0.0;
        for (int i = 0; i < R; ++i) md = fmax(md, V[i + R * i]);
        const double thr = md > 0.0 ? kEps * R * md : INFINITY;
        const int rk = block_chol_inv64(V, R, R, thr, Lf, R, Ev, R, red);
        if (threadIdx.x == 0) rank = rk;
    }
    __syncthreads();
    double* out = d.Vinv + (size_t)prob * R * R;
    if (rank == R) {
        // Vi = L^-T L^-1 on the FP64 tensor cores: Vi(i, j) = sum_k Ev(k, i) Ev(k, j)
        block_dmma_small(R, R, R, Ev, R, 1, Ev, 1, R, Vi, 1, R);
    } else {
        TeamDev team;
        jacobi_eig_sym(team, R, V, Ev, cs, iw);
        __syncthreads();
        double wmax = 0.0;
        for (int i = 0; i < R; ++i) wmax = fmax(wmax, fabs(V[i + R * i]));
        const double thr = kEps * R * wmax;
        for (int e = threadIdx.x; e < R * R; e += blockDim.x) {
            const int i = e % R, j = e / R;
            double s = 0.0;
            for (int k = 0; k < R; ++k) {
                const double w = V[k + R * k];
                if (w > thr) s += Ev[i + R * k] * Ev[j + R * k] / w;
            }
            Vi[e] = s;
        }
    }
    __syncthreads();
    for (int e = threadIdx.x; e < R * R; e += blockDim.x) out[e] = Vi[e];
}

// MTTKRP from a partial contraction T(u, v, r) (row u + Q v of the
// per-replica T, column s R + r): contract_first == 0 gives
// M(u, r) = sum_v T(u,v,r) F_fsrc(v,r), contract_first == 1 gives
// M(v, r) = sum_u T(u,v,r) F_fsrc(u,r).  One block per (problem, r); the 8
// warps split the v range, lanes run along the contiguous u index of T; the
// contract-v partials are combined across warps in fixed order.
// One mode update per problem: raw = M V^-1 (COD of the Hadamard Gram;
// cp_als.cpp:298-323), non-finite check, normalize into lambda with the
// seeded rescue, new Gram; after mode 2 the fit and the convergence test
// (cp_als.cpp:325-345).  V^-1 (als_vinv_block, formed during the MTTKRP)
// makes raw = M V^-1 a parallel (Q x R)(R x R) product.
__device__ void als_update_block(const AlsDev& d, int prob, int mode, int sweep, double* sm) {
    AlsState* st = d.state + prob;
    if (!st->active) return;
    const int Q = d.Q, R = d.R;
    double* Vi = sm;                // R*R  (V^-1 or V^+, from als_vinv_block)
    double* raw = Vi + R * R;       // Q*R
    double* Ms = raw + Q * R;       // Q*R  (staged MTTKRP)
    double* nrm = Ms + Q * R;       // R
    double* cs = nrm + R;           // 2(R+2)
    double* red = cs + 2 * (R + 2); // blockDim
    __shared__ int bad;
    const double* M = Ms;
#define OCTEN_TSC(i) \
    if (d.tsc && threadIdx.x == 0 && prob == 0) d.tsc[(i)] = clock64();
    OCTEN_TSC(0)
    {
        g2s_copy(Ms, d.Mb + (size_t)prob * Q * R, Q * R);
    }
    g2s_copy(Vi, d.Vinv + (size_t)prob * R * R, R * R);
    if (threadIdx.x == 0) bad = 0;
    __syncthreads();
    OCTEN_TSC(1)
    // raw = M Vi on the FP64 tensor cores (Q x R x R)
    block_dmma_small(Q, R, R, M, 1, Q, Vi, 1, R, raw, 1, Q);
    __syncthreads();
    for (int e = threadIdx.x; e < Q * R; e += blockDim.x)
        if (!isfinite(raw[e])) bad = 1;
    __syncthreads();
    OCTEN_TSC(4)
    if (bad) {
        if (threadIdx.x == 0) {
            d.err[prob].code = kAlsNonFiniteFactor;
            d.err[prob].problem = prob;
            d.err[prob].a = sweep + 1;
            d.err[prob].b = mode + 1;
            st->active = 0;
            st->failed = 1;
        }
        return;
    }
    {
        // column norms: one warp per column
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
        for (int c = warp; c < R; c += nw) {
            double sacc = 0.0;
            for (int q = lane; q < Q; q += 32) sacc += raw[q + Q * c] * raw[q + Q * c];
            for (int o = 16; o > 0; o >>= 1) sacc += __shfl_xor_sync(0xffffffffu, sacc, o);
            if (lane == 0) nrm[c] = sqrt(sacc);
        }
    }
    __syncthreads();
    OCTEN_TSC(5)
    // degenerate columns are re-drawn from the problem's sequential rescue
    // stream (column order); the common case (none) skips the serial loop
    __shared__ int any_degenerate;
    if (threadIdx.x == 0) any_degenerate = 0;
    __syncthreads();
    for (int c = threadIdx.x; c < R; c += blockDim.x)
        if (nrm[c] < kDegenerateNorm) any_degenerate = 1;
    __syncthreads();
    if (!any_degenerate) {
        for (int c = threadIdx.x; c < R; c += blockDim.x) {
            d.lam[(size_t)prob * R + c] = nrm[c];
            cs[c] = 1.0 / nrm[c];
        }
    } else if (threadIdx.x == 0) {
        for (int c = 0; c < R; ++c) {
            if (nrm[c] < kDegenerateNorm) {
                Mt64* g = d.rngs + prob;
                if (!st->rng_init) {
                    g->seed(d.rescue_seed[prob]);
                    st->rng_init = 1;
                }
                double s = 0.0;
                for (int q = 0; q < Q; ++q) {
                    raw[q + Q * c] = g->uniform01();
                    s += raw[q + Q * c] * raw[q + Q * c];
                }
                nrm[c] = sqrt(s);
                st->rescued = 1;
            }
            d.lam[(size_t)prob * R + c] = nrm[c];
            cs[c] = 1.0 / nrm[c];
        }
    }
    __syncthreads();
    OCTEN_TSC(6)
    double* f = d.f(prob, mode);
    for (int e = threadIdx.x; e < Q * R; e += blockDim.x) {
        const double v = raw[e] * cs[e / Q];  // cs: 1 / column norm
        raw[e] = v;
        f[e] = v;
    }
    __syncthreads();
    OCTEN_TSC(7)
    double* g = d.g(prob, mode);
    // Gram of the new factor on the FP64 tensor cores: g(i, j) = sum_q raw(q, i) raw(q, j)
    block_dmma_small(R, R, Q, raw, Q, 1, raw, 1, Q, g, 1, R);
    if (d.Fd) {  // the new factor's digits for the next T-GEMM that contracts this mode
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
        for (int r = warp; r < R; r += nw)
            oz::factor_column_digits(d.Fd, d.Fcs, d.oz_G, d.S, R, Q, prob, mode, r, raw + (size_t)Q * r, lane);
    }
    __syncthreads();
    OCTEN_TSC(8)
    if (mode != 2) return;
    // fit (cp_als.cpp:325-345)
    const double* lam = d.lam + (size_t)prob * R;
    double part = 0.0;
    for (int e = threadIdx.x; e < Q * R; e += blockDim.x) part += M[e] * raw[e] * lam[e / Q];
    const double inner = block_sum(part, red);
    double part2 = 0.0;
    for (int e = threadIdx.x; e < R * R; e += blockDim.x) {
        const int i = e % R, j = e / R;
        part2 += lam[i] * (d.g(prob, 0)[e] * d.g(prob, 1)[e] * d.g(prob, 2)[e]) * lam[j];
    }
    const double norm_m_sq = block_sum(part2, red);
    if (threadIdx.x == 0) {
        const int p = prob / d.S;
        const double nx2 = d.normx2[p];
        const double norm_x = sqrt(nx2);
        const double res_sq = fmax(0.0, nx2 - 2.0 * inner + norm_m_sq);
        const double residual = sqrt(res_sq);
        const double fit = 1.0 - residual / norm_x;
        if (!isfinite(fit)) {
            d.err[prob].code = kAlsNonFiniteFit;
            d.err[prob].problem = prob;
            d.err[prob].a = sweep + 1;
            st->active = 0;
            st->failed = 1;
            return;
        }
        d.fit_hist[(size_t)prob * d.max_iters + sweep] = fit;
        d.res_hist[(size_t)prob * d.max_iters + sweep] = residual;
        bool stop = false;
        if (sweep > 0 && fabs(fit - st->prev_fit) < d.rel_tol) stop = true;
        st->prev_fit = fit;
        if (stop || sweep + 1 >= d.max_iters) {
            st->iterations = sweep + 1;
            st->active = 0;
        } else {
            d.hact[(size_t)sweep * kAlsMaxLanes] = 1;  // host-mapped; visible once the sweep's event completes
        }
    }
#undef OCTEN_TSC
}

__global__ void als_update_kernel(AlsDev d, int mode, int sweep) {
    pdl_trigger();
    pdl_wait();
    extern __shared__ double sm[];
    als_update_block(d, blockIdx.x, mode, sweep, sm);
}

// One T column (Q x Q, u fastest) against the weight vector w: warps take
// rows v (U rows per round, all loads issued first), lanes run along u.
template <int NA>
__device__ __forceinline__ void mttkrp_column(const double* __restrict__ tcol, const double* __restrict__ w,
                                              double* __restrict__ M, int Q, int contract_first) {
    constexpr int U = 4;
    __shared__ double part[8][257];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    if (!contract_first) {  // M(u) = sum_v T(u, v) w(v)
        double acc[NA];
#pragma unroll
        for (int i = 0; i < NA; ++i) acc[i] = 0.0;
        for (int b0 = warp; b0 < Q; b0 += U * nw) {
            double x[U][NA], wv[U];
#pragma unroll
            for (int j = 0; j < U; ++j) {
                const int b = b0 + j * nw;
                const bool vb = b < Q;
                wv[j] = vb ? __ldg(w + b) : 0.0;
                const double* row = tcol + (size_t)Q * b;
#pragma unroll
                for (int i = 0; i < NA; ++i) {
                    const int a = lane + 32 * i;
                    x[j][i] = (vb && a < Q) ? __ldg(row + a) : 0.0;
                }
            }
#pragma unroll
            for (int j = 0; j < U; ++j)
#pragma unroll
                for (int i = 0; i < NA; ++i) acc[i] += x[j][i] * wv[j];
        }
#pragma unroll
        for (int i = 0; i < NA; ++i) {
            const int a = lane + 32 * i;
            if (a < Q) part[warp][a] = acc[i];
        }
        __syncthreads();
        for (int a = threadIdx.x; a < Q; a += blockDim.x) {
            double sum = 0.0;
            for (int v = 0; v < nw; ++v) sum += part[v][a];
            M[a] = sum;
        }
    } else {  // M(v) = sum_u T(u, v) w(u)
        double av[NA];
#pragma unroll
        for (int i = 0; i < NA; ++i) {
            const int a = lane + 32 * i;
            av[i] = a < Q ? __ldg(w + a) : 0.0;
        }
        for (int b0 = warp; b0 < Q; b0 += U * nw) {
            double acc[U];
#pragma unroll
            for (int j = 0; j < U; ++j) {
                const int b = b0 + j * nw;
                const bool vb = b < Q;
                const double* row = tcol + (size_t)Q * b;
                double x[NA];
#pragma unroll
                for (int i = 0; i < NA; ++i) {
                    const int a = lane + 32 * i;
                    x[i] = (vb && a < Q) ? __ldg(row + a) : 0.0;
                }
                acc[j] = 0.0;
#pragma unroll
                for (int i = 0; i < NA; ++i) acc[j] += x[i] * av[i];
            }
#pragma unroll
            for (int j = 0; j < U; ++j) {
                double v = acc[j];
                for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
                const int b = b0 + j * nw;
                if (lane == 0 && b < Q) M[b] = v;
            }
        }
    }
}

// The same contraction with 16-byte loads, eight of them in flight per thread
// before their first use (Q even, Q <= 128, 256 threads).  contract_first ==
// 0: thread (pair pu, group vg) sums rows v = vg, vg + 4, ... of pairs
// (2 pu, 2 pu + 1); the four group partials are added in group order.
// contract_first == 1: warp w takes rows v = w, w + 8, ...; its lanes hold
// pairs pu = lane, lane + 32 of each row and the row sum is a fixed shuffle
// tree.
__device__ __forceinline__ void mttkrp_column_v2(const double* __restrict__ tcol, const double* __restrict__ w,
                                                 double* __restrict__ M, int Q, int contract_first) {
    constexpr int B = 8;  // rows of a thread in flight per batch (registers: 80 at 3 CTAs per SM)
    __shared__ double2 part2[4][64];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int QP = Q >> 1;  // pairs per row
    if (!contract_first) {  // M(u) = sum_v T(u, v) w(v)
        const int pu = tid & 63, vg = tid >> 6;
        double2 acc = make_double2(0.0, 0.0);
        if (pu < QP) {
#pragma unroll 1
            for (int v0 = vg; v0 < Q; v0 += 4 * B) {
                double2 x[B];
                double wv[B];
#pragma unroll
                for (int j = 0; j < B; ++j) {
                    const int v = v0 + 4 * j;
                    x[j] = make_double2(0.0, 0.0);
                    wv[j] = 0.0;
                    if (v < Q) {
                        x[j] = __ldg(reinterpret_cast<const double2*>(tcol + (size_t)Q * v) + pu);
                        wv[j] = __ldg(w + v);
                    }
                }
#pragma unroll
                for (int j = 0; j < B; ++j) {
                    acc.x += x[j].x * wv[j];
                    acc.y += x[j].y * wv[j];
                }
            }
        }
        part2[vg][pu] = acc;
        __syncthreads();
        for (int e = tid; e < QP; e += blockDim.x) {
            double2 sacc = part2[0][e];
            for (int g = 1; g < 4; ++g) {
                sacc.x += part2[g][e].x;
                sacc.y += part2[g][e].y;
            }
            M[2 * e] = sacc.x;
            M[2 * e + 1] = sacc.y;
        }
    } else {  // M(v) = sum_u T(u, v) w(u)
        double2 wa = make_double2(0.0, 0.0), wb = make_double2(0.0, 0.0);
        if (lane < QP) wa = __ldg(reinterpret_cast<const double2*>(w) + lane);
        if (lane + 32 < QP) wb = __ldg(reinterpret_cast<const double2*>(w) + lane + 32);
#pragma unroll 1
        for (int v0 = warp; v0 < Q; v0 += 8 * (B / 2)) {
            double2 xa[B / 2], xb[B / 2];
#pragma unroll
            for (int j = 0; j < B / 2; ++j) {
                const int v = v0 + 8 * j;
                xa[j] = xb[j] = make_double2(0.0, 0.0);
                if (v < Q) {
                    const double2* row = reinterpret_cast<const double2*>(tcol + (size_t)Q * v);
                    if (lane < QP) xa[j] = __ldg(row + lane);
                    if (lane + 32 < QP) xb[j] = __ldg(row + lane + 32);
                }
            }
#pragma unroll
            for (int j = 0; j < B / 2; ++j) {
                const int v = v0 + 8 * j;
                double sacc = (xa[j].x * wa.x + xa[j].y * wa.y) + (xb[j].x * wb.x + xb[j].y * wb.y);
                for (int o = 16; o > 0; o >>= 1) sacc += __shfl_xor_sync(0xffffffffu, sacc, o);
                if (lane == 0 && v < Q) M[v] = sacc;
            }
        }
    }
}

// Diagnostics, compiled in with -DOCTEN_ALS_GT_STAMPS only (the stamps cost the
// contraction kernel registers): %globaltimer marks (ns) of problem 0's V^-1
// block, first column block and mode update within one MTTKRP launch.
__device__ __forceinline__ void als_gt_stamp(const AlsDev& d, int i) {
#ifdef OCTEN_ALS_GT_STAMPS
    if (d.tsc && threadIdx.x == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
        d.tsc[i] = (long long)t;
    }
#endif
}

// The first NP blocks instead form Vi of `mode` (als_vinv_block).  With
// `fused`, the last of a problem's R + 1 blocks to finish (fence + counter)
// runs the mode update for it (als_update_block), so the update needs no
// launch of its own and overlaps the other problems' contractions.
template <int NA>
__global__ void __launch_bounds__(256, 3) als_mttkrp_T_kernel(AlsDev d, int contract_first, int fsrc, int mode,
                                                              int sweep, int fused) {
    pdl_trigger();
    pdl_wait();
    extern __shared__ double vsm[];
    const int R = d.R, Q = d.Q;
    int prob;
    if ((int)blockIdx.x < d.NP) {
        prob = blockIdx.x;
        if (!d.state[prob].active) return;
        if (prob == 0) als_gt_stamp(d, 32);
        als_vinv_block(d, prob, mode, vsm);
        if (prob == 0) als_gt_stamp(d, 33);
    } else {
        const int bid = blockIdx.x - d.NP;
        prob = bid / R;
        const int r = bid % R;
        if (!d.state[prob].active) return;
        const int p = prob / d.S, s = prob % d.S;
        const double* tcol = d.T + (size_t)p * d.q2() * d.S * R + (size_t)d.q2() * (s * R + r);
        double* M = d.Mb + (size_t)prob * Q * R + (size_t)Q * r;
        const double* w = d.f(prob, fsrc) + (size_t)Q * r;
        if (bid == 0) als_gt_stamp(d, 34);
        if (NA == 0)
            mttkrp_column_v2(tcol, w, M, Q, contract_first);
        else
            mttkrp_column<NA == 0 ? 4 : NA>(tcol, w, M, Q, contract_first);
    }
#ifdef OCTEN_ALS_GT_STAMPS
    if (d.tsc && blockIdx.x == (unsigned)d.NP) { __syncthreads(); als_gt_stamp(d, 35); }
#endif
    if (!fused) return;
    __shared__ int last;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        last = atomicAdd(d.mcount + prob, 1) == R;
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    if (threadIdx.x == 0) d.mcount[prob] = 0;
    if (prob == 0) als_gt_stamp(d, 36);
    als_update_block(d, prob, mode, sweep, vsm);
#ifdef OCTEN_ALS_GT_STAMPS
    if (prob == 0) { __syncthreads(); als_gt_stamp(d, 37); }
#endif
}


// Best restart per replica (strictly greater final fit wins; cp_als.cpp:347-356).
__global__ void als_select_kernel(AlsDev d, double* Mf, double* Mlam, int* best_out) {
    const int p = blockIdx.x;
    __shared__ int best;
    if (threadIdx.x == 0) {
        double bf = -INFINITY;
        best = 0;
        for (int s = 0; s < d.S; ++s) {
            const int prob = p * d.S + s;
            const AlsState& st = d.state[prob];
            const double ff = st.iterations > 0 ? d.fit_hist[(size_t)prob * d.max_iters + st.iterations - 1] : -INFINITY;
            if (ff > bf) {
                bf = ff;
                best = s;
            }
        }
        best_out[p] = best;
    }
    __syncthreads();
    const int prob = p * d.S + best;
    const size_t fsz = (size_t)3 * d.Q * d.R;
    for (size_t e = threadIdx.x; e < fsz; e += blockDim.x) Mf[(size_t)p * fsz + e] = d.F[(size_t)prob * fsz + e];
    for (int c = threadIdx.x; c < d.R; c += blockDim.x) Mlam[(size_t)p * d.R + c] = d.lam[(size_t)prob * d.R + c];
}

// ---- GEMM functors ----
struct YmatA {  // A(p, m, k) = Y[p][m + Q^2 k]   (Y as Q^2 x Q)
    const double* Y;
    size_t q3, q2;
    int S;
    bool per_problem;
    __device__ double operator()(int b, int m, int k) const {
        const int p = per_problem ? b / S : b;
        return Y[(size_t)p * q3 + m + q2 * k];
    }
};
struct YmidA {  // A(p, m, k) = Y[p][i + Q k + Q^2 c], m = i + Q c   (rows of Y x2)
    const double* Y;
    size_t q3;
    int Q;
    __device__ double operator()(int p, int m, int k) const {
        const int c = m / Q, i = m - c * Q;
        return Y[(size_t)p * q3 + i + (size_t)Q * (k + (size_t)Q * c)];
    }
};
struct Y0tA {  // A(p, m, k) = Y[p][k + Q m]   (rows of Y x1: m = b + Q c)
    const double* Y;
    size_t q3;
    int Q;
    __device__ double operator()(int p, int m, int k) const { return Y[(size_t)p * q3 + k + (size_t)Q * m]; }
};
struct FacB {  // B(p, k, n) = F[(p S + n / R)][mode][k + Q (n % R)]
    const double* F;
    int S, Q, R, mode;
    __device__ double operator()(int p, int k, int n) const {
        const int prob = p * S + n / R;
        return F[((size_t)prob * 3 + mode) * Q * R + k + (size_t)Q * (n % R)];
    }
};
struct TStore {  // T[p][m + Q^2 n]
    double* T;
    size_t q2;
    int SR;
    __device__ void operator()(int p, int m, int n, double v) const { T[(size_t)p * q2 * SR + m + q2 * n] = v; }
};
// element-pointer twins for the pipelined DMMA GEMM (16-byte pairs along the
// fast index; used when Q is even)
struct YmatP {  // &Y[p][m + Q^2 k]   (M-fast)
    const double* Y;
    size_t q3, q2;
    __device__ const double* operator()(int p, int m, int k) const { return Y + (size_t)p * q3 + m + q2 * k; }
};
struct FacP {  // &F[(p S + n / R)][mode][k + Q (n % R)]   (K-fast)
    const double* F;
    int S, Q, R, mode;
    __device__ const double* operator()(int p, int k, int n) const {
        const int prob = p * S + n / R;
        return F + ((size_t)prob * 3 + mode) * Q * R + k + (size_t)Q * (n % R);
    }
};
struct YmidP {  // &Y[p][i + Q k + Q^2 c], m = i + Q c   (Y x2: rows (i, c), M-fast in runs of Q)
    const double* Y;
    size_t q3;
    unsigned Q, qinv;  // qinv = ceil(2^32 / Q): m / Q = umulhi(m, qinv) for m Q < 2^32
    __device__ const double* operator()(int p, int m, int k) const {
        const unsigned c = __umulhi((unsigned)m, qinv), i = (unsigned)m - c * Q;
        return Y + (size_t)p * q3 + i + (size_t)Q * (k + (size_t)Q * c);
    }
};
// GEVD Grams
struct Y0A {  // A(p, a, k) = Y[p][a + Q k]   (Y_(0): Q x Q^2)
    const double* Y;
    size_t q3;
    int Q;
    __device__ double operator()(int p, int a, int k) const { return Y[(size_t)p * q3 + a + (size_t)Q * k]; }
};
struct Y0B {  // B(p, k, a') = Y[p][a' + Q k]
    const double* Y;
    size_t q3;
    int Q;
    __device__ double operator()(int p, int k, int a) const { return Y[(size_t)p * q3 + a + (size_t)Q * k]; }
};
struct Y1A {  // A(p, b, k), k = a + Q c -> Y[a + Q b + Q^2 c]   (Y_(1))
    const double* Y;
    size_t q3;
    int Q;
    __device__ double operator()(int p, int b, int k) const {
        const int a = k % Q, c = k / Q;
        return Y[(size_t)p * q3 + a + (size_t)Q * b + (size_t)Q * Q * c];
    }
};
struct Y1B {
    const double* Y;
    size_t q3;
    int Q;
    __device__ double operator()(int p, int k, int b) const {
        const int a = k % Q, c = k / Q;
        return Y[(size_t)p * q3 + a + (size_t)Q * b + (size_t)Q * Q * c];
    }
};
struct GevStore {
    double* G;
    int Q, which;
    __device__ void operator()(int p, int i, int j, double v) const {
        G[((size_t)p * 2 + which) * Q * Q + i + (size_t)Q * j] = v;
    }
};
// mixtures
struct MixB {  // B(prob, c, j) = Wmix[prob][j][c]
    const double* W;
    int Q;
    __device__ double operator()(int prob, int c, int j) const { return W[((size_t)prob * 6 + j) * Q + c]; }
};
struct MixStore {
    double* S;
    size_t q2;
    __device__ void operator()(int prob, int m, int j, double v) const { S[((size_t)prob * 6 + j) * q2 + m] = v; }
};
struct SmA {  // A(bj, a, b) = Smix[bj][a + Q b]
    const double* S;
    int Q;
    __device__ double operator()(int bj, int a, int b) const { return S[(size_t)bj * Q * Q + a + (size_t)Q * b]; }
};
struct UrB {  // B(bj, b, r) = Ur[p][which][b + Q r], p = (bj/6)/S
    const double* Ur;
    int Q, R, S, which;
    __device__ double operator()(int bj, int b, int r) const {
        const int p = (bj / 6) / S;
        return Ur[((size_t)p * 2 + which) * Q * R + b + (size_t)Q * r];
    }
};
struct Tmp6Store {
    double* T;
    int Q, R;
    __device__ void operator()(int bj, int a, int r, double v) const { T[(size_t)bj * Q * R + a + (size_t)Q * r] = v; }
};
struct UrTA {  // A(bj, i, a) = Ur[p][0][a + Q i]
    const double* Ur;
    int Q, R, S;
    __device__ double operator()(int bj, int i, int a) const {
        const int p = (bj / 6) / S;
        return Ur[((size_t)p * 2) * Q * R + a + (size_t)Q * i];
    }
};
struct Tmp6B {
    const double* T;
    int Q, R;
    __device__ double operator()(int bj, int a, int r) const { return T[(size_t)bj * Q * R + a + (size_t)Q * r]; }
};
struct PmStore {
    double* Pm;
    int R;
    __device__ void operator()(int bj, int i, int r, double v) const { Pm[(size_t)bj * R * R + i + (size_t)R * r] = v; }
};
// h = a1^T Y_(0)
struct A1tA {  // A(prob, r, a) = F[prob][0][a + Q r]
    const double* F;
    int Q, R;
    __device__ double operator()(int prob, int r, int a) const { return F[((size_t)prob * 3) * Q * R + a + (size_t)Q * r]; }
};
struct Y0Bp {  // B(prob, a, k) = Y[p][a + Q k]
    const double* Y;
    size_t q3;
    int Q, S;
    __device__ double operator()(int prob, int a, int k) const {
        return Y[(size_t)(prob / S) * q3 + a + (size_t)Q * k];
    }
};
struct VpA {  // A(prob, i, j) = Vp[prob][i + R j]   (the R x R solve operator)
    const double* G;
    int R;
    __device__ double operator()(int prob, int i, int j) const {
        return G[(size_t)prob * (6 * R * R + 4 * R) + 3 * R * R + i + (size_t)R * j];
    }
};
struct HrowB {  // B(prob, j, k) = H[prob][j][k]
    const double* H;
    int R;
    size_t q2;
    __device__ double operator()(int prob, int j, int k) const { return H[(size_t)prob * R * q2 + (size_t)j * q2 + k]; }
};
// pointer functors for the pipelined GEVD GEMMs (Q even)
struct Y0PA {  // &Y[p][m + Q k]   (Y_(0), M-fast)
    const double* Y;
    size_t q3;
    int Q;
    __device__ const double* operator()(int p, int m, int k) const { return Y + (size_t)p * q3 + m + (size_t)Q * k; }
};
struct Y0PB {  // &Y[p][n + Q k]   (Y_(0)^T, N-fast)
    const double* Y;
    size_t q3;
    int Q;
    __device__ const double* operator()(int p, int k, int n) const { return Y + (size_t)p * q3 + n + (size_t)Q * k; }
};
struct Y1PA {  // &Y[p][a + Q b + Q^2 c], k = a + Q c   (Y_(1), K-fast)
    const double* Y;
    size_t q3;
    int Q;
    __device__ const double* operator()(int p, int b, int k) const {
        const int a = k % Q, c = k / Q;
        return Y + (size_t)p * q3 + a + (size_t)Q * b + (size_t)Q * Q * c;
    }
};
struct Y1PB {
    const double* Y;
    size_t q3;
    int Q;
    __device__ const double* operator()(int p, int k, int b) const {
        const int a = k % Q, c = k / Q;
        return Y + (size_t)p * q3 + a + (size_t)Q * b + (size_t)Q * Q * c;
    }
};
struct Y0tP {  // &Y[p][k + Q m]   (Y_(0)^T rows: m = b + Q c, K = a contiguous)
    const double* Y;
    size_t q3;
    int Q;
    __device__ const double* operator()(int p, int m, int k) const { return Y + (size_t)p * q3 + k + (size_t)Q * m; }
};
struct HtStore {  // C(p, m, n) -> H[p S + n / R][n % R][m]
    double* H;
    int S, R;
    size_t q2;
    __device__ void operator()(int p, int m, int n, double v) const {
        const int prob = p * S + n / R;
        H[(size_t)prob * R * q2 + (size_t)(n % R) * q2 + m] = v;
    }
};
struct HStore {  // H[prob][r][k]: row r of h contiguous (the peel reads H_r = h(r, :) whole)
    double* H;
    int R;
    size_t q2;
    __device__ void operator()(int prob, int r, int k, double v) const { H[(size_t)prob * R * q2 + (size_t)r * q2 + k] = v; }
};

}  // namespace

AlsHostDraws als_host_draws(const std::vector<std::uint64_t>& seeds, int S, int Q) {
    const int P = (int)seeds.size(), NP = P * S;
    AlsHostDraws d;
    d.S = S;
    d.Q = Q;
    d.seeds = seeds;
    d.restart_seed.resize(NP);
    d.hres.resize(NP);
    d.hw.resize((size_t)NP * 6 * Q);
    for (int p = 0; p < P; ++p)
        for (int s = 0; s < S; ++s) {
            const int prob = p * S + s;
            d.restart_seed[prob] = rng::derive(seeds[p], {rng::kAlsRestart, (std::uint64_t)s});
            d.hres[prob] = rng::derive(d.restart_seed[prob], {rng::kAlsRescue});
            for (int a = 0; a < 3; ++a) {
                rng::Substream ws(rng::derive(d.restart_seed[prob], {rng::kAlsGevd, (std::uint64_t)a}));
                double* w1 = d.hw.data() + ((size_t)prob * 6 + a * 2 + 0) * Q;
                double* w2 = d.hw.data() + ((size_t)prob * 6 + a * 2 + 1) * Q;
                for (int i = 0; i < Q; ++i) w1[i] = ws.uniform01() * 2 - 1;
                for (int i = 0; i < Q; ++i) w2[i] = ws.uniform01() * 2 - 1;
            }
        }
    return d;
}

void AlsEngine::prefetch_host_draws(const std::vector<std::uint64_t>& seeds, int S, int Q) {
    if (next_draws.valid()) next_draws.wait();
    next_draws = std::async(std::launch::async, als_host_draws, seeds, S, Q);
}

void AlsEngine::alloc(int P, int S, int Q, int R, int max_iters) {
    const size_t NP = (size_t)P * S, q2 = (size_t)Q * Q;
    P_ = P;
    S_ = S;
    Q_ = Q;
    R_ = R;
    I_ = max_iters;
    normx2.reserve(P);
    F.reserve(NP * 3 * Q * R);
    G.reserve(NP * 3 * R * R);
    lam.reserve(NP * R);
    T.reserve((size_t)P * q2 * S * R);
    KR.reserve((size_t)P * q2 * S * R);
    Mb.reserve(NP * Q * R);
    Vinv.reserve(NP * R * R);
    fit_hist.reserve(NP * max_iters);
    res_hist.reserve(NP * max_iters);
    state.reserve(NP);
    err.reserve(NP);
    rngs.reserve(NP);
    rescue_seed.reserve(NP);
    Gev.reserve((size_t)P * 2 * q2);
    EV.reserve((size_t)P * 2 * q2);
    Ur.reserve((size_t)P * 2 * Q * R);
    Wmix.reserve(NP * 6 * Q);
    Smix.reserve(NP * 6 * q2);
    Tmp6.reserve(NP * 6 * Q * R);
    Pm.reserve(NP * 6 * R * R);
    Hh.reserve(NP * R * q2);
    gscr.reserve(NP * (6 * R * R + 4 * R));
    usable.reserve(P);
    att_start.reserve(NP);
    att_used.reserve(NP);
    todo.reserve(NP);
    peel_fail.reserve(NP);
    Mf.reserve((size_t)P * 3 * Q * R);
    Mlam.reserve((size_t)P * R);
}

std::string als_failure_message(int kind, int a, int b) {
    // cp_als.cpp:305-307 (non-finite factor), 335-336 (non-finite fit), 251 (zero input)
    if (kind == 1) return "cp_als: input tensor is identically zero";
    if (kind == 2) return "cp_als: non-finite factor at sweep " + std::to_string(a) + ", mode " + std::to_string(b);
    return "cp_als: non-finite fit at sweep " + std::to_string(a);
}

AlsEngine::~AlsEngine() {
    for (cudaStream_t ls : lane_st)
        if (ls) {
            cudaStreamSynchronize(ls);
            cudaStreamDestroy(ls);
        }
    for (cudaStream_t ls : lane_hp)
        if (ls) {
            cudaStreamSynchronize(ls);
            cudaStreamDestroy(ls);
        }
    if (gemm_st) {
        cudaStreamSynchronize(gemm_st);
        cudaStreamDestroy(gemm_st);
    }
    for (cudaStream_t ls : lane_gemm)
        if (ls) {
            cudaStreamSynchronize(ls);
            cudaStreamDestroy(ls);
        }
    if (hact) cudaFreeHost(hact);
    if (res_pin) cudaFreeHost(res_pin);
    for (cudaEvent_t e : kev)
        if (e) cudaEventDestroy(e);
    for (cudaEvent_t e : lane_ev)
        if (e) cudaEventDestroy(e);
}

namespace {
// What run_init hands to run_sweeps.
struct AlsPending {
    AlsDev d;
    int P, S, Q, R, max_iters;
    double rel_tol;
    const double* dY;
    std::vector<int> used;  // GEVD attempt per problem (-1: random start)
};
}  // namespace

void AlsEngine::run(int P, int S, int Q, int R, int max_iters, double rel_tol, const double* dY,
                    const std::vector<std::uint64_t>& seeds, cudaStream_t st) {
    run_init(P, S, Q, R, max_iters, rel_tol, dY, seeds, st);
    run_sweeps(st);
}

void AlsEngine::run_init(int P, int S, int Q, int R, int max_iters, double rel_tol, const double* dY,
                         const std::vector<std::uint64_t>& seeds, cudaStream_t st) {
    failure = {};
    pend.reset();
    if (R < 1) throw ConfigError("cp_als: rank must be >= 1");
    if (max_iters < 1) throw ConfigError("cp_als: max_iters must be >= 1");
    if (!(rel_tol > 0.0)) throw ConfigError("cp_als: rel_tol must be > 0");
    if (S < 1) throw ConfigError("cp_als: n_restarts must be >= 1");
    if ((long long)R > (long long)Q * Q)
        throw ConfigError("cp_als: rank " + std::to_string(R) + " exceeds solvability bound for mode 1");
    if (R > 64) throw ConfigError("octen: device CP-ALS supports rank <= 64");
    if (Q > 256) throw ConfigError("octen: device CP-ALS supports Q <= 256");
    alloc(P, S, Q, R, max_iters);
    const int NP = P * S;
    const size_t q2 = (size_t)Q * Q, q3 = q2 * Q;

    AlsDev d;
    d.P = P;
    d.S = S;
    d.Q = Q;
    d.R = R;
    d.NP = NP;
    d.max_iters = max_iters;
    d.rel_tol = rel_tol;
    d.Y = dY;
    d.normx2 = normx2.p;
    d.F = F.p;
    d.G = G.p;
    d.lam = lam.p;
    d.T = T.p;
    d.KR = KR.p;
    d.Mb = Mb.p;
    d.Vinv = Vinv.p;
    mcount.reserve(NP);
    d.mcount = mcount.p;
    d.fit_hist = fit_hist.p;
    d.res_hist = res_hist.p;
    d.state = state.p;
    d.err = err.p;
    d.rngs = rngs.p;
    d.rescue_seed = rescue_seed.p;
    d.Fd = nullptr;
    d.Fcs = nullptr;
    d.oz_G = 0;
    d.Gev = Gev.p;
    d.EV = EV.p;
    d.Ur = Ur.p;
    d.Wmix = Wmix.p;
    d.Smix = Smix.p;
    d.Tmp6 = Tmp6.p;
    d.Pm = Pm.p;
    d.Hh = Hh.p;
    eigdbg.reserve(4);
    eigdbg.zero(4, st);
    d.eigdbg = eigdbg.p;
    static const bool want_tsc = std::getenv("OCTEN_DEBUG_ALS_TSC") != nullptr;
    if (want_tsc) {
        tscbuf.reserve(64);
        tscbuf.zero(64, st);
    }
    d.tsc = want_tsc ? reinterpret_cast<long long*>(tscbuf.p) : nullptr;
    d.gscr = gscr.p;
    d.usable = usable.p;
    d.att_start = att_start.p;
    d.att_used = att_used.p;
    d.todo = todo.p;
    d.peel_fail = peel_fail.p;
    host_syncs = 0;

    // ---- norms; the zero-tensor check (cp_als.cpp:255-256) reads them with
    // the results at the end (no host round trip here: a zero summary only
    // produces garbage in buffers this run owns, and its error takes
    // precedence over any later one)
    OCTEN_PROF("begin", st);
    ws.reserve((size_t)P * 64);
    als_norm_kernel<<<dim3(64, P), 256, 0, st>>>(d, ws.p); OCTEN_LAUNCHED(1);
    als_norm_finish_kernel<<<(P + 127) / 128, 128, 0, st>>>(d, ws.p, 64); OCTEN_LAUNCHED(1);
    OCTEN_CUDA(cudaGetLastError());

    // ---- host RNG: restart seeds, GEVD mixtures, rescue seeds (drawn ahead
    // by prefetch_host_draws when the caller knew the seeds)
    AlsHostDraws draws;
    if (next_draws.valid()) {
        AlsHostDraws nd = next_draws.get();
        if (nd.seeds == seeds && nd.S == S && nd.Q == Q) draws = std::move(nd);
    }
    if (draws.seeds.empty()) draws = als_host_draws(seeds, S, Q);
    const std::vector<std::uint64_t>& restart_seed = draws.restart_seed;
    const std::vector<std::uint64_t>& hres = draws.hres;
    const std::vector<double>& hw = draws.hw;
    Wmix.reserve(hw.size());
    h2d_param(Wmix.p, hw.data(), hw.size() * sizeof(double), st);
    rescue_seed.reserve(NP);
    h2d_param(rescue_seed.p, hres.data(), NP * sizeof(std::uint64_t), st);

    // ---- GEVD init (usable when Q >= R and Q >= 2; cp_als.cpp:64)
    std::vector<int> used(NP, -1);
    const bool shape_ok = (Q >= R) && (Q >= 2);
    if (shape_ok) {
        std::vector<int> ones(P, 1);
        usable.reserve(P);
        h2d_param(usable.p, ones.data(), P * sizeof(int), st);
        const int ks = pick_ksplit(P, Q, Q, (int)q2);
        ws.reserve((size_t)P * ks * q2);
        const bool gpipe = (Q % 2 == 0) && ((uintptr_t)dY % 16 == 0);
        if (gpipe) {
            gemm_f64_pipe<false, Y0PA, Y0PB, GevStore, false>(P, Q, Q, (int)q2, Y0PA{dY, q3, Q}, Y0PB{dY, q3, Q},
                                                              GevStore{Gev.p, Q, 0}, st, ks, ws.p);
            gemm_f64_pipe<true>(P, Q, Q, (int)q2, Y1PA{dY, q3, Q}, Y1PB{dY, q3, Q}, GevStore{Gev.p, Q, 1}, st, ks,
                                ws.p);
        } else {
            gemm_f64<false, false>(P, Q, Q, (int)q2, Y0A{dY, q3, Q}, Y0B{dY, q3, Q}, GevStore{Gev.p, Q, 0}, st, ks,
                                   ws.p);
            gemm_f64<true, true>(P, Q, Q, (int)q2, Y1A{dY, q3, Q}, Y1B{dY, q3, Q}, GevStore{Gev.p, Q, 1}, st, ks,
                                 ws.p);
        }
        size_t smem_eig = (q2 + 2 * (Q + 2) + 1024 / 32 + 4) * sizeof(double) + (2 * Q + 16) * sizeof(int) + 64;
        const int v_in_smem = (smem_eig + q2 * sizeof(double) <= 220 * 1024) ? 1 : 0;
        if (v_in_smem) smem_eig += q2 * sizeof(double);
        // subspace iteration for the top-R block when the matrix is large
        // enough for it to pay and its scratch fits the V region
        const int mblk = std::min(Q, R + 4);
        // Q <= 64: the dense top-R solve (sym_eig_top_tridiag, 0.9 ms at Q = 64)
        // beats a subspace attempt that may have to give up on a gapless
        // spectrum first (c4: 1.3 ms); at larger Q subspace iteration wins
        // when there is a gap (c3 0.59 vs 1.45 ms, c5 1.28 vs 3.3 ms)
        static const bool force_dense = std::getenv("OCTEN_EIG_DENSE") != nullptr;  // diagnostics
        const int use_sub =
            (!force_dense && Q > 64 && Q >= 2 * mblk && (size_t)2 * Q * mblk + 2 * mblk * mblk + mblk <= q2) ? mblk : 0;
        OCTEN_CUDA(cudaFuncSetAttribute(gevd_eig_sym_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_eig));
        OCTEN_PROF("grams", st);
        gevd_eig_sym_kernel<<<P * 2, 256, smem_eig, st>>>(d, v_in_smem, use_sub); OCTEN_LAUNCHED(1);
        OCTEN_CUDA(cudaGetLastError());
        OCTEN_PROF("eig", st);
        // mixtures -> p1/p2 for all attempts
        if (S <= 4) {
            const size_t smem_mix = (size_t)S * 6 * Q * sizeof(double);
            if (smem_mix > 48 * 1024)
                OCTEN_CUDA(cudaFuncSetAttribute(gevd_mix_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                (int)smem_mix));
            gevd_mix_kernel<<<dim3((unsigned)((q2 + 255) / 256), P), 256, smem_mix, st>>>(d);
            OCTEN_LAUNCHED(1);
        } else {
            gemm_f64<false, true>(NP, (int)q2, 6, Q, YmatA{dY, q3, q2, S, true}, MixB{Wmix.p, Q}, MixStore{Smix.p, q2},
                                  st);
        }
        gemm_f64<false, false>(NP * 6, Q, R, Q, SmA{Smix.p, Q}, UrB{Ur.p, Q, R, S, 1},
                                                Tmp6Store{Tmp6.p, Q, R}, st);
        gemm_f64<true, false>(NP * 6, R, R, Q, UrTA{Ur.p, Q, R, S}, Tmp6B{Tmp6.p, Q, R},
                                               PmStore{Pm.p, R}, st);
        // round 0 starts from the device's usability flags (no host round
        // trip); the host learns them with the round's outcome
        std::vector<int> start(NP, 0), td(NP, 0);
        att_start.reserve(NP);
        todo.reserve(NP);
        for (int round = 0; round < 3; ++round) {
            if (round == 0) {
                gevd_round0_kernel<<<(NP + 127) / 128, 128, 0, st>>>(d); OCTEN_LAUNCHED(1);
            } else {
                bool any = false;
                for (int prob = 0; prob < NP; ++prob) any |= td[prob] != 0;
                if (!any) break;
                h2d_param(att_start.p, start.data(), NP * sizeof(int), st);
                h2d_param(todo.p, td.data(), NP * sizeof(int), st);
            }
            peel_fail.zero(NP, st);
            const size_t smem_pen = (size_t)(5 * R * R + 7 * R + 72) * sizeof(double);
            OCTEN_PROF("mix", st);
            gevd_pencil_kernel<<<NP, 128, smem_pen, st>>>(d); OCTEN_LAUNCHED(1);
            OCTEN_CUDA(cudaGetLastError());
            OCTEN_PROF("pencil", st);
            // h = a1^T Y_(0) for all restarts of a replica at once:
            // H^T (Q^2 x S R) = Y_(0)^T [a1_s...]
            if (gpipe)
                gemm_f64_pipe<true>(P, (int)q2, S * R, Q, Y0tP{dY, q3, Q}, FacP{F.p, S, Q, R, 0},
                                    HtStore{Hh.p, S, R, q2}, st);
            else
                gemm_f64<false, false>(NP, R, (int)q2, Q, A1tA{F.p, Q, R}, Y0Bp{dY, q3, Q, S}, HStore{Hh.p, R, q2},
                                       st);
            const size_t smem_h = (size_t)(3 * R * R + 2 * (R + 2) + (R + 8)) * sizeof(double) + 16;
            OCTEN_CUDA(cudaFuncSetAttribute(gevd_hsolve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_h));
            gevd_hsolve_kernel<<<NP, 256, smem_h, st>>>(d); OCTEN_LAUNCHED(1);
            OCTEN_CUDA(cudaGetLastError());
            // h2 = Vp h into the KR scratch (same size, unused before the sweeps)
            gemm_f64<false, false>(NP, R, (int)q2, R, VpA{gscr.p, R}, HrowB{Hh.p, R, q2}, HStore{KR.p, R, q2}, st);
            const int peel_threads = 128;
            const size_t smem_peel = (q2 + 2 * Q + peel_threads + 2 + Q) * sizeof(double);
            OCTEN_CUDA(cudaFuncSetAttribute(gevd_peel_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_peel));
            OCTEN_PROF("hsolve", st);
            gevd_peel_kernel<<<NP * R, peel_threads, smem_peel, st>>>(d); OCTEN_LAUNCHED(1);
            OCTEN_CUDA(cudaGetLastError());
            OCTEN_PROF("peel", st);
            std::vector<int> au(NP), pf(NP);
            {
                // one read: this round's attempts and peel flags (+ the
                // usability flags after round 0)
                const size_t nb = (size_t)NP * sizeof(int);
                if (3 * nb + P * sizeof(int) > res_cap) {
                    if (res_pin) OCTEN_CUDA(cudaFreeHost(res_pin));
                    res_cap = 2 * (3 * nb + P * sizeof(int));
                    OCTEN_CUDA(cudaHostAlloc((void**)&res_pin, res_cap, cudaHostAllocDefault));
                }
                OCTEN_CUDA(cudaMemcpyAsync(res_pin, att_used.p, nb, cudaMemcpyDeviceToHost, st));
                OCTEN_CUDA(cudaMemcpyAsync(res_pin + nb, peel_fail.p, nb, cudaMemcpyDeviceToHost, st));
                if (round == 0)
                    OCTEN_CUDA(cudaMemcpyAsync(res_pin + 2 * nb, usable.p, P * sizeof(int), cudaMemcpyDeviceToHost, st));
                OCTEN_CUDA(cudaStreamSynchronize(st));
                std::memcpy(au.data(), res_pin, nb);
                std::memcpy(pf.data(), res_pin + nb, nb);
                if (round == 0) {
                    const int* hus = reinterpret_cast<const int*>(res_pin + 2 * nb);
                    for (int prob = 0; prob < NP; ++prob) td[prob] = hus[prob / S] ? 1 : 0;
                }
            }
            ++host_syncs;
            for (int prob = 0; prob < NP; ++prob) {
                if (!td[prob]) continue;
                if (au[prob] < 0) {  // exhausted: random fallback
                    td[prob] = 0;
                    used[prob] = -1;
                } else if (pf[prob]) {  // non-finite peel: next attempt
                    start[prob] = au[prob] + 1;
                    if (start[prob] >= 3) {
                        td[prob] = 0;
                        used[prob] = -1;
                    }
                } else {
                    td[prob] = 0;
                    used[prob] = au[prob];
                }
            }
        }
    }
    // random fallback factors (cp_als.cpp:275-283)
    {
        std::vector<double> fac((size_t)3 * Q * R);
        for (int prob = 0; prob < NP; ++prob) {
            if (used[prob] >= 0) continue;
            for (int n = 0; n < 3; ++n) {
                rng::Substream rs(rng::derive(restart_seed[prob], {rng::kAlsFactor, (std::uint64_t)n}));
                rs.fill_uniform(fac.data() + (size_t)n * Q * R, Q, R, Q);
            }
            OCTEN_CUDA(cudaMemcpyAsync(F.p + (size_t)prob * 3 * Q * R, fac.data(), fac.size() * sizeof(double),
                                       cudaMemcpyHostToDevice, st));
            OCTEN_CUDA(cudaStreamSynchronize(st));
        }
    }
    als_init_state_kernel<<<NP, 128, 0, st>>>(d); OCTEN_LAUNCHED(1);
    OCTEN_CUDA(cudaGetLastError());
    OCTEN_PROF("init", st);
    pend = std::make_shared<AlsPending>(AlsPending{d, P, S, Q, R, max_iters, rel_tol, dY, used});
}

// The sweeps of the run prepared by run_init (on `st`, which must be ordered
// after run_init's stream), best restart selection and the results.
void AlsEngine::run_sweeps(cudaStream_t st) {
    if (!pend) throw ConfigError("octen: CP-ALS sweeps without an initialised run");
    const AlsPending pd = *static_cast<const AlsPending*>(pend.get());
    pend.reset();
    AlsDev d = pd.d;
    const int P = pd.P, S = pd.S, Q = pd.Q, R = pd.R, max_iters = pd.max_iters;
    const double rel_tol = pd.rel_tol;
    const double* dY = pd.dY;
    (void)rel_tol;
    const int NP = P * S;
    const size_t q2 = (size_t)Q * Q, q3 = q2 * Q;

    // ---- sweeps
    const int SR = S * R;
    static const bool use_pdl = std::getenv("OCTEN_NO_PDL") == nullptr;
    const unsigned qinv = (unsigned)((0x100000000ull + (unsigned)Q - 1) / (unsigned)Q);
    const int upd_threads = 256;
    const size_t smem_upd = (size_t)(R * R + 2 * Q * R + R + 2 * (R + 2) + upd_threads) * sizeof(double) + 16;
    OCTEN_CUDA(cudaFuncSetAttribute(als_update_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_upd));
    const size_t smem_vinv = (size_t)(4 * R * R + 2 * (R + 2) + 256) * sizeof(double) + (R + 8) * sizeof(int) + 16;
    // 16-byte, one-round-trip contraction when Q is even and <= 128
    static const bool mk_v1 = std::getenv("OCTEN_ALS_MTTKRP_V1") != nullptr;  // diagnostics: the round-1 kernel
    const bool v2_ok = !mk_v1 && Q % 2 == 0 && Q <= 128 && ((uintptr_t)T.p % 16 == 0) && ((uintptr_t)F.p % 16 == 0);
    auto mttkrp_kernel = v2_ok ? als_mttkrp_T_kernel<0> : (Q <= 128 ? als_mttkrp_T_kernel<4> : als_mttkrp_T_kernel<8>);
    // MTTKRP + update fused in one launch unless OCTEN_ALS_NOFUSE (diagnostics)
    static const bool fuse_update = std::getenv("OCTEN_ALS_NOFUSE") == nullptr;
    const size_t smem_mk = fuse_update ? std::max(smem_vinv, smem_upd) : smem_vinv;
    OCTEN_CUDA(cudaFuncSetAttribute(mttkrp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_mk));
    mcount.reserve(NP);
    mcount.zero(NP, st);
    // 16-byte pairs along every fast index need an even Q (and aligned bases)
    const bool pipe_ok = (Q % 2 == 0) && ((uintptr_t)dY % 16 == 0) && ((uintptr_t)F.p % 16 == 0) &&
                         ((uintptr_t)KR.p % 16 == 0);

    // Up to four lanes (replica slices, each on its own stream): the
    // latency-bound per-problem kernels of one lane overlap the DMMA GEMMs of
    // the other.  Lane 1 starts half a phase late (after lane 0's first
    // T-GEMM) and the lanes run free: the convergence count of sweep s is
    // read while sweep s+1 is already queued (converged problems are masked
    // inside every kernel, so the one extra sweep is harmless).
    int L = 4;  // measured: 1 lane 14.1 ms, 2 lanes 13.5, 4 lanes 13.4 (c3 CP-ALS stage)
    if (const char* ev = std::getenv("OCTEN_ALS_LANES")) L = std::max(1, std::min(kMaxLanes, std::atoi(ev)));
    L = std::min(L, P);
    int lp0[kMaxLanes], lp1[kMaxLanes];
    for (int l = 0; l < L; ++l) {
        lp0[l] = (int)((long long)P * l / L);
        lp1[l] = (int)((long long)P * (l + 1) / L);
    }
    // With several lanes, the T-GEMMs of all lanes go through one
    // low-priority stream (so they run one at a time, in enqueue order) while
    // the latency-bound MTTKRP / update kernels stay on high-priority lane
    // streams: lane l's mode updates overlap the other lanes' GEMMs.
    // (Measured slower at c3: a lane's 4-replica GEMM alone is ~1.07 waves.
    // Off unless OCTEN_ALS_GEMM_STREAM=1.)
    // OCTEN_ALS_GEMM_STREAM=2: the same split with one low-priority GEMM
    // stream per lane, so the lanes' GEMMs still run side by side while the
    // update kernels take the SMs first when both are ready.
    static const int gsplit_env = [] {
        const char* e = std::getenv("OCTEN_ALS_GEMM_STREAM");
        return e ? std::atoi(e) : 0;
    }();
    const bool gsplit = gsplit_env >= 1 && L > 1;
    const bool gper = gsplit_env == 2;
    if (!lane_st[1]) {
        for (int l = 0; l < kMaxLanes; ++l)
            OCTEN_CUDA(cudaStreamCreateWithPriority(&lane_st[l], cudaStreamNonBlocking, critical_stream_priority()));
    }
    if (gsplit && !gemm_st) {
        int least = 0, greatest = 0;
        OCTEN_CUDA(cudaDeviceGetStreamPriorityRange(&least, &greatest));
        OCTEN_CUDA(cudaStreamCreateWithPriority(&gemm_st, cudaStreamNonBlocking, least));
        for (int l = 0; l < kMaxLanes; ++l) {
            OCTEN_CUDA(cudaStreamCreateWithPriority(&lane_hp[l], cudaStreamNonBlocking, greatest));
            OCTEN_CUDA(cudaStreamCreateWithPriority(&lane_gemm[l], cudaStreamNonBlocking, least));
        }
    }
    for (cudaEvent_t& e : lane_ev)
        if (!e) OCTEN_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    cudaStream_t ls[kMaxLanes];
    ls[0] = gsplit ? lane_hp[0] : st;
    for (int l = 1; l < L; ++l) ls[l] = gsplit ? lane_hp[l] : lane_st[l];
    if (hact_n < (size_t)max_iters * kMaxLanes) {
        if (hact) cudaFreeHost(hact);
    for (cudaEvent_t e : kev)
        if (e) cudaEventDestroy(e);
        hact = nullptr;
        hact_n = (size_t)max_iters * kMaxLanes;
        OCTEN_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&hact), hact_n * sizeof(int), cudaHostAllocMapped));
    }
    std::memset(hact, 0, (size_t)max_iters * kMaxLanes * sizeof(int));
    int* hact_dev = nullptr;
    OCTEN_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&hact_dev), hact, 0));
    AlsDev dl[kMaxLanes];
    for (int l = 0; l < L; ++l) {
        const int pb = lp0[l], pn = lp1[l] - lp0[l], qb = pb * S;
        AlsDev& x = dl[l];
        x = d;
        x.P = pn;
        x.NP = pn * S;
        x.Y = dY + (size_t)pb * q3;
        x.normx2 = normx2.p + pb;
        x.F = F.p + (size_t)qb * 3 * Q * R;
        x.G = G.p + (size_t)qb * 3 * R * R;
        x.lam = lam.p + (size_t)qb * R;
        x.T = T.p + (size_t)pb * q2 * SR;
        x.KR = KR.p + (size_t)pb * q2 * SR;
        x.Mb = Mb.p + (size_t)qb * Q * R;
        x.Vinv = Vinv.p + (size_t)qb * R * R;
        x.mcount = mcount.p + qb;
        x.fit_hist = fit_hist.p + (size_t)qb * max_iters;
        x.res_hist = res_hist.p + (size_t)qb * max_iters;
        x.state = state.p + qb;
        x.err = err.p + qb;
        x.rngs = rngs.p + qb;
        x.rescue_seed = rescue_seed.p + qb;
        x.hact = hact_dev + l;
    }
    // The T-GEMMs run on the int8 tensor cores with exact digit splitting
    // (ozaki.cu): the summaries are sliced once here, in all three
    // orientations, before the lanes fork (a normal launch, so every
    // programmatic dependent launch after it sees the slices).
    const bool use_oz = ozaki_selected(Q);
    CUtensorMap ozmap[3][kMaxLanes], ozbmap[kMaxLanes];
    if (use_oz) {
        const size_t pitch = (size_t)ozaki_pitch(Q);
        const int G = ozaki_groups(S, R);
        oz_a.reserve((size_t)3 * P * kOzSlices * q2 * pitch);
        oz_e.reserve((size_t)3 * P * q2);
        oz_fd.reserve(ozaki_fd_bytes(P, S, R));
        oz_fcs.reserve(ozaki_fcs_count(P, S, R));
        oz_fd.zero(ozaki_fd_bytes(P, S, R), st);  // (padding columns stay zero)
        ozaki_slice_y(dY, P, Q, oz_a.p, oz_e.p, st);
        ozaki_slice_factors(F.p, P, S, Q, R, oz_fd.p, oz_fcs.p, st);
        const size_t plane_bytes = ozaki_fd_bytes(1, 1, 1) / 3, plane_cols = ozaki_fcs_count(1, 1, 1) / 3;
        for (int l = 0; l < L; ++l) {
            for (int o = 0; o < 3; ++o)
                if (!ozaki_make_map(&ozmap[o][l], oz_a.p, P, Q, o, lp0[l], lp1[l] - lp0[l]))
                    throw CudaError("octen: tensor map of the CP-ALS digit slices could not be encoded");
            if (!ozaki_make_fmap(&ozbmap[l], oz_fd.p, Q, G, lp0[l], lp1[l] - lp0[l]))
                throw CudaError("octen: tensor map of the CP-ALS factor digits could not be encoded");
            AlsDev& x = dl[l];
            x.Fd = oz_fd.p + (size_t)lp0[l] * 3 * G * plane_bytes;
            x.Fcs = oz_fcs.p + (size_t)lp0[l] * 3 * G * plane_cols;
            x.oz_G = G;
        }
    }
    if (L > 1) {
        OCTEN_CUDA(cudaEventRecord(lane_ev[0], st));
        for (int l = 0; l < L; ++l)
            if (ls[l] != st) OCTEN_CUDA(cudaStreamWaitEvent(ls[l], lane_ev[0], 0));
        if (gsplit) OCTEN_CUDA(cudaStreamWaitEvent(gemm_st, lane_ev[0], 0));
        if (gsplit && gper)
            for (int l = 0; l < L; ++l) OCTEN_CUDA(cudaStreamWaitEvent(lane_gemm[l], lane_ev[0], 0));
    }
    // OCTEN_ALS_PROFILE: CUDA events between the kernels of lane 0's sweeps,
    // averaged per sweep parity and label (diagnostics)
    static const bool want_prof = std::getenv("OCTEN_ALS_PROFILE") != nullptr;
    struct ProfMark {
        int sweep;
        const char* label;
        cudaEvent_t ev;
    };
    std::vector<ProfMark> pmarks;
    if (want_prof) pmarks.reserve((size_t)max_iters * 16);
    auto mark = [&](int l, int sw, const char* label, cudaStream_t ss) {
        if (!want_prof || l != 0) return;
        ProfMark m{sw, label, nullptr};
        OCTEN_CUDA(cudaEventCreate(&m.ev));
        OCTEN_CUDA(cudaEventRecord(m.ev, ss));
        pmarks.push_back(m);
    };
    // Dimension tree over sweep pairs: consecutive mode updates that leave
    // one factor untouched share the partial contraction with it.
    //   even sweep: T = Y x3 C -> modes 0 (contract v with B), 1 (contract
    //               u with A); T = Y x2 B -> mode 2 (contract u with A)
    //   odd sweep:  the same T -> mode 0 (contract v with C); T = Y x1 A ->
    //               modes 1 (contract v with C), 2 (contract u with B)
    // 1.5 Q^3 S R GEMMs per sweep instead of 2 (or 3 without a tree).  Each
    // sweep is enqueued as two segments, each segment for every lane in turn,
    // so the GEMM stream alternates between lanes.
    krec.clear();
    // sampled: lane 0, every fifth sweep (an event between two programmatic
    // dependent launches costs the overlap PDL buys: timing every launch
    // measured +2 ms per c3 batch)
    auto ktime_on = [&](int l, int sw) { return l == 0 && sw % 5 == 2; };
    auto ktime_begin = [&](cudaStream_t ss) {
        const int i = (int)krec.size() * 2;
        while ((int)kev.size() < i + 2) {
            cudaEvent_t e;
            OCTEN_CUDA(cudaEventCreate(&e));
            kev.push_back(e);
        }
        OCTEN_CUDA(cudaEventRecord(kev[i], ss));
        return i;
    };
    auto ktime_end = [&](int i, cudaStream_t ss, bool gemm, double work) {
        OCTEN_CUDA(cudaEventRecord(kev[i + 1], ss));
        krec.push_back(KevRec{i, gemm, work});
    };
    auto launch_seg = [&](int l, int sw, int seg) {
        const AlsDev& x = dl[l];
        cudaStream_t ss = ls[l];
        const int pn = x.P, npn = x.NP;
        auto tgemm = [&](int contracted) {
            cudaStream_t gs = ss;
            bool pd = use_pdl;
            if (gsplit) {
                gs = gper ? lane_gemm[l] : gemm_st;
                OCTEN_CUDA(cudaEventRecord(lane_ev[kGin + l], ss));
                OCTEN_CUDA(cudaStreamWaitEvent(gs, lane_ev[kGin + l], 0));
                pd = false;
            }
            const bool kt_on = ktime_on(l, sw);
            const int kt0 = kt_on ? ktime_begin(gs) : -1;
            if (use_oz) {
                ozaki_tgemm(ozmap[contracted][l], ozbmap[l], oz_e.p + ((size_t)contracted * P + lp0[l]) * q2, x.Fcs,
                            x.T, pn, Q, S, R, contracted, gs, pd);
            } else if (contracted == 2) {  // rows (i, j)
                if (pipe_ok)
                    gemm_f64_pipe<false>(pn, (int)q2, SR, Q, YmatP{x.Y, q3, q2}, FacP{x.F, S, Q, R, 2},
                                         TStore{x.T, q2, SR}, gs, 1, nullptr, pd);
                else
                    gemm_f64<false, true>(pn, (int)q2, SR, Q, YmatA{x.Y, q3, q2, S, false}, FacB{x.F, S, Q, R, 2},
                                          TStore{x.T, q2, SR}, gs);
            } else if (contracted == 1) {  // rows (i, k)
                if (pipe_ok)
                    gemm_f64_pipe<false>(pn, (int)q2, SR, Q, YmidP{x.Y, q3, (unsigned)Q, qinv}, FacP{x.F, S, Q, R, 1},
                                         TStore{x.T, q2, SR}, gs, 1, nullptr, pd);
                else
                    gemm_f64<false, true>(pn, (int)q2, SR, Q, YmidA{x.Y, q3, Q}, FacB{x.F, S, Q, R, 1},
                                          TStore{x.T, q2, SR}, gs);
            } else {  // rows (j, k)
                if (pipe_ok)
                    gemm_f64_pipe<true>(pn, (int)q2, SR, Q, Y0tP{x.Y, q3, Q}, FacP{x.F, S, Q, R, 0},
                                        TStore{x.T, q2, SR}, gs, 1, nullptr, pd);
                else
                    gemm_f64<true, true>(pn, (int)q2, SR, Q, Y0tA{x.Y, q3, Q}, FacB{x.F, S, Q, R, 0},
                                         TStore{x.T, q2, SR}, gs);
            }
            if (kt_on) ktime_end(kt0, gs, true, 2.0 * (double)pn * (double)q2 * SR * Q);
            if (gsplit) {
                OCTEN_CUDA(cudaEventRecord(lane_ev[kGout + l], gs));
                OCTEN_CUDA(cudaStreamWaitEvent(ss, lane_ev[kGout + l], 0));
            }
            mark(l, sw, contracted == 2 ? "gemm Yx3C" : contracted == 1 ? "gemm Yx2B" : "gemm Yx1A", ss);
        };
        auto mode_step = [&](int contract_first, int fsrc, int mode) {
            const int fz = fuse_update ? 1 : 0;
            const bool kt_on = ktime_on(l, sw);
            const int kt1 = kt_on ? ktime_begin(ss) : -1;
            if (use_pdl) {
                launch_pdl(mttkrp_kernel, dim3(npn * (R + 1)), dim3(256), smem_mk, ss, x, contract_first, fsrc, mode,
                           sw, fz);
            } else {
                mttkrp_kernel<<<npn * (R + 1), 256, smem_mk, ss>>>(x, contract_first, fsrc, mode, sw, fz);
                OCTEN_LAUNCHED(1);
            }
            if (kt_on) ktime_end(kt1, ss, false, (double)npn * R * q2 * sizeof(double));  // T columns read (active problems at most)
            mark(l, sw, mode == 0 ? "mttkrp0" : mode == 1 ? "mttkrp1" : "mttkrp2", ss);
            if (fuse_update) return;
            if (use_pdl) {
                launch_pdl(als_update_kernel, dim3(npn), dim3(upd_threads), smem_upd, ss, x, mode, sw);
            } else {
                als_update_kernel<<<npn, upd_threads, smem_upd, ss>>>(x, mode, sw);
                OCTEN_LAUNCHED(1);
            }
            mark(l, sw, mode == 0 ? "update0" : mode == 1 ? "update1" : "update2", ss);
        };
        if (seg == 0) mark(l, sw, "start", ss);
        if ((sw & 1) == 0) {
            if (seg == 0) {
                tgemm(2);
                mode_step(0, 1, 0);
                mode_step(1, 0, 1);
            } else {
                tgemm(1);
                mode_step(1, 0, 2);
            }
        } else {
            if (seg == 0) {
                mode_step(0, 2, 0);
            } else {
                tgemm(0);
                mode_step(0, 2, 1);
                mode_step(1, 1, 2);
            }
        }
        OCTEN_CUDA(cudaGetLastError());
        if (seg == 1) OCTEN_CUDA(cudaEventRecord(lane_ev[kSweepEv + kMaxLanes * (sw & 3) + l], ss));
    };
    // The host stays `ahead` sweeps in front of the device (a ring of four
    // sweep events): the sweeps queued past the one every problem stopped in
    // find no active problem and return at once, so the results do not depend
    // on the depth.
    static const int ahead = [] {
        const char* e = std::getenv("OCTEN_ALS_LOOKAHEAD");
        return e ? std::max(1, std::min(3, std::atoi(e))) : 1;
    }();
    int sweep = 0;
    for (; sweep < max_iters; ++sweep) {
        for (int seg = 0; seg < 2; ++seg)
            for (int l = 0; l < L; ++l) launch_seg(l, sweep, seg);
        if (sweep >= ahead) {
            // problems still active after sweep `sweep - ahead`
            int left = 0;
            for (int l = 0; l < L; ++l) {
                OCTEN_CUDA(cudaEventSynchronize(lane_ev[kSweepEv + kMaxLanes * ((sweep - ahead) & 3) + l]));
                left += reinterpret_cast<volatile int*>(hact)[(size_t)(sweep - ahead) * kMaxLanes + l];
            }
            ++host_syncs;
            if (left == 0) {
                ++sweep;
                break;
            }
        }
    }
    for (int l = 0; l < L; ++l)
        if (ls[l] != st) {
            OCTEN_CUDA(cudaEventRecord(lane_ev[0], ls[l]));
            OCTEN_CUDA(cudaStreamWaitEvent(st, lane_ev[0], 0));
        }
    // best restart per replica and every result the host needs, in one
    // read (the select kernel is harmless when a failure is raised below)
    DevBuf<int> best;
    best.reserve(P);
    als_select_kernel<<<P, 256, 0, st>>>(d, Mf.p, Mlam.p, best.p); OCTEN_LAUNCHED(1);
    OCTEN_CUDA(cudaGetLastError());
    const size_t o_norm = 0, o_err = o_norm + P * sizeof(double), o_state = o_err + NP * sizeof(DevStatus),
                 o_best = o_state + NP * sizeof(AlsState), o_fh = (o_best + P * sizeof(int) + 7) & ~size_t(7),
                 o_rh = o_fh + (size_t)NP * max_iters * sizeof(double), o_end = o_rh + (size_t)NP * max_iters * sizeof(double);
    if (o_end > res_cap) {
        if (res_pin) OCTEN_CUDA(cudaFreeHost(res_pin));
        res_cap = 2 * o_end;
        OCTEN_CUDA(cudaHostAlloc((void**)&res_pin, res_cap, cudaHostAllocDefault));
    }
    OCTEN_CUDA(cudaMemcpyAsync(res_pin + o_norm, normx2.p, P * sizeof(double), cudaMemcpyDeviceToHost, st));
    OCTEN_CUDA(cudaMemcpyAsync(res_pin + o_err, err.p, NP * sizeof(DevStatus), cudaMemcpyDeviceToHost, st));
    OCTEN_CUDA(cudaMemcpyAsync(res_pin + o_state, state.p, NP * sizeof(AlsState), cudaMemcpyDeviceToHost, st));
    OCTEN_CUDA(cudaMemcpyAsync(res_pin + o_best, best.p, P * sizeof(int), cudaMemcpyDeviceToHost, st));
    OCTEN_CUDA(cudaMemcpyAsync(res_pin + o_fh, fit_hist.p, (size_t)NP * max_iters * sizeof(double),
                               cudaMemcpyDeviceToHost, st));
    OCTEN_CUDA(cudaMemcpyAsync(res_pin + o_rh, res_hist.p, (size_t)NP * max_iters * sizeof(double),
                               cudaMemcpyDeviceToHost, st));
    OCTEN_CUDA(cudaStreamSynchronize(st));
    ++host_syncs;
    last_sweeps = sweep;
    for (const KevRec& k : krec) {
        float ms = 0.f;
        OCTEN_CUDA(cudaEventElapsedTime(&ms, kev[k.ev], kev[k.ev + 1]));
        if (k.gemm) {
            kstats.gemm_ms += ms;
            kstats.gemm_flops += k.work;
            ++kstats.gemm_launches;
        } else {
            kstats.mttkrp_ms += ms;
            kstats.mttkrp_bytes += k.work;
            ++kstats.mttkrp_launches;
        }
    }
    kstats.sweeps += sweep;
    if (want_prof) {
        // duration of each label = time since the previous mark (any sweep)
        std::vector<std::string> lab[2];
        std::vector<double> acc[2];
        int cnt[2] = {0, 0};
        int last_sw = -1;
        for (size_t i = 1; i < pmarks.size(); ++i) {
            const int e = pmarks[i].sweep & 1;
            if (pmarks[i].sweep != last_sw && std::string(pmarks[i].label) == "start") ++cnt[pmarks[i].sweep & 1];
            last_sw = pmarks[i].sweep;
            float ms = 0.f;
            OCTEN_CUDA(cudaEventElapsedTime(&ms, pmarks[i - 1].ev, pmarks[i].ev));
            const std::string key = std::string(pmarks[i].label) == "start" ? "gap" : pmarks[i].label;
            size_t k = 0;
            while (k < lab[e].size() && lab[e][k] != key) ++k;
            if (k == lab[e].size()) {
                lab[e].push_back(key);
                acc[e].push_back(0.0);
            }
            acc[e][k] += ms;
        }
        cnt[0] += 1;  // sweep 0's start mark is the first mark
        for (int e = 0; e < 2; ++e) {
            std::fprintf(stderr, "octen als lane0 (L=%d, %d sweeps) %s sweeps, us:", L, sweep, e ? "odd" : "even");
            for (size_t k = 0; k < lab[e].size(); ++k)
                std::fprintf(stderr, " %s %.1f", lab[e][k].c_str(), cnt[e] ? acc[e][k] * 1e3 / cnt[e] : 0.0);
            std::fprintf(stderr, "\n");
        }
        for (ProfMark& m : pmarks) cudaEventDestroy(m.ev);
    }
    if (d.tsc) {
        std::vector<double> raw = tscbuf.to_host(64, st);
        const long long* t = reinterpret_cast<const long long*>(raw.data());
        std::fprintf(stderr, "octen als update phases (cycles from start):");
        for (int i = 1; i < 32; ++i)
            if (t[i]) std::fprintf(stderr, " [%d] %lld", i, t[i] - t[0]);
        std::fprintf(stderr, "\n");
#ifdef OCTEN_ALS_GT_STAMPS
        const long long b = t[32] ? t[32] : t[34];
        std::fprintf(stderr, "octen als mttkrp launch, problem 0 (ns from the earlier start): vinv %lld..%lld, column block 0 %lld..%lld, update %lld..%lld\n",
                     t[32] - b, t[33] - b, t[34] - b, t[35] - b, t[36] - b, t[37] - b);
#endif
    }
    if (std::getenv("OCTEN_DEBUG_ALS")) {
        const std::vector<int> ed = eigdbg.to_host(1, st);
        std::fprintf(stderr, "octen als: %d problems, %d sweeps, %d GEVD eigen fallbacks\n", NP, sweep, ed[0]);
    }

    // ---- errors: a zero input first (cp_als.cpp:255-256), then the lowest
    // replica, then restart
    {
        const double* hn = reinterpret_cast<const double*>(res_pin + o_norm);
        for (int p = 0; p < P; ++p)
            if (hn[p] == 0.0) {
                failure = {1, 0, 0};
                throw NumericError(als_failure_message(1, 0, 0));
            }
    }
    const DevStatus* he = reinterpret_cast<const DevStatus*>(res_pin + o_err);
    const AlsState* hs = reinterpret_cast<const AlsState*>(res_pin + o_state);
    for (int prob = 0; prob < NP; ++prob) {
        if (!hs[prob].failed) continue;
        const DevStatus& e = he[prob];
        if (e.code == kAlsNonFiniteFactor) {
            failure = {2, e.a, e.b};
            throw NumericError(als_failure_message(2, e.a, e.b));
        }
        if (e.code == kAlsNonFiniteFit) {
            failure = {3, e.a, 0};
            throw NumericError(als_failure_message(3, e.a, 0));
        }
    }
    OCTEN_PROF("sweeps+select", st);
    EvProf::get().report("als");
    const int* hb = reinterpret_cast<const int*>(res_pin + o_best);
    const double* fh = reinterpret_cast<const double*>(res_pin + o_fh);
    const double* rh = reinterpret_cast<const double*>(res_pin + o_rh);
    results.assign(P, AlsReplicaResult{});
    for (int p = 0; p < P; ++p) {
        const int prob = p * S + hb[p];
        AlsReplicaResult& r = results[p];
        r.restart = hb[p];
        r.iterations = hs[prob].iterations;
        r.rescued = hs[prob].rescued != 0;
        r.gevd_attempt = pd.used[prob];
        r.fit_history.assign(fh + (size_t)prob * max_iters, fh + (size_t)prob * max_iters + r.iterations);
        r.residual_history.assign(rh + (size_t)prob * max_iters, rh + (size_t)prob * max_iters + r.iterations);
        r.fit = r.fit_history.empty() ? -INFINITY : r.fit_history.back();
    }
}


// One T-GEMM of the dimension tree (the partial MTTKRP contraction
// T = Y x_mode F of every restart), on the engine the sweeps use (engine 1:
// int8 tcgen05 digit split, ozaki.cu) or the DMMA GEMM (engine 0), for the
// kernel-level parity tests.  Device pointers: Y P x Q^3, F P x S x 3 x Q x R,
// T P x Q^2 x S R (T[p][m + Q^2 n], n = s R + r).
void als_tgemm(int P, int Q, int S, int R, int mode, const double* Y, const double* F, double* T, int engine,
               cudaStream_t st) {
    if (mode < 0 || mode > 2 || P < 1 || Q < 1 || S < 1 || R < 1) throw ConfigError("als_tgemm: bad shape");
    const size_t q2 = (size_t)Q * Q, q3 = q2 * Q;
    const int SR = S * R;
    if (engine == 1) {
        if (!ozaki_supported(Q)) throw ConfigError("als_tgemm: the tcgen05 digit-split GEMM needs Q <= 128 on sm_100");
        DevBuf<std::uint8_t> a, fd;
        DevBuf<int> e;
        DevBuf<double> fcs;
        a.reserve((size_t)3 * P * kOzSlices * q2 * ozaki_pitch(Q));
        e.reserve((size_t)3 * P * q2);
        fd.reserve(ozaki_fd_bytes(P, S, R));
        fcs.reserve(ozaki_fcs_count(P, S, R));
        fd.zero(ozaki_fd_bytes(P, S, R), st);
        ozaki_slice_y(Y, P, Q, a.p, e.p, st);
        ozaki_slice_factors(F, P, S, Q, R, fd.p, fcs.p, st);
        CUtensorMap map, fmap;
        if (!ozaki_make_map(&map, a.p, P, Q, mode, 0, P) || !ozaki_make_fmap(&fmap, fd.p, Q, ozaki_groups(S, R), 0, P))
            throw CudaError("als_tgemm: tensor map");
        ozaki_tgemm(map, fmap, e.p + (size_t)mode * P * q2, fcs.p, T, P, Q, S, R, mode, st, false);
        OCTEN_CUDA(cudaStreamSynchronize(st));
        return;
    }
    const unsigned qinv = (unsigned)((0x100000000ull + Q - 1) / Q);
    if (mode == 2)
        gemm_f64<false, true>(P, (int)q2, SR, Q, YmatA{Y, q3, q2, S, false}, FacB{F, S, Q, R, 2}, TStore{T, q2, SR}, st);
    else if (mode == 1)
        gemm_f64_pipe<false>(P, (int)q2, SR, Q, YmidP{Y, q3, (unsigned)Q, qinv}, FacP{F, S, Q, R, 1},
                             TStore{T, q2, SR}, st, 1, nullptr, false);
    else
        gemm_f64<true, true>(P, (int)q2, SR, Q, Y0tA{Y, q3, Q}, FacB{F, S, Q, R, 0}, TStore{T, q2, SR}, st);
    OCTEN_CUDA(cudaStreamSynchronize(st));
}

}  // namespace octen
