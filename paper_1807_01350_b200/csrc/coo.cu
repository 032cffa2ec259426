// Sparse (COO) compression of one temporal batch into the P replica summaries.
//
// The reference ingests COO data through SparseTensor (proj/include/cpstream/
// tensor.hpp:66-90): the constructor validates every entry
// (proj/src/tensor.cpp:87-102: index out of bounds -> ConfigError, non-finite
// value -> NumericError, duplicate index -> ConfigError), and read_tensor_any
// densifies it (proj/src/io.cpp:124-132, tensor.cpp:118-122) before the dense
// compress / update_summaries (proj/src/compression.cpp:108-153).  Here the
// batch is never densified:
//
//   Y_p += sum_e v_e  U_p(i_e,:) (x) V_p(j_e,:) (x) W_p(k_e,:)
//
// which equals compress(to_dense(batch)) in exact arithmetic.  Per batch:
//
//   coo_keys_kernel   validate (bounds, finiteness), key = (k I + i) J + j
//   radix sort        (key, entry) pairs -> slice-major, then i, then j
//   coo_scan_kernel   duplicates (adjacent equal keys), slice offsets,
//                     decoded entries, count of distinct (k, i) groups
//   coo_slice_kernel  per (slice k, replica block):
//                       S_p(:,:,k) = sum_i U_p(i,:)^T r_i,  r_i = sum_{j in (k,i)} v V_p(j,:)
//                     written as the mode-1/2 output Z2 of the dense path
//   accumulate        Y_p += Z2_p (Q^2 x t) W_p (t x Q), fp64 DMMA (compress.cu)
//
// Grouping by (k, i) turns the per-entry rank-1 update of the Q x Q slice
// matrix (2 Q^2 flop per entry) into a gather-accumulate of V rows (2 Q flop
// per entry, the HBM/L2-bound part) plus one rank-1 update per distinct row i
// of the slice (2 Q^2 flop per group, the FFMA-bound part).
#include <cuda_runtime.h>

#include <cub/device/device_radix_sort.cuh>

#include <algorithm>
#include <climits>
#include <cstring>
#include <string>
#include <vector>

#include "engine.hpp"

namespace octen {

namespace {

constexpr int kChunkE = 256;  // entries staged per round of a slice CTA
constexpr int kChunkG = 48;   // distinct rows i (groups) per round

__global__ void coo_keys_kernel(const int* __restrict__ ci, const int* __restrict__ cj, const int* __restrict__ ck,
                                const float* __restrict__ cv, long long nnz, int I, int J, int t,
                                unsigned long long* __restrict__ keys, int* __restrict__ idx, CooStatus* err) {
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < nnz;
         e += (long long)gridDim.x * blockDim.x) {
        const int i = ci[e], j = cj[e], k = ck[e];
        const float v = cv[e];
        const bool ok = (unsigned)i < (unsigned)I && (unsigned)j < (unsigned)J && (unsigned)k < (unsigned)t;
        // tensor.cpp:94-98: bounds are checked before finiteness
        if (!ok)
            atomicMin(&err->bounds, (int)e);
        else if (!isfinite(v))
            atomicMin(&err->nonfinite, (int)e);
        keys[e] = ok ? ((unsigned long long)k * (unsigned)I + (unsigned)i) * (unsigned)J + (unsigned)j : 0ull;
        idx[e] = (int)e;
    }
}

// After the (stable) sort: the reference throws at the first entry, in input
// order, whose index was already seen (tensor.cpp:99-100): the smallest
// original position among the non-first members of equal-key runs.
__global__ void coo_scan_kernel(const unsigned long long* __restrict__ keys, const int* __restrict__ idx,
                                const float* __restrict__ cv, long long nnz, unsigned long long IJ, int J, int t,
                                int4* __restrict__ ent, int* __restrict__ off, CooStatus* err) {
    int groups = 0;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < nnz;
         e += (long long)gridDim.x * blockDim.x) {
        const unsigned long long key = keys[e];
        const unsigned long long kk = key / IJ;
        const unsigned long long rem = key - kk * IJ;
        const int i = (int)(rem / (unsigned)J), j = (int)(rem - (unsigned long long)i * (unsigned)J);
        long long kprev = -1;
        bool head = true;
        if (e > 0) {
            const unsigned long long prev = keys[e - 1];
            if (prev == key) atomicMin(&err->dup, idx[e]);
            kprev = (long long)(prev / IJ);
            head = prev / (unsigned)J != key / (unsigned)J;  // (k, i) changes
        }
        for (long long q = kprev + 1; q <= (long long)kk; ++q) off[q] = (int)e;
        if (e == nnz - 1)
            for (long long q = (long long)kk + 1; q <= t; ++q) off[q] = (int)nnz;
        groups += head;
        ent[e] = make_int4(i, j, __float_as_int(cv[idx[e]]), 0);
    }
    // warp-aggregated group count
    for (int o = 16; o > 0; o >>= 1) groups += __shfl_xor_sync(0xffffffffu, groups, o);
    if ((threadIdx.x & 31) == 0 && groups) atomicAdd(&err->groups, (unsigned long long)groups);
}

// One CTA per (slice k, block of RB replicas); 256 threads.  QP = Q padded
// to the tile (32, 64 or 128), TM x TM accumulators per thread.  The slice's
// entries are consumed in rounds of <= kChunkE entries / kChunkG groups:
//   phase A' Us[g][c] = U(i_g, c)            (cp.async, overlapping phase A)
//   phase A  Rs[g][c] = sum_{e in g} v_e V(j_e, c)   (float4 gathers; NS thread
//            sets each take an equal contiguous share of the round's entries;
//            partial sums of groups split across sets are added afterwards in
//            set order: fixed summation order)
//   phase B  acc += Us[g][rows]^T Rs[g][cols] over the round's groups
// A group split across two rounds is simply two groups (the sum is linear).
template <int QP, int TM>
__global__ void __launch_bounds__(256) coo_slice_kernel(const int4* __restrict__ ent, const int* __restrict__ off,
                                                        const float* __restrict__ U, const float* __restrict__ V,
                                                        int ldp, int P, int Q, long long zs,
                                                        float* __restrict__ Z2) {
    constexpr int TD = QP / TM;         // threads per tile dimension
    constexpr int TPR = TD * TD;        // threads per replica
    constexpr int RB = 256 / TPR;       // replicas per CTA
    constexpr int NC = RB * QP;         // staged columns
    constexpr int H = TM / 4;           // float4 segments per thread row/col
    constexpr int NQ = NC / 4;          // float4 column quads
    constexpr int NS = 256 / NQ;        // entry sets of phase A
    static_assert(NC == 128 || NC == 256, "tile");
    extern __shared__ __align__(16) float sm[];
    float* Rs = sm;                     // [kChunkG][NC]
    float* Us = sm + kChunkG * NC;      // [kChunkG][NC]
    __shared__ int s_j[kChunkE], s_g[kChunkE], s_gi[kChunkG], s_gs[kChunkG];
    __shared__ float s_v[kChunkE];
    __shared__ int s_wsum[8], s_nused, s_cg[8];
    __shared__ float4 s_carry[256];  // NS x NQ continuation partial sums

    const int k = blockIdx.x, p0 = blockIdx.y * RB;
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int rp = tid / TPR, tt = tid % TPR, ty = tt / TD, tx = tt % TD;
    const int sset = tid / NQ, cq = tid % NQ;
    const int cols_valid = min(RB, P - p0) * QP;
    const size_t colbase = (size_t)p0 * QP;

    float acc[TM][TM];
#pragma unroll
    for (int x = 0; x < TM; ++x)
#pragma unroll
        for (int y = 0; y < TM; ++y) acc[x][y] = 0.f;

    long long pos = off[k];
    const long long end = off[k + 1];
    while (pos < end) {
        const int n = (int)(end - pos < kChunkE ? end - pos : kChunkE);
        int head = 0, ei = 0;
        if (tid == 0) s_nused = n;
        if (tid < n) {
            const int4 en = ent[pos + tid];
            ei = en.x;
            s_j[tid] = en.y;
            s_v[tid] = __int_as_float(en.z);
            head = tid == 0 || __ldg(&ent[pos + tid - 1].x) != ei;
        }
        const unsigned b = __ballot_sync(0xffffffffu, head);
        const int incl = __popc(b & (0xffffffffu >> (31 - lane)));
        if (lane == 31) s_wsum[w] = incl;
        __syncthreads();
        int base = 0, total = 0;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const int s = s_wsum[q];
            base += q < w ? s : 0;
            total += s;
        }
        const int gid = base + incl - 1;
        if (tid < n) {
            s_g[tid] = gid;
            if (head && gid < kChunkG) {
                s_gi[gid] = ei;
                s_gs[gid] = tid;
            }
            if (head && gid == kChunkG) s_nused = tid;
        }
        __syncthreads();
        const int nused = s_nused, ng = min(total, kChunkG);

        // phase A': the U rows of the groups, 16-byte cp.async (zero-filled
        // past the last replica), in flight while phase A gathers
        for (int x = tid; x < ng * NQ; x += 256) {
            const int g = x / NQ, cq = x - g * NQ;
            const float* src = U + (size_t)s_gi[g] * ldp + colbase + 4 * cq;
            const unsigned d = (unsigned)__cvta_generic_to_shared(Us + g * NC + 4 * cq);
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(src),
                         "r"(4 * cq < cols_valid ? 16 : 0)
                         : "memory");
        }
        asm volatile("cp.async.commit_group;\n" ::: "memory");
        // phase A: thread set s accumulates the V rows (float4 column quad cq)
        // of entries [nused s / NS, nused (s+1) / NS).  A group is stored by
        // the set in which it starts; a set whose range begins inside a group
        // (a continuation) leaves that partial sum in carry[s], and the
        // carries are added in set order after the barrier -- equal work per
        // set and a fixed summation order (run-to-run deterministic)
        const int e_lo = nused * sset / NS, e_hi = nused * (sset + 1) / NS;
        const bool cont = e_lo > 0 && e_lo < e_hi && s_g[e_lo - 1] == s_g[e_lo];
        if (cq == 0) s_cg[sset] = cont ? s_g[e_lo] : -1;
        if (4 * cq < cols_valid) {
            const float* vc = V + colbase + 4 * cq;
            float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
            int gc = e_lo < e_hi ? s_g[e_lo] : 0;
            bool carry = cont;
            auto flush = [&](int g) {
                if (carry)
                    s_carry[sset * NQ + cq] = a;
                else
                    *reinterpret_cast<float4*>(Rs + gc * NC + 4 * cq) = a;
                carry = false;
                a = make_float4(0.f, 0.f, 0.f, 0.f);
                gc = g;
            };
            int e = e_lo;
            for (; e + 8 <= e_hi; e += 8) {
                float4 x[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) x[u] = __ldg(reinterpret_cast<const float4*>(vc + (size_t)s_j[e + u] * ldp));
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const int g = s_g[e + u];
                    if (g != gc) flush(g);
                    const float sv = s_v[e + u];
                    a.x = fmaf(sv, x[u].x, a.x);
                    a.y = fmaf(sv, x[u].y, a.y);
                    a.z = fmaf(sv, x[u].z, a.z);
                    a.w = fmaf(sv, x[u].w, a.w);
                }
            }
            for (; e < e_hi; ++e) {
                const float4 x = __ldg(reinterpret_cast<const float4*>(vc + (size_t)s_j[e] * ldp));
                const int g = s_g[e];
                if (g != gc) flush(g);
                const float sv = s_v[e];
                a.x = fmaf(sv, x.x, a.x);
                a.y = fmaf(sv, x.y, a.y);
                a.z = fmaf(sv, x.z, a.z);
                a.w = fmaf(sv, x.w, a.w);
            }
            if (e_lo < e_hi) flush(gc);
        }
        asm volatile("cp.async.wait_all;\n" ::: "memory");
        __syncthreads();
        // carries, in set order (the owner's store came first)
        if (sset == 0 && 4 * cq < cols_valid) {
#pragma unroll
            for (int s2 = 1; s2 < NS; ++s2) {
                const int g = s_cg[s2];
                if (g < 0) continue;
                float4* r = reinterpret_cast<float4*>(Rs + g * NC + 4 * cq);
                const float4 c = s_carry[s2 * NQ + cq];
                float4 v = *r;
                v.x += c.x;
                v.y += c.y;
                v.z += c.z;
                v.w += c.w;
                *r = v;
            }
        }
        __syncthreads();

        // phase B: rank-1 updates of the replica's Q x Q slice matrix.  Thread
        // (ty, tx) owns rows {h TD 4 + 4 ty + u} and columns {h TD 4 + 4 tx + u}
        // so a quarter-warp's float4 loads cover 128 contiguous bytes.
        const float* ub = Us + rp * QP + 4 * ty;
        const float* rb = Rs + rp * QP + 4 * tx;
#pragma unroll 2
        for (int g = 0; g < ng; ++g) {
            float av[TM], bv[TM];
#pragma unroll
            for (int h = 0; h < H; ++h) {
                const float4 a4 = *reinterpret_cast<const float4*>(ub + g * NC + h * TD * 4);
                const float4 b4 = *reinterpret_cast<const float4*>(rb + g * NC + h * TD * 4);
                av[4 * h] = a4.x, av[4 * h + 1] = a4.y, av[4 * h + 2] = a4.z, av[4 * h + 3] = a4.w;
                bv[4 * h] = b4.x, bv[4 * h + 1] = b4.y, bv[4 * h + 2] = b4.z, bv[4 * h + 3] = b4.w;
            }
#pragma unroll
            for (int x = 0; x < TM; ++x)
#pragma unroll
                for (int y = 0; y < TM; ++y) acc[x][y] = fmaf(av[x], bv[y], acc[x][y]);
        }
        __syncthreads();
        pos += nused;
    }

    const int p = p0 + rp;
    if (p >= P) return;
    float* z = Z2 + (size_t)p * zs + (size_t)Q * Q * k;
#pragma unroll
    for (int y = 0; y < TM; ++y) {
        const int bcol = (y / 4) * TD * 4 + 4 * tx + (y & 3);
        if (bcol >= Q) continue;
#pragma unroll
        for (int x = 0; x < TM; ++x) {
            const int arow = (x / 4) * TD * 4 + 4 * ty + (x & 3);
            if (arow < Q) z[arow + (size_t)Q * bcol] = acc[x][y];
        }
    }
}

template <int QP, int TM>
void launch_slices(const CooEngine& e, std::int64_t t, float* Z2, cudaStream_t st) {
    constexpr int TPR = (QP / TM) * (QP / TM);
    constexpr int RB = 256 / TPR;
    constexpr int NC = RB * QP;
    const size_t smem = (size_t)2 * kChunkG * NC * sizeof(float);
    static PerDevice attr;
    attr.once([&] {
        OCTEN_CUDA(cudaFuncSetAttribute(coo_slice_kernel<QP, TM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)smem));
    });
    dim3 grid((unsigned)t, (unsigned)((e.P + RB - 1) / RB));
    coo_slice_kernel<QP, TM><<<grid, 256, smem, st>>>(e.ent.p, e.off.p, e.U32.p, e.V32.p, e.ldp, e.P, e.Q,
                                                      (long long)e.Q * e.Q * t, Z2);
    OCTEN_LAUNCHED(1);
}

}  // namespace

CooEngine::CooEngine() {
    for (auto& ev : evs) OCTEN_CUDA(cudaEventCreate(&ev));
}

CooEngine::~CooEngine() {
    for (auto& ev : evs)
        if (ev) cudaEventDestroy(ev);
}

void CooEngine::set_projections(int P_, int Q_, std::int64_t I_, std::int64_t J_, const double* hU, const double* hV,
                                cudaStream_t st) {
    if (P_ < 1 || Q_ < 1 || I_ < 1 || J_ < 1) throw ConfigError("compress: bad sparse compression shape");
    if (Q_ > 128) throw ConfigError("octen: sparse compression supports Q <= 128");
    if (I_ > INT_MAX || J_ > INT_MAX) throw ConfigError("octen: sparse extents must fit int32");
    P = P_;
    Q = Q_;
    I = I_;
    J = J_;
    QP = Q <= 32 ? 32 : Q <= 64 ? 64 : 128;
    ldp = P * QP;
    // row-major fp32 copies, one row per index holding every replica's
    // (zero-padded) projection row: the gathers read NC contiguous floats
    auto pack = [&](const double* h, std::int64_t d, DevBuf<float>& out) {
        std::vector<float> r((size_t)d * ldp, 0.f);
        for (int p = 0; p < P; ++p)
            for (int a = 0; a < Q; ++a) {
                const double* col = h + (size_t)p * d * Q + (size_t)d * a;
                float* dst = r.data() + (size_t)p * QP + a;
                for (std::int64_t i = 0; i < d; ++i) dst[(size_t)i * ldp] = (float)col[i];
            }
        out.upload(r.data(), r.size(), st);
        OCTEN_CUDA(cudaStreamSynchronize(st));
    };
    pack(hU, I, U32);
    pack(hV, J, V32);
}

void CooEngine::compress(std::int64_t t, std::int64_t nnz, const int* di, const int* dj, const int* dk,
                         const float* dv, const double* dW, double* dY, cudaStream_t st) {
    if (t < 1) throw ConfigError("compress: temporal extent must be >= 1");
    if (nnz < 0 || nnz >= INT_MAX) throw ConfigError("octen: nnz must be in [0, 2^31 - 1)");
    if ((unsigned long long)I * (unsigned long long)J > (~0ull) / (unsigned long long)t)
        throw ConfigError("octen: sparse batch index space exceeds 64 bits");
    OCTEN_CUDA(cudaEventRecord(evs[0], st));
    err.reserve(1);
    CooStatus init{INT_MAX, INT_MAX, INT_MAX, 0, 0ull};
    OCTEN_CUDA(cudaMemcpyAsync(err.p, &init, sizeof(init), cudaMemcpyHostToDevice, st));
    off.reserve((size_t)t + 1);
    OCTEN_CUDA(cudaMemsetAsync(off.p, 0, ((size_t)t + 1) * sizeof(int), st));
    if (nnz > 0) {
        // grow with headroom: batches differ slightly in nnz, and a fresh
        // pool allocation per batch would cost more than the batch
        const size_t cap = keys.n >= (size_t)nnz ? keys.n : (size_t)nnz + (size_t)nnz / 4;
        keys.reserve(cap);
        keys2.reserve(cap);
        idx.reserve(cap);
        idx2.reserve(cap);
        ent.reserve(cap);
        const int blocks = (int)std::min<long long>((nnz + 255) / 256, 148 * 16);
        coo_keys_kernel<<<blocks, 256, 0, st>>>(di, dj, dk, dv, nnz, (int)I, (int)J, (int)t, keys.p, idx.p, err.p);
        OCTEN_LAUNCHED(1);
        const unsigned long long maxkey = (unsigned long long)I * J * t - 1;
        int end_bit = 1;
        while (end_bit < 64 && (maxkey >> end_bit)) ++end_bit;
        size_t tmp_bytes = 0;
        OCTEN_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, keys.p, keys2.p, idx.p, idx2.p, (int)nnz, 0,
                                                   end_bit, st));
        sort_tmp.reserve(tmp_bytes);
        OCTEN_CUDA(cub::DeviceRadixSort::SortPairs(sort_tmp.p, tmp_bytes, keys.p, keys2.p, idx.p, idx2.p, (int)nnz,
                                                   0, end_bit, st));
        OCTEN_LAUNCHED(2 * ((end_bit + 7) / 8) + 2);  // CUB onesweep: histogram + one pass per digit (estimate)
        coo_scan_kernel<<<blocks, 256, 0, st>>>(keys2.p, idx2.p, dv, nnz, (unsigned long long)I * J, (int)J, (int)t,
                                                ent.p, off.p, err.p);
        OCTEN_LAUNCHED(1);
    }
    CooStatus hs;
    OCTEN_CUDA(cudaMemcpyAsync(&hs, err.p, sizeof(hs), cudaMemcpyDeviceToHost, st));
    OCTEN_CUDA(cudaStreamSynchronize(st));
    // the first offending entry in input order wins; on the same entry the
    // bounds check precedes the finiteness check (tensor.cpp:91-100)
    const int first = std::min(hs.bounds, std::min(hs.nonfinite, hs.dup));
    if (first != INT_MAX) {
        if (hs.bounds == first) throw ConfigError("SparseTensor: index out of bounds");
        if (hs.nonfinite == first) throw NumericError("SparseTensor: non-finite value");
        throw ConfigError("SparseTensor: duplicate index");
    }
    groups_total += (double)hs.groups;
    nnz_total += (double)nnz;
    Z2.reserve((size_t)P * Q * Q * t);
    OCTEN_CUDA(cudaEventRecord(evs[1], st));
    if (QP == 32)
        launch_slices<32, 4>(*this, t, Z2.p, st);
    else if (QP == 64)
        launch_slices<64, 8>(*this, t, Z2.p, st);
    else
        launch_slices<128, 8>(*this, t, Z2.p, st);
    OCTEN_CUDA(cudaEventRecord(evs[2], st));
    accumulate_z2_f32(P, Q, t, Z2.p, dW, dY, st);
    OCTEN_CUDA(cudaEventRecord(evs[3], st));
    OCTEN_CUDA(cudaGetLastError());
    pending = true;
}

void CooEngine::collect(cudaStream_t st) {
    if (!pending) return;
    OCTEN_CUDA(cudaStreamSynchronize(st));
    float a = 0.f, b = 0.f, c = 0.f;
    OCTEN_CUDA(cudaEventElapsedTime(&a, evs[0], evs[1]));
    OCTEN_CUDA(cudaEventElapsedTime(&b, evs[1], evs[2]));
    OCTEN_CUDA(cudaEventElapsedTime(&c, evs[2], evs[3]));
    ms_prep += a;
    ms_slice += b;
    ms_accum += c;
    ++batches;
    pending = false;
}

}  // namespace octen
