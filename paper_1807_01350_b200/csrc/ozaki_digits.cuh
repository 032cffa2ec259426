// Digit splitting of fp64 values for the int8 tensor-core T-GEMM (ozaki.cu),
// shared by the kernels that produce digits: the summaries' pre-slicing
// (ozaki.cu) and the CP-ALS mode update, which writes its new factor's
// digits next to the factor (als.cu).
#pragma once

#include <cstdint>

#include "ozaki.hpp"

namespace octen {
namespace oz {

constexpr int NS = kOzSlices;
constexpr int kBadExp = 0x7fffffff;  // a non-finite row / column: its outputs are NaN
constexpr int kGroupCols = 64;       // factor columns per T-GEMM CTA (two halves of 32)
constexpr int kRowBytes = 128;       // one K row of digits (Q <= 128)

// Scale exponent of a row / column with largest magnitude `mx`: mx < 2^e.
__device__ __forceinline__ int oz_exponent(double mx, bool bad) {
    if (bad) return kBadExp;
    if (mx == 0.0) return 0;
    return ilogb(mx) + 1;
}
// 2^k as a double, for k in the normal range.
__device__ __forceinline__ double pow2i(int k) { return __longlong_as_double((long long)(k + 1023) << 52); }
// The two power-of-two factors whose product is 2^(54 - e) (each in range
// for any finite e, so x s1 s2 is an exact scaling).
__device__ __forceinline__ void oz_scales(int e, double& s1, double& s2) {
    const int k = 54 - e, h = k / 2;
    s1 = pow2i(h);
    s2 = pow2i(k - h);
}
// Balanced signed base-256 digits of N = rint(x 2^(54 - e)), |x| < 2^e so
// |N| <= 2^54: N = sum_i d_i 256^(7 - i), every d_i in [-128, 127] (the top
// one in [-65, 65]), i.e. y = x 2^-e = sum_i d_i 2^(2 - 8 i) up to half a
// unit of 2^-54 (round to nearest: no bias).  With M = N + 128 (1 + 256 +
// ... + 256^5) the low six bytes of M are d_i + 128 and M >> 48 is the top
// digit, so byte 7 - i of M ^ 0x808080808080 is d_i (two's complement): one
// exact scaling, one rounding conversion, two integer operations.
__device__ __forceinline__ unsigned long long oz_digits(double x, double s1, double s2) {
    const long long n = __double2ll_rn(x * s1 * s2);
    return (unsigned long long)(n + 0x808080808080LL) ^ 0x808080808080ULL;
}

// Factor digits for the T-GEMM's B operand, laid out for its TMA: per
// (lane-local replica p, mode, 64-column group g) a plane of 2 halves x NS
// slices x 32 rows of kRowBytes bytes (row = column n of the group, byte k =
// digit of F(k, n)); the column scale 2^e goes to Fcs[plane * 64 + n % 64].
// Column n = s R + r of replica p is column r of problem p S + s.
__host__ __device__ __forceinline__ size_t factor_plane(int p, int mode, int g, int G) {
    return ((size_t)p * 3 + mode) * G + g;
}
// One warp converts column r (Q values at col[q], q < Q) of problem `prob`'s
// factor of `mode`.
__device__ __forceinline__ void factor_column_digits(uint8_t* Fd, double* Fcs, int G, int S, int R, int Q, int prob,
                                                     int mode, int r, const double* col, int lane) {
    const int p = prob / S, n = (prob % S) * R + r;
    const size_t plane = factor_plane(p, mode, n / kGroupCols, G);
    const int c = n % kGroupCols;
    double v[4];
    double mx = 0.0;
    bool bad = false;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        const int k = lane + 32 * u;
        v[u] = k < Q ? col[k] : 0.0;
        bad |= !isfinite(v[u]);
        mx = fmax(mx, fabs(v[u]));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    bad = __any_sync(0xffffffffu, bad);
    const int e = oz_exponent(mx, bad);
    if (lane == 0) Fcs[plane * kGroupCols + c] = e == kBadExp ? __longlong_as_double(0x7ff8000000000000LL) : ldexp(1.0, e);
    double c1 = 0.0, c2 = 0.0;
    if (e != kBadExp) oz_scales(e, c1, c2);
    uint8_t* row = Fd + (plane * 2 * NS * 32 + (size_t)(c >> 5) * NS * 32 + (c & 31)) * kRowBytes;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        const int k = lane + 32 * u;
        if (k < Q) {
            const unsigned long long dg = e != kBadExp ? oz_digits(v[u], c1, c2) : 0ull;
#pragma unroll
            for (int i = 0; i < NS; ++i) row[(size_t)i * 32 * kRowBytes + k] = (uint8_t)(dg >> (8 * (NS - 1 - i)));
        }
    }
}

}  // namespace oz
}  // namespace octen
