// CP-ALS partial contractions T = Y x_n F in fp64 on the int8 tensor cores
// (tcgen05 kind::i8, sm_100a) by exact digit splitting (Ozaki scheme).
//
// The fp64 products of cp_als.cpp:296-303 (MTTKRP = Y_(n) KR(others), here
// the dimension-tree partial T of als.cu) are formed as
//     A(m, k) = 2^ea(m) sum_i a_i(m, k) 2^(2 - 8 i),  F(k, n) = 2^eb(n) sum_j b_j(k, n) 2^(2 - 8 j)
// with balanced signed byte digits a_i, b_j in [-128, 127], i, j = 1..7:
// the digits hold rint(x 2^(54 - e)) exactly, 54 bits of each row's
// (column's) largest value (fp64 has 53), and every digit product is summed
// in int32 with no rounding at all.  The pairs with i + j <= 9 are kept (the
// first dropped diagonal weighs 2^-76 of the scale product, per K term); the
// int32 sums of each diagonal d = i + j are combined in fp64 in the epilogue.
// Error per dot product: a few units of 2^-54 of (max|a| sum|b| + sum|a| max|b|).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

namespace octen {

constexpr int kOzSlices = 7;

// Shapes the kernel covers (Q <= 128: one 128-byte K row; any S R).
bool ozaki_supported(int Q);
// Whether the CP-ALS sweeps use it (supported, unless OCTEN_ALS_TGEMM=dmma).
bool ozaki_selected(int Q);
// Bytes of one row of the sliced operand (Q rounded up to 16).
int ozaki_pitch(int Q);
// Slice all three orientations of the P summaries Y (P x Q^3, first index
// fastest): As[o][p][slice][m][pitch] (int8 / uint8 digits), Ea[o][p][m]
// (row exponents).  Orientation o is the contracted mode:
//   o = 2: A(i + Q j, k) = Y(i, j, k);  o = 1: A(i + Q k, j);  o = 0: A(j + Q k, i).
void ozaki_slice_y(const double* Y, int P, int Q, uint8_t* As, int* Ea, cudaStream_t st);
// Tensor map over the sliced operand of orientation o for replicas
// [p0, p0 + pn) of a P-replica slicing.
bool ozaki_make_map(CUtensorMap* map, const uint8_t* As, int P, int Q, int o, int p0, int pn);
// Factor digits (the T-GEMM's B operand, ozaki_digits.cuh layout): 64-column
// groups per replica, their buffer sizes, the slicing of whole factor sets
// F (P S problems x 3 modes x Q x R) and the tensor map over replicas
// [p0, p0 + pn).
int ozaki_groups(int S, int R);
size_t ozaki_fd_bytes(int P, int S, int R);
size_t ozaki_fcs_count(int P, int S, int R);
void ozaki_slice_factors(const double* F, int P, int S, int Q, int R, uint8_t* Fd, double* Fcs, cudaStream_t st);
bool ozaki_make_fmap(CUtensorMap* map, const uint8_t* Fd, int Q, int G, int p0, int pn);
// T[p][m + Q^2 n] = sum_k A_o(p; m, k) F(p; k, n), n = s R + r over the S
// restarts, with F of mode o given by its digits (bmap, Fcs_lane: the lane's
// first replica).  Ea_lane / T point at the lane's first replica.
void ozaki_tgemm(const CUtensorMap& amap, const CUtensorMap& bmap, const int* Ea_lane, const double* Fcs_lane,
                 double* T, int pn, int Q, int S, int R, int mode, cudaStream_t st, bool pdl);

}  // namespace octen
