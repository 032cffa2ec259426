// tcgen05 split-TF32 GEMM (see tc_gemm.hpp).  Round-1 bring-up: not yet
// enabled; the SIMT path carries the contraction.
#include "tc_gemm.hpp"

namespace octen {

bool tc_gemm_f32_nt(const float*, const float*, float*, int, long long, int, cudaStream_t) { return false; }

}  // namespace octen
