// TEST INFRASTRUCTURE ONLY (oracle/).  The two declarations
// proj/src/streaming.cpp:111,115 call but no reference header provides
// (SURVEY F2(b)); force-included (-include) when the reference sources are
// compiled, so those sources stay byte-for-byte unmodified.  Signatures as
// defined at proj/src/recovery.cpp:321-322 and :464-465.
#pragma once
#include "cpstream/recovery.hpp"

namespace cpstream {
Matrix refine_stack(AlignedStack& aligned, const ReplicaSet& rs, const std::vector<Matrix>& nontemporal_solved);
Matrix recover_nontemporal_weighted(const Matrix& stacked_factor, const Matrix& stacked_projection, int mode, int q,
                                    const Matrix& col_weights);
}  // namespace cpstream
