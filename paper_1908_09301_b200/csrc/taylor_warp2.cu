// Warp kernel, two columns per lane (32 < Lf + 4 <= 64; W up to 34 digits).
// See taylor_warp_impl.cuh for the algorithm.
#include "taylor_warp_impl.cuh"

namespace mpt {
const void* warp_fn_mc2(const Params& p) { return wp::warp_fn_mc<2>(p); }
}  // namespace mpt
