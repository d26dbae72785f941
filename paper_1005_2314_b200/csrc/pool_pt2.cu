// Pool-kernel instantiations for pass type 2 (rotation + stride_transpose).
// rotation passes are ping-pong only (measurement variants may set the
// in-place knobs for the wallace4 pass types)
#undef WB_INPLACE_F32
#undef WB_INPLACE_F64
#include "wallace_pool.cuh"

namespace wb {
template <>
cudaError_t launch_pool_pt<2>(int dtype, int log2n, const FillArgs& a, uint64_t n_pools, cudaStream_t s) {
  return dtype == 0 ? launch_pool_dispatch<float, 2>(log2n, a, n_pools, s)
                    : launch_pool_dispatch<double, 2>(log2n, a, n_pools, s);
}
}  // namespace wb
