// Pool-kernel instantiations for pass type 0 (wallace4 + stride_transpose).
#include "wallace_pool.cuh"

namespace wb {
template <>
cudaError_t launch_pool_pt<0>(int dtype, int log2n, const FillArgs& a, uint64_t n_pools, cudaStream_t s) {
  return dtype == 0 ? launch_pool_dispatch<float, 0>(log2n, a, n_pools, s)
                    : launch_pool_dispatch<double, 0>(log2n, a, n_pools, s);
}
}  // namespace wb
