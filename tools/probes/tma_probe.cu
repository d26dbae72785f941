// Probe: which way of passing a CUtensorMap works for a 2-D TMA store on this
// driver (measurement/debug helper, not product code).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstring>
#include <vector>

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                                   CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                                   CUtensorMapFloatOOBfill);
struct Args {
  int x0;
  int pad[15];
  CUtensorMap tmap;
};

__device__ void store_box(const CUtensorMap* map, int x, int y) {
  __shared__ __align__(1024) float buf[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) buf[i] = float(i + 1000 * y);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t src = static_cast<uint32_t>(__cvta_generic_to_shared(buf));
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                     reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(src) : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
#ifndef NOWAIT
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
#endif
  }
  __syncthreads();
}
__global__ void k_load(const __grid_constant__ CUtensorMap map, int x0, float* res) {
  __shared__ __align__(1024) float buf[256];
  __shared__ __align__(8) unsigned long long bar;
  const uint32_t b = static_cast<uint32_t>(__cvta_generic_to_shared(&bar));
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], 1024;" ::"r"(b) : "memory");
    const uint32_t dst = static_cast<uint32_t>(__cvta_generic_to_shared(buf));
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                 ::"r"(dst), "l"(reinterpret_cast<uint64_t>(&map)), "r"(x0), "r"((int)blockIdx.x), "r"(b) : "memory");
  }
  uint32_t ok = 0;
  while (!ok) {
    asm volatile("{ .reg .pred P1; mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], 0; selp.b32 %0, 1, 0, P1; }"
                 : "=r"(ok) : "r"(b) : "memory");
  }
  if (threadIdx.x == 0) res[blockIdx.x] = buf[0];
}
__global__ void k_param(const __grid_constant__ CUtensorMap map, int x0) { store_box(&map, x0, blockIdx.x); }
__global__ void k_struct(const __grid_constant__ Args a) { store_box(&a.tmap, a.x0, blockIdx.x); }
__global__ void k_global(const CUtensorMap* map, int x0) { store_box(map, x0, blockIdx.x); }

int main(int argc, char** argv) {
  const int mode = argc > 1 ? atoi(argv[1]) : 0;
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  auto enc = reinterpret_cast<EncodeTiledFn>(p);
  const int count = 4096, rows = 4;
  float* out;
  cudaMalloc(&out, count * rows * 4);
  cudaMemset(out, 0, count * rows * 4);
  CUtensorMap map;
  const cuuint64_t dims[2] = {(cuuint64_t)count, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)count * 4};
  const cuuint32_t box[2] = {256, 1}, es[2] = {1, 1};
  CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, out, dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("mode %d encode=%d\n", mode, (int)r);
  const int x0 = argc > 2 ? atoi(argv[2]) : 37;
  if (mode == 0) k_param<<<rows, 128>>>(map, x0);
  if (mode == 3) {
    float* res; cudaMalloc(&res, 64);
    cudaMemset(out, 0, count * rows * 4);
    k_load<<<rows, 128>>>(map, x0, res);
    cudaError_t e3 = cudaDeviceSynchronize();
    float hr[4]; cudaMemcpy(hr, res, 16, cudaMemcpyDeviceToHost);
    printf("load sync=%s res=%g\n", cudaGetErrorString(e3), hr[0]);
    return 0;
  }
  if (mode == 1) {
    Args a{};
    a.x0 = x0;
    a.tmap = map;
    k_struct<<<rows, 128>>>(a);
  }
  if (mode == 2) {
    CUtensorMap* d;
    cudaMalloc(&d, sizeof(map));
    cudaMemcpy(d, &map, sizeof(map), cudaMemcpyHostToDevice);
    k_global<<<rows, 128>>>(d, x0);
  }
  cudaError_t e = cudaDeviceSynchronize();
  std::vector<float> h(count * rows);
  cudaMemcpy(h.data(), out, h.size() * 4, cudaMemcpyDeviceToHost);
  printf("mode %d sync=%s out[1][36..39]=%g %g %g %g out[1][292]=%g out[1][293]=%g\n", mode, cudaGetErrorString(e),
         h[count + 36], h[count + 37], h[count + 38], h[count + 39], h[count + 292], h[count + 293]);
  return e == cudaSuccess ? 0 : 1;
}
