// Store-only HBM peak on this box: 16 GiB of 128-bit streaming stores (the
// output pattern of pool_kernel), best of 10 with CUDA events; and a copy
// (read + write bytes, the MEASURED_PEAKS.json convention) for comparison.
// Measurement helper for the roofline denominator; not product code.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void store_kernel(float4* out, size_t n4, float v) {
  const size_t stride = size_t(gridDim.x) * blockDim.x;
  for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n4; i += stride)
    __stcs(out + i, make_float4(v, v + 1, v + 2, v + 3));
}

__global__ void copy_kernel(const float4* in, float4* out, size_t n4) {
  const size_t stride = size_t(gridDim.x) * blockDim.x;
  for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n4; i += stride)
    __stcs(out + i, __ldcs(in + i));
}

int main() {
  const size_t bytes = size_t(16) << 30, n4 = bytes / 16;
  float4* out;
  if (cudaMalloc(&out, bytes) != cudaSuccess) return 1;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float best = 1e30f;
  for (int blocks_per_sm : {4, 8, 16}) {
    for (int it = 0; it < 10; ++it) {
      cudaEventRecord(a);
      store_kernel<<<sms * blocks_per_sm, 256>>>(out, n4, float(it));
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (ms < best) best = ms;
    }
  }
  printf("{\"store_only_gbs\": %.1f, \"bytes\": %zu, \"best_ms\": %.4f}\n", bytes / (best * 1e-3) / 1e9,
         bytes, best);
  float4* o2 = out + n4 / 2;
  float bestc = 1e30f;
  for (int it = 0; it < 10; ++it) {
    cudaEventRecord(a);
    copy_kernel<<<sms * 8, 256>>>(out, o2, n4 / 2);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < bestc) bestc = ms;
  }
  printf("{\"copy_gbs\": %.1f}\n", bytes / (bestc * 1e-3) / 1e9);
  return 0;
}
