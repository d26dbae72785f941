// Which write pattern reaches the HBM store peak? 16 GiB per launch, best of 8.
//  gridstride : persistent grid-stride float4 stores
//  blocked<U> : torch-style, one short block per 256*U float4 chunk, U stores per thread
//  pools<C>   : pool_kernel's pattern: one CTA per 1 MiB pool row, 16 KiB per
//               "emission", C CTAs per SM (occupancy pinned with dynamic smem)
// Measurement helper; not product code.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void gridstride(float4* out, size_t n4, float v) {
  const size_t stride = size_t(gridDim.x) * blockDim.x;
  for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n4; i += stride)
    __stcs(out + i, make_float4(v, v + 1, v + 2, v + 3));
}
template <int U>
__global__ void blocked(float4* out, float v) {
  float4* p = out + size_t(blockIdx.x) * 256 * U + threadIdx.x;
#pragma unroll
  for (int i = 0; i < U; ++i) __stcs(p + i * 256, make_float4(v, v + i, v + 2, v + 3));
}
// 128 threads; pool row = 65536 float4; emission = 1024 float4 (16 KiB)
__global__ void pools(float4* out, float v, int spin) {
  extern __shared__ float sm[];
  float4* row = out + size_t(blockIdx.x) * 65536;
  float x = v + threadIdx.x;
  for (int e = 0; e < 64; ++e) {
    for (int k = 0; k < spin; ++k) x = x * 1.0001f + 0.5f;  // stand-in for the passes
    if (threadIdx.x == 0) sm[0] = x;
    float4* p = row + e * 1024 + threadIdx.x;
#pragma unroll
    for (int i = 0; i < 8; ++i) __stcs(p + i * 128, make_float4(x, x + i, x + 2, x + 3));
  }
}

int main() {
  const size_t bytes = size_t(16) << 30, n4 = bytes / 16;
  float4* out;
  if (cudaMalloc(&out, bytes) != cudaSuccess) return 1;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute(pools, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(pools, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto run = [&](const char* name, auto launch) {
    float best = 1e30f;
    for (int it = 0; it < 8; ++it) {
      cudaEventRecord(a);
      launch(it);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (ms < best) best = ms;
    }
    cudaError_t e = cudaGetLastError();
    printf("{\"pattern\": \"%s\", \"gbs\": %.1f, \"ms\": %.4f, \"err\": \"%s\"}\n", name,
           bytes / (best * 1e-3) / 1e9, best, cudaGetErrorString(e));
  };
  run("gridstride x16", [&](int it) { gridstride<<<sms * 16, 256>>>(out, n4, it); });
  run("blocked U=4", [&](int it) { blocked<4><<<n4 / 1024, 256>>>(out, it); });
  run("blocked U=8", [&](int it) { blocked<8><<<n4 / 2048, 256>>>(out, it); });
  run("blocked U=16", [&](int it) { blocked<16><<<n4 / 4096, 256>>>(out, it); });
  for (int c : {4, 6, 8, 12, 16})
    for (int spin : {0, 64}) {
      char nm[64];
      snprintf(nm, sizeof nm, "pools %d/SM spin %d", c, spin);
      const int smem = (220 * 1024) / c - 1024;
      run(nm, [&](int it) { pools<<<16384, 128, smem>>>(out, it, spin); });
    }
  return 0;
}
