// Store-only HBM peak on this box: 16 GiB of 128-bit stores (the output
// pattern of pool_kernel), best of 10 with CUDA events, for each store cache
// hint (default st.global / .cs streaming / .cg) and for constant vs varying
// data; plus a copy (read + write bytes, the MEASURED_PEAKS.json convention).
// Measurement helper for the roofline denominator; not product code.
#include <cstdio>
#include <cuda_runtime.h>

template <int HINT, bool VARY>
__global__ void store_kernel(float4* out, size_t n4, float v) {
  const size_t stride = size_t(gridDim.x) * blockDim.x;
  for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n4; i += stride) {
    const float x = VARY ? v + float(i & 0xffff) * 1e-3f : v;
    const float4 q = make_float4(x, x + 1, x + 2, x + 3);
    if (HINT == 0) out[i] = q;
    if (HINT == 1) __stcs(out + i, q);
    if (HINT == 2) __stcg(out + i, q);
  }
}

__global__ void copy_kernel(const float4* in, float4* out, size_t n4) {
  const size_t stride = size_t(gridDim.x) * blockDim.x;
  for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n4; i += stride)
    __stcs(out + i, __ldcs(in + i));
}

template <int HINT, bool VARY>
float best_store(float4* out, size_t n4, int sms, int* best_bps) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e30f;
  for (int blocks_per_sm : {4, 8, 16}) {
    for (int it = 0; it < 10; ++it) {
      cudaEventRecord(a);
      store_kernel<HINT, VARY><<<sms * blocks_per_sm, 256>>>(out, n4, float(it));
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (ms < best) best = ms, *best_bps = blocks_per_sm;
    }
  }
  return best;
}

int main() {
  const size_t bytes = size_t(16) << 30, n4 = bytes / 16;
  float4* out;
  if (cudaMalloc(&out, bytes) != cudaSuccess) return 1;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const char* names[3] = {"default", "cs", "cg"};
  float t[3][2];
  int bps[3][2];
  t[0][0] = best_store<0, false>(out, n4, sms, &bps[0][0]);
  t[0][1] = best_store<0, true>(out, n4, sms, &bps[0][1]);
  t[1][0] = best_store<1, false>(out, n4, sms, &bps[1][0]);
  t[1][1] = best_store<1, true>(out, n4, sms, &bps[1][1]);
  t[2][0] = best_store<2, false>(out, n4, sms, &bps[2][0]);
  t[2][1] = best_store<2, true>(out, n4, sms, &bps[2][1]);
  for (int h = 0; h < 3; ++h)
    for (int v = 0; v < 2; ++v)
      printf("{\"store\": \"%s\", \"data\": \"%s\", \"gbs\": %.1f, \"ms\": %.4f, \"blocks_per_sm\": %d}\n",
             names[h], v ? "varying" : "constant", bytes / (t[h][v] * 1e-3) / 1e9, t[h][v], bps[h][v]);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
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
