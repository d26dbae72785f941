// Timing probe: one-thread sequential Neumaier (neumaier_sq, both forms) vs
// the warp-parallel neumaier_warp over a 1024-element fp32 pool in shared
// memory; cycles per call and bit-equality of the results.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -I../../paper_1005_2314_b200/csrc neum_probe.cu -o neum_probe
#include <cstdio>
#include "wallace_pool.cuh"
using namespace wb;

__global__ void probe(const float* in, double* out, long long* cyc) {
  __shared__ __align__(16) float pool[1024];
  __shared__ __align__(16) double scr[288];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) pool[i] = in[i];
  __syncthreads();
  long long t0 = clock64();
  double a = 0, b = 0, c = 0;
  if (threadIdx.x == 0) a = neumaier_sq<float, true>(pool, 1024);
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) b = neumaier_sq<float, false>(pool, 1024);
  __syncthreads();
  long long t2 = clock64();
  if (threadIdx.x < 32) c = neumaier_warp<float, 1024>(pool, scr, threadIdx.x);
  __syncthreads();
  long long t3 = clock64();
  long long t4 = clock64();
  double d = a;
  if (threadIdx.x == 0) {
#pragma unroll 64
    for (int i = 0; i < 1024; ++i) d = __dadd_rn(d, scr[i & 7]);
  }
  __syncthreads();
  long long t5 = clock64();
  float f = (float)a;
  if (threadIdx.x == 0) {
#pragma unroll 64
    for (int i = 0; i < 1024; ++i) f = __fadd_rn(f, pool[i & 7]);
  }
  __syncthreads();
  long long t6 = clock64();
  if (threadIdx.x == 0) {
    out[3] = d + f; cyc[3] = t5 - t4; cyc[4] = t6 - t5;
    out[0] = a; out[1] = b; out[2] = c;
    cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2;
  }
}

int main() {
  float h[1024];
  unsigned s = 12345;
  for (int i = 0; i < 1024; ++i) { s = s * 1664525u + 1013904223u; h[i] = (float)((int)(s >> 8) - (1 << 23)) / (1 << 22); }
  float* d; double* o; long long* c;
  cudaMalloc(&d, 4096); cudaMalloc(&o, 64); cudaMalloc(&c, 64);
  cudaMemcpy(d, h, 4096, cudaMemcpyHostToDevice);
  for (int it = 0; it < 3; ++it) probe<<<1, 256>>>(d, o, c);
  double ho[8]; long long hc[8];
  cudaMemcpy(ho, o, 64, cudaMemcpyDeviceToHost); cudaMemcpy(hc, c, 64, cudaMemcpyDeviceToHost);
  printf("1024 dependent DADD %lld cyc, FADD %lld cyc\n", hc[3], hc[4]);
  printf("select-form %lld cyc, branch-form %lld cyc, warp %lld cyc; equal %d %d (%.17g)\n", hc[0], hc[1], hc[2],
         ho[0] == ho[2], ho[1] == ho[2], ho[2]);
  return 0;
}
