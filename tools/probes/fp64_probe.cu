// fp64 pipe probe: cycles per dependent DADD, per DADD with 2/4/8 independent
// chains, and per DFMA/DMUL, one warp and 4 warps per SM sub-partition.
#include <cstdio>
template <int C>
__global__ void chains(double* out, long long* cyc, double a) {
  double x[C];
#pragma unroll
  for (int c = 0; c < C; ++c) x[c] = a + c + threadIdx.x;
  __syncthreads();
  long long t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < 1024; ++i)
#pragma unroll
    for (int c = 0; c < C; ++c) x[c] = __dadd_rn(x[c], a);
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int c = 0; c < C; ++c) s += x[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 1 << 20); cudaMalloc(&c, 64);
  long long h;
  for (int w : {32, 128, 512}) {
    chains<1><<<1, w>>>(o, c, 1e-3); chains<1><<<1, w>>>(o, c, 1e-3); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("threads %d: 1 chain  %.2f cyc/DADD-step\n", w, h / 1024.0);
    chains<2><<<1, w>>>(o, c, 1e-3); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("threads %d: 2 chains %.2f cyc/step (%.2f per DADD)\n", w, h / 1024.0, h / 2048.0);
    chains<4><<<1, w>>>(o, c, 1e-3); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("threads %d: 4 chains %.2f cyc/step (%.2f per DADD)\n", w, h / 1024.0, h / 4096.0);
    chains<8><<<1, w>>>(o, c, 1e-3); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("threads %d: 8 chains %.2f cyc/step (%.2f per DADD)\n", w, h / 1024.0, h / 8192.0);
  }
  return 0;
}
