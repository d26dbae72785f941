// Probe: latency (cycles) of the per-emission fp64 chain on one thread, and of
// its parts (measurement helper, not product code).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double x0, double ss, double a, double c, double nu, int iters, long long* out, double* sink) {
  double x = x0;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {  // full chain
    const double t1 = __dmul_rn(a, __dsub_rn(__dmul_rn(x, x), 1.0));
    const double S = __dadd_rn(__dadd_rn(t1, __dmul_rn(c, x)), nu);
    const double r = __dsqrt_rn(__ddiv_rn(S, ss));
    x = __dmul_rn(0.7, r);
  }
  long long t1 = clock64();
  for (int i = 0; i < iters; ++i) x = __ddiv_rn(x, ss);  // division only
  long long t2 = clock64();
  for (int i = 0; i < iters; ++i) x = __dsqrt_rn(x);  // sqrt only
  long long t3 = clock64();
  for (int i = 0; i < iters; ++i) x = __dadd_rn(x, 1e-3);  // dependent DADD
  long long t4 = clock64();
  for (int i = 0; i < iters; ++i) x = __fma_rn(x, 0.999, 1e-3);  // dependent DFMA
  long long t5 = clock64();
  out[0] = (t1 - t0) / iters; out[1] = (t2 - t1) / iters; out[2] = (t3 - t2) / iters;
  out[3] = (t4 - t3) / iters; out[4] = (t5 - t4) / iters;
  *sink = x;
}
int main() {
  long long* d; double* s;
  cudaMalloc(&d, 64); cudaMalloc(&s, 8);
  k<<<1, 1>>>(0.3, 1024.0, 0.6667631591704396, 45.2, 1024.0, 20000, d, s);
  long long h[5];
  cudaMemcpy(h, d, 40, cudaMemcpyDeviceToHost);
  printf("cycles/iter: chain %lld  ddiv %lld  dsqrt %lld  dadd %lld  dfma %lld\n", h[0], h[1], h[2], h[3], h[4]);
  return 0;
}
