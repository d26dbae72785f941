// Device streams of the reference's conventional normal generators
// (baselines.cpp:51-92): the Polar method and streaming Box-Muller, one
// thread per BaselineState, fp64 like the reference.
//
// The uniform words are exact: each thread walks its stream's xoshiro256**
// state (baselines.cpp:33-49) and consumes words exactly as polar_next /
// boxmuller_next do (the Polar acceptance loop, u1 == 0 -> 2^-53, the cached
// twin), so draw counts and the accept/reject sequence equal the
// reference's.  The values use CUDA's fp64 log / sqrt / sincos, within a few
// ulps of glibc's (tests/test_gpu_baselines.py states the measured bound);
// every other operation is an explicit round-to-nearest in the reference's
// order (-fmad=false, like -ffp-contract=off).
//
//   baseline_fill_kernel     -> wallace_baseline_fill: values to HBM, the
//                               states advanced (a stream continues across calls)
//   baseline_consume_kernel  -> wallace_baseline_consume: config-5 comparator,
//                               the same fused moment/histogram consumer as
//                               the Wallace consumer kernel, in fp64
#include <cuda_runtime.h>

#include <cstdint>

#include "wallace_pool.cuh"

namespace wb {

// wallace_baseline_state (include/wallace_b200.h): UniformState + cached twin
struct BaselineDev {
  uint64_t s[4];
  uint64_t draws;
  int32_t has_cached;
  int32_t pad;
  double cached;
};
static_assert(sizeof(BaselineDev) == 56, "wallace_baseline_state layout");

struct Xoshiro {
  uint64_t s[4];
  uint64_t draws;
  __device__ __forceinline__ uint64_t bits() {  // baselines.cpp:33-45
    const uint64_t w = rotl64(s[1] * 5, 7) * 9;
    const uint64_t t = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= t;
    s[3] = rotl64(s[3], 45);
    ++draws;
    return w;
  }
  // baselines.cpp:47-49
  __device__ __forceinline__ double next() { return static_cast<double>(bits() >> 11) * 0x1.0p-53; }
};

constexpr double kTwoPi = 6.283185307179586;  // 2.0 * std::numbers::pi, exact doubling

// One pair of the method: (first, twin).  METHOD 0: polar_next's acceptance
// loop (baselines.cpp:55-65); 1: boxmuller_next + boxmuller_pair
// (baselines.cpp:68-92).
template <int METHOD>
__device__ __forceinline__ void baseline_pair(Xoshiro& u, double& z1, double& z2) {
  if constexpr (METHOD == 0) {
    for (;;) {
      const double a = __dsub_rn(__dmul_rn(2.0, u.next()), 1.0);
      const double b = __dsub_rn(__dmul_rn(2.0, u.next()), 1.0);
      const double s2 = __dadd_rn(__dmul_rn(a, a), __dmul_rn(b, b));
      if (s2 >= 1.0 || s2 == 0.0) continue;
      const double scale = __dsqrt_rn(__ddiv_rn(__dmul_rn(-2.0, log(s2)), s2));
      z1 = __dmul_rn(a, scale);
      z2 = __dmul_rn(b, scale);
      return;
    }
  } else {
    double u1 = u.next();
    if (u1 == 0.0) u1 = 0x1.0p-53;
    const double u2 = u.next();
    const double r = __dsqrt_rn(__dmul_rn(-2.0, log(u1)));
    double sn, cs;
    sincos(__dmul_rn(kTwoPi, u2), &sn, &cs);
    z1 = __dmul_rn(r, cs);
    z2 = __dmul_rn(r, sn);
  }
}

template <int METHOD>
__global__ void __launch_bounds__(128)
    baseline_fill_kernel(BaselineDev* st, uint64_t n_streams, uint64_t count, double* out) {
  const uint64_t p = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (p >= n_streams) return;
  BaselineDev b = st[p];
  Xoshiro u{{b.s[0], b.s[1], b.s[2], b.s[3]}, b.draws};
  double* o = out + p * count;
  uint64_t i = 0;
  if (b.has_cached && count > 0) {
    o[i++] = b.cached;
    b.has_cached = 0;
  }
  while (i < count) {
    double z1, z2;
    baseline_pair<METHOD>(u, z1, z2);
    o[i++] = z1;
    if (i < count) {
      o[i++] = z2;
    } else {
      b.cached = z2;
      b.has_cached = 1;
    }
  }
  for (int k = 0; k < 4; ++k) b.s[k] = u.s[k];
  b.draws = u.draws;
  st[p] = b;
}

// Config-5 comparator: stream p = BaselineState(seeds[p] or seed_base + p),
// `count` values into sums of x..x^4 (fp64) and the 258-bin histogram
// (bin = floor((x + 8) * 16) in fp64).  One thread per stream.
template <int METHOD>
__global__ void __launch_bounds__(128)
    baseline_consume_kernel(const uint64_t* seeds, uint64_t seed_base, uint64_t n_streams, uint64_t count,
                            double* part_sums, uint32_t* part_hist) {
  __shared__ uint32_t hist[258];
  __shared__ double red[4][4];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < 258; i += 128) hist[i] = 0;
  __syncthreads();
  Consumer<double> cons;
  cons.hist = hist;
  const uint64_t p = uint64_t(blockIdx.x) * 128 + tid;
  if (p < n_streams) {
    uint64_t sm = seeds ? seeds[p] : seed_base + p;
    Xoshiro u{};
    for (int k = 0; k < 4; ++k) u.s[k] = splitmix64_dev(sm);  // baselines.cpp:26-31
    for (uint64_t i = 0; i < count; i += 2) {
      double z[2];
      baseline_pair<METHOD>(u, z[0], z[1]);
      cons.add_group(z, (i + 1 < count) ? 2 : 1);
      if ((i & 255) == 254) cons.flush();  // fp64 partials folded every 256 values
    }
    cons.flush();
  }
  double v[4] = {cons.s1, cons.s2, cons.s3, cons.s4};
#pragma unroll
  for (int k = 0; k < 4; ++k)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v[k] = __dadd_rn(v[k], __shfl_down_sync(0xffffffffu, v[k], o));
  if (lane == 0)
    for (int k = 0; k < 4; ++k) red[k][warp] = v[k];
  __syncthreads();
  if (tid < 4) {
    double acc = 0.0;
    for (int w = 0; w < 4; ++w) acc = __dadd_rn(acc, red[tid][w]);
    part_sums[blockIdx.x * 4 + tid] = acc;
  }
  for (int i = tid; i < 258; i += 128) part_hist[blockIdx.x * 258 + i] = hist[i];
}

cudaError_t launch_baseline_fill(int method, void* states, uint64_t n_streams, uint64_t count, double* out,
                                 cudaStream_t s) {
  const unsigned blocks = unsigned((n_streams + 127) / 128);
  BaselineDev* st = static_cast<BaselineDev*>(states);
  if (method == 0) baseline_fill_kernel<0><<<blocks, 128, 0, s>>>(st, n_streams, count, out);
  else baseline_fill_kernel<1><<<blocks, 128, 0, s>>>(st, n_streams, count, out);
  return cudaGetLastError();
}

cudaError_t launch_baseline_consume(int method, const uint64_t* d_seeds, uint64_t seed_base, uint64_t n_streams,
                                    uint64_t count, double* part_sums, uint32_t* part_hist, uint64_t n_blocks,
                                    cudaStream_t s) {
  if (method == 0)
    baseline_consume_kernel<0><<<unsigned(n_blocks), 128, 0, s>>>(d_seeds, seed_base, n_streams, count, part_sums,
                                                                  part_hist);
  else
    baseline_consume_kernel<1><<<unsigned(n_blocks), 128, 0, s>>>(d_seeds, seed_base, n_streams, count, part_sums,
                                                                  part_hist);
  return cudaGetLastError();
}

}  // namespace wb
