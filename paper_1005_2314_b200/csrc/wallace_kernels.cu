// Non-pool kernels and the host-callable launch table (the pool kernel
// templates are in wallace_pool.cuh, instantiated per pass type in
// pool_pt*.cu so the instantiations compile in parallel).
#include <algorithm>

#include "wallace_pool.cuh"

namespace wb {

// ---------------------------------------------------------------------------
// plan_kernel: one thread per pool walks its xoshiro256** stream two words
// per pass (generator.cpp:335-339) and writes the decoded plans.  A warp
// stages 32 pools x 32 passes in shared memory so the pool-major plan rows
// are written with coalesced 128-byte stores.
// ---------------------------------------------------------------------------

// w mod 384 (decode_pass_plan's variant, generator.cpp:249) in 32-bit
// arithmetic: 2^32 = 256 (mod 384), so w = hi*2^32 + lo = (hi mod 384)*256 +
// lo (mod 384) -- three constant 32-bit remainders instead of a 64-bit one
__device__ __forceinline__ uint32_t mod384(uint64_t w) {
  const uint32_t hi = static_cast<uint32_t>(w >> 32), lo = static_cast<uint32_t>(w);
  return ((hi % 384u) * 256u + lo % 384u) % 384u;
}

// LARGE / ROT are compile-time (a.large / a.rotation): a single pool's
// walk is one thread's dependent chain, exposed once per latency fill, so its
// loop carries no branches or parameter reloads.
template <bool LARGE, bool ROT>
__global__ void __launch_bounds__(128) plan_kernel(const PlanArgs a) {
  __shared__ uint32_t tile[4][32][33];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint64_t pool = uint64_t(blockIdx.x) * 128 + threadIdx.x;
  const uint64_t warp_pool0 = uint64_t(blockIdx.x) * 128 + w * 32;
  const bool live = pool < a.n_pools;
  uint64_t s0 = 0, s1 = 0, s2 = 0, s3 = 0;
  if (live) {
    const PoolState& st = a.st_in[pool];
    s0 = st.s[0];
    s1 = st.s[1];
    s2 = st.s[2];
    s3 = st.s[3];
  }
  // plan words of this launch: one per pass (wallace4: offset | variant << 16)
  // or two (rotation: per sweep offset | t_index << 16 | negate << 20;
  // decode_pass_plan, generator.cpp:238-257)
  constexpr uint32_t pw = LARGE ? (ROT ? 3u : 2u) : (ROT ? 2u : 1u);
  const uint32_t off_mask = a.off_mask;
  const bool fixed = a.fixed_transform != 0;
  const uint32_t n_words = a.n_passes * pw;
  constexpr uint32_t step = 32u - 32u % pw;  // whole passes per staged tile
  // one pass's plan words into the tile at word index i
  auto one_pass = [&](uint32_t i) {
    uint64_t w2[2];
#pragma unroll
    for (int q = 0; q < 2; ++q) {  // baselines.cpp:33-45
      w2[q] = rotl64(s1 * 5, 7) * 9;
      const uint64_t t = s1 << 17;
      s2 ^= s0;
      s3 ^= s1;
      s1 ^= s2;
      s0 ^= s3;
      s2 ^= t;
      s3 = rotl64(s3, 45);
    }
    if constexpr (LARGE) {
      // wallace_large.cu plan words: offsets need up to 31 bits
      uint32_t o0 = static_cast<uint32_t>(w2[1]) & off_mask;
      uint32_t o1 = static_cast<uint32_t>(w2[1] >> 32) & off_mask;
      uint32_t x = ROT ? static_cast<uint32_t>((w2[0] & 15u) | ((w2[0] >> 4) & 1u) << 4 |
                                               ((w2[0] >> 5) & 15u) << 8 | ((w2[0] >> 9) & 1u) << 12)
                       : mod384(w2[0]);
      if (fixed) o0 = o1 = x = 0;
      tile[w][lane][i] = o0;
      if constexpr (ROT) {
        tile[w][lane][i + 1] = o1;
        tile[w][lane][i + 2] = x;
      } else {
        tile[w][lane][i + 1] = x;
      }
    } else if constexpr (!ROT) {
      const uint32_t word = (static_cast<uint32_t>(w2[1]) & off_mask) | (mod384(w2[0]) << 16);
      tile[w][lane][i] = fixed ? 0u : word;  // PassPlan{} (generator.cpp:336-338)
    } else {
      uint32_t x0 = (static_cast<uint32_t>(w2[1]) & off_mask) |
                    static_cast<uint32_t>(w2[0] & 15u) << 16 | static_cast<uint32_t>((w2[0] >> 4) & 1u) << 20;
      uint32_t x1 = (static_cast<uint32_t>(w2[1] >> 32) & off_mask) |
                    static_cast<uint32_t>((w2[0] >> 5) & 15u) << 16 |
                    static_cast<uint32_t>((w2[0] >> 9) & 1u) << 20;
      if (fixed) x0 = x1 = 0;
      tile[w][lane][i] = x0;
      tile[w][lane][i + 1] = x1;
    }
  };
  for (uint32_t base = 0; base < n_words; base += step) {
    const uint32_t cnt = min(step, n_words - base);
    if (cnt == step) {
#pragma unroll
      for (uint32_t i = 0; i < step; i += pw) one_pass(i);
    } else {
      for (uint32_t i = 0; i < cnt; i += pw) one_pass(i);
    }
    __syncwarp();
    for (int q = 0; q < 32; ++q) {
      const uint64_t pq = warp_pool0 + q;
      if (pq < a.n_pools && uint32_t(lane) < cnt)
        a.plans[pq * a.plan_stride + base + lane] = tile[w][q][lane];
    }
    __syncwarp();
  }
  if (live) {
    PoolState& so = a.st_out[pool];
    so.s[0] = s0;
    so.s[1] = s1;
    so.s[2] = s2;
    so.s[3] = s3;
    so.draws = a.st_in[pool].draws + 2ull * a.n_passes;
  }
}

// ---------------------------------------------------------------------------
// Device seeding (WALLACE_CREATE_DEVICE_SEED): the constructor's Polar fill
// and normalisation (generator.cpp:309-331, baselines.cpp:19-66) for one pool
// per CTA.  Thread 0 walks the pool's xoshiro256** stream and records the
// accepted Polar pairs (u, v) -- the integer stream and the acceptance test
// are exact; all threads then form the values u*f, v*f with
// f = sqrt(-2 log(s)/s) using CUDA's log (within ~1 ulp of glibc's, so this
// is NOT a parity path); thread 0 runs the sequential Neumaier normalisation.
// Shared memory: (N + 2) doubles (pairs, then values in place) + N T values.
// ---------------------------------------------------------------------------
template <typename T>
__global__ void __launch_bounds__(128) seed_kernel(const uint64_t* seeds, uint64_t seed_base, uint32_t N,
                                                   T* pools, PoolState* st) {
  extern __shared__ __align__(16) unsigned char seed_smem[];
  double* x = reinterpret_cast<double*>(seed_smem);             // N + 2
  T* t = reinterpret_cast<T*>(seed_smem + (N + 2) * sizeof(double));  // N
  __shared__ uint64_t s_state[4];
  __shared__ uint64_t s_draws;
  __shared__ double s_k;
  const uint64_t pool = blockIdx.x;
  const uint64_t seed = seeds ? seeds[pool] : seed_base + pool;
  const uint32_t pairs = N / 2 + 1;  // N values + the reserved one (N even)
  if (threadIdx.x == 0) {
    uint64_t sm = seed, s[4];
    for (int k = 0; k < 4; ++k) s[k] = splitmix64_dev(sm);  // baselines.cpp:19-31 seeding
    uint64_t draws = 0;
    auto next_u = [&]() -> double {  // uniform_next (baselines.cpp:33-49)
      const uint64_t w = rotl64(s[1] * 5, 7) * 9;
      const uint64_t tt = s[1] << 17;
      s[2] ^= s[0];
      s[3] ^= s[1];
      s[1] ^= s[2];
      s[0] ^= s[3];
      s[2] ^= tt;
      s[3] = rotl64(s[3], 45);
      ++draws;
      return __dmul_rn(static_cast<double>(w >> 11), 0x1.0p-53);
    };
    for (uint32_t i = 0; i < pairs;) {  // polar_next's acceptance loop
      const double u = __dsub_rn(__dmul_rn(2.0, next_u()), 1.0);
      const double v = __dsub_rn(__dmul_rn(2.0, next_u()), 1.0);
      const double s2 = __dadd_rn(__dmul_rn(u, u), __dmul_rn(v, v));
      if (s2 >= 1.0 || s2 == 0.0) continue;
      x[2 * i] = u;
      x[2 * i + 1] = v;
      ++i;
    }
    for (int k = 0; k < 4; ++k) s_state[k] = s[k];
    s_draws = draws;
  }
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < pairs; i += blockDim.x) {
    const double u = x[2 * i], v = x[2 * i + 1];
    const double s2 = __dadd_rn(__dmul_rn(u, u), __dmul_rn(v, v));
    const double f = __dsqrt_rn(__ddiv_rn(__dmul_rn(-2.0, log(s2)), s2));
    x[2 * i] = __dmul_rn(u, f);
    x[2 * i + 1] = __dmul_rn(v, f);
  }
  __syncthreads();
  if (threadIdx.x == 0) {  // generator.cpp:318-327: Neumaier, k = sqrt(n / ss)
    double sum = 0.0, comp = 0.0;
    for (uint32_t i = 0; i < N; ++i) {
      const double term = __dmul_rn(x[i], x[i]);
      const double tt = __dadd_rn(sum, term);
      comp = fabs(sum) >= fabs(term) ? __dadd_rn(comp, __dadd_rn(__dsub_rn(sum, tt), term))
                                     : __dadd_rn(comp, __dadd_rn(__dsub_rn(term, tt), sum));
      sum = tt;
    }
    s_k = __dsqrt_rn(__ddiv_rn(static_cast<double>(N), __dadd_rn(sum, comp)));
  }
  __syncthreads();
  T* dst = pools + pool * N;
  for (uint32_t i = threadIdx.x; i < N; i += blockDim.x) {
    const T v = static_cast<T>(__dmul_rn(x[i], s_k));
    t[i] = v;
    dst[i] = v;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double sum = 0.0, comp = 0.0;  // recompute_sum_sq over the stored values
    for (uint32_t i = 0; i < N; ++i) {
      const double xi = static_cast<double>(t[i]);
      const double term = __dmul_rn(xi, xi);
      const double tt = __dadd_rn(sum, term);
      comp = fabs(sum) >= fabs(term) ? __dadd_rn(comp, __dadd_rn(__dsub_rn(sum, tt), term))
                                     : __dadd_rn(comp, __dadd_rn(__dsub_rn(term, tt), sum));
      sum = tt;
    }
    PoolState ps{};
    ps.reserved_prev = x[N];
    ps.sum_sq = __dadd_rn(sum, comp);
    for (int k = 0; k < 4; ++k) ps.s[k] = s_state[k];
    ps.draws = s_draws;
    ps.cursor = N - 1;
    ps.seed = seed;
    st[pool] = ps;
  }
}

// Snapshot of the current emission before the pool is advanced outside
// fill(): Generator::out_ keeps the old values until the next refill.
template <typename T>
__global__ void materialize_kernel(const T* pools, PoolState* st, T* leftover, uint64_t n_pools,
                                   uint32_t N, double mean) {
  const uint64_t pool = blockIdx.x;
  if (pool >= n_pools) return;
  const PoolState& ps = st[pool];
  if (ps.cursor >= N - 1 || (ps.flags & kFlagLeftover)) return;
  const T sc = from_double<T>(ps.scale);
  const T mt = from_double<T>(mean);
  const bool mz = mean == 0.0 && !signbit(mean);
  for (uint32_t i = threadIdx.x; i < N - 1; i += blockDim.x)
    leftover[pool * (N - 1) + i] = emit_value(pools[pool * N + i], sc, mt, mz);
  __syncthreads();
  if (threadIdx.x == 0) st[pool].flags |= kFlagLeftover;
}

// kModeFillLat epilogue: the passes sent each emission's raw pool to a
// pitched row; write x*scale + mean of its first N-1 values to the output
// (generator.cpp:366-368, the same rounding as emit_value in pool_kernel).
// Emission e of pool p covers elements [lead + e*(N-1), lead + (e+1)*(N-1))
// of the launch's slice (the last one last_limit values).  blockIdx.y = pool.
template <typename T, bool MZ>
__global__ void __launch_bounds__(256) rescale_kernel(const FillArgs a, uint32_t N) {
  const uint64_t pool = blockIdx.y;
  const uint64_t n1 = N - 1;
  const uint64_t count = a.n_emit ? (a.n_emit - 1) * n1 + a.last_limit : 0;
  T* const out = static_cast<T*>(a.out) + pool * a.out_stride + a.out_offset + a.lead;
  const T* const raw = static_cast<const T*>(a.lat_raw) + pool * a.lat_rows * N;
  const double* const scl = a.scales + pool * a.scale_stride;
  const T mean = from_double<T>(a.mean);
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < count;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t e = static_cast<uint32_t>(i / n1);
    const uint64_t k = i - e * n1;
    out[i] = emit_value(__ldcs(raw + e * uint64_t(N) + k), from_double<T>(scl[e]), mean, MZ);
  }
}

cudaError_t launch_rescale(int dtype, const FillArgs& a, uint32_t N, uint64_t n_pools, cudaStream_t s) {
  const uint64_t count = a.n_emit ? uint64_t(a.n_emit - 1) * (N - 1) + a.last_limit : 0;
  if (count == 0) return cudaSuccess;
  const unsigned bx = unsigned(std::min<uint64_t>(1024, (count + 1023) / 1024));
  const dim3 grid(bx, unsigned(n_pools));
  if (dtype == 0) {
    if (a.mean_is_zero) rescale_kernel<float, true><<<grid, 256, 0, s>>>(a, N);
    else rescale_kernel<float, false><<<grid, 256, 0, s>>>(a, N);
  } else {
    if (a.mean_is_zero) rescale_kernel<double, true><<<grid, 256, 0, s>>>(a, N);
    else rescale_kernel<double, false><<<grid, 256, 0, s>>>(a, N);
  }
  return cudaGetLastError();
}

// Fixed-order reduction of the consumer partials: block k sums pools
// [k*chunk, (k+1)*chunk) in order; the host adds the block results in order.
__global__ void reduce_consumer_kernel(const double* part_sums, const uint32_t* part_hist,
                                       uint64_t n_pools, uint64_t chunk, double* blk_sums,
                                       unsigned long long* blk_hist) {
  const uint64_t k = blockIdx.x;
  const uint64_t p0 = k * chunk, p1 = min(n_pools, p0 + chunk);
  for (int i = threadIdx.x; i < 258 + 4; i += blockDim.x) {
    if (i < 258) {
      unsigned long long acc = 0;
      for (uint64_t p = p0; p < p1; ++p) acc += part_hist[p * 258 + i];
      blk_hist[k * 258 + i] = acc;
    } else {
      const int m = i - 258;
      double acc = 0.0;
      for (uint64_t p = p0; p < p1; ++p) acc = __dadd_rn(acc, part_sums[p * 4 + m]);
      blk_sums[k * 4 + m] = acc;
    }
  }
}

cudaError_t launch_pool_large(int dtype, const FillArgs& a, uint64_t n_pools, cudaStream_t s);

size_t large_state_bytes() { return sizeof(SState); }

cudaError_t launch_pool_kernel(int dtype, int log2n, const FillArgs& a, uint64_t n_pools,
                               cudaStream_t s) {
  if (log2n >= 64) return launch_pool_large(dtype, a, n_pools, s);  // HBM-resident pools
  switch (a.pass_type) {
    case 0: return launch_pool_pt<0>(dtype, log2n, a, n_pools, s);
    case 1: return launch_pool_pt<1>(dtype, log2n, a, n_pools, s);
    case 2: return launch_pool_pt<2>(dtype, log2n, a, n_pools, s);
    case 3: return launch_pool_pt<3>(dtype, log2n, a, n_pools, s);
    default: return cudaErrorInvalidValue;
  }
}

// generator.cpp:286-294 default_multipliers as compiled into the kernels
void affine_multipliers(int log2n, uint32_t* alpha, uint32_t* beta) {
  const uint32_t n = 1u << log2n;
  *alpha = affine_alpha_c(n);
  *beta = affine_beta_c(n);
}

int pool_kernel_threads(int dtype, int log2n) {
#define WB_T(T)                                    \
  switch (log2n) {                                 \
    case 5: return Geo<T, 5>::THREADS;             \
    case 6: return Geo<T, 6>::THREADS;             \
    case 7: return Geo<T, 7>::THREADS;             \
    case 8: return Geo<T, 8>::THREADS;             \
    case 9: return Geo<T, 9>::THREADS;             \
    case 10: return Geo<T, 10>::THREADS;           \
    case 11: return Geo<T, 11>::THREADS;           \
    case 12: return Geo<T, 12>::THREADS;           \
    case 13: return Geo<T, 13>::THREADS;           \
    case 14: return Geo<T, 14>::THREADS;           \
    default: return 0;                             \
  }
  if (dtype == 0) { WB_T(float) } else { WB_T(double) }
#undef WB_T
}

cudaError_t launch_plan_kernel(const PlanArgs& a, cudaStream_t s) {
  const unsigned blocks = unsigned((a.n_pools + 127) / 128);
  if (a.large) {
    if (a.rotation) plan_kernel<true, true><<<blocks, 128, 0, s>>>(a);
    else plan_kernel<true, false><<<blocks, 128, 0, s>>>(a);
  } else {
    if (a.rotation) plan_kernel<false, true><<<blocks, 128, 0, s>>>(a);
    else plan_kernel<false, false><<<blocks, 128, 0, s>>>(a);
  }
  return cudaGetLastError();
}

cudaError_t launch_seed(int dtype, const uint64_t* d_seeds, uint64_t seed_base, uint32_t N, void* pools,
                        PoolState* st, uint64_t n_pools, cudaStream_t s) {
  const size_t smem = (N + 2) * sizeof(double) + N * (dtype == 0 ? 4 : 8);
  if (dtype == 0) {
    cudaError_t e = cudaFuncSetAttribute(seed_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e != cudaSuccess) return e;
    seed_kernel<float><<<unsigned(n_pools), 128, smem, s>>>(d_seeds, seed_base, N, static_cast<float*>(pools), st);
  } else {
    cudaError_t e = cudaFuncSetAttribute(seed_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e != cudaSuccess) return e;
    seed_kernel<double><<<unsigned(n_pools), 128, smem, s>>>(d_seeds, seed_base, N, static_cast<double*>(pools), st);
  }
  return cudaGetLastError();
}

cudaError_t launch_materialize(int dtype, const void* pools, PoolState* st, void* leftover,
                               uint64_t n_pools, uint32_t N, double mean, cudaStream_t s) {
  if (dtype == 0)
    materialize_kernel<float><<<unsigned(n_pools), 256, 0, s>>>(
        static_cast<const float*>(pools), st, static_cast<float*>(leftover), n_pools, N, mean);
  else
    materialize_kernel<double><<<unsigned(n_pools), 256, 0, s>>>(
        static_cast<const double*>(pools), st, static_cast<double*>(leftover), n_pools, N, mean);
  return cudaGetLastError();
}

cudaError_t launch_reduce_consumer(const double* part_sums, const uint32_t* part_hist,
                                   uint64_t n_pools, uint64_t chunk, double* blk_sums,
                                   unsigned long long* blk_hist, cudaStream_t s) {
  const unsigned blocks = unsigned((n_pools + chunk - 1) / chunk);
  reduce_consumer_kernel<<<blocks, 288, 0, s>>>(part_sums, part_hist, n_pools, chunk, blk_sums,
                                                blk_hist);
  return cudaGetLastError();
}

}  // namespace wb
