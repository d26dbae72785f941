// Pools larger than shared memory (N > 2^14 fp32 / 2^13 fp64): an
// HBM-resident executor with exactly the per-launch semantics of pool_kernel
// (prologue draw, lead drain, passes with renormalisation every 256 passes,
// emissions with the one-ahead chi2 chain, epilogue state), issued as a
// sequence of small kernels over two HBM pool buffers: one kernel per pass
// (a thread per 4-block, gathering from L2/HBM), one-thread-per-pool chain
// and state kernels, grid-wide emission and scaling kernels, and a staged
// sequential Neumaier per pool.  Same explicit-rounding arithmetic as the
// on-chip kernel, so parity is unchanged; the work per pass is a gather over
// the whole pool from L2/HBM instead of shared memory.
//
// Plan words for this path (plan_kernel with PlanArgs::large): wallace4 two
// per pass (offset, variant), rotation three (offset0, offset1,
// t0 | negate0 << 4 | t1 << 8 | negate1 << 12) -- offsets need 31 bits here.
#include "wallace_pool.cuh"

namespace wb {

namespace {

constexpr int kLgThreads = 256;

__device__ __forceinline__ const uint32_t* plan_at(const FillArgs& a, uint64_t pool, uint32_t p, uint32_t pw) {
  return a.plans + pool * a.plan_stride + uint64_t(p) * pw;
}

template <typename T>
__global__ void lg_prologue(const FillArgs a, uint64_t n_pools) {
  const uint64_t pool = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (pool >= n_pools) return;
  SState s{};
  const PoolState& st = a.st_in[pool];
  s.reserved_prev = st.reserved_prev;
  s.sum_sq = st.sum_sq;
  s.cur_scale = st.scale;
  s.last_chi2 = st.last_chi2;
  s.last_r = st.r;
  s.last_scale = st.scale;
  s.flags = st.flags;
  if (a.mode != kModePasses && a.n_emit > 0) chain_draw(s, 0, a.chi2, a.sigma);
  static_cast<SState*>(a.lg_state)[pool] = s;
}

// drain the partially consumed emission (pool_kernel's lead)
template <typename T>
__global__ void lg_lead(const FillArgs a, const T* pool_buf, uint64_t N) {
  const uint64_t pool = blockIdx.y;
  const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= a.lead) return;
  const SState& s = static_cast<const SState*>(a.lg_state)[pool];
  const PoolState& st = a.st_in[pool];
  const uint64_t idx = st.cursor + i;
  const bool mz = a.mean_is_zero != 0;
  T v;
  if (st.flags & kFlagLeftover) v = static_cast<const T*>(a.leftover)[pool * (N - 1) + idx];
  else v = emit_value(pool_buf[pool * N + idx], from_double<T>(s.cur_scale), from_double<T>(a.mean), mz);
  static_cast<T*>(a.out)[pool * a.out_stride + a.out_offset + i] = v;
}

// Fused emission (emit_slot >= 0): the pass's outputs x, scaled, are the
// emission (values i < limit at output offset gofs) -- valid when no
// renormalisation follows the pass.
template <typename T>
__device__ __forceinline__ void lg_emit4(const FillArgs& a, uint64_t pool, uint64_t i0, const T* x, int slot,
                                         uint64_t gofs, uint32_t limit) {
  const SState& s = static_cast<const SState*>(a.lg_state)[pool];
  const T sc = from_double<T>(s.scale[slot]);
  const T mean = from_double<T>(a.mean);
  T* o = static_cast<T*>(a.out) + pool * a.out_stride + gofs;
#pragma unroll
  for (int k = 0; k < 4; ++k)
    if (i0 + k < limit) o[i0 + k] = emit_value(x[k], sc, mean, a.mean_is_zero != 0);
}

// One wallace4 pass (generator.cpp:52-110), a thread per 4-block.
template <typename T, int MIX>
__global__ void lg_pass_wallace(const FillArgs a, const T* in, T* out, uint32_t p, uint64_t N, int emit_slot,
                                uint64_t gofs, uint32_t limit) {
  const uint64_t pool = blockIdx.y;
  const uint64_t rows = N / 4;
  const uint64_t b = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (b >= rows) return;
  const uint32_t* w = plan_at(a, pool, p, 2);
  const uint64_t off = w[0];
  const uint32_t variant = w[1];
  const T* src = in + pool * N;
  T v[4];
  if (MIX == 0) {
    const uint64_t r = (off + b * a.lg_stride) & (rows - 1);
#pragma unroll
    for (int c = 0; c < 4; ++c) v[c] = src[c * rows + r];
  } else {
#pragma unroll
    for (int c = 0; c < 4; ++c) v[c] = src[(off + (4 * b + c) * a.lg_alpha) & (N - 1)];
  }
  const T aa = add_rn(v[0], v[1]), bb = sub_rn(v[0], v[1]), cc = add_rn(v[2], v[3]), dd = sub_rn(v[2], v[3]);
  const T z[4] = {sub_rn(aa, dd), add_rn(bb, cc), sub_rn(bb, cc), sub_rn(-aa, dd)};
  const int perm = int(variant >> 4);
  T* dst = out + pool * N + 4 * b;
  T x[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const T h = ((variant >> k) & 1u) ? T(-0.5) : T(0.5);
    x[k] = mul_rn(h, z[perm_at(perm, k)]);
    dst[k] = x[k];
  }
  if (emit_slot >= 0) lg_emit4(a, pool, 4 * b, x, emit_slot, gofs, limit);
}

// One rotation half-sweep (generator.cpp:113-172), a thread per 4-block of
// the output; sweep 1 gathers the block's neighbours g[4b-1], g[4b+4] too.
template <typename T, int MIX, int SWEEP>
__global__ void lg_pass_rotation(const FillArgs a, const T* in, T* out, uint32_t p, uint64_t N, int emit_slot,
                                 uint64_t gofs, uint32_t limit) {
  const uint64_t pool = blockIdx.y;
  const uint64_t rows = N / 4;
  const uint64_t b = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (b >= rows) return;
  const uint32_t* w = plan_at(a, pool, p, 3);
  const uint64_t off = w[SWEEP];
  const uint32_t tb = (w[2] >> (8 * SWEEP)) & 0xffu;
  const uint32_t t = tb & 15u;
  const bool neg = (tb >> 4) & 1u;
  const T ce = from_double<T>(neg ? -a.rot_c[t] : a.rot_c[t]);
  const T se = from_double<T>(neg ? -a.rot_s[t] : a.rot_s[t]);
  const T nse = -se;
  const T* src = in + pool * N;
  // element j of the gathered sequence (mod N)
  auto g = [&](uint64_t j) -> T {
    j &= N - 1;
    if (MIX == 0) {
      const uint64_t q = j >> 2, c = j & 3;
      return src[c * rows + ((off + q * a.lg_stride) & (rows - 1))];
    }
    return src[(off + j * (SWEEP == 0 ? a.lg_alpha : a.lg_beta)) & (N - 1)];
  };
  T* dst = out + pool * N + 4 * b;
  if (SWEEP == 0) {
    const T g0 = g(4 * b), g1 = g(4 * b + 1), g2 = g(4 * b + 2), g3 = g(4 * b + 3);
    dst[0] = add_rn(mul_rn(ce, g0), mul_rn(se, g1));
    dst[1] = add_rn(mul_rn(nse, g0), mul_rn(ce, g1));
    dst[2] = add_rn(mul_rn(ce, g2), mul_rn(se, g3));
    dst[3] = add_rn(mul_rn(nse, g2), mul_rn(ce, g3));
  } else {
    const T hm = g(4 * b + N - 1), h0 = g(4 * b), h1 = g(4 * b + 1), h2 = g(4 * b + 2), h3 = g(4 * b + 3),
            hp = g(4 * b + 4);
    T x[4];
    x[0] = add_rn(mul_rn(nse, hm), mul_rn(ce, h0));
    x[1] = add_rn(mul_rn(ce, h1), mul_rn(se, h2));
    x[2] = add_rn(mul_rn(nse, h1), mul_rn(ce, h2));
    x[3] = add_rn(mul_rn(ce, h3), mul_rn(se, hp));
#pragma unroll
    for (int k = 0; k < 4; ++k) dst[k] = x[k];
    if (emit_slot >= 0) lg_emit4(a, pool, 4 * b, x, emit_slot, gofs, limit);
  }
}

// Sequential Neumaier over a pool in HBM (generator.cpp:20-34): the CTA
// stages chunks in shared memory, thread 0 adds them in order.
template <typename T>
__device__ double lg_neumaier(const T* v, uint64_t N) {
  constexpr int CH = 4096;
  __shared__ T chunk[CH];
  double sum = 0.0, comp = 0.0;
  for (uint64_t c0 = 0; c0 < N; c0 += CH) {
    const uint64_t n = N - c0 < CH ? N - c0 : CH;
    for (uint64_t i = threadIdx.x; i < n; i += blockDim.x) chunk[i] = v[c0 + i];
    __syncthreads();
    if (threadIdx.x == 0)
      for (uint64_t i = 0; i < n; ++i) neumaier_add<false>(sum, comp, static_cast<double>(chunk[i]));
    __syncthreads();
  }
  return __dadd_rn(sum, comp);
}

// renormalize_ (generator.cpp:345-351), part 1: ss and k
template <typename T>
__global__ void lg_renorm_begin(const FillArgs a, const T* pool_buf, uint64_t N) {
  const uint64_t pool = blockIdx.x;
  const double ss = lg_neumaier(pool_buf + pool * N, N);
  if (threadIdx.x == 0) {
    SState& s = static_cast<SState*>(a.lg_state)[pool];
    s.renorm_ok = ss > 0.0;
    s.renorm_k = ss > 0.0 ? __dsqrt_rn(__ddiv_rn(static_cast<double>(N), ss)) : 0.0;
  }
}
template <typename T>
__global__ void lg_renorm_scale(const FillArgs a, T* pool_buf, uint64_t N) {
  const uint64_t pool = blockIdx.y;
  const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const SState& s = static_cast<const SState*>(a.lg_state)[pool];
  if (i >= N || !s.renorm_ok) return;
  T& x = pool_buf[pool * N + i];
  x = from_double<T>(__dmul_rn(static_cast<double>(x), s.renorm_k));
}
// part 2: sum_sq of the scaled pool; in an emission run the current
// emission's r / scale follow (refill_ reads sum_sq after the renormalisation)
template <typename T>
__global__ void lg_renorm_end(const FillArgs a, const T* pool_buf, uint64_t N, int slot, int rescale) {
  const uint64_t pool = blockIdx.x;
  SState* ls = static_cast<SState*>(a.lg_state);
  if (!ls[pool].renorm_ok) {
    if (threadIdx.x == 0 && rescale) chain_rescale(ls[pool], slot, a.chi2, a.sigma);
    return;
  }
  const double ss = lg_neumaier(pool_buf + pool * N, N);
  if (threadIdx.x == 0) {
    ls[pool].sum_sq = ss;
    if (rescale) chain_rescale(ls[pool], slot, a.chi2, a.sigma);
  }
}

template <typename T>
__global__ void lg_emit(const FillArgs a, const T* pool_buf, uint64_t N, uint64_t gofs, uint32_t limit, int slot) {
  const uint64_t pool = blockIdx.y;
  const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= limit) return;
  const SState& s = static_cast<const SState*>(a.lg_state)[pool];
  static_cast<T*>(a.out)[pool * a.out_stride + gofs + i] =
      emit_value(pool_buf[pool * N + i], from_double<T>(s.scale[slot]), from_double<T>(a.mean), a.mean_is_zero != 0);
}

template <typename T>
__global__ void lg_chain(const FillArgs a, const T* pool_buf, uint64_t N, int slot, int draw, uint64_t n_pools) {
  const uint64_t pool = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (pool >= n_pools) return;
  SState& s = static_cast<SState*>(a.lg_state)[pool];
  chain_close(s, slot, static_cast<double>(pool_buf[pool * N + N - 1]));
  if (draw) chain_draw(s, slot ^ 1, a.chi2, a.sigma);
}

template <typename T>
__global__ void lg_epilogue(const FillArgs a, uint64_t n_pools) {
  const uint64_t pool = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (pool >= n_pools) return;
  const SState& s = static_cast<const SState*>(a.lg_state)[pool];
  const PoolState in = a.st_in[pool];
  PoolState& so = a.st_out[pool];
  so.reserved_prev = s.reserved_prev;
  so.sum_sq = s.sum_sq;
  so.pass_count = in.pass_count + a.n_passes;
  so.clamp_count = in.clamp_count + s.clamp;
  uint32_t flags = s.flags;
  so.scale = s.last_scale;
  so.r = s.last_r;
  so.last_chi2 = s.last_chi2;
  if (a.mode != kModePasses && a.n_emit > 0) {
    so.cursor = a.last_limit;
    flags &= ~kFlagLeftover;
  } else {
    so.cursor = in.cursor + (a.mode != kModePasses ? a.lead : 0);
  }
  so.flags = flags;
  so.seed = in.seed;
  if (a.n_passes == 0 && &so != &a.st_in[pool]) {
    for (int k = 0; k < 4; ++k) so.s[k] = in.s[k];
    so.draws = in.draws;
  }
}

template <typename T>
cudaError_t run_large(const FillArgs& a, uint64_t n_pools, cudaStream_t st) {
  const uint64_t N = uint64_t(1) << a.lg_log2n;
  const uint64_t rows = N / 4;
  const int pt = a.pass_type;
  const bool rot = pt >= 2;
  const unsigned pool_blocks = unsigned((n_pools + 127) / 128);
  const dim3 grid_rows(unsigned((rows + kLgThreads - 1) / kLgThreads), unsigned(n_pools));
  const dim3 grid_vals(unsigned((N + kLgThreads - 1) / kLgThreads), unsigned(n_pools));
  T* w[2] = {static_cast<T*>(a.pools_out), static_cast<T*>(a.lg_pool2)};
  int cur = 0;
  if (a.pools_in != a.pools_out)
    cudaMemcpyAsync(w[0], a.pools_in, n_pools * N * sizeof(T), cudaMemcpyDeviceToDevice, st);
  lg_prologue<T><<<pool_blocks, 128, 0, st>>>(a, n_pools);
  if (a.mode != kModePasses && a.lead > 0) {
    const dim3 g(unsigned((a.lead + kLgThreads - 1) / kLgThreads), unsigned(n_pools));
    lg_lead<T><<<g, kLgThreads, 0, st>>>(a, w[0], N);
  }
  // one pass; emit_slot >= 0 fuses the emission (values i < limit at gofs)
  auto pass = [&](uint32_t p, int es = -1, uint64_t go = 0, uint32_t lim = 0) {
    if (!rot) {
      if (pt == 0) lg_pass_wallace<T, 0><<<grid_rows, kLgThreads, 0, st>>>(a, w[cur], w[cur ^ 1], p, N, es, go, lim);
      else lg_pass_wallace<T, 1><<<grid_rows, kLgThreads, 0, st>>>(a, w[cur], w[cur ^ 1], p, N, es, go, lim);
    } else if (pt == 2) {
      lg_pass_rotation<T, 0, 0><<<grid_rows, kLgThreads, 0, st>>>(a, w[cur], w[cur ^ 1], p, N, -1, 0, 0);
      lg_pass_rotation<T, 0, 1><<<grid_rows, kLgThreads, 0, st>>>(a, w[cur ^ 1], w[cur], p, N, es, go, lim);
    } else {
      lg_pass_rotation<T, 1, 0><<<grid_rows, kLgThreads, 0, st>>>(a, w[cur], w[cur ^ 1], p, N, -1, 0, 0);
      lg_pass_rotation<T, 1, 1><<<grid_rows, kLgThreads, 0, st>>>(a, w[cur ^ 1], w[cur], p, N, es, go, lim);
    }
    if (!rot) cur ^= 1;
  };
  auto renorm = [&](int slot, int rescale) {
    lg_renorm_begin<T><<<unsigned(n_pools), kLgThreads, 0, st>>>(a, w[cur], N);
    lg_renorm_scale<T><<<grid_vals, kLgThreads, 0, st>>>(a, w[cur], N);
    lg_renorm_end<T><<<unsigned(n_pools), kLgThreads, 0, st>>>(a, w[cur], N, slot, rescale);
  };
  uint32_t pc = static_cast<uint32_t>(a.lg_pass0 + 1) & 255u;  // pass count after the next pass, mod 256
  uint32_t p = 0;
  if (a.mode == kModePasses) {
    for (; p < a.n_passes; ++p) {
      pass(p);
      if (pc == 0) renorm(0, 0);
      pc = (pc + 1) & 255u;
    }
  } else {
    uint64_t gofs = a.out_offset + a.lead;
    for (uint32_t e = 0; e < a.n_emit; ++e, gofs += N - 1) {
      const int slot = e & 1;
      const uint32_t limit = (e + 1 == a.n_emit) ? a.last_limit : uint32_t(N - 1);
      for (uint32_t q = 1; q <= a.d; ++q, ++p) {
        const bool emit = q == a.d;
        const bool fuse = emit && pc != 0;  // no renormalisation between the pass and its emission
        if (fuse) pass(p, slot, gofs, limit);
        else pass(p);
        if (pc == 0) renorm(slot, 1);
        if (emit) {
          if (!fuse) {
            const dim3 g(unsigned((limit + kLgThreads - 1) / kLgThreads), unsigned(n_pools));
            lg_emit<T><<<g, kLgThreads, 0, st>>>(a, w[cur], N, gofs, limit, slot);
          }
          lg_chain<T><<<pool_blocks, 128, 0, st>>>(a, w[cur], N, slot, e + 1 < a.n_emit ? 1 : 0, n_pools);
        }
        pc = (pc + 1) & 255u;
      }
    }
  }
  if (cur != 0) cudaMemcpyAsync(w[0], w[1], n_pools * N * sizeof(T), cudaMemcpyDeviceToDevice, st);
  lg_epilogue<T><<<pool_blocks, 128, 0, st>>>(a, n_pools);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_pool_large(int dtype, const FillArgs& a, uint64_t n_pools, cudaStream_t s) {
  if (a.mode != kModeFill && a.mode != kModePasses) return cudaErrorNotSupported;
  return dtype == 0 ? run_large<float>(a, n_pools, s) : run_large<double>(a, n_pools, s);
}

}  // namespace wb
