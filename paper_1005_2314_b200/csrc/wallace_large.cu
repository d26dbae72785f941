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

// 2-D launches over (blocks of a pool) x (pools): gridDim.y/z are limited to
// 65535, so the pool index spans y and z
__device__ __forceinline__ uint64_t lg_pool_index() { return blockIdx.y + uint64_t(blockIdx.z) * 65535u; }
inline dim3 lg_grid(uint64_t bx, uint64_t n_pools) {
  const uint64_t y = n_pools < 65535 ? n_pools : 65535;
  return dim3{unsigned(bx), unsigned(y), unsigned((n_pools + 65534) / 65535)};
}

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
  s.flags = st.flags & ~kFlagChi2NonFinite;
  if (a.mode != kModePasses && a.n_emit > 0) chain_draw(s, 0, a.chi2, a.sigma);
  static_cast<SState*>(a.lg_state)[pool] = s;
}

// drain the partially consumed emission (pool_kernel's lead)
template <typename T>
__global__ void lg_lead(const FillArgs a, const T* pool_buf, uint64_t N) {
  const uint64_t pool = lg_pool_index();
  if (pool >= a.lg_npools) return;
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
  const uint64_t pool = lg_pool_index();
  if (pool >= a.lg_npools) return;
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

// The same pass with a thread per gathered *row*: row r holds elements
// r, r+rows, r+2rows, r+3rows, the inputs of the 4-block b whose row is
// r = (off + b*stride) mod rows, i.e. b = (r - off) * stride^-1 mod rows.
// Consecutive threads then load consecutive addresses (every sector fully
// used, against one 4-byte value per 32-byte sector for a thread per block),
// and each thread stores its block as one 16-byte vector.  Same arithmetic,
// same results.
template <typename T>
__global__ void lg_pass_wallace_rows(const FillArgs a, const T* in, T* out, uint32_t p, uint64_t N,
                                     int emit_slot, uint64_t gofs, uint32_t limit) {
  const uint64_t pool = lg_pool_index();
  if (pool >= a.lg_npools) return;
  const uint64_t rows = N / 4;
  const uint64_t r = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= rows) return;
  const uint32_t* w = plan_at(a, pool, p, 2);
  const uint64_t off = w[0];
  const uint32_t variant = w[1];
  const T* src = in + pool * N;
  T v[4];
#pragma unroll
  for (int c = 0; c < 4; ++c) v[c] = src[c * rows + r];
  const uint64_t b = ((r - off) * a.lg_stride_inv) & (rows - 1);
  const T aa = add_rn(v[0], v[1]), bb = sub_rn(v[0], v[1]), cc = add_rn(v[2], v[3]), dd = sub_rn(v[2], v[3]);
  const T z[4] = {sub_rn(aa, dd), add_rn(bb, cc), sub_rn(bb, cc), sub_rn(-aa, dd)};
  const int perm = int(variant >> 4);
  T x[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const T h = ((variant >> k) & 1u) ? T(-0.5) : T(0.5);
    x[k] = mul_rn(h, z[perm_at(perm, k)]);
  }
  T* dst = out + pool * N + 4 * b;
  if constexpr (sizeof(T) == 4) {
    *reinterpret_cast<float4*>(dst) = make_float4(x[0], x[1], x[2], x[3]);
  } else {
    reinterpret_cast<double2*>(dst)[0] = make_double2(x[0], x[1]);
    reinterpret_cast<double2*>(dst)[1] = make_double2(x[2], x[3]);
  }
  if (emit_slot >= 0) lg_emit4(a, pool, 4 * b, x, emit_slot, gofs, limit);
}

// One rotation half-sweep (generator.cpp:113-172), a thread per 4-block of
// the output; sweep 1 gathers the block's neighbours g[4b-1], g[4b+4] too.
template <typename T, int MIX, int SWEEP>
__global__ void lg_pass_rotation(const FillArgs a, const T* in, T* out, uint32_t p, uint64_t N, int emit_slot,
                                 uint64_t gofs, uint32_t limit) {
  const uint64_t pool = lg_pool_index();
  if (pool >= a.lg_npools) return;
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
    s.renorm_ok = !(ss <= 0.0);  // generator.cpp:347: a NaN sum still rescales
    s.renorm_k = s.renorm_ok ? __dsqrt_rn(__ddiv_rn(static_cast<double>(N), ss)) : 0.0;
  }
}
template <typename T>
__global__ void lg_renorm_scale(const FillArgs a, T* pool_buf, uint64_t N) {
  const uint64_t pool = lg_pool_index();
  if (pool >= a.lg_npools) return;
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
  const uint64_t pool = lg_pool_index();
  if (pool >= a.lg_npools) return;
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
  if (flags & kFlagChi2NonFinite) atomicOr(a.err_word, 1u);  // see pool_kernel's epilogue
  flags &= ~kFlagChi2NonFinite;
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

// ---- fused consumers (kModeConsume, kModeDefect) and probes on the large path
// aux layout per pool (doubles): [0..3] consumer totals, [4] defect mark,
// [8..39] probe x, [40...] per-block partials (4 per block).
constexpr int kAuxTotals = 0, kAuxMark = 4, kAuxProbe = 8, kAuxPart = 40;
constexpr int kLgVpt = 16;                     // values per thread in the consumer kernels
constexpr int kLgBlockVals = kLgThreads * kLgVpt;

__device__ __forceinline__ double block_sum(double v, double* red) {
  v = warp_sum_f64(v);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x == 0)
    for (int w = 0; w < kLgThreads / 32; ++w) t = __dadd_rn(t, red[w]);
  return t;
}

// values [i0, i0 + n) of pool `pool`: emitted (scale sc) from the pool or the
// materialized leftover, fed to the consumer (moments + histogram) or the
// defect statistics (sum of squares + rare-event mark); one block partial
template <typename T, int MODE>
__global__ void lg_consume(const FillArgs a, const T* src, uint64_t src_stride, uint64_t n, int use_cur_scale,
                           int slot) {
  __shared__ double red[kLgThreads / 32];
  const uint64_t pool = lg_pool_index(), blk = blockIdx.x;
  if (pool >= a.lg_npools) return;
  const SState& s = static_cast<const SState*>(a.lg_state)[pool];
  const T sc = from_double<T>(use_cur_scale ? s.cur_scale : s.scale[slot]);
  const T mean = from_double<T>(a.mean);
  const bool mz = a.mean_is_zero != 0, raw = use_cur_scale == 2;  // 2: leftover values are already emitted
  double m[4] = {0.0, 0.0, 0.0, 0.0};
  bool mark = false;
  for (int k = 0; k < kLgVpt; ++k) {
    const uint64_t i = blk * kLgBlockVals + uint64_t(k) * kLgThreads + threadIdx.x;
    if (i >= n) break;
    const T x = src[pool * src_stride + i];
    const T y = raw ? x : emit_value(x, sc, mean, mz);
    const double v = static_cast<double>(y);
    if (MODE == kModeConsume) {
      const double v2 = __dmul_rn(v, v);
      m[0] = __dadd_rn(m[0], v);
      m[1] = __dadd_rn(m[1], v2);
      m[2] = __dadd_rn(m[2], __dmul_rn(v2, v));
      m[3] = __dadd_rn(m[3], __dmul_rn(v2, v2));
      const T t = fma_rn(y, T(16), T(128));  // floor((y + 8) * 16), as the on-chip consumer
      int bin = sizeof(T) == 4 ? __float2int_rd(static_cast<float>(t)) : __double2int_rd(static_cast<double>(t));
      bin = max(-1, min(bin, 256));
      atomicAdd(&a.part_hist[pool * 258 + bin + 1], 1u);
    } else {
      m[0] = __dadd_rn(m[0], __dmul_rn(v, v));
      mark |= fabs(v) > a.def_threshold;
    }
  }
  double* part = a.lg_aux + pool * a.lg_aux_stride + kAuxPart + blk * 4;
  for (int q = 0; q < (MODE == kModeConsume ? 4 : 1); ++q) {
    const double t = block_sum(m[q], red);
    if (threadIdx.x == 0) part[q] = t;
  }
  if (MODE == kModeDefect && __syncthreads_or(mark) && threadIdx.x == 0)
    a.lg_aux[pool * a.lg_aux_stride + kAuxMark] = 1.0;
}

// fold the block partials of one emission (or of the lead) in block order
template <int MODE>
__global__ void lg_fold(const FillArgs a, uint64_t nblk, uint64_t e, uint64_t n_pools) {
  const uint64_t pool = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (pool >= n_pools) return;
  double* aux = a.lg_aux + pool * a.lg_aux_stride;
  if (MODE == kModeConsume) {
    for (int q = 0; q < 4; ++q) {
      double t = aux[kAuxTotals + q];
      for (uint64_t b = 0; b < nblk; ++b) t = __dadd_rn(t, aux[kAuxPart + b * 4 + q]);
      aux[kAuxTotals + q] = t;
    }
  } else {
    // pool_sum_squares_test's total: reserved^2 (chain_close ran) + sum v^2
    const SState& s = static_cast<const SState*>(a.lg_state)[pool];
    double t = __dmul_rn(s.reserved_prev, s.reserved_prev);
    for (uint64_t b = 0; b < nblk; ++b) t = __dadd_rn(t, aux[kAuxPart + b * 4]);
    a.def_totals[pool * a.def_stride + a.def_e0 + e] = t;
    a.def_marks[pool * a.def_stride + a.def_e0 + e] = aux[kAuxMark] != 0.0 ? 1 : 0;
    aux[kAuxMark] = 0.0;
  }
}

__global__ void lg_consume_begin(const FillArgs a, uint64_t n_pools) {
  const uint64_t pool = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (pool >= n_pools) return;
  double* aux = a.lg_aux + pool * a.lg_aux_stride;
  for (int q = 0; q < 5; ++q) aux[q] = 0.0;
  if (a.mode == kModeConsume)
    for (int i = 0; i < 258; ++i) a.part_hist[pool * 258 + i] = 0;
}
__global__ void lg_consume_end(const FillArgs a, uint64_t n_pools) {
  const uint64_t pool = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (pool >= n_pools) return;
  for (int q = 0; q < 4; ++q) a.part_sums[pool * 4 + q] = a.lg_aux[pool * a.lg_aux_stride + kAuxTotals + q];
}

// cross-pool probes (stats.cpp:310-338): x before the pass, y after it (and
// after a renormalisation), ProbeAccumulator sums in pass order
template <typename T>
__global__ void lg_probe_x(const FillArgs a, const T* pool_buf, uint64_t N, uint64_t n_pools) {
  const uint64_t pool = blockIdx.x;
  const uint32_t k = threadIdx.x;
  if (pool >= n_pools || k >= a.n_probes) return;
  a.lg_aux[pool * a.lg_aux_stride + kAuxProbe + k] = static_cast<double>(pool_buf[pool * N + a.probe_in[k]]);
}
template <typename T>
__global__ void lg_probe_y(const FillArgs a, const T* pool_buf, uint64_t N, uint64_t n_pools) {
  const uint64_t pool = blockIdx.x;
  const uint32_t k = threadIdx.x;
  if (pool >= n_pools || k >= a.n_probes) return;
  const double x = a.lg_aux[pool * a.lg_aux_stride + kAuxProbe + k];
  const double y = static_cast<double>(pool_buf[pool * N + a.probe_out[k]]);
  double* pa = a.probe_acc + (pool * a.n_probes + k) * 6;
  pa[0] = __dadd_rn(pa[0], x);
  pa[1] = __dadd_rn(pa[1], __dmul_rn(x, x));
  pa[2] = __dadd_rn(pa[2], y);
  pa[3] = __dadd_rn(pa[3], __dmul_rn(y, y));
  const double w = __dmul_rn(x, y);
  pa[4] = __dadd_rn(pa[4], w);
  pa[5] = __dadd_rn(pa[5], __dmul_rn(w, w));
}

template <typename T>
cudaError_t run_large(const FillArgs& args, uint64_t n_pools, cudaStream_t st) {
  FillArgs a = args;
  a.lg_npools = n_pools;
  const uint64_t N = uint64_t(1) << a.lg_log2n;
  const uint64_t rows = N / 4;
  const int pt = a.pass_type;
  const bool rot = pt >= 2;
  const unsigned pool_blocks = unsigned((n_pools + 127) / 128);
  const dim3 grid_rows = lg_grid((rows + kLgThreads - 1) / kLgThreads, n_pools);
  const dim3 grid_vals = lg_grid((N + kLgThreads - 1) / kLgThreads, n_pools);
  T* w[2] = {static_cast<T*>(a.pools_out), static_cast<T*>(a.lg_pool2)};
  int cur = 0;
  if (a.pools_in != a.pools_out)
    cudaMemcpyAsync(w[0], a.pools_in, n_pools * N * sizeof(T), cudaMemcpyDeviceToDevice, st);
  lg_prologue<T><<<pool_blocks, 128, 0, st>>>(a, n_pools);
  const bool cons = a.mode == kModeConsume || a.mode == kModeDefect;
  if (cons) lg_consume_begin<<<pool_blocks, 128, 0, st>>>(a, n_pools);
  if (a.mode == kModeConsume && a.lead > 0) {
    // the lead: from the materialized leftover (already emitted values) or the
    // pool with the current emission's scale; pools agree on both (uniform cursor)
    cudaError_t e0 = cudaSuccess;
    PoolState st0{};
    e0 = cudaMemcpyAsync(&st0, a.st_in, sizeof(st0), cudaMemcpyDeviceToHost, st);
    if (e0 == cudaSuccess) e0 = cudaStreamSynchronize(st);
    if (e0 != cudaSuccess) return e0;
    const uint64_t nb = (a.lead + kLgBlockVals - 1) / kLgBlockVals;
    const dim3 g = lg_grid(nb, n_pools);
    if (st0.flags & kFlagLeftover)
      lg_consume<T, kModeConsume><<<g, kLgThreads, 0, st>>>(
          a, static_cast<const T*>(a.leftover) + st0.cursor, N - 1, a.lead, 2, 0);
    else
      lg_consume<T, kModeConsume><<<g, kLgThreads, 0, st>>>(a, w[0] + st0.cursor, N, a.lead, 1, 0);
    lg_fold<kModeConsume><<<pool_blocks, 128, 0, st>>>(a, nb, 0, n_pools);
  } else if (a.mode != kModePasses && a.lead > 0 && !cons) {
    const dim3 g = lg_grid((a.lead + kLgThreads - 1) / kLgThreads, n_pools);
    lg_lead<T><<<g, kLgThreads, 0, st>>>(a, w[0], N);
  }
  // one pass; emit_slot >= 0 fuses the emission (values i < limit at gofs)
  auto pass = [&](uint32_t p, int es = -1, uint64_t go = 0, uint32_t lim = 0) {
    if (!rot) {
      if (pt == 0 && a.lg_row_major)
        lg_pass_wallace_rows<T><<<grid_rows, kLgThreads, 0, st>>>(a, w[cur], w[cur ^ 1], p, N, es, go, lim);
      else if (pt == 0)
        lg_pass_wallace<T, 0><<<grid_rows, kLgThreads, 0, st>>>(a, w[cur], w[cur ^ 1], p, N, es, go, lim);
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
      if (a.n_probes) lg_probe_x<T><<<unsigned(n_pools), 32, 0, st>>>(a, w[cur], N, n_pools);
      pass(p);
      if (pc == 0) renorm(0, 0);
      if (a.n_probes) lg_probe_y<T><<<unsigned(n_pools), 32, 0, st>>>(a, w[cur], N, n_pools);
      pc = (pc + 1) & 255u;
    }
  } else {
    uint64_t gofs = a.out_offset + a.lead;
    for (uint32_t e = 0; e < a.n_emit; ++e, gofs += N - 1) {
      const int slot = e & 1;
      const uint32_t limit = (e + 1 == a.n_emit) ? a.last_limit : uint32_t(N - 1);
      for (uint32_t q = 1; q <= a.d; ++q, ++p) {
        const bool emit = q == a.d;
        // the emission fused into the pass when no renormalisation intervenes
        const bool fuse = emit && pc != 0 && !cons;
        if (fuse) pass(p, slot, gofs, limit);
        else pass(p);
        if (pc == 0) renorm(slot, 1);
        if (emit) {
          const uint64_t nb = (limit + kLgBlockVals - 1) / kLgBlockVals;
          const dim3 gc = lg_grid(nb, n_pools);
          if (a.mode == kModeConsume) {
            lg_consume<T, kModeConsume><<<gc, kLgThreads, 0, st>>>(a, w[cur], N, limit, 0, slot);
            lg_fold<kModeConsume><<<pool_blocks, 128, 0, st>>>(a, nb, e, n_pools);
          } else if (a.mode == kModeDefect) {
            lg_consume<T, kModeDefect><<<gc, kLgThreads, 0, st>>>(a, w[cur], N, limit, 0, slot);
          } else if (!fuse) {
            const dim3 g = lg_grid((limit + kLgThreads - 1) / kLgThreads, n_pools);
            lg_emit<T><<<g, kLgThreads, 0, st>>>(a, w[cur], N, gofs, limit, slot);
          }
          lg_chain<T><<<pool_blocks, 128, 0, st>>>(a, w[cur], N, slot, e + 1 < a.n_emit ? 1 : 0, n_pools);
          if (a.mode == kModeDefect) lg_fold<kModeDefect><<<pool_blocks, 128, 0, st>>>(a, nb, e, n_pools);
        }
        pc = (pc + 1) & 255u;
      }
    }
  }
  if (cur != 0) cudaMemcpyAsync(w[0], w[1], n_pools * N * sizeof(T), cudaMemcpyDeviceToDevice, st);
  if (a.mode == kModeConsume) lg_consume_end<<<pool_blocks, 128, 0, st>>>(a, n_pools);
  lg_epilogue<T><<<pool_blocks, 128, 0, st>>>(a, n_pools);
  return cudaGetLastError();
}

}  // namespace

// One pass (generator.cpp:259-271 run_pass) over n_pools pools in buf_a with
// the plan words in a.plans (large format, p = 0), scratch buf_b.  Returns
// through *in_b whether the result sits in buf_b (wallace4) or buf_a
// (rotation ends where it started).
cudaError_t launch_single_pass(int dtype, const FillArgs& a, void* buf_a, void* buf_b, uint64_t n_pools,
                               cudaStream_t st, int* in_b) {
  const uint64_t N = uint64_t(1) << a.lg_log2n;
  const dim3 grid = lg_grid((N / 4 + kLgThreads - 1) / kLgThreads, n_pools);
  FillArgs b = a;
  b.lg_npools = n_pools;
  auto go = [&](auto tag) {
    using T = decltype(tag);
    T* A = static_cast<T*>(buf_a);
    T* B = static_cast<T*>(buf_b);
    switch (a.pass_type) {
      case 0: lg_pass_wallace<T, 0><<<grid, kLgThreads, 0, st>>>(b, A, B, 0, N, -1, 0, 0); break;
      case 1: lg_pass_wallace<T, 1><<<grid, kLgThreads, 0, st>>>(b, A, B, 0, N, -1, 0, 0); break;
      case 2:
        lg_pass_rotation<T, 0, 0><<<grid, kLgThreads, 0, st>>>(b, A, B, 0, N, -1, 0, 0);
        lg_pass_rotation<T, 0, 1><<<grid, kLgThreads, 0, st>>>(b, B, A, 0, N, -1, 0, 0);
        break;
      default:
        lg_pass_rotation<T, 1, 0><<<grid, kLgThreads, 0, st>>>(b, A, B, 0, N, -1, 0, 0);
        lg_pass_rotation<T, 1, 1><<<grid, kLgThreads, 0, st>>>(b, B, A, 0, N, -1, 0, 0);
    }
  };
  if (dtype == 0) go(float{});
  else go(double{});
  *in_b = a.pass_type < 2 ? 1 : 0;
  return cudaGetLastError();
}

// doubles of aux scratch per pool for pool size N
uint64_t large_aux_stride(uint64_t N) { return kAuxPart + 4 * ((N + kLgBlockVals - 1) / kLgBlockVals); }

cudaError_t launch_pool_large(int dtype, const FillArgs& a, uint64_t n_pools, cudaStream_t s) {
  return dtype == 0 ? run_large<float>(a, n_pools, s) : run_large<double>(a, n_pools, s);
}

}  // namespace wb
