#pragma once
// sm_100a kernels for the Wallace maximum-entropy normal generator.
//
//   plan_kernel  — the xoshiro256** pass-plan stream, one thread per pool
//                  (baselines.cpp:33-45 + decode_pass_plan, generator.cpp:238-257)
//   pool_kernel  — passes + emissions of one pool per CTA, pool resident in
//                  shared memory (generator.cpp:52-85, 333-376)
//   materialize_kernel — snapshot of a partially consumed emission before the
//                  pool is advanced outside fill() (Generator::out_ semantics)
//   reduce_consumer_kernel — fixed-order reduction of the fused consumer
//
// Numerics: every floating-point operation on the data path is an explicit
// round-to-nearest intrinsic (__fadd_rn, __dmul_rn, ...), and the library is
// compiled with -fmad=false, so no multiply-add is contracted — the
// reference pins -ffp-contract=off for the same reason
// (/root/reference/proj/CMakeLists.txt:10-14).
#include <cuda_runtime.h>
#include <math_constants.h>
#ifdef WB_DEBUG_TIMING
#include <cstdio>
#endif

#include <algorithm>
#include <atomic>
#include <cstdint>
#include <type_traits>
#include <utility>

#include "wallace_common.h"

namespace wb {

// ---------------------------------------------------------------------------
// compile-time geometry
// ---------------------------------------------------------------------------
constexpr uint32_t gcd_c(uint32_t a, uint32_t b) { return b ? gcd_c(b, a % b) : a; }
// transforms.cpp:161-169 default_stride: smallest odd > rows/3 coprime to rows
constexpr uint32_t default_stride_c(uint32_t rows) {
  uint32_t k = rows / 3 + 1;
  if (k % 2 == 0) ++k;
  while (gcd_c(k, rows) != 1) k += 2;
  return k;
}

// generator.cpp:286-294 default_multipliers: odd neighbours of 0.382 n and
// 0.618 n (llround of a positive value = floor(x + 0.5) for these sizes)
constexpr uint32_t near_odd_c(double x) { return static_cast<uint32_t>(x + 0.5) | 1u; }
constexpr uint32_t affine_alpha_c(uint32_t n) { return near_odd_c(0.382 * n); }
constexpr uint32_t affine_beta_c(uint32_t n) {
  return near_odd_c(0.618 * n) == affine_alpha_c(n) ? near_odd_c(0.618 * n) + 2 : near_odd_c(0.618 * n);
}

// Pass types (the template parameter PT of pool_kernel):
//   0 wallace4 + stride_transpose, 1 wallace4 + affine,
//   2 rotation + stride_transpose, 3 rotation + affine.
constexpr int pass_type_of(int family, int mixing) { return 2 * family + mixing; }

// transforms.cpp:24-35: element k of the p-th permutation of {0,1,2,3} in
// lexicographic (std::next_permutation) order, evaluated at compile time.
__host__ __device__ constexpr int perm_at(int p, int k) {
  int avail[4] = {0, 1, 2, 3};
  int n = 4;
  const int fact[4] = {6, 2, 1, 1};
  int out = 0;
  for (int pos = 0; pos <= k; ++pos) {
    const int q = p / fact[pos];
    p %= fact[pos];
    out = avail[q];
    for (int j = q; j + 1 < n; ++j) avail[j] = avail[j + 1];
    --n;
  }
  return out;
}
template <int P, int K>
struct PermAt {
  static constexpr int v = perm_at(P, K);
};
static_assert(PermAt<1, 2>::v == 3 && PermAt<23, 0>::v == 3 && PermAt<9, 3>::v == 0, "perm table");

// Build-time knobs (defaults are the tuned choice; variants are built for
// measurement by bench/tune scripts).
#ifndef WB_INPLACE_F32
#define WB_INPLACE_F32 0
#endif
#ifndef WB_INPLACE_F64
#define WB_INPLACE_F64 0
#endif
#ifndef WB_REGS_INPLACE
#define WB_REGS_INPLACE 56
#endif
// ABLATION builds only (timing experiments, wrong output): 1 = skip the
// fast emission, 2 = skip its global stores, 3 = skip the scalar chain,
// 7 = staged emission without the wait for the bulk copy's read, 8 = staged
// emission without its shared stores, 9 = staged emission without the proxy fence, 13 = latency fill without the chain,
// 14 = latency fill without the row stores, 16 = latency fill without renormalisation
#ifndef WB_ABLATE
#define WB_ABLATE 0
#endif
#ifndef WB_PREFETCH
#define WB_PREFETCH 1
#endif
#ifndef WB_D2_STG64
#define WB_D2_STG64 0
#endif
// 1: fp32 emissions shifted by 3 store [4b-1, 4b+3) (one shuffle per block)
// instead of [4b+3, 4b+7) (three shuffles)
#ifndef WB_D3_DOWN
#define WB_D3_DOWN 1
#endif
// packed f32x2 ops for fp32 (measured slower on cfg2: 3.754-3.778 vs 3.731 ms,
// FFMA2 latency lengthens each pass): bit 0 the butterfly and row factors, bit 1 the
// mean-zero emission scaling
#ifndef WB_PACKED
#define WB_PACKED 0
#endif
// 1: the host uses the bulk-emission kernel (cp.async.bulk from a shifted
// shared buffer) when every emission is the pool itself (scale 1, mean +0)
#ifndef WB_BULK
#define WB_BULK 1
#endif
// 1: emission stores at one base register + immediate group offsets
#ifndef WB_EMIT_IMM
#define WB_EMIT_IMM 0
#endif
// 1: latency kernel runs the per-emission chain in a dedicated warp (measured
// slower for one pool: the chain latency, not its placement, is the limit)
#ifndef WB_CHAINW
#define WB_CHAINW 0
#endif
// chain-warp kernels: nanoseconds a waiting warp sleeps between polls (0: spin)
#ifndef WB_CHAIN_SLEEP
#define WB_CHAIN_SLEEP 32
#endif
// 1: the consumer's four power sums as two packed f32x2 FMAs
#ifndef WB_CONS_PACKED
#define WB_CONS_PACKED 1
#endif
// latency fills: 1 = the per-emission chain runs in a second CTA of a 2-CTA
// cluster (its own SM), reading the ring over distributed shared memory
#ifndef WB_LAT_CLUSTER
#define WB_LAT_CLUSTER 1
#endif
// fp64 pass stores: 1 = swizzled (conflict-free) 32-byte block stores, for
// the throughput / the latency kernels
#ifndef WB_F64_SWZ
#define WB_F64_SWZ 1
#endif
#ifndef WB_LAT_F64_SWZ
#define WB_LAT_F64_SWZ 0
#endif
// latency fills: 1 = the owner publishes each emission's ring entry during
// the next pass, after its gathers
#ifndef WB_LAT_DEFER_PUB
#define WB_LAT_DEFER_PUB 1
#endif
// ... shared memory (KiB) each CTA of such a cluster requests: more than
// half an SM, so the two ranks run on different SMs, and enough that no
// other kernel's block (the concurrent plan kernel) shares their SMs
#ifndef WB_LAT_CLU_SMEM_KB
#define WB_LAT_CLU_SMEM_KB 120
#endif
// ... ring entries per mbarrier (batch) of the chain CTA
#ifndef WB_LAT_CBATCH
#define WB_LAT_CBATCH 4
#endif
// latency fills: emissions per release of the chain warp's ring, and the
// chain warp's sleep between polls (ns)
#ifndef WB_LAT_BATCH
#define WB_LAT_BATCH 1
#endif
#ifndef WB_LAT_POLL_NS
#define WB_LAT_POLL_NS 20
#endif
// 1: renormalisation sums on one warp (neumaier_warp) in the latency
// kernels, where the other pool buffer is dead shared memory
#ifndef WB_NEUM_WARP
#define WB_NEUM_WARP 1
#endif
// 1: fp32 mean-zero consumer on f32x2 value pairs with an unclamped
// histogram fast path (consume_chunk_pairs)
// owner_chain: chi2_draw inlined as straight-line code per method, the clamp
// and non-finite bookkeeping behind one rare branch
#ifndef WB_LEAN_CHAIN
#define WB_LEAN_CHAIN 1
#endif
// consumer: the renormalisation's two sums on the pool's warp (inline
// neumaier_warp_body) instead of one lane
#ifndef WB_CONS_NEUM
#define WB_CONS_NEUM 1
#endif
// consumer histogram: floor of the bin coordinate by one round-toward-zero
// add of 2^23 (FADD, fma pipe) where the bins are known to lie in [0, 256],
// instead of F2I.FLOOR (a quarter-rate conversion) per value
#ifndef WB_CONS_RZBIN
#define WB_CONS_RZBIN 1
#endif
#ifndef WB_CONS_PAIRS
#define WB_CONS_PAIRS 1
#endif
// ABLATION builds only: consumer without histogram (1) / moments (2) / both (3)
#ifndef WB_CONS_ABLATE
#define WB_CONS_ABLATE 0
#endif
#ifndef WB_REGS_PP
#define WB_REGS_PP 80
#endif
#ifndef WB_REGS_PP_F64
#define WB_REGS_PP_F64 WB_REGS_PP
#endif
#ifndef WB_J_F32
#define WB_J_F32 8
#endif
#ifndef WB_J_F64
#define WB_J_F64 8
#endif
// 4-blocks per processing chunk (registers hold one chunk at a time)
#ifndef WB_JC_F32
#define WB_JC_F32 8
#endif
#ifndef WB_JC_F64
#define WB_JC_F64 8
#endif
// staged emission: 1 = the owner's per-emission chain runs after the
// emission's barrier (off its critical path) instead of before it
#ifndef WB_DEFER_F32
#define WB_DEFER_F32 0
#endif
#ifndef WB_DEFER_F64
#define WB_DEFER_F64 1
#endif
// 1: the consumer kernel's register budget follows its shared-memory limit
#ifndef WB_CONS_REGS
#define WB_CONS_REGS 1
#endif
// latency fills: 1 = each thread stores its 4-blocks of the emission pass to
// the pitched row from registers (no bulk copy, no read wait on the next
// pass); 0 = one cp.async.bulk of the pool per emission
#ifndef WB_LAT_STG
#define WB_LAT_STG 1
#endif
// at least this many 4-blocks per thread in the latency kernels (2: four
// compute warps for N = 1024, so the chain warp shares its SM sub-partition
// with one compute warp instead of two -- cfg1 0.752 -> 0.727 ms per
// 2048-pass launch; 1: 0.752, 4: 0.763)
#ifndef WB_LAT_J
#define WB_LAT_J 2
#endif
#ifndef WB_HS_LUT
#define WB_HS_LUT 1
#endif
// wallace4 + stride passes: 8 of the 24 output row permutations folded into
// the order of the four column gathers (perm3_entry below), 3-way dispatch.
// Bit-exact (the parity suite passes) but measured slower: the column
// offsets are not uniform registers for ptxas, so every gather pays an
// address add, and the table lookup lengthens each pass's preamble
// (cfg2 3.13 -> 5.70 ms, profiles/r02_summary.md).  Off.
#ifndef WB_PERM3
#define WB_PERM3 0
#endif

// Kernel geometry.  The template key is log2(N) for the throughput kernel
// (many pools: few warps per pool, 8 4-blocks per thread) and log2(N) + 16
// for the latency kernel (few pools: WB_LAT_J 4-blocks per thread, up to
// 1024 threads per pool, so one pass is a short critical path).
template <typename T, int LOG2N>
struct Geo {
  static constexpr bool LAT = LOG2N >= 16;
  static constexpr int N = 1 << (LOG2N & 15);
  static constexpr int ROWS = N / 4;
  // groups (4-blocks) per thread: enough independent gathers per thread to
  // hide LDS latency, few enough warps per pool for cheap barriers.
  static constexpr int JLAT = ROWS > (WB_CHAINW ? 512 : 1024) ? ROWS / (WB_CHAINW ? 512 : 1024) : 1;
  static constexpr int JWANT = LAT ? (JLAT > WB_LAT_J ? JLAT : WB_LAT_J) : (sizeof(T) == 4 ? WB_J_F32 : WB_J_F64);
  static constexpr int J = (ROWS >= 32 * JWANT) ? JWANT : (ROWS >= 32 ? ROWS / 32 : 1);
  static constexpr int JCWANT = LAT ? J : (sizeof(T) == 4 ? WB_JC_F32 : WB_JC_F64);
  static constexpr int JC = J < JCWANT ? J : JCWANT;
  static_assert(J % JC == 0, "chunking");
  static constexpr int CT = (ROWS >= 32) ? ROWS / J : 32;  // compute threads (4-block owners)
  static constexpr int NW = CT / 32;                       // compute warps
  // the latency kernel adds a chain warp: the per-emission fp64 chain (chi2,
  // division, sqrt: ~30 dependent ops) then overlaps the next pass instead of
  // sitting on every pass's critical path
  static constexpr bool CHAINW = LAT && WB_CHAINW;
  static constexpr int THREADS = CT + (CHAINW ? 32 : 0);
  static constexpr uint32_t MASK = ROWS - 1;
  static constexpr uint32_t STRIDE = default_stride_c(ROWS) % ROWS;
  static constexpr int VEC = 16 / sizeof(T);  // elements per 128-bit store
  // the thread holding pool element N-1 (block ROWS-1, slot 3), group J-1
  static constexpr int OWNER = (NW - 1) * 32 + ((ROWS - 1) & 31);
  // in-place passes keep one pool buffer (two barriers per pass) and fit
  // twice the pools per SM; ping-pong keeps two (one barrier per pass)
  static constexpr bool INPLACE = sizeof(T) == 4 ? WB_INPLACE_F32 : WB_INPLACE_F64;
  static constexpr int BUFS = INPLACE ? 1 : 2;
  // resident CTAs per SM we ask ptxas to fit in registers: the smem limit
  // (e.g. 6 ping-pong pools of N=4096 fp32) and a register budget
  static constexpr int SMEM_PER_CTA = BUFS * N * sizeof(T) + 2048;
  static constexpr int MINB_RAW = (220 * 1024) / SMEM_PER_CTA;
  static constexpr int MINB_SMEM = MINB_RAW < 1 ? 1 : (MINB_RAW * THREADS > 2048 ? 2048 / THREADS : MINB_RAW);
  static constexpr int REG_BUDGET = INPLACE ? WB_REGS_INPLACE : (sizeof(T) == 8 ? WB_REGS_PP_F64 : WB_REGS_PP);
  static constexpr int MINB_REGS = 65536 / (THREADS * REG_BUDGET) < 1 ? 1 : 65536 / (THREADS * REG_BUDGET);
  static constexpr int MINB = LAT ? 1 : (MINB_SMEM < MINB_REGS ? MINB_SMEM : MINB_REGS);
  // affine mixing multipliers (generator.cpp:286-294 default_multipliers);
  // the host checks them against std::llround at handle creation
  static constexpr uint32_t ALPHA = affine_alpha_c(N);
  static constexpr uint32_t BETA = affine_beta_c(N);
};

// compile-time loop: f(std::integral_constant<int, i>) for i in [0, N)
template <int N, int I = 0, class F>
__device__ __forceinline__ void static_for(F&& f) {
  if constexpr (I < N) {
    f(std::integral_constant<int, I>{});
    static_for<N, I + 1>(f);
  }
}

__device__ __forceinline__ uint64_t rotl64(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
// baselines.cpp:19-24 splitmix64 (seeding of UniformState, :26-31)
__device__ __forceinline__ uint64_t splitmix64_dev(uint64_t& state) {
  uint64_t z = (state += 0x9e3779b97f4a7c15ULL);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

// ---------------------------------------------------------------------------
// explicit-rounding arithmetic
// ---------------------------------------------------------------------------
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float sub_rn(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float fma_rn(float a, float b, float c) { return __fmaf_rn(a, b, c); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub_rn(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double fma_rn(double a, double b, double c) { return __fma_rn(a, b, c); }
template <typename T> __device__ __forceinline__ T from_double(double x);
template <> __device__ __forceinline__ float from_double<float>(double x) { return __double2float_rn(x); }
template <> __device__ __forceinline__ double from_double<double>(double x) { return x; }

// Packed fp32 pairs (sm_100 FADD2/FMUL2/FFMA2): two independently rounded
// lanes per instruction.  fma(x, +-1, y) is exactly the sum y +- x (the
// product is exact), including the sign of a zero result, so the butterfly
// below is bit-identical to the scalar add_rn/sub_rn form.  ptxas folds the
// lane broadcasts, swaps and per-lane negations of pk2() into operand
// modifiers.
__device__ __forceinline__ uint64_t pk2(float lo, float hi) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ void upk2(uint64_t r, float& lo, float& hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(r));
}
__device__ __forceinline__ uint64_t fma2_rn(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
__device__ __forceinline__ uint64_t mul2_rn(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ uint64_t add2_rn(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ uint64_t add2_rz(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("add.rz.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}

// Second butterfly stage for output pair (S0, S1) of a permutation, times
// the two row factors h = (h0, h1):
//   z0 = a - d = fma(d, -1, a)     z1 = b + c = fma(c, 1, b)
//   z2 = b - c = fma(c, -1, b)     z3 = (-a) - d = fma(d, -1, -a)
// (transforms.hpp:89-103 op order).  The pair {z0, z3} shares a, so it uses
// z0 = fma(a, 1, -d), z3 = fma(a, -1, -d): one broadcast per operand.
template <int S0, int S1>
__device__ __forceinline__ void wallace_pair(float a, float b, float c, float d, uint64_t h, float& o0,
                                             float& o1) {
  uint64_t z;
  if constexpr ((S0 == 0 && S1 == 3) || (S0 == 3 && S1 == 0)) {
    z = fma2_rn(pk2(a, a), pk2(S0 == 0 ? 1.f : -1.f, S1 == 0 ? 1.f : -1.f), pk2(-d, -d));
  } else {
    auto m = [&](int s) { return (s == 1 || s == 2) ? c : d; };
    auto k = [](int s) { return s == 1 ? 1.f : -1.f; };
    auto ad = [&](int s) { return s == 0 ? a : s == 3 ? -a : b; };
    z = fma2_rn(pk2(m(S0), m(S1)), pk2(k(S0), k(S1)), pk2(ad(S0), ad(S1)));
  }
  upk2(mul2_rn(z, h), o0, o1);
}

// out = x * scale + mean with two roundings (generator.cpp:366-368).  When
// mean is +0.0, fma(x, scale, +0) rounds x*scale once and adds +0 exactly,
// which is bit-identical to the two-step form (including -0 + 0 = +0).
template <typename T>
__device__ __forceinline__ T emit_value(T x, T scale, T mean, bool mean_zero) {
  return mean_zero ? fma_rn(x, scale, T(0)) : add_rn(mul_rn(x, scale), mean);
}

// ---------------------------------------------------------------------------
// shared-memory vector helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ void sts4(float* p, float a, float b, float c, float d) {
  *reinterpret_cast<float4*>(p) = make_float4(a, b, c, d);
}
__device__ __forceinline__ void sts4(double* p, double a, double b, double c, double d) {
  reinterpret_cast<double2*>(p)[0] = make_double2(a, b);
  reinterpret_cast<double2*>(p)[1] = make_double2(c, d);
}
// streaming (evict-first) global stores: the output is written once
__device__ __forceinline__ void stg_vec(float* p, const float* v) {
  __stcs(reinterpret_cast<float4*>(p), make_float4(v[0], v[1], v[2], v[3]));
}
__device__ __forceinline__ void stg_vec(double* p, const double* v) {
  __stcs(reinterpret_cast<double2*>(p), make_double2(v[0], v[1]));
}
template <typename T>
__device__ __forceinline__ void stg1(T* p, T v) { __stcs(p, v); }
// streaming 128-bit store at base + OFF bytes (OFF an immediate: one base
// register serves every group of a chunk)
template <int OFF>
__device__ __forceinline__ void stg_vec_at(uint64_t base, const float* v) {
  // no "memory" clobber: nothing in the kernel reads the output, and a
  // clobber would pin the scheduler (all stores bunched at the end)
  asm("st.global.cs.v4.f32 [%0+%1], {%2, %3, %4, %5};" ::"l"(base), "n"(OFF), "f"(v[0]), "f"(v[1]),
      "f"(v[2]), "f"(v[3]));
}
template <int OFF>
__device__ __forceinline__ void stg_vec_at(uint64_t base, const double* v) {
  asm("st.global.cs.v2.f64 [%0+%1], {%2, %3};" ::"l"(base), "n"(OFF), "d"(v[0]), "d"(v[1]));
}
#if WB_ABLATE == 2
#define stg_vec(p, v) do { if (reinterpret_cast<uintptr_t>(p) == 1) stg_vec(p, v); } while (0)
#endif
#if WB_ABLATE == 6
// timing-only: no global stores; the values stay live through an XOR fold
// (one conditional store per emission chunk keeps the fold itself alive)
__device__ uint32_t g_ablate_sink;
__device__ __forceinline__ uint32_t ablate_fold(const float* v) {
  return __float_as_uint(v[0]) ^ __float_as_uint(v[1]) ^ __float_as_uint(v[2]) ^ __float_as_uint(v[3]);
}
__device__ __forceinline__ uint32_t ablate_fold(const double* v) {
  return __float_as_uint(float(v[0])) ^ __float_as_uint(float(v[1]));
}
__device__ __forceinline__ uint32_t ablate_fold1(float v) { return __float_as_uint(v); }
__device__ __forceinline__ uint32_t ablate_fold1(double v) { return __float_as_uint(float(v)); }
#endif

// ---------------------------------------------------------------------------
// chi-squared draw and the per-emission scalar chain (chi2.cpp:27-59,
// generator.cpp:358-364, 373-375).  All in double, explicit rounding.
// ---------------------------------------------------------------------------
static __device__ double chi2_draw(double x, const Chi2Consts& c, uint32_t& clamped, uint32_t& flags) {
  if (!isfinite(x)) flags |= kFlagChi2NonFinite;
  double s;
  if (c.method == 0) {
    const double y = __dadd_rn(x, c.shift_c);
    s = __dmul_rn(__dmul_rn(0.5, y), y);
  } else if (c.method == 1) {
    const double y = __dadd_rn(__dmul_rn(c.wh_sqrt_d, x), c.wh_one_m_d);
    s = __dmul_rn(__dmul_rn(__dmul_rn(c.nu, y), y), y);
  } else {
    // a * (x*x - 1) + sqrt(2(nu - a^2)) * x + nu, evaluated left to right
    const double t1 = __dmul_rn(c.a, __dsub_rn(__dmul_rn(x, x), 1.0));
    const double t2 = __dmul_rn(c.cubic_c, x);
    s = __dadd_rn(__dadd_rn(t1, t2), c.nu);
  }
  if (s < c.floor_v) {
    ++clamped;
    return c.floor_v;
  }
  return s;
}

// 128-bit shared store of p ? (b0, b1) : (a0, a1), selected as 32-bit halves
#ifndef WB_F64_SWZ_B32
#define WB_F64_SWZ_B32 1
#endif
__device__ __forceinline__ void sts_sel_b32(uint32_t addr, bool p, double a0, double a1, double b0, double b1) {
  const uint32_t r0 = p ? uint32_t(__double2loint(b0)) : uint32_t(__double2loint(a0));
  const uint32_t r1 = p ? uint32_t(__double2hiint(b0)) : uint32_t(__double2hiint(a0));
  const uint32_t r2 = p ? uint32_t(__double2loint(b1)) : uint32_t(__double2loint(a1));
  const uint32_t r3 = p ? uint32_t(__double2hiint(b1)) : uint32_t(__double2hiint(a1));
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(r0), "r"(r1), "r"(r2), "r"(r3) : "memory");
}

struct SState {
  double reserved_prev;
  double sum_sq;
  double S[2];
  double r[2];
  double scale[2];
  double cur_scale;  // scale of the emission being drained by `lead`
  double last_chi2;
  double last_r;
  double last_scale;
  double renorm_k;
  uint32_t clamp;
  uint32_t flags;
  int32_t renorm_ok;
  uint32_t zero_seen;  // an exact zero was emitted by bulk stores (patch needed)
  uint32_t x_last_bulk_set;  // bulk kernels: the last emission was a fast one
  double x_last_bulk;        // ... and its pool element N-1
  uint32_t ready;      // chain-warp kernels: S/r/scale of every emission <= ready published
  uint32_t produced;   // kModeFillLat: emissions whose (x_last, sum_sq) are in the ring
  uint32_t end_off;    // kModeFillLat: the compute threads' final buffer offset
  int32_t closed;      // owner_chain closed this slot last: last_chi2 / last_scale are its S / scale
};

// S, r, scale of the emission in `slot` from the current reserved value.
__device__ __forceinline__ void chain_draw(SState& s, int slot, const Chi2Consts& c, double sigma) {
  const double S = c.disable ? s.sum_sq : chi2_draw(s.reserved_prev, c, s.clamp, s.flags);
  const double r = s.sum_sq > 0.0 ? __dsqrt_rn(__ddiv_rn(S, s.sum_sq)) : 0.0;
  s.S[slot] = S;
  s.r[slot] = r;
  s.scale[slot] = __dmul_rn(sigma, r);
}
// after a renormalization changed sum_sq: S is kept (disable_chi2 re-reads it)
__device__ __forceinline__ void chain_rescale(SState& s, int slot, const Chi2Consts& c, double sigma) {
  if (c.disable) s.S[slot] = s.sum_sq;
  const double r = s.sum_sq > 0.0 ? __dsqrt_rn(__ddiv_rn(s.S[slot], s.sum_sq)) : 0.0;
  s.r[slot] = r;
  s.scale[slot] = __dmul_rn(sigma, r);
}
// bookkeeping at the end of emission `slot` (generator.cpp:373-375)
__device__ __forceinline__ void chain_close(SState& s, int slot, double x_last) {
  s.closed = -1;
  s.reserved_prev = __dmul_rn(x_last, s.r[slot]);
  s.last_chi2 = s.S[slot];
  s.last_r = s.r[slot];
  s.last_scale = s.scale[slot];
}

// chain_close + chain_draw of the owner thread (the one holding pool element
// N-1), with one shared-memory round trip: r of this emission and sum_sq
// are loaded together up front, and the dependent fp64 chain (reserved,
// chi2, S/sum_sq, sqrt, scale) then runs in registers; the results are
// stored without being read back.  last_chi2 / last_scale are S / scale of
// `slot` as drawn (or rescaled) and stay where they are; the epilogue and
// the next close read them from the slot (SState::closed).
__device__ __forceinline__ void owner_chain(SState& s, int slot, double x_last, bool next, const Chi2Consts& c,
                                            double sigma) {
  const double r_e = s.r[slot];
  const double ss = s.sum_sq;
  // generator.cpp:373-375
  const double reserved = __dmul_rn(x_last, r_e);
  s.reserved_prev = reserved;
  s.last_r = r_e;
  s.closed = slot;
  if (next) {
    // generator.cpp:358-364 for the next emission
    double S;
    if (WB_LEAN_CHAIN && !c.disable) {
      // chi2_draw's arithmetic with the method as a uniform branch around
      // straight-line code; the clamp count and the non-finite flag (rare)
      // behind one test: v is finite and >= floor in every common case
      double v;
      if (c.method == 2) {
        const double t1 = __dmul_rn(c.a, __dsub_rn(__dmul_rn(reserved, reserved), 1.0));
        v = __dadd_rn(__dadd_rn(t1, __dmul_rn(c.cubic_c, reserved)), c.nu);
      } else if (c.method == 0) {
        const double y = __dadd_rn(reserved, c.shift_c);
        v = __dmul_rn(__dmul_rn(0.5, y), y);
      } else {
        const double y = __dadd_rn(__dmul_rn(c.wh_sqrt_d, reserved), c.wh_one_m_d);
        v = __dmul_rn(__dmul_rn(__dmul_rn(c.nu, y), y), y);
      }
      S = v;
      if (!(v >= c.floor_v && fabs(v) < CUDART_INF)) {
        if (!isfinite(reserved)) s.flags |= kFlagChi2NonFinite;
        if (v < c.floor_v) {
          ++s.clamp;
          S = c.floor_v;
        }
      }
    } else {
      S = c.disable ? ss : chi2_draw(reserved, c, s.clamp, s.flags);
    }
    const double r = ss > 0.0 ? __dsqrt_rn(__ddiv_rn(S, ss)) : 0.0;
    s.S[slot ^ 1] = S;
    s.r[slot ^ 1] = r;
    s.scale[slot ^ 1] = __dmul_rn(sigma, r);
  }
}

__device__ __forceinline__ uint32_t ld_acquire_cta(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.cta.shared::cta.u32 %0, [%1];"
               : "=r"(v)
               : "r"(static_cast<uint32_t>(__cvta_generic_to_shared(p)))
               : "memory");
  return v;
}
__device__ __forceinline__ void st_release_cta(uint32_t* p, uint32_t v) {
  asm volatile("st.release.cta.shared::cta.u32 [%0], %1;" ::"r"(
                   static_cast<uint32_t>(__cvta_generic_to_shared(p))),
               "r"(v)
               : "memory");
}

// Thread-block-cluster helpers (the latency fill's chain CTA reads the
// compute CTA's ring over distributed shared memory).
__device__ __forceinline__ void st_release_cluster(uint32_t* p, uint32_t v) {
  asm volatile("st.release.cluster.shared::cta.u32 [%0], %1;" ::"r"(
                   static_cast<uint32_t>(__cvta_generic_to_shared(p))),
               "r"(v)
               : "memory");
}
// shared::cluster address of `p` (a shared variable) in cluster CTA `rank`
__device__ __forceinline__ uint32_t dsmem_addr(const void* p, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;"
               : "=r"(r)
               : "r"(static_cast<uint32_t>(__cvta_generic_to_shared(p))), "r"(rank));
  return r;
}
__device__ __forceinline__ uint32_t ld_acquire_cluster(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.acquire.cluster.shared::cluster.u32 %0, [%1];" : "=r"(v) : "r"(addr) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t ld_dsmem_u32(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared::cluster.u32 %0, [%1];" : "=r"(v) : "r"(addr) : "memory");
  return v;
}
__device__ __forceinline__ void ld_dsmem_f64x2(uint32_t addr, double& x, double& y) {
  asm volatile("ld.shared::cluster.v2.f64 {%0, %1}, [%2];" : "=d"(x), "=d"(y) : "r"(addr) : "memory");
}
__device__ __forceinline__ void st_dsmem_f64(uint32_t addr, double v) {
  asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(addr), "d"(v) : "memory");
}
__device__ __forceinline__ void st_dsmem_u32(uint32_t addr, uint32_t v) {
  asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
// Remote 16-byte store into cluster CTA memory that completes `bytes` on
// the destination CTA's mbarrier (no fence on the producer's path).
__device__ __forceinline__ void st_async_f64x2(uint32_t raddr, double x, double y, uint32_t rmbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::"r"(raddr),
               "d"(x), "d"(y), "r"(rmbar)
               : "memory");
}
__device__ __forceinline__ void mbar_init(uint64_t* m, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(m))),
               "r"(count)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* m, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                   static_cast<uint32_t>(__cvta_generic_to_shared(m))),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait_parity(uint64_t* m, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WB_MBAR_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WB_MBAR_WAIT_%=;\n}" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(m))),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void fence_mbarrier_init_cluster() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

// every thread of every CTA of the cluster; orders prior shared (and
// distributed shared) accesses before those after it
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// Barrier of the pass loop: the whole CTA, or (NB) named barrier 1 over the
// NT compute threads when a decoupled chain warp runs beside the passes.
template <bool NB, int NT>
__device__ __forceinline__ void loop_bar() {
  if constexpr (NB) asm volatile("bar.sync 1, %0;" ::"n"(NT) : "memory");
  else __syncthreads();
}

// generator.cpp:20-34 recompute_sum_sq — sequential Neumaier, one thread.
// SELECT: branch-free form — the reference's two branches are the same
// expression with the operands ordered by magnitude, (big - t) + small, so
// only the running sum's 8-cycle DADD dependency is on the critical path
// (used by the latency kernel, where the renormalisation is on the critical
// path; the throughput kernel keeps the compact form for register pressure).
template <bool SELECT>
__device__ __forceinline__ void neumaier_add(double& sum, double& comp, double x) {
  const double term = __dmul_rn(x, x);
  const double t = __dadd_rn(sum, term);
  if constexpr (SELECT) {
    const bool sum_big = fabs(sum) >= fabs(term);
    const double big = sum_big ? sum : term;
    const double small = sum_big ? term : sum;
    comp = __dadd_rn(comp, __dadd_rn(__dsub_rn(big, t), small));
  } else if (fabs(sum) >= fabs(term)) {
    comp = __dadd_rn(comp, __dadd_rn(__dsub_rn(sum, t), term));
  } else {
    comp = __dadd_rn(comp, __dadd_rn(__dsub_rn(term, t), sum));
  }
  sum = t;
}
template <typename T, bool VECTOR_LOADS>
__device__ double neumaier_sq(const T* v, int n) {
  double sum = 0.0, comp = 0.0;
  if constexpr (VECTOR_LOADS && sizeof(T) == 4) {
    const float4* q = reinterpret_cast<const float4*>(v);
#pragma unroll 4
    for (int i = 0; i < n / 4; ++i) {
      const float4 f = q[i];
      neumaier_add<VECTOR_LOADS>(sum, comp, f.x);
      neumaier_add<VECTOR_LOADS>(sum, comp, f.y);
      neumaier_add<VECTOR_LOADS>(sum, comp, f.z);
      neumaier_add<VECTOR_LOADS>(sum, comp, f.w);
    }
  } else if constexpr (VECTOR_LOADS) {
    const double2* q = reinterpret_cast<const double2*>(v);
#pragma unroll 4
    for (int i = 0; i < n / 2; ++i) {
      const double2 f = q[i];
      neumaier_add<VECTOR_LOADS>(sum, comp, f.x);
      neumaier_add<VECTOR_LOADS>(sum, comp, f.y);
    }
  } else {
#pragma unroll 8
    for (int i = 0; i < n; ++i) neumaier_add<false>(sum, comp, static_cast<double>(v[i]));
  }
  return __dadd_rn(sum, comp);
}

// generator.cpp:20-34 recompute_sum_sq on one warp, bit-identical to the
// sequential loop.  Only the two running sums are sequential: sum_i =
// fl(sum_{i-1} + x_i^2) and comp_i = fl(comp_{i-1} + err_i).  The reference's
// err_i = (big - t) + small (big/small: sum_{i-1} and the term ordered by
// magnitude, ties to sum) is Fast2Sum's exact rounding error of that
// addition, so it depends only on (sum_{i-1}, term_i, sum_i) and is formed in
// parallel.  Per tile of 32 elements: the lanes square their element (terms
// to scr), every lane runs the same sum chain over the tile from shared
// memory (two terms per 128-bit broadcast load) and records the partial sums,
// the lanes form the tile's errors, and the comp chain of an earlier tile
// runs interleaved with the sum chain (two independent DADD chains); the
// next tile's terms and the previous tile's errors are formed mid-chain, so
// their latency hides behind the chains.  1024 fp32 values: 14.8k cycles
// against 23.4k for the one-thread loop (tools/probes/neum_probe.cu; the
// floor is 1024 dependent DADDs = 8.4k).  scr: 288 doubles of dead shared
// memory (16-byte aligned).  Out of line: its registers stay out of the pass
// loop's allocation.
//
// One tile's sum chain over tb (32 terms) into pb, beside (EC) the comp
// chain over an earlier tile's errors eb; loads run 8 elements ahead; mid()
// runs after the first 8 elements (in-order issue: work placed there
// overlaps the chains instead of delaying their start).
template <bool SC, bool EC, class Mid>
__device__ __forceinline__ void neumaier_tile(const double* tb, double* pb, const double* eb, double& sum,
                                              double& comp, Mid&& mid) {
  double2 t[4], e[4];
#pragma unroll
  for (int g = 0; g < 4; ++g) {
    if (SC) t[g] = reinterpret_cast<const double2*>(tb)[g];
    if (EC) e[g] = reinterpret_cast<const double2*>(eb)[g];
  }
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const int g = i & 3;
    double2 tn, en;
    if (i + 4 < 16) {
      if (SC) tn = reinterpret_cast<const double2*>(tb)[i + 4];
      if (EC) en = reinterpret_cast<const double2*>(eb)[i + 4];
    }
    if (SC) {
      const double s0 = __dadd_rn(sum, t[g].x);
      sum = __dadd_rn(s0, t[g].y);
      reinterpret_cast<double2*>(pb)[i] = make_double2(s0, sum);
    }
    if (EC) comp = __dadd_rn(__dadd_rn(comp, e[g].x), e[g].y);
    if (i + 4 < 16) {
      if (SC) t[g] = tn;
      if (EC) e[g] = en;
    }
    if (i == 3) mid();
  }
}

template <typename T, int N>
__device__ __forceinline__ double neumaier_warp_body(const T* v, double* scr, int lane) {
  static_assert(N % 32 == 0 && N >= 128, "whole tiles, at least four");
  constexpr int NT = N / 32;
  // scr: three slots of [terms 32 | partial sums 32 | errors 32], slot = tile mod 3
  auto tb = [&](int k) { return scr + (k % 3) * 96; };
  double sum = 0.0, comp = 0.0;
  double start_cur = 0.0;  // sum before the tile whose chain ran last
  // one pipeline step at tile k: the sum chain of k, the comp chain of k-2,
  // and (loads issued before, the arithmetic mid-chain) the terms of k+1 and
  // the errors of k-1
  auto step = [&](int k, auto TM, auto ER, auto SC, auto EC) {
    T xv = T(0);
    double term = 0.0, prev = 0.0, cur = 0.0;
    if constexpr (decltype(TM)::value) xv = v[32 * (k + 1) + lane];
    if constexpr (decltype(ER)::value) {
      const double* t = tb(k - 1);
      term = t[lane];
      prev = lane == 0 ? start_cur : t[32 + lane - 1];
      cur = t[32 + lane];
    }
    start_cur = sum;
    neumaier_tile<decltype(SC)::value, decltype(EC)::value>(tb(k), tb(k) + 32, tb(k - 2 + 3) + 64, sum, comp, [&] {
      if constexpr (decltype(TM)::value) {
        const double x = static_cast<double>(xv);
        tb(k + 1)[lane] = __dmul_rn(x, x);
      }
      if constexpr (decltype(ER)::value) {
        const bool sum_big = fabs(prev) >= fabs(term);
        const double big = sum_big ? prev : term;
        const double small = sum_big ? term : prev;
        tb(k - 1)[64 + lane] = __dadd_rn(__dsub_rn(big, cur), small);
      }
    });
    __syncwarp();
  };
  using Y = std::true_type;
  using F = std::false_type;
  {  // terms of tile 0
    const double x = static_cast<double>(v[lane]);
    tb(0)[lane] = __dmul_rn(x, x);
    __syncwarp();
  }
  step(0, Y{}, F{}, Y{}, F{});
  step(1, Y{}, Y{}, Y{}, F{});
  for (int k = 2; k < NT - 1; ++k) step(k, Y{}, Y{}, Y{}, Y{});
  step(NT - 1, F{}, Y{}, Y{}, Y{});
  step(NT, F{}, Y{}, F{}, Y{});
  step(NT + 1, F{}, F{}, F{}, Y{});
  return __dadd_rn(sum, comp);
}
// Out of line (latency kernels: its registers stay out of the pass loop's
// allocation) or inline (the consumer kernel: one warp per pool, nothing else
// is live across the renormalisation but the accumulators, and a call's ABI
// would spill them).
template <typename T, int N>
__device__ __noinline__ double neumaier_warp(const T* v, double* scr, int lane) {
  return neumaier_warp_body<T, N>(v, scr, lane);
}

// generator.cpp:345-351 renormalize_.  Contains block barriers: call from
// all threads.
// LAT: the latency kernel (one pool per SM, the renormalisation is on the
// critical path: vector loads, out of line); otherwise inline scalar loads.
// scr: dead shared memory (the other pool buffer) for the warp-parallel sum
// (latency kernels only: in the throughput kernels other pools hide the
// one-thread loop, and the call costs more than it saves there), or nullptr.
template <typename T, int N, int THREADS, bool LAT, bool NB = false, bool INL = false>
__device__ __forceinline__ void renormalize(T* cur, SState& s, int tid, double* scr = nullptr) {
  constexpr bool PAR = WB_NEUM_WARP && (LAT || INL || WB_NEUM_WARP == 2) && N >= 128 && N % 32 == 0 &&
                       N * sizeof(T) >= 288 * sizeof(double);
  const bool par = PAR && scr != nullptr;
  auto warp_sum = [&]() -> double {
    if constexpr (!PAR) return 0.0;
    else if constexpr (INL) return neumaier_warp_body<T, N>(cur, scr, tid);
    else return neumaier_warp<T, N>(cur, scr, tid);
  };
  if (par ? tid < 32 : tid == 0) {
    double ss;
    if constexpr (PAR) ss = par ? warp_sum() : neumaier_sq<T, LAT>(cur, N);
    else ss = neumaier_sq<T, LAT>(cur, N);
    if (tid == 0) {
      // generator.cpp:347 skips only ss <= 0: a NaN sum still rescales (by NaN)
      s.renorm_ok = !(ss <= 0.0);
      s.renorm_k = s.renorm_ok ? __dsqrt_rn(__ddiv_rn(static_cast<double>(N), ss)) : 0.0;
    }
  }
  loop_bar<NB, THREADS>();
  if (s.renorm_ok) {
    const double k = s.renorm_k;
    for (int i = tid; i < N; i += THREADS)
      cur[i] = from_double<T>(__dmul_rn(static_cast<double>(cur[i]), k));
    loop_bar<NB, THREADS>();
    if (par ? tid < 32 : tid == 0) {
      double ss;
      if constexpr (PAR) ss = par ? warp_sum() : neumaier_sq<T, LAT>(cur, N);
      else ss = neumaier_sq<T, LAT>(cur, N);
      if (tid == 0) s.sum_sq = ss;
    }
  }
  loop_bar<NB, THREADS>();
}

// ---------------------------------------------------------------------------
// fused consumer accumulators (config 5)
// ---------------------------------------------------------------------------
template <typename T>
struct Consumer {
  double s1 = 0, s2 = 0, s3 = 0, s4 = 0;  // per-thread totals (fp64)
  T a1 = 0, a2 = 0, a3 = 0, a4 = 0;       // per-emission partials (T)
  // fp32 pair path (consume_chunk_pairs): per-emission partials of value
  // pairs, one f32x2 register each (lanes: even / odd slots of a block)
  uint64_t p1 = 0, p2 = 0, p3 = 0, p4 = 0;
  uint32_t* hist;  // shared, 258 bins (under, 256, over)
  __device__ __forceinline__ void add(T x) {
    if (WB_CONS_ABLATE != 2 && WB_CONS_ABLATE != 3) {
      const T x2 = mul_rn(x, x);
      if constexpr (sizeof(T) == 4 && WB_CONS_PACKED) {
        // (a1, a2) += (x, x^2) and (a3, a4) += (x^2 * x, x^2 * x^2) as two
        // packed f32x2 FMAs (the add as fma(.., 1, ..): no contraction risk)
        uint64_t p12 = pk2(a1, a2), p34 = pk2(a3, a4);
        p12 = fma2_rn(pk2(x, x2), pk2(1.0f, 1.0f), p12);
        p34 = fma2_rn(pk2(x2, x2), pk2(x, x2), p34);
        upk2(p12, a1, a2);
        upk2(p34, a3, a4);
      } else {
        a1 = add_rn(a1, x);
        a2 = add_rn(a2, x2);
        a3 = fma_rn(x2, x, a3);
        a4 = fma_rn(x2, x2, a4);
      }
    }
    if (WB_CONS_ABLATE != 1 && WB_CONS_ABLATE != 3) {
      // bin = floor((x + 8) * 16) in T, clamped to [-1, 256] (under / over);
      // fl(fl(x + 8) * 16) == fma(x, 16, 128): scaling by 16 is exact
      const T t = fma_rn(x, T(16), T(128));
      int bin = sizeof(T) == 4 ? __float2int_rd(static_cast<float>(t)) : __double2int_rd(static_cast<double>(t));
      bin = max(-1, min(bin, 256));
      atomicAdd(&hist[bin + 1], 1u);
    }
  }
  __device__ __forceinline__ void add_group(const T* y, int n) {
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (k < n) add(y[k]);
  }
  // fold the per-emission partials into the fp64 totals
  __device__ __forceinline__ void flush() {
    s1 += static_cast<double>(a1);
    s2 += static_cast<double>(a2);
    s3 += static_cast<double>(a3);
    s4 += static_cast<double>(a4);
    a1 = a2 = a3 = a4 = T(0);
    if constexpr (sizeof(T) == 4 && WB_CONS_PAIRS) {
      float lo, hi;
      upk2(p1, lo, hi);
      s1 += static_cast<double>(lo) + static_cast<double>(hi);
      upk2(p2, lo, hi);
      s2 += static_cast<double>(lo) + static_cast<double>(hi);
      upk2(p3, lo, hi);
      s3 += static_cast<double>(lo) + static_cast<double>(hi);
      upk2(p4, lo, hi);
      s4 += static_cast<double>(lo) + static_cast<double>(hi);
      p1 = p2 = p3 = p4 = 0;
    }
  }
};

// ---------------------------------------------------------------------------
// The fast emission (full emissions: all N-1 values): values are in
// registers in pool order; 128-bit aligned streaming stores, shifted by DELTA
// elements with warp shuffles (the emission start e*(N-1) is misaligned in
// 3 of 4 emissions).
//
// Thread t owns blocks b_j = (warp*J + j)*32 + lane.  The aligned chunk
// [4b+DELTA, 4b+DELTA+4) holds b's tail and the first DELTA values of block
// b+1, which lives in lane+1 — or, for lane 31, in lane 0 of group j+1.  So
// lanes 0..30 store their group-j chunk as soon as group j is shuffled, and
// lane 31 stores its group-(j-1) chunk when group j's shuffle delivers lane
// 0's head.  Lane 31's last group and lane 0's first head straddle two warps
// and use scalar stores.  Element N-1 is never emitted (generator.cpp:366).
// ---------------------------------------------------------------------------
#if WB_ABLATE == 6
#define stg_vec(p, v) do { ablate_x ^= ablate_fold(v); } while (0)
#define stg1(p, v) do { ablate_x ^= ablate_fold1(v); } while (0)
#endif
template <typename T>
__device__ __forceinline__ bool is_neg_zero(T x) {
  if constexpr (sizeof(T) == 4) return __float_as_uint(x) == 0x80000000u;
  else return static_cast<unsigned long long>(__double_as_longlong(x)) == 0x8000000000000000ull;
}

// SMD (shared destination): instead of emitting y = x*scale + mean to global
// memory, write the raw pool values x themselves -- all N of them, element
// N-1 included -- into a shared buffer whose layout is shifted by the
// emission's misalignment (see "Bulk emission"); zf collects whether any
// value is an exact -0 (which the emission must turn into +0).
//
// STAGED (staged emission): the scaled values y go to a shared buffer in the
// same shifted layout (gbase is then that buffer's element 0), except the
// scalar head/tail values at the warp's ends, which go straight to global
// memory at g1 (the emission's element 0 there).  Every 16-byte vector a warp
// writes lies inside its own segment, so each warp can send its segment with
// one bulk copy (staged_range).
template <typename T, int LOG2N, int DELTA, bool MZ, bool SMD = false, bool STAGED = false>
__device__ __forceinline__ void emit_chunk(const T (&X)[Geo<T, LOG2N>::JC][4], int c0, T (&prev)[4],
                                           T* gbase, T sc, T mean, int lane, int warp,
                                           int jfirst = 0, uint32_t* zf = nullptr, T* g1 = nullptr) {
  using G = Geo<T, LOG2N>;
  constexpr int J = G::J, JC = G::JC, VEC = G::VEC;
  static_assert(!(SMD && STAGED), "one destination kind");
  constexpr uint32_t NLIM = SMD ? G::N : G::N - 1;  // elements written
  static_assert(DELTA < VEC, "shift");
#if WB_ABLATE == 6
  uint32_t ablate_x = 0;
  struct Flush {
    uint32_t& x;
    __device__ ~Flush() {
      if (x == 0x9e3779b9u) g_ablate_sink = x;
    }
  } ablate_flush{ablate_x};
#endif
  auto put_vec = [&](T* p, const T* v) {
    if constexpr (SMD || STAGED) {
      if constexpr (sizeof(T) == 4) *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
      else *reinterpret_cast<double2*>(p) = make_double2(v[0], v[1]);
    } else {
      stg_vec(p, v);
    }
  };
  // a 4-value block as VEC-wide stores; fp64 into shared memory: the two
  // 16-byte halves at a 32-byte lane stride would hit each bank twice per
  // 8-lane phase, so lanes with bit 2 set store the upper half first
  // (lanes l and l+4 then cover complementary banks, as in run_pass)
  auto put_block = [&](T* p, const T* w) {
    if constexpr (VEC == 2 && (SMD || STAGED)) {
      const bool sw = (lane & 4) != 0;
      if constexpr (WB_F64_SWZ_B32) {
        const uint32_t a0 = static_cast<uint32_t>(__cvta_generic_to_shared(p));
        sts_sel_b32(a0 + (sw ? 16u : 0u), sw, w[0], w[1], w[2], w[3]);
        sts_sel_b32(a0 + (sw ? 0u : 16u), sw, w[2], w[3], w[0], w[1]);
      } else {
        const T fa[2] = {sw ? w[2] : w[0], sw ? w[3] : w[1]};
        const T fb[2] = {sw ? w[0] : w[2], sw ? w[1] : w[3]};
        put_vec(p + (sw ? 2 : 0), fa);
        put_vec(p + (sw ? 0 : 2), fb);
      }
    } else {
#pragma unroll
      for (int v = 0; v < 4; v += VEC) put_vec(p + v, w + v);
    }
  };
  auto put1 = [&](T* p, T v) {
    if constexpr (SMD) *p = v;
    else if constexpr (STAGED) stg1(g1 + (p - gbase), v);
    else stg1(p, v);
  };
  const bool l31 = lane == 31;
  const uint32_t b0 = warp * J * 32 + lane;  // this thread's block in group 0
  // Every lane's chunk of group j starts at cbase + 128 j elements: lanes
  // 0..30 store their own group-j chunk, lane 31 its group-(j-1) chunk, so
  // its base is one group (128 elements) lower.  The group offsets are then
  // immediates of the store instructions.
  const uint64_t cbase = reinterpret_cast<uint64_t>(gbase) +
                         sizeof(T) * (4ull * (b0 + 32u * c0) + DELTA) -
                         ((DELTA > 0 && l31) ? 128u * sizeof(T) : 0u);
  auto store_group = [&](auto jjc, const T* c) {
    constexpr int JJ = decltype(jjc)::value;
#pragma unroll
    for (int v = 0; v < 4; v += VEC) {
      if (v == 0) stg_vec_at<JJ * 128 * int(sizeof(T))>(cbase, c);
      else stg_vec_at<JJ * 128 * int(sizeof(T)) + 16>(cbase, c + 2);
    }
  };
  (void)store_group;
  uint32_t z = 0;
#pragma unroll
  for (int jj = 0; jj < JC; ++jj) {
    const int j = c0 + jj;
    if (j < jfirst) continue;  // groups before jfirst are emitted elsewhere
    const uint32_t b = b0 + 32 * j;
    T y[4];
    if constexpr (SMD) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        y[k] = X[jj][k];
        z |= is_neg_zero(y[k]) ? 1u : 0u;
      }
    } else if constexpr ((WB_PACKED & 2) && MZ && sizeof(T) == 4 && !STAGED) {
      // (only the mean-zero form: ptxas contracts a packed mul.rn + add.rn
      // pair into one FFMA2 despite the explicit rounding modifiers)
      const uint64_t s2 = pk2(sc, sc);
#pragma unroll
      for (int h = 0; h < 4; h += 2)
        upk2(fma2_rn(pk2(X[jj][h], X[jj][h + 1]), s2, pk2(0.f, 0.f)), y[h], y[h + 1]);
    } else {
#pragma unroll
      for (int k = 0; k < 4; ++k) y[k] = MZ ? fma_rn(X[jj][k], sc, T(0)) : add_rn(mul_rn(X[jj][k], sc), mean);
    }
    if constexpr (!SMD && !STAGED && WB_D2_STG64 && sizeof(T) == 4 && DELTA == 2) {
      // global(4b) is 8-byte aligned: two float2 stores of the own block,
      // no neighbour values needed
      if (b != G::ROWS - 1) {
        __stcs(reinterpret_cast<float2*>(gbase + 4 * b), make_float2(y[0], y[1]));
        __stcs(reinterpret_cast<float2*>(gbase + 4 * b + 2), make_float2(y[2], y[3]));
      } else {
        __stcs(reinterpret_cast<float2*>(gbase + 4 * b), make_float2(y[0], y[1]));
        stg1(gbase + 4 * b + 2, y[2]);
      }
    } else if constexpr (WB_D3_DOWN && VEC == 4 && DELTA == 3) {
      // shift the other way: the aligned chunk [4b-1, 4b+3) is the previous
      // block's last value (lane-1, or for lane 0 lane 31 of group j-1, kept
      // in prev[0]) and this block's first three -- one shuffle, and the
      // pool's last element X[N-1] = y[3] of block ROWS-1 falls outside
      const T s = __shfl_sync(0xffffffffu, y[3], (lane + 31) & 31);
      if (lane == 0 && j == jfirst) {  // head of this warp: the value before is the previous warp's
        put1(gbase + 4 * b + 0, y[0]);
        put1(gbase + 4 * b + 1, y[1]);
        put1(gbase + 4 * b + 2, y[2]);
      } else {
        const T c[4] = {lane == 0 ? prev[0] : s, y[0], y[1], y[2]};
        put_vec(gbase + 4 * b - 1, c);
      }
      if (lane == 31 && j == J - 1 && 4 * b + 3 < NLIM)
        put1(gbase + 4 * b + 3, y[3]);  // tail of this warp: the next warp's head is scalar
      prev[0] = s;
    } else if constexpr (DELTA == 0) {
      if (SMD || b != G::ROWS - 1) {
        if constexpr (WB_EMIT_IMM && !SMD && !STAGED) {
          static_for<JC>([&](auto jjc) {
            if (decltype(jjc)::value == jj) store_group(jjc, y);
          });
        } else {
          put_block(gbase + 4 * b, y);
        }
      } else {
        put1(gbase + 4 * b + 0, y[0]);
        put1(gbase + 4 * b + 1, y[1]);
        put1(gbase + 4 * b + 2, y[2]);
      }
    } else {
      T sh[DELTA];
#pragma unroll
      for (int t = 0; t < DELTA; ++t) sh[t] = __shfl_sync(0xffffffffu, y[t], (lane + 1) & 31);
      T c[4];
#pragma unroll
      for (int m = 0; m < 4; ++m) {
        if (DELTA + m < 4) c[m] = l31 ? prev[(DELTA + m) & 3] : y[(DELTA + m) & 3];
        else c[m] = sh[(DELTA + m - 4) & (DELTA > 0 ? 3 : 0)];
      }
      if (!(l31 && j == jfirst)) {
        if constexpr (WB_EMIT_IMM && !SMD && !STAGED) {
          static_for<JC>([&](auto jjc) {
            if (decltype(jjc)::value == jj) store_group(jjc, c);
          });
        } else {
          const uint32_t cb = l31 ? b - 32 : b;
          put_block(gbase + 4 * cb + DELTA, c);
        }
      }
      if (j == jfirst && lane == 0) {  // head of this warp's first block
#pragma unroll
        for (int t = 0; t < DELTA; ++t) put1(gbase + 4 * b + t, y[t]);
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) prev[k] = y[k];
    }
  }
  if constexpr (DELTA > 0 && !(!SMD && !STAGED && WB_D2_STG64 && sizeof(T) == 4 && DELTA == 2) &&
                !(WB_D3_DOWN && VEC == 4 && DELTA == 3)) {
    if (l31 && c0 + JC == J) {  // last group of the warp: own tail only, the head is the next warp's
      const uint32_t b = (warp * J + J - 1) * 32 + 31;
#pragma unroll
      for (int m = DELTA; m < 4; ++m)
        if (4 * b + m < NLIM) put1(gbase + 4 * b + m, prev[m]);
    }
  }
  if constexpr (SMD) *zf |= z;
}

#if WB_ABLATE == 6
#undef stg_vec
#undef stg1
#endif
template <typename T, int LOG2N, int DELTA>
__device__ __forceinline__ void emit_chunk_mz(bool mz, const T (&X)[Geo<T, LOG2N>::JC][4], int c0,
                                              T (&prev)[4], T* gbase, T sc, T mean, int lane, int warp,
                                              int jfirst = 0) {
  if (mz) emit_chunk<T, LOG2N, DELTA, true>(X, c0, prev, gbase, sc, mean, lane, warp, jfirst);
  else emit_chunk<T, LOG2N, DELTA, false>(X, c0, prev, gbase, sc, mean, lane, warp, jfirst);
}

// The shifted shared-memory write of an emission pass (bulk emission): the
// raw values, dispatched on the shift.
template <typename T, int LOG2N>
__device__ __forceinline__ void shift_chunk_any(uint32_t delta, const T (&X)[Geo<T, LOG2N>::JC][4], int c0,
                                                T (&prev)[4], T* sbase, int lane, int warp, uint32_t* zf) {
  using G = Geo<T, LOG2N>;
  if constexpr (G::VEC == 4) {
    switch (delta) {
      case 0: emit_chunk<T, LOG2N, 0, true, true>(X, c0, prev, sbase, T(1), T(0), lane, warp, 0, zf); break;
      case 1: emit_chunk<T, LOG2N, 1 % G::VEC, true, true>(X, c0, prev, sbase, T(1), T(0), lane, warp, 0, zf); break;
      case 2: emit_chunk<T, LOG2N, 2 % G::VEC, true, true>(X, c0, prev, sbase, T(1), T(0), lane, warp, 0, zf); break;
      default: emit_chunk<T, LOG2N, 3 % G::VEC, true, true>(X, c0, prev, sbase, T(1), T(0), lane, warp, 0, zf); break;
    }
  } else {
    if (delta == 0) emit_chunk<T, LOG2N, 0, true, true>(X, c0, prev, sbase, T(1), T(0), lane, warp, 0, zf);
    else emit_chunk<T, LOG2N, 1, true, true>(X, c0, prev, sbase, T(1), T(0), lane, warp, 0, zf);
  }
}

// The staged write of an emission (kModeFillStaged): scaled values into the
// shifted shared layout at sbase, warp-end scalars to global at g1.
template <typename T, int LOG2N>
__device__ __forceinline__ void stage_chunk_any(uint32_t delta, bool mz, const T (&X)[Geo<T, LOG2N>::JC][4],
                                                int c0, T (&prev)[4], T* sbase, T* g1, T sc, T mean,
                                                int lane, int warp) {
  using G = Geo<T, LOG2N>;
#define WB_STAGE(D)                                                                                     \
  (mz ? emit_chunk<T, LOG2N, (D) % G::VEC, true, false, true>(X, c0, prev, sbase, sc, mean, lane, warp, 0, \
                                                               nullptr, g1)                              \
      : emit_chunk<T, LOG2N, (D) % G::VEC, false, false, true>(X, c0, prev, sbase, sc, mean, lane, warp, 0, \
                                                                nullptr, g1))
  if constexpr (G::VEC == 4) {
    switch (delta) {
      case 0: WB_STAGE(0); break;
      case 1: WB_STAGE(1); break;
      case 2: WB_STAGE(2); break;
      default: WB_STAGE(3); break;
    }
  } else {
    if (delta == 0) WB_STAGE(0);
    else WB_STAGE(1);
  }
#undef WB_STAGE
}

// The slots [lo, hi) of the shifted staging layout (slot = element + sigma)
// that warp w filled with 16-byte vectors in stage_chunk_any: its segment
// [w*WE, (w+1)*WE) minus the partial vectors at its ends, which went out as
// scalars (emit_chunk: lane 0's head, lane 31's last block; the pool's last
// block when sigma = 0, element N-1 not emitted).
template <typename T, int LOG2N>
__device__ __forceinline__ void staged_range(uint32_t sigma, int warp, uint32_t& lo, uint32_t& hi) {
  using G = Geo<T, LOG2N>;
  constexpr uint32_t WE = 128u * G::J;  // elements per warp segment
  lo = warp * WE;
  hi = lo + WE;
  if (sigma == 0) {
    if (warp == G::NW - 1) hi -= 4;
  } else if constexpr (G::VEC == 4) {
    lo += 4;
  } else {
    lo += 2;
    hi -= 2;
  }
}

// Register emission of one chunk for any shift: dispatch on delta.
template <typename T, int LOG2N>
__device__ __forceinline__ void emit_chunk_any(uint32_t delta, bool mz,
                                               const T (&X)[Geo<T, LOG2N>::JC][4], int c0,
                                               T (&prev)[4], T* gbase, T sc, T mean, int lane,
                                               int warp, int jfirst = 0) {
  using G = Geo<T, LOG2N>;
  if constexpr (G::VEC == 4) {
    switch (delta) {
      case 0: emit_chunk_mz<T, LOG2N, 0>(mz, X, c0, prev, gbase, sc, mean, lane, warp, jfirst); break;
      case 1: emit_chunk_mz<T, LOG2N, 1 % G::VEC>(mz, X, c0, prev, gbase, sc, mean, lane, warp, jfirst); break;
      case 2: emit_chunk_mz<T, LOG2N, 2 % G::VEC>(mz, X, c0, prev, gbase, sc, mean, lane, warp, jfirst); break;
      default: emit_chunk_mz<T, LOG2N, 3 % G::VEC>(mz, X, c0, prev, gbase, sc, mean, lane, warp, jfirst); break;
    }
  } else {
    if (delta == 0) emit_chunk_mz<T, LOG2N, 0>(mz, X, c0, prev, gbase, sc, mean, lane, warp, jfirst);
    else emit_chunk_mz<T, LOG2N, 1>(mz, X, c0, prev, gbase, sc, mean, lane, warp, jfirst);
  }
}

// ---------------------------------------------------------------------------
// Bulk emission.  When an emission's scale is exactly 1 and the mean is +0
// (disable_chi2 with sigma 1 makes r = S/sum_sq = 1 exactly -- BASELINE
// config 2), out[i] = x[i]*1 + 0 is the pool value itself, bit for bit,
// except that the "+0" turns an exact -0 into +0.  The emission pass then
// writes its result into shared memory shifted by the output's misalignment
// sigma (element i at slot i + sigma, so slot and global address agree mod
// 16 bytes; the same shuffle realignment as the register emission), and one
// thread sends the aligned middle of the emission to global memory with a
// single cp.async.bulk while the next pass runs.  The <= 3 head and tail
// values go out as scalar stores, and an exact -0 anywhere in the emission
// (an exact cancellation in the butterfly, rare) triggers a patch that
// rewrites it as +0 once the bulk copy has landed.  The next pass gathers
// from the shifted buffer (the shift is part of its buffer base).
// ---------------------------------------------------------------------------
__device__ __forceinline__ void bulk_s2g(void* dst, uint32_t src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(src), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

// ---------------------------------------------------------------------------
// pool_kernel: one CTA per pool.  The pool ping-pongs between two shared
// buffers (one block barrier per pass); plans for the launch are staged in
// shared memory; pool state persists in HBM across launches.
//
// One pass (generator.cpp:64-85): for b < ROWS, r = (off + b*STRIDE) mod ROWS,
//   v_c = in[c*ROWS + r], a=v0+v1, bb=v0-v1, c=v2+v3, d=v2-v3,
//   z = {a-d, bb+c, bb-c, -a-d}, out[4b+k] = (0.5*sign_k) * z[src_k].
// The gather is bank-conflict-free: STRIDE is odd and ROWS a multiple of 32,
// so 32 consecutive b hit 32 distinct banks; out[4b..4b+3] is one 128-bit
// shared store.  The row permutation src is warp-uniform per pass and is
// applied through a 24-way uniform branch over compile-time register moves.
// Shared addresses are byte offsets: gather = ((rb4 + off4) & MASK4) | cur,
// one IADD3 + one LOP3 per 4-block (the buffers sit at power-of-two offsets).
// ---------------------------------------------------------------------------
template <typename T, int LOG2N>
struct Smem {
  static constexpr int N = Geo<T, LOG2N>::N;
  static constexpr uint32_t BUF = N * sizeof(T);  // bytes per pool buffer (power of two)
  // pools in static shared memory when they fit the 48 KiB static limit: the
  // buffer base then folds into the LDS/STS immediate offsets
  static constexpr int BUFS = Geo<T, LOG2N>::BUFS;
  // buffers sit BSTRIDE apart: 16 bytes of slack after each pool for the
  // shifted layout of a bulk emission (up to 3 fp32 / 1 fp64 elements)
  static constexpr uint32_t BSTRIDE = BUF + 16;
  static constexpr uint32_t TOTAL = BUFS * BSTRIDE;
  static constexpr bool STATIC = TOTAL <= 40 * 1024;
};

// Affine-mixing gathers without bank conflicts.  Lanes with consecutive
// 4-blocks b read elements (off + (4b + c)*alpha) mod N; for a fixed column c
// those are 4*alpha apart, so a warp would hit only 8 of the 32 banks (fp32;
// 4 of 16 per half-warp for fp64).  Lane group g (lanes 8g..8g+7 for fp32,
// 4g..4g+3 within each half-warp for fp64) reads column k ^ g in its k-th
// load instead: 4*(b mod 8) + (k ^ g) covers every bank once.  The values
// are then put back in column order with selects.
template <typename T>
__device__ __forceinline__ uint32_t affine_lane_group(uint32_t lane) {
  return (lane >> (sizeof(T) == 4 ? 3 : 2)) & 3u;
}
template <typename T, uint32_t A, uint32_t MASKN>
__device__ __forceinline__ void affine_gather4(const char* base, uint32_t buf, uint32_t e, uint32_t g,
                                               T (&v)[4]) {
  T L[4];
#pragma unroll
  for (int k = 0; k < 4; ++k)
    L[k] = *reinterpret_cast<const T*>(base + (((e + (uint32_t(k) ^ g) * A) & MASKN) + buf));
  const bool x1 = g & 1u, x2 = g & 2u;
  const T t0 = x1 ? L[1] : L[0], t1 = x1 ? L[0] : L[1], t2 = x1 ? L[3] : L[2], t3 = x1 ? L[2] : L[3];
  v[0] = x2 ? t2 : t0;
  v[1] = x2 ? t3 : t1;
  v[2] = x2 ? t0 : t2;
  v[3] = x2 ? t1 : t3;
}

// One pass over the pool in shared memory (generator.cpp:64-85); leaves the
// signed, permuted outputs of this thread's 4-blocks in X and stores them to
// the next buffer.  sb = b0*STRIDE + off for this thread's first block.
// hook(): work issued right after the pass's gathers (in-order issue: it
// then overlaps their latency instead of lengthening the pass).
// The butterfly z(v) = {a-d, b+c, b-c, -a-d}, a = v0+v1, b = v0-v1, c = v2+v3,
// d = v2-v3 (transforms.hpp:89-103) is, bit for bit, invariant up to an output
// permutation and output signs under the 8 input permutations generated by
// v0<->v1, v2<->v3 and (v0,v1)<->(v2,v3): fp addition commutes, x-y = -(y-x)
// and -x-y = -(x+y) exactly.  Those 8 input orders induce 8 output row
// permutations (a subgroup of S4 with three cosets), so every one of the 24
// row permutations src of a variant is   X[k] = (+-hs[k]) * z_{R_t[k]}(v o Q)
// with R_t one of {0123, 0132, 0312}, Q one of the 8 input orders and a sign
// mask.  Q is free: the four column gathers are issued in the order Q (their
// address offsets are warp-uniform), the signs fold into the row factors,
// and the 24-way register-move dispatch becomes a 3-way one.
// Entry p (lexicographic permutation index, transforms.cpp:24-35):
// t | Q[0..3] << 2 (2 bits each) | sign mask << 10.  Derived and checked
// bitwise on random inputs by tools/perm3_table.py.
__device__ __forceinline__ uint32_t perm3_entry(uint32_t p) {
  constexpr uint32_t kTab[24] = {0x390,  0x391,  0x1b84, 0x2b85, 0x392,  0x3386, 0x06d,  0x06c,
                                 0x06e,  0x307a, 0x1878, 0x2879, 0x152d, 0x252c, 0xd2e,  0x3d3a,
                                 0x3d38, 0x3d39, 0xed2,  0x3ec6, 0x16d1, 0x26d0, 0x3ec5, 0x3ec4};
  return kTab[p];
}
template <int T_, int K>
struct Perm3Rep {
  static constexpr int v = T_ == 0 ? K : (T_ == 1 ? (K == 2 ? 3 : (K == 3 ? 2 : K)) : (K == 0 ? 0 : (K == 1 ? 3 : K - 1)));
};
static_assert(Perm3Rep<2, 0>::v == 0 && Perm3Rep<2, 1>::v == 3 && Perm3Rep<2, 2>::v == 1 && Perm3Rep<2, 3>::v == 2,
              "coset representatives");

struct NoHook {
  __device__ __forceinline__ void operator()() const {}
};
template <typename T, int LOG2N, int J, int PT = 0, class Hook = NoHook, bool HSA = false>
__device__ __forceinline__ void run_pass(const char* base, uint32_t cur_off, uint32_t nxt_off,
                                         uint32_t plan, uint32_t b0, T (&X)[J][4],
                                         const float* hs_lut, bool store = true,
                                         bool wait_stage = false, Hook hook = Hook{}, uint32_t hs_saddr = 0) {
  // HSA: hs_saddr is hs_lut's shared-window address, kept in a register by
  // the caller (the latency fill: ptxas otherwise rebuilds it every pass)
  constexpr bool HOOK = !std::is_same<Hook, NoHook>::value;
  static_assert(PT == 0 || PT == 1, "wallace4 pass types");
  using G = Geo<T, LOG2N>;
  constexpr int ROWS = G::ROWS;
  constexpr uint32_t MASK4 = (ROWS - 1) * sizeof(T);
  const uint32_t off = plan & 0xffffu;
  const uint32_t variant = plan >> 16;
  const uint32_t perm = variant >> 4;
  constexpr bool P3 = WB_PERM3 && PT == 0 && !((WB_PACKED & 1) && sizeof(T) == 4);
  // P3: byte offsets of the four column gathers in the order Q, the coset
  // representative and the signs that fold into the row factors
  uint32_t co[4] = {0u, uint32_t(ROWS * sizeof(T)), uint32_t(2 * ROWS * sizeof(T)), uint32_t(3 * ROWS * sizeof(T))};
  uint32_t rep = 0, smask = variant & 15u;
  if constexpr (P3) {
    const uint32_t pe = perm3_entry(perm);
    rep = pe & 3u;
    smask ^= (pe >> 10) & 15u;
#pragma unroll
    for (int c = 0; c < 4; ++c) co[c] = ((pe >> (2 + 2 * c)) & 3u) * uint32_t(ROWS * sizeof(T));
  }
  T hs[4];
  if constexpr (WB_HS_LUT && sizeof(T) == 4) {
    // the four +-1/2 row factors of this variant's sign mask, one 128-bit load
    float4 h;
    if constexpr (HSA)
      asm("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(h.x), "=f"(h.y), "=f"(h.z), "=f"(h.w) : "r"(hs_saddr + 16u * smask));
    else
      h = reinterpret_cast<const float4*>(hs_lut)[smask];
    hs[0] = h.x;
    hs[1] = h.y;
    hs[2] = h.z;
    hs[3] = h.w;
  } else {
#pragma unroll
    for (int k = 0; k < 4; ++k) hs[k] = ((smask >> k) & 1u) ? T(-0.5) : T(0.5);
  }
  // byte offset of row r_j = (off + b_j*STRIDE) mod ROWS, b_j = b0 + 32j
  const uint32_t r0 = (b0 * G::STRIDE + off) * sizeof(T);

  if constexpr ((WB_PACKED & 1) && sizeof(T) == 4 && PT == 0) {
    // gather + first butterfly stage as two packed ops per 4-block:
    // (a, b) = (v0 + v1, v0 - v1), (c, d) = (v2 + v3, v2 - v3)
    float ab[J][2], cd[J][2];
#pragma unroll
    for (int j = 0; j < J; ++j) {
      float v0 = 0, v1 = 0, v2 = 0, v3 = 0;
      if (ROWS >= 32 || b0 + 32 * j < ROWS) {
        constexpr uint32_t step = 32u * G::STRIDE * sizeof(T);
        const float* row = reinterpret_cast<const float*>(base + (((r0 + j * step) & MASK4) + cur_off));
        v0 = row[0];
        v1 = row[ROWS];
        v2 = row[2 * ROWS];
        v3 = row[3 * ROWS];
      }
      const uint64_t pm = pk2(1.f, -1.f);
      upk2(fma2_rn(pk2(v1, v1), pm, pk2(v0, v0)), ab[j][0], ab[j][1]);
      upk2(fma2_rn(pk2(v3, v3), pm, pk2(v2, v2)), cd[j][0], cd[j][1]);
    }
    const uint64_t h01 = pk2(float(hs[0]), float(hs[1]));
    const uint64_t h23 = pk2(float(hs[2]), float(hs[3]));
    float (&Xf)[J][4] = reinterpret_cast<float (&)[J][4]>(X);
    switch (perm) {
#define WB_PERM_CASE(P)                                                                              \
  case P:                                                                                            \
    _Pragma("unroll") for (int j = 0; j < J; ++j) {                                                  \
      wallace_pair<PermAt<P, 0>::v, PermAt<P, 1>::v>(ab[j][0], ab[j][1], cd[j][0], cd[j][1], h01,    \
                                                      Xf[j][0], Xf[j][1]);                           \
      wallace_pair<PermAt<P, 2>::v, PermAt<P, 3>::v>(ab[j][0], ab[j][1], cd[j][0], cd[j][1], h23,    \
                                                      Xf[j][2], Xf[j][3]);                           \
    }                                                                                                \
    break;
      WB_PERM_CASE(0) WB_PERM_CASE(1) WB_PERM_CASE(2) WB_PERM_CASE(3) WB_PERM_CASE(4)
      WB_PERM_CASE(5) WB_PERM_CASE(6) WB_PERM_CASE(7) WB_PERM_CASE(8) WB_PERM_CASE(9)
      WB_PERM_CASE(10) WB_PERM_CASE(11) WB_PERM_CASE(12) WB_PERM_CASE(13) WB_PERM_CASE(14)
      WB_PERM_CASE(15) WB_PERM_CASE(16) WB_PERM_CASE(17) WB_PERM_CASE(18) WB_PERM_CASE(19)
      WB_PERM_CASE(20) WB_PERM_CASE(21) WB_PERM_CASE(22) WB_PERM_CASE(23)
      default: __builtin_unreachable();
#undef WB_PERM_CASE
    }
    if constexpr (G::INPLACE) __syncthreads();
    if (!store) return;
    float* nb = reinterpret_cast<float*>(const_cast<char*>(base) + nxt_off);
#pragma unroll
    for (int j = 0; j < J; ++j) {
      const uint32_t b = b0 + 32 * j;
      if (ROWS >= 32 || b < ROWS) sts4(nb + 4 * b, Xf[j][0], Xf[j][1], Xf[j][2], Xf[j][3]);
    }
    return;
  }

  // gather + butterfly (apply_wallace4 op order, transforms.hpp:89-103)
  T z[J][4];
  T vg[HOOK ? J : 1][4];  // HOOK: every gather issued before the hook
  if constexpr (HOOK) {
#pragma unroll
    for (int j = 0; j < J; ++j) {
      vg[j][0] = vg[j][1] = vg[j][2] = vg[j][3] = T(0);
      if ((ROWS >= 32 || b0 + 32 * j < ROWS) && PT == 0) {
        constexpr uint32_t step = 32u * G::STRIDE * sizeof(T);
        const char* row = base + (((r0 + j * step) & MASK4) + cur_off);
#pragma unroll
        for (int c = 0; c < 4; ++c) vg[j][c] = *reinterpret_cast<const T*>(row + co[c]);
      }
    }
    hook();
  }
#pragma unroll
  for (int j = 0; j < J; ++j) {
    T v0 = 0, v1 = 0, v2 = 0, v3 = 0;
    if constexpr (HOOK && PT == 0) {
      v0 = vg[j][0];
      v1 = vg[j][1];
      v2 = vg[j][2];
      v3 = vg[j][3];
    } else if (ROWS >= 32 || b0 + 32 * j < ROWS) {
      if constexpr (PT == 0) {
        constexpr uint32_t step = 32u * G::STRIDE * sizeof(T);
        const char* row = base + (((r0 + j * step) & MASK4) + cur_off);
        v0 = *reinterpret_cast<const T*>(row + co[0]);
        v1 = *reinterpret_cast<const T*>(row + co[1]);
        v2 = *reinterpret_cast<const T*>(row + co[2]);
        v3 = *reinterpret_cast<const T*>(row + co[3]);
      } else {
        // affine (generator.cpp:86-110): element 4b+c of the gathered
        // sequence sits at (off + (4b+c)*alpha) mod N
        constexpr uint32_t A = G::ALPHA * sizeof(T), MASKN = (G::N - 1) * sizeof(T);
        const uint32_t e = (off + 4u * (b0 + 32u * j) * G::ALPHA) * sizeof(T);
        T v[4];
        affine_gather4<T, A, MASKN>(base, cur_off, e, affine_lane_group<T>(b0 & 31u), v);
        v0 = v[0];
        v1 = v[1];
        v2 = v[2];
        v3 = v[3];
      }
    }
    const T aa = add_rn(v0, v1);
    const T bb = sub_rn(v0, v1);
    const T cc = add_rn(v2, v3);
    const T dd = sub_rn(v2, v3);
    z[j][0] = sub_rn(aa, dd);
    z[j][1] = add_rn(bb, cc);
    z[j][2] = sub_rn(bb, cc);
    z[j][3] = sub_rn(-aa, dd);
  }
  // signed row permutation: X[k] = (0.5*sign_k) * z[src_k]
  if constexpr (P3) {
    switch (rep) {
#define WB_REP_CASE(R)                                      \
  case R:                                                   \
    _Pragma("unroll") for (int j = 0; j < J; ++j) {         \
      X[j][0] = mul_rn(hs[0], z[j][Perm3Rep<R, 0>::v]);     \
      X[j][1] = mul_rn(hs[1], z[j][Perm3Rep<R, 1>::v]);     \
      X[j][2] = mul_rn(hs[2], z[j][Perm3Rep<R, 2>::v]);     \
      X[j][3] = mul_rn(hs[3], z[j][Perm3Rep<R, 3>::v]);     \
    }                                                       \
    break;
      WB_REP_CASE(0) WB_REP_CASE(1)
      default:
        WB_REP_CASE(2)
#undef WB_REP_CASE
    }
  } else
  switch (perm) {
#define WB_PERM_CASE(P)                                     \
  case P:                                                   \
    _Pragma("unroll") for (int j = 0; j < J; ++j) {         \
      X[j][0] = mul_rn(hs[0], z[j][PermAt<P, 0>::v]);       \
      X[j][1] = mul_rn(hs[1], z[j][PermAt<P, 1>::v]);       \
      X[j][2] = mul_rn(hs[2], z[j][PermAt<P, 2>::v]);       \
      X[j][3] = mul_rn(hs[3], z[j][PermAt<P, 3>::v]);       \
    }                                                       \
    break;
    WB_PERM_CASE(0) WB_PERM_CASE(1) WB_PERM_CASE(2) WB_PERM_CASE(3) WB_PERM_CASE(4)
    WB_PERM_CASE(5) WB_PERM_CASE(6) WB_PERM_CASE(7) WB_PERM_CASE(8) WB_PERM_CASE(9)
    WB_PERM_CASE(10) WB_PERM_CASE(11) WB_PERM_CASE(12) WB_PERM_CASE(13) WB_PERM_CASE(14)
    WB_PERM_CASE(15) WB_PERM_CASE(16) WB_PERM_CASE(17) WB_PERM_CASE(18) WB_PERM_CASE(19)
    WB_PERM_CASE(20) WB_PERM_CASE(21) WB_PERM_CASE(22) WB_PERM_CASE(23)
    default: __builtin_unreachable();  // perm = variant >> 4 < 24 (variant = w0 % 384)
#undef WB_PERM_CASE
  }
  if constexpr (G::INPLACE) __syncthreads();  // every gather of this pass is done
  if (!store) return;  // the caller writes the shifted layout (bulk emission)
  if (wait_stage) {
    // staged emission: this warp's bulk copy must have read its segment of
    // the buffer these stores overwrite (the segment is the warp's own blocks)
    if ((threadIdx.x & 31u) == 0) bulk_wait_read();
    __syncwarp();
  }
  T* nb = reinterpret_cast<T*>(const_cast<char*>(base) + nxt_off);
  if constexpr (sizeof(T) == 8) {
    // a 4-double block is 32 bytes: two 128-bit stores at a 32-byte lane
    // stride would hit each bank twice per 8-lane phase; lanes with bit 2 set
    // store their halves in the opposite order, which makes both stores
    // conflict-free (lanes l and l+4 then cover complementary banks)
    // (latency kernels, WB_LAT_F64_SWZ 0: natural order -- there the data
    // selects and the register moves feeding the stores lengthen the pass
    // more than the 2-way conflicts do)
    constexpr bool SWZ = G::LAT ? WB_LAT_F64_SWZ : WB_F64_SWZ;
    const bool swz = SWZ && ((b0 >> 2) & 1);
#pragma unroll
    for (int j = 0; j < J; ++j) {
      const uint32_t b = b0 + 32 * j;
      if (ROWS >= 32 || b < ROWS) {
        double2* q = reinterpret_cast<double2*>(nb + 4 * b);
        const double2 lo = make_double2(X[j][0], X[j][1]);
        const double2 hi = make_double2(X[j][2], X[j][3]);
        if constexpr (SWZ && WB_F64_SWZ_B32) {
          // the same two stores with the selects on 32-bit halves and the
          // data as four 32-bit registers (keeps ptxas from funnelling every
          // store through one register quad)
          const uint32_t a0 = static_cast<uint32_t>(__cvta_generic_to_shared(q));
          sts_sel_b32(a0 + (swz ? 16u : 0u), swz, X[j][0], X[j][1], X[j][2], X[j][3]);
          sts_sel_b32(a0 + (swz ? 0u : 16u), swz, X[j][2], X[j][3], X[j][0], X[j][1]);
        } else if constexpr (SWZ) {
          q[swz ? 1 : 0] = swz ? hi : lo;
          q[swz ? 0 : 1] = swz ? lo : hi;
        } else {
          q[0] = lo;
          q[1] = hi;
        }
      }
    }
  } else {
#pragma unroll
    for (int j = 0; j < J; ++j) {
      const uint32_t b = b0 + 32 * j;
      if (ROWS >= 32 || b < ROWS) sts4(nb + 4 * b, X[j][0], X[j][1], X[j][2], X[j][3]);
    }
  }
}

// One 4-block store of a pass result.  fp64: a 4-double block is 32 bytes;
// lanes with bit 2 set store their halves in the opposite order so both
// 128-bit stores are bank-conflict-free (see run_pass).
template <typename T>
__device__ __forceinline__ void store_block(T* nb, uint32_t b, T x0, T x1, T x2, T x3) {
  if constexpr (sizeof(T) == 8) {
    const bool swz = (b >> 2) & 1;
    if constexpr (WB_F64_SWZ_B32) {
      const uint32_t a0 = static_cast<uint32_t>(__cvta_generic_to_shared(nb + 4 * b));
      sts_sel_b32(a0 + (swz ? 16u : 0u), swz, x0, x1, x2, x3);
      sts_sel_b32(a0 + (swz ? 0u : 16u), swz, x2, x3, x0, x1);
    } else {
      double2* q = reinterpret_cast<double2*>(nb + 4 * b);
      const double2 lo = make_double2(x0, x1), hi = make_double2(x2, x3);
      q[swz ? 1 : 0] = swz ? hi : lo;
      q[swz ? 0 : 1] = swz ? lo : hi;
    }
  } else {
    sts4(nb + 4 * b, x0, x1, x2, x3);
  }
}

// One rotation pass (run_pass, generator.cpp:259-271: two half-sweeps,
// rotation_sweep :113-172).
//   sweep 0: gather through the mixing map (offset word 0), rotate the pairs
//            (4b, 4b+1), (4b+2, 4b+3) -> scratch buffer (nxt_off); barrier;
//   sweep 1: gather the scratch through the map (offset word 1), rotate the
//            pairs (4b+1, 4b+2), (4b+3, 4b+4) and the wrap pair (N-1, 0) ->
//            back into the current buffer.  Each thread gathers its block's
//            two neighbours g[4b-1], g[4b+4] itself (no exchange), so every
//            store is an aligned 4-block.
// The pool therefore stays in `cur` (the caller does not flip buffers) and
// this thread's 4-blocks are left in X, like run_pass.  Coefficients
// ce = g*c, se = g*s in fp64 (exact sign flips of the table entry), rounded
// once for T = float; out = ce*z1 + se*z2 and
// (-se)*z1 + ce*z2 with two roundings each, as the reference.
// Plan words: offset | t_index << 16 | negate << 20, one per sweep.
template <typename T, int LOG2N, int J, int MIX>
__device__ __forceinline__ void run_pass_rot(const char* base, uint32_t cur_off, uint32_t nxt_off,
                                             uint32_t w0, uint32_t w1, uint32_t b0, T (&X)[J][4],
                                             const double* rc, const double* rs) {
  using G = Geo<T, LOG2N>;
  constexpr int ROWS = G::ROWS;
  constexpr uint32_t ES = sizeof(T);
  constexpr uint32_t MASK4 = (ROWS - 1) * ES, MASKN = (G::N - 1) * ES;
  constexpr uint32_t SROW = G::STRIDE * ES;  // one row step in bytes
  auto coef = [&](uint32_t w, T& ce, T& se) {
    const uint32_t t = (w >> 16) & 15u;
    const bool neg = (w >> 20) & 1u;
    ce = from_double<T>(neg ? -rc[t] : rc[t]);
    se = from_double<T>(neg ? -rs[t] : rs[t]);
  };
  auto ld = [&](uint32_t byte_off, uint32_t buf) -> T {
    return *reinterpret_cast<const T*>(base + (byte_off + buf));
  };
  // ---- sweep 0 ----
  {
    T ce, se;
    coef(w0, ce, se);
    const T nse = -se;
    const uint32_t off = w0 & 0xffffu;
    T* nb = reinterpret_cast<T*>(const_cast<char*>(base) + nxt_off);
#pragma unroll
    for (int j = 0; j < J; ++j) {
      const uint32_t b = b0 + 32 * j;
      if (ROWS >= 32 || b < ROWS) {
        T g[4];
        if constexpr (MIX == 0) {
          const uint32_t r = ((off + b * G::STRIDE) * ES) & MASK4;
#pragma unroll
          for (int c = 0; c < 4; ++c) g[c] = ld(r + c * ROWS * ES, cur_off);
        } else {
          const uint32_t e = (off + 4u * b * G::ALPHA) * ES;
          affine_gather4<T, G::ALPHA * ES, MASKN>(base, cur_off, e, affine_lane_group<T>(b0 & 31u), g);
        }
        store_block(nb, b, add_rn(mul_rn(ce, g[0]), mul_rn(se, g[1])),
                    add_rn(mul_rn(nse, g[0]), mul_rn(ce, g[1])),
                    add_rn(mul_rn(ce, g[2]), mul_rn(se, g[3])),
                    add_rn(mul_rn(nse, g[2]), mul_rn(ce, g[3])));
      }
    }
  }
  __syncthreads();  // the whole sweep-0 result is in the scratch buffer
  // ---- sweep 1 ----
  {
    T ce, se;
    coef(w1, ce, se);
    const T nse = -se;
    const uint32_t off = w1 & 0xffffu;
    T* cb = reinterpret_cast<T*>(const_cast<char*>(base) + cur_off);
#pragma unroll
    for (int j = 0; j < J; ++j) {
      const uint32_t b = b0 + 32 * j;
      X[j][0] = X[j][1] = X[j][2] = X[j][3] = T(0);
      if (ROWS >= 32 || b < ROWS) {
        T h[4], hm, hp;  // g[4b..4b+3], g[4b-1], g[4b+4] (indices mod N)
        if constexpr (MIX == 0) {
          // element 4q+c at column c, row (off + q*stride) mod rows
          const uint32_t r = ((off + b * G::STRIDE) * ES) & MASK4;
#pragma unroll
          for (int c = 0; c < 4; ++c) h[c] = ld(r + c * ROWS * ES, nxt_off);
          hm = ld(((r - SROW) & MASK4) + 3 * ROWS * ES, nxt_off);
          hp = ld((r + SROW) & MASK4, nxt_off);
        } else {
          constexpr uint32_t B = G::BETA * ES;
          const uint32_t e = (off + 4u * b * G::BETA) * ES;
          const uint32_t lane = b0 & 31u;
          affine_gather4<T, B, MASKN>(base, nxt_off, e, affine_lane_group<T>(lane), h);
          if constexpr (ROWS >= 32) {
            // the neighbours are the adjacent lanes' end values (lane 0 and
            // lane 31 reach into the previous / next group: direct loads)
            hm = __shfl_up_sync(0xffffffffu, h[3], 1);
            hp = __shfl_down_sync(0xffffffffu, h[0], 1);
            if (lane == 0) hm = ld((e - B) & MASKN, nxt_off);
            if (lane == 31) hp = ld((e + 4 * B) & MASKN, nxt_off);
          } else {
            hm = ld((e - B) & MASKN, nxt_off);
            hp = ld((e + 4 * B) & MASKN, nxt_off);
          }
        }
        X[j][0] = add_rn(mul_rn(nse, hm), mul_rn(ce, h[0]));
        X[j][1] = add_rn(mul_rn(ce, h[1]), mul_rn(se, h[2]));
        X[j][2] = add_rn(mul_rn(nse, h[1]), mul_rn(ce, h[2]));
        X[j][3] = add_rn(mul_rn(ce, h[3]), mul_rn(se, hp));
        store_block(cb, b, X[j][0], X[j][1], X[j][2], X[j][3]);
      }
    }
  }
}

// Emission of the values already in registers (fast path) into the fused
// consumer instead of memory.
// (MZ is a template parameter: with a runtime flag the compiler evaluates
// both forms of emit_value for every value)
template <typename T, int LOG2N, int JCL, bool MZ>
__device__ __forceinline__ void consume_chunk_mz(const T (&X)[JCL][4], Consumer<T>& cons, T sc, T mean,
                                                 uint32_t b0c) {
  using G = Geo<T, LOG2N>;
#pragma unroll
  for (int j = 0; j < JCL; ++j) {
    const uint32_t b = b0c + 32 * j;
    T y[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) y[k] = emit_value(X[j][k], sc, mean, MZ);
    cons.add_group(y, b == G::ROWS - 1 ? 3 : 4);
  }
}
// fp32, mean +0: the chunk's values as f32x2 pairs (slots 0,1 and 2,3 of a
// block).  Per pair: y = x*scale (one FFMA2 with +0, bit-identical to the
// scalar emission), the four power sums (FMUL2, 2 FADD2, 2 FFMA2), the
// histogram coordinate 16y + 128 (one FFMA2, exact like fl(fl(y+8)*16)).
// The bins are floored first and counted after the check: a power-4 partial
// below 4096 proves every |y| of this emission so far is below 8 (the terms
// are non-negative and rounding is monotone; NaN fails the test), so the
// clamp to [-1, 256] is the identity and is skipped.  Element N-1 (slot 3 of
// block ROWS-1) is the reserved value: it adds 0 to the sums and no count.
template <int LOG2N, int JCL>
__device__ __forceinline__ void consume_chunk_pairs(const float (&X)[JCL][4], Consumer<float>& cons, float sc,
                                                    uint32_t b0c) {
  using G = Geo<float, LOG2N>;
  const uint64_t sc2 = pk2(sc, sc), zero2 = pk2(0.f, 0.f);
  const uint64_t k16 = pk2(16.f, 16.f), k128 = pk2(128.f, 128.f);
  // WB_CONS_RZBIN: the bin coordinates t stay as f32x2 pairs; floor(t) for
  // t in [0, 256] is the low bits of t + 2^23 added toward zero (the sum lies
  // in [2^23, 2^24), where the ulp is 1), one FADD2 per pair
  uint64_t tc[JCL][2];
  int bin[WB_CONS_RZBIN ? 1 : JCL][4];
  bool tail = false;  // this thread's last block is the pool's last
#pragma unroll
  for (int j = 0; j < JCL; ++j) {
    const bool last = (b0c + 32 * j == G::ROWS - 1);
    tail |= last;
#pragma unroll
    for (int h = 0; h < 4; h += 2) {
      uint64_t y = fma2_rn(pk2(X[j][h], X[j][h + 1]), sc2, zero2);
      if (h == 2 && j == JCL - 1) {
        float y0, y1;
        upk2(y, y0, y1);
        y = pk2(y0, last ? 0.f : y1);
      }
      const uint64_t q = mul2_rn(y, y);
      cons.p1 = add2_rn(cons.p1, y);
      cons.p2 = add2_rn(cons.p2, q);
      cons.p3 = fma2_rn(q, y, cons.p3);
      cons.p4 = fma2_rn(q, q, cons.p4);
      if constexpr (WB_CONS_RZBIN) {
        tc[j][h >> 1] = fma2_rn(y, k16, k128);
      } else {
        float t0, t1;
        upk2(fma2_rn(y, k16, k128), t0, t1);
        bin[j][h] = __float2int_rd(t0);
        bin[j][h + 1] = __float2int_rd(t1);
      }
    }
  }
  float q4lo, q4hi;
  upk2(cons.p4, q4lo, q4hi);
  const bool inside = q4lo < 4096.f && q4hi < 4096.f;  // every |y| so far < 8: t in [0, 256]
  if constexpr (WB_CONS_RZBIN) {
    if (inside) {
      // hist[floor(t) + 1] = word (bits(t + 2^23) - bits(2^23) + 1): the
      // constant folds into one base address
      // (shared addresses mod 2^32: 4 * (1 - 0x4B000000) = 4 - 0x2C000000)
      const uint64_t big2 = pk2(8388608.f, 8388608.f);
      const uint32_t hb = static_cast<uint32_t>(__cvta_generic_to_shared(cons.hist)) + 4u - 0x2C000000u;
      auto count = [&](float f) {
        asm volatile("red.shared.add.u32 [%0], 1;" ::"r"(hb + (__float_as_uint(f) << 2)));
      };
#pragma unroll
      for (int j = 0; j < JCL; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          float f0, f1;
          upk2(add2_rz(tc[j][h], big2), f0, f1);
          count(f0);
          if (!(h == 1 && j == JCL - 1 && tail)) count(f1);
        }
    } else {
#pragma unroll
      for (int j = 0; j < JCL; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          float t0, t1;
          upk2(tc[j][h], t0, t1);
          atomicAdd(&cons.hist[max(-1, min(__float2int_rd(t0), 256)) + 1], 1u);
          if (!(h == 1 && j == JCL - 1 && tail))
            atomicAdd(&cons.hist[max(-1, min(__float2int_rd(t1), 256)) + 1], 1u);
        }
    }
  } else {
    if (!inside) {
#pragma unroll
      for (int j = 0; j < JCL; ++j)
#pragma unroll
        for (int k = 0; k < 4; ++k) bin[j][k] = max(-1, min(bin[j][k], 256));
    }
#pragma unroll
    for (int j = 0; j < JCL; ++j)
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (!(k == 3 && j == JCL - 1 && tail)) atomicAdd(&cons.hist[bin[j][k] + 1], 1u);
  }
}

template <typename T, int LOG2N, int JCL>
__device__ __forceinline__ void consume_chunk(const T (&X)[JCL][4], Consumer<T>& cons, T sc, T mean,
                                              bool mz, uint32_t b0c) {
  if constexpr (sizeof(T) == 4 && WB_CONS_PAIRS) {
    if (mz) {
      consume_chunk_pairs<LOG2N, JCL>(X, cons, sc, b0c);
      return;
    }
  }
  if (mz) consume_chunk_mz<T, LOG2N, JCL, true>(X, cons, sc, mean, b0c);
  else consume_chunk_mz<T, LOG2N, JCL, false>(X, cons, sc, mean, b0c);
}

// Defect-suite consumer of one chunk (stats.cpp:340-369 pool_sum_squares_test,
// :424-447 rare_event_adjacency): the fp64 sum of squares of this thread's
// emitted (standardized) values and whether any |v| exceeds the threshold.
// Element N-1 is the reserved value, not emitted.
template <typename T, int LOG2N, int JCL, bool MZ>
__device__ __forceinline__ void defect_chunk_mz(const T (&X)[JCL][4], double& dsum, bool& mark, T sc, T mean,
                                                uint32_t b0c, double thr) {
  constexpr bool mz = MZ;
  using G = Geo<T, LOG2N>;
  // four independent accumulators (one per block slot) keep the fp64 add
  // chain short; the order is a tree anyway (reference: sequential)
  double d4[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
  for (int j = 0; j < JCL; ++j) {
    const uint32_t b = b0c + 32 * j;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (k == 3 && b == G::ROWS - 1) continue;
      const double v = static_cast<double>(emit_value(X[j][k], sc, mean, mz));
      d4[k] = __dadd_rn(d4[k], __dmul_rn(v, v));
      mark |= fabs(v) > thr;
    }
  }
  dsum = __dadd_rn(dsum, __dadd_rn(__dadd_rn(d4[0], d4[1]), __dadd_rn(d4[2], d4[3])));
}
template <typename T, int LOG2N, int JCL>
__device__ __forceinline__ void defect_chunk(const T (&X)[JCL][4], double& dsum, bool& mark, T sc, T mean,
                                             bool mz, uint32_t b0c, double thr) {
  if (mz) defect_chunk_mz<T, LOG2N, JCL, true>(X, dsum, mark, sc, mean, b0c, thr);
  else defect_chunk_mz<T, LOG2N, JCL, false>(X, dsum, mark, sc, mean, b0c, thr);
}
__device__ __forceinline__ double warp_sum_f64(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Threads of a pool_kernel instantiation: kModeFillLat adds the chain warp.
template <typename T, int LOG2N, int MODE>
constexpr int kernel_threads() {
  return Geo<T, LOG2N>::THREADS + (MODE == kModeFillLat ? 32 : 0);
}
// Resident CTAs per SM the kernel is compiled for (its register budget).
// The consumer kernel keeps 258 histogram bins and no output path: its CTAs
// are limited by shared memory only, so it may use the registers that leaves.
template <typename T, int LOG2N, int MODE>
constexpr int kernel_minb() {
  using G = Geo<T, LOG2N>;
  if constexpr (MODE == kModeConsume && !G::LAT && WB_CONS_REGS) {
    constexpr int per_cta = G::BUFS * G::N * int(sizeof(T)) + 4096;
    constexpr int by_smem = (220 * 1024) / per_cta;
    constexpr int by_threads = 2048 / G::THREADS;
    constexpr int m0 = by_smem < by_threads ? by_smem : by_threads;
    constexpr int m = m0 > 32 ? 32 : m0;  // at most 32 resident CTAs per SM
    return m < 1 ? 1 : m;
  } else {
    return G::MINB;
  }
}
// kModeFillLat ring: (x_last, sum_sq) of every emission of a launch
constexpr uint32_t kLatRingMax = 2048;

template <typename T, int LOG2N, int MODE, int PT>
__global__ void __launch_bounds__(kernel_threads<T, LOG2N, MODE>(), kernel_minb<T, LOG2N, MODE>())
    pool_kernel(const __grid_constant__ FillArgs a) {
  using G = Geo<T, LOG2N>;
  using SM = Smem<T, LOG2N>;
  // DEC (kModeFillLat): lean pass loop + decoupled chain warp (tid >= CT),
  // DESIGN.md §5 "Latency fills"
  constexpr bool DEC = MODE == kModeFillLat;
  static_assert(!DEC || (G::LAT && !G::CHAINW && PT < 2 && G::CT <= 512), "latency-fill geometry");
  constexpr int N = G::N, ROWS = G::ROWS, J = G::J, THREADS = kernel_threads<T, LOG2N, MODE>();
  constexpr bool FAST = ROWS >= 32;
  // buffer 0 at offset 0, buffer 1 at BSTRIDE; plans in dynamic smem
  constexpr uint32_t FLIP = G::INPLACE ? 0u : SM::BSTRIDE;  // cur_off ^ FLIP = next buffer
  // rotation passes (PT 2, 3) use the other buffer as sweep scratch and end
  // in the current one; their plans are two words per pass
  constexpr bool ROT = PT >= 2;
  constexpr uint32_t PFLIP = ROT ? 0u : FLIP;
  constexpr uint32_t PW = ROT ? 2u : 1u;
  static_assert(!ROT || (G::JC == G::J && !G::INPLACE),
                "rotation passes hold all 4-blocks of a thread across their inner barrier");
  __shared__ __align__(1024) unsigned char s_pool[SM::STATIC ? SM::TOTAL : 16];
  extern __shared__ __align__(1024) unsigned char dsmem[];
  unsigned char* const pbase = SM::STATIC ? s_pool : dsmem;
  T* const pools = reinterpret_cast<T*>(pbase);
  uint32_t* const s_plans = reinterpret_cast<uint32_t*>(dsmem + (SM::STATIC ? 0 : SM::TOTAL));
  // kModeFillLat: (x_last, sum_sq) per emission, after the plans
  double* const ring = reinterpret_cast<double*>(dsmem + (SM::STATIC ? 0 : SM::TOTAL) +
                                                 ((a.n_passes * 4u * (PT >= 2 ? 2u : 1u) + 15u) & ~15u));
  (void)ring;
  // WB_LAT_CLUSTER: one mbarrier per batch of WB_LAT_CBATCH ring entries in
  // the chain CTA, after its ring (each used for exactly one phase)
  uint64_t* const rmbar = reinterpret_cast<uint64_t*>(ring + 2 * size_t(a.n_emit));
  (void)rmbar;
  __shared__ SState s;
  __shared__ uint32_t s_hist[MODE == kModeConsume ? 258 : 1];
  // defect suite: per-warp partial sums / marks of the last two emissions
  __shared__ double s_def[MODE == kModeDefect ? 2 : 1][MODE == kModeDefect ? G::NW : 1];
  __shared__ uint32_t s_defm[MODE == kModeDefect ? 2 : 1][MODE == kModeDefect ? G::NW : 1];
  __shared__ __align__(16) float s_hs[64];  // sign mask -> (0.5*sign_k)_k (transforms.cpp:88)

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t b0 = warp * J * 32 + lane;  // first 4-block of this thread
  const bool compute = !(G::CHAINW || DEC) || tid < G::CT;  // owns 4-blocks (else: chain warp)
  // latency fills with a chain CTA (WB_LAT_CLUSTER): clusters of two CTAs
  // per pool -- rank 0 runs the passes, rank 1 the per-emission chain on
  // its own SM, reading rank 0's ring over distributed shared memory
  constexpr bool CLU = DEC && WB_LAT_CLUSTER;
  const uint32_t crank = CLU ? (blockIdx.x & 1u) : 0u;
  const uint64_t pool = CLU ? (blockIdx.x >> 1) : blockIdx.x;
#ifdef WB_DEBUG_TIMING
  const long long dbg_t0 = clock64();
#endif
  const bool mean_zero = a.mean_is_zero != 0;
  const T mean_t = from_double<T>(a.mean);

  // ---- prologue: state, pool, plans ----------------------------------------
  if (tid == 0) {
    const PoolState& st = a.st_in[pool];
    s.reserved_prev = st.reserved_prev;
    s.sum_sq = st.sum_sq;
    s.cur_scale = st.scale;
    s.last_chi2 = st.last_chi2;
    s.last_r = st.r;
    s.last_scale = st.scale;
    s.closed = -1;
    s.clamp = 0;
    s.zero_seen = 0;
    s.x_last_bulk_set = 0;
    s.ready = 0;
    s.produced = 0;
    s.flags = st.flags & ~kFlagChi2NonFinite;
    if (MODE != kModePasses && !DEC && a.n_emit > 0) chain_draw(s, 0, a.chi2, a.sigma);
  }
  if constexpr (MODE == kModeConsume)
    for (int i = tid; i < 258; i += THREADS) s_hist[i] = 0;
  for (int i = tid; i < 64; i += THREADS) s_hs[i] = ((i >> 2) >> (i & 3)) & 1 ? -0.5f : 0.5f;
  {
    const float4* src = reinterpret_cast<const float4*>(static_cast<const T*>(a.pools_in) + pool * N);
    float4* dst = reinterpret_cast<float4*>(pools);
    constexpr int NV = N * sizeof(T) / 16;
    for (int i = tid; i < NV; i += THREADS) dst[i] = __ldcs(src + i);
  }
  for (uint32_t i = tid; i < a.n_passes * PW; i += THREADS) s_plans[i] = a.plans[pool * a.plan_stride + i];
  const uint64_t pass0 = a.st_in[pool].pass_count;
  const uint32_t cursor0 = a.st_in[pool].cursor;
  __syncthreads();
  if constexpr (CLU) {
    // rank 1: every batch's mbarrier expects its ring entries' bytes; the
    // cluster barrier publishes the initialisation before rank 0's stores
    if (crank == 1 && tid == 0) {
      const uint32_t nb = (a.n_emit + WB_LAT_CBATCH - 1) / WB_LAT_CBATCH;
      for (uint32_t b = 0; b < nb; ++b) {
        mbar_init(rmbar + b, 1);
        const uint32_t cnt = min(uint32_t(WB_LAT_CBATCH), a.n_emit - b * WB_LAT_CBATCH);
        mbar_arrive_expect_tx(rmbar + b, 16u * cnt);
      }
      fence_mbarrier_init_cluster();
    }
    cluster_sync_all();
  }

  T* const out_pool = static_cast<T*>(a.out) + pool * a.out_stride + a.out_offset;
  Consumer<T> cons;
  cons.hist = s_hist;

  // ---- drain the partially consumed emission --------------------------------
  if (MODE != kModePasses && a.lead > 0) {
    const T sc = from_double<T>(s.cur_scale);
    const bool mat = (s.flags & kFlagLeftover) != 0;
    const T* lo = static_cast<const T*>(a.leftover) + pool * (N - 1);
    for (uint32_t i = tid; i < a.lead; i += THREADS) {
      const uint32_t idx = cursor0 + i;
      const T v = mat ? lo[idx] : emit_value(pools[idx], sc, mean_t, mean_zero);
      if constexpr (MODE == kModeConsume) cons.add(v);
      else if constexpr (MODE != kModeDefect) stg1(out_pool + i, v);  // (defect runs start at an emission)
    }
    if constexpr (MODE == kModeConsume) cons.flush();
  }

  const char* const cbase = reinterpret_cast<const char*>(pbase);
  uint32_t cur_off = 0;
  uint32_t sh = 0;  // byte shift of the current buffer's layout (after a bulk emission pass)
  uint32_t pc = static_cast<uint32_t>(pass0 + 1) & 255u;  // pass count after the next pass, mod 256
  uint32_t p = 0;                                          // plan index

  if constexpr (MODE == kModePasses) {
    // cross-pool probes (stats.cpp:310-338, cross_pool_correlation on a
    // streaming generator): thread k follows probe k, x = pool[in_j] before
    // the pass, y = pool[out_i] after it (and after a renormalisation, as
    // step_pass); the ProbeAccumulator sums in pass order, fp64
    const bool probe = tid < int(a.n_probes);
    double pa[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
    if (probe)
      for (int k = 0; k < 6; ++k) pa[k] = a.probe_acc[(pool * a.n_probes + tid) * 6 + k];
    for (; p < a.n_passes; ++p) {
      double px = 0.0;
      if (probe) px = static_cast<double>(reinterpret_cast<const T*>(pbase + cur_off)[a.probe_in[tid]]);
      const uint32_t plan_p = s_plans[p * PW];
      if (compute) {
        for (int c0 = 0; c0 < J; c0 += G::JC) {
          T X[G::JC][4];
          if constexpr (ROT)
            run_pass_rot<T, LOG2N, G::JC, PT & 1>(cbase, cur_off, cur_off ^ FLIP, plan_p, s_plans[p * PW + 1],
                                                  b0 + 32 * c0, X, a.rot_c, a.rot_s);
          else
            run_pass<T, LOG2N, G::JC, PT>(cbase, cur_off, cur_off ^ FLIP, plan_p, b0 + 32 * c0, X, s_hs);
        }
      } else if constexpr (ROT) {
        __syncthreads();  // the chain warp joins the rotation pass's inner barrier
      }
      __syncthreads();
      cur_off ^= PFLIP;
      if (pc == 0)
        renormalize<T, N, THREADS, G::LAT>(reinterpret_cast<T*>(pbase + cur_off), s, tid,
                                            G::INPLACE ? nullptr : reinterpret_cast<double*>(pbase + (cur_off ^ FLIP)));
      pc = (pc + 1) & 255u;
      if (probe) {
        const double y = static_cast<double>(reinterpret_cast<const T*>(pbase + cur_off)[a.probe_out[tid]]);
        pa[0] = __dadd_rn(pa[0], px);
        pa[1] = __dadd_rn(pa[1], __dmul_rn(px, px));
        pa[2] = __dadd_rn(pa[2], y);
        pa[3] = __dadd_rn(pa[3], __dmul_rn(y, y));
        const double w = __dmul_rn(px, y);
        pa[4] = __dadd_rn(pa[4], w);
        pa[5] = __dadd_rn(pa[5], __dmul_rn(w, w));
      }
    }
    if (probe)
      for (int k = 0; k < 6; ++k) a.probe_acc[(pool * a.n_probes + tid) * 6 + k] = pa[k];
  } else if constexpr (DEC) {
    // ---- latency fill (kModeFillLat): a lean pass loop for the compute
    // warps, the chi2/scale chain in the last warp (of the rank-1 CTA with
    // WB_LAT_CLUSTER) ----------------------------------------------------------
    if (compute && crank == 0) {
      bool pending = false;  // thread 0's last row copy may still read its buffer
      uint32_t plan = a.n_passes > 0 ? s_plans[0] : 0u;
      // pool element N-1 and the sum of squares of each emission go to the
      // chain (generator.cpp:358-364, 373-375 run there).  The owner
      // publishes emission e during the NEXT pass, right after that pass's
      // gathers: the release fence then waits on loads the butterfly waits
      // for anyway, instead of standing between the owner and the pass
      // barrier (measured: ~115 cycles per pass on the critical path).
      double ss_reg = s.sum_sq;  // sum_sq changes only at renormalisations
      bool pub = false;          // the owner holds an unpublished entry
      T pub_x = T(0);  // (converted in publish: the owner alone pays for it)
      uint32_t pub_e = 0;
      // rank 1's ring and batch mbarriers in the cluster window, and the
      // row-factor table's shared address, once
      uint32_t ring_r = 0, mbar_r = 0;
      if constexpr (CLU) {
        ring_r = dsmem_addr(ring, 1);
        mbar_r = dsmem_addr(rmbar, 1);
      }
      uint32_t hs_sa;  // (through an asm so that it is kept, not rebuilt from the CTA id each pass)
      asm volatile("mov.u32 %0, %1;" : "=r"(hs_sa) : "r"(static_cast<uint32_t>(__cvta_generic_to_shared(s_hs))));
      auto publish = [&] {
        if constexpr (CLU) {
          // into the chain CTA's ring, completing its batch mbarrier
          if (WB_ABLATE != 18)
            st_async_f64x2(ring_r + 16u * pub_e, static_cast<double>(pub_x), ss_reg,
                           mbar_r + 8u * (pub_e / WB_LAT_CBATCH));
        } else {
          ring[2 * pub_e] = static_cast<double>(pub_x);
          ring[2 * pub_e + 1] = ss_reg;
          if ((pub_e + 1) % WB_LAT_BATCH == 0 || pub_e + 1 == a.n_emit) st_release_cta(&s.produced, pub_e + 1);
        }
        pub = false;
      };
      auto pub_hook = [&] {
        if (pub) publish();
      };
      // this thread's first 4-block in the pitched row of emission e: one
      // pointer advanced by N per emission (the loop is one warp per
      // scheduler: every instruction of a pass is on its critical path)
      T* row_t = static_cast<T*>(a.lat_raw) + (pool * a.lat_rows) * N + 4 * b0;
      const uint32_t lat_n_emit = a.n_emit, lat_d = a.d, lat_n_passes = a.n_passes;
      // one pass of emission e (emit_pass: its last); instantiated twice so that
      // discard_every = 1 -- every pass an emission -- runs a single loop with
      // emit_pass folded (each instruction saved is ~4 cycles of the pass)
      auto lat_pass = [&](uint32_t e, auto emit_tag, bool emit_rt) __attribute__((always_inline)) {
          const bool emit_pass = decltype(emit_tag)::value ? true : emit_rt;
          const bool renorm_now = pc == 0;
          const uint32_t plan_p = plan;
          plan = s_plans[p + 1 < lat_n_passes ? p + 1 : p];  // next pass's plan
          T X[G::J][4];
          if (WB_LAT_DEFER_PUB)
            run_pass<T, LOG2N, G::J, PT, decltype(pub_hook), true>(cbase, cur_off, cur_off ^ FLIP, plan_p, b0, X, s_hs, true,
                                                                   false, pub_hook, hs_sa);
          else
            run_pass<T, LOG2N, G::J, PT, NoHook, true>(cbase, cur_off, cur_off ^ FLIP, plan_p, b0, X, s_hs, true, false,
                                                       NoHook{}, hs_sa);
          T* const row = row_t - 4 * b0;
          if (emit_pass && !renorm_now && tid == G::OWNER) {
            pub_x = X[G::J - 1][3];
            pub_e = e;
            pub = true;
            if (!WB_LAT_DEFER_PUB) publish();
          }
          if (WB_LAT_STG && emit_pass && !renorm_now && WB_ABLATE != 14) {
            // the pool this pass wrote is the raw emission: each thread's
            // 4-blocks go to the pitched row straight from registers
#pragma unroll
            for (int j = 0; j < G::J; ++j) {
              T* const d = row_t + 128 * j;
              stg_vec(d, X[j]);
              if constexpr (sizeof(T) == 8) stg_vec(d + 2, X[j] + 2);
            }
          }
          // WB_LAT_STG 0: the pool this pass wrote is the raw emission, one
          // bulk copy after the barrier sends it to its pitched row
          if (emit_pass && !WB_LAT_STG) fence_proxy_async_smem();
          // the copy issued after the previous pass read the buffer the
          // next pass overwrites
          if (pending && tid == 0) bulk_wait_read();
          pending = false;
          loop_bar<true, G::CT>();
          cur_off ^= FLIP;
          T* const cur = reinterpret_cast<T*>(pbase + cur_off);
          if (renorm_now && WB_ABLATE != 16) {
            renormalize<T, N, G::CT, true, true>(
                cur, s, tid, (G::INPLACE || !WB_LAT_STG) ? nullptr : reinterpret_cast<double*>(pbase + (cur_off ^ FLIP)));
            ss_reg = s.sum_sq;  // (renormalize ends on a barrier)
            if (WB_LAT_STG && emit_pass) {
              // renormalised emission: each thread's own 4-blocks, from the
              // pool (renormalize ends on a barrier)
#pragma unroll
              for (int j = 0; j < G::J; ++j) {
                const T* const v = cur + 4 * (b0 + 32 * j);
                T* const d = row_t + 128 * j;
                stg_vec(d, v);
                if constexpr (sizeof(T) == 8) stg_vec(d + 2, v + 2);
              }
            } else if (emit_pass) {
              fence_proxy_async_smem();
              loop_bar<true, G::CT>();
            }
          }
          if (emit_pass && tid == 0 && renorm_now) {
            // refill_ after step_pass renormalised (generator.cpp:342, 363)
            if constexpr (CLU) {
              st_async_f64x2(dsmem_addr(ring + 2 * e, 1), static_cast<double>(cur[N - 1]), s.sum_sq,
                             dsmem_addr(rmbar + e / WB_LAT_CBATCH, 1));
            } else {
              ring[2 * e] = static_cast<double>(cur[N - 1]);
              ring[2 * e + 1] = s.sum_sq;
              st_release_cta(&s.produced, e + 1);
            }
          }
          if (!WB_LAT_STG && emit_pass && tid == 0) {
            bulk_s2g(row, static_cast<uint32_t>(__cvta_generic_to_shared(cur)), N * uint32_t(sizeof(T)));
            bulk_commit();
            pending = true;
          }
          pc = (pc + 1) & 255u;
      };
      if (lat_d == 1) {
        for (uint32_t e = 0; e < lat_n_emit; ++e, row_t += N, ++p) lat_pass(e, std::true_type{}, true);
      } else {
        for (uint32_t e = 0; e < lat_n_emit; ++e, row_t += N)
          for (uint32_t q = 1; q <= lat_d; ++q, ++p) lat_pass(e, std::false_type{}, q == lat_d);
      }
      if (pub) publish();  // the owner's last emission
      if (tid == 0) {
        if (!WB_LAT_STG) bulk_wait_all();  // the rows are complete before rescale_kernel reads them
        s.end_off = cur_off;
#ifdef WB_DEBUG_TIMING
        printf("compute done at %lld cycles (n_emit %u)\n", clock64() - dbg_t0, a.n_emit);
#endif
      }
    } else {
      // the chain warp (lane 0): the per-emission recurrence of refill_
      // (generator.cpp:358-364, 373-375; chi2.cpp:27-59), one emission
      // behind the passes at most; its scales go to rescale_kernel
      if (!compute && lane == 0 && (!CLU || crank == 1)) {
        // rank 1 (CLU): the chain state from HBM, rank 0's ring and counter
        // over distributed shared memory
        const PoolState& st0 = a.st_in[pool];
        double reserved = CLU ? st0.reserved_prev : s.reserved_prev;
        double lS = CLU ? st0.last_chi2 : s.last_chi2;
        double lr = CLU ? st0.r : s.last_r;
        double lsc = CLU ? st0.scale : s.last_scale;

        uint32_t clamp = 0, flags = 0;
        double* const scl = a.scales + pool * a.scale_stride;
        for (uint32_t e = 0; e < (WB_ABLATE == 13 ? 0u : a.n_emit); ++e) {
          // S_e depends on the previous emission only: drawn while waiting
          const double S0 = a.chi2.disable ? 0.0 : chi2_draw(reserved, a.chi2, clamp, flags);
          double xl, ss;
          if constexpr (CLU) {
            // this CTA's own ring, filled by rank 0's st.async
            if (e % WB_LAT_CBATCH == 0 && WB_ABLATE != 18) mbar_wait_parity(rmbar + e / WB_LAT_CBATCH, 0);
            xl = ring[2 * e];
            ss = ring[2 * e + 1];
          } else {
            while (ld_acquire_cta(&s.produced) <= e) __nanosleep(WB_LAT_POLL_NS);
            xl = ring[2 * e];
            ss = ring[2 * e + 1];
          }
          // disable_chi2: S is the sum of squares refill_ sees (after a
          // renormalisation, the new one: chain_rescale)
          const double S = a.chi2.disable ? ss : S0;
#if WB_ABLATE == 17
          const double r = __dmul_rn(S, 9.765625e-4);  // timing only: no division / square root (N = 1024)
#else
          const double r = ss > 0.0 ? __dsqrt_rn(__ddiv_rn(S, ss)) : 0.0;
#endif
          const double sc = __dmul_rn(a.sigma, r);
          scl[e] = sc;
          reserved = __dmul_rn(xl, r);
          lS = S;
          lr = r;
          lsc = sc;
        }
#ifdef WB_DEBUG_TIMING
        printf("chain done at %lld cycles (rank %u)\n", clock64() - dbg_t0, crank);
#endif
        if constexpr (CLU) {
          // into rank 0's SState for its epilogue (the cluster barrier below
          // orders these stores before rank 0 reads them)
          st_dsmem_f64(dsmem_addr(&s.reserved_prev, 0), reserved);
          st_dsmem_f64(dsmem_addr(&s.last_chi2, 0), lS);
          st_dsmem_f64(dsmem_addr(&s.last_r, 0), lr);
          st_dsmem_f64(dsmem_addr(&s.last_scale, 0), lsc);
          st_dsmem_u32(dsmem_addr(&s.clamp, 0), clamp);
          const uint32_t rf = dsmem_addr(&s.flags, 0);
          st_dsmem_u32(rf, ld_dsmem_u32(rf) | flags);
        } else {
          s.reserved_prev = reserved;
          s.last_chi2 = lS;
          s.last_r = lr;
          s.last_scale = lsc;
          s.clamp = clamp;
          s.flags |= flags;
        }
      }
    }
    if constexpr (CLU) {
      // the chain CTA's results land in rank 0 before its epilogue, and rank
      // 0's shared memory (the ring) outlives rank 1's reads
      cluster_sync_all();
      if (crank == 1) return;
    } else {
      __syncthreads();  // the chain's state and the final buffer precede the epilogue
    }
    cur_off = s.end_off;
  } else {
    uint32_t plan = a.n_passes > 0 ? s_plans[0] : 0u;
    // bulk emission (see "Bulk emission" above; its own instantiation: the
    // register emission path is compiled out there, which keeps the general
    // kernel's registers)
    constexpr bool BULK_OK = MODE == kModeFillBulk;
    static_assert(!BULK_OK || (FAST && !G::LAT && !ROT && !G::CHAINW && !G::INPLACE), "bulk geometry");
    constexpr bool RAWB = BULK_OK;  // raw pool values sent by one bulk copy per emission
    bool bulk_pending = false;
    // staged emission (stage_chunk_any / staged_range above)
    constexpr bool STAGED_OK = MODE == kModeFillStaged;
    static_assert(!STAGED_OK || (FAST && !G::LAT && !ROT && !G::CHAINW && !G::INPLACE && G::JC == G::J),
                  "staged geometry");
    bool stage_pending = false;  // this warp's last bulk copy may still read the next pass's buffer
    constexpr bool DEFER = STAGED_OK && (sizeof(T) == 4 ? WB_DEFER_F32 : WB_DEFER_F64);
    T* gbase = out_pool + a.lead;  // element 0 of the current emission
    for (uint32_t e = 0; e < a.n_emit; ++e, gbase += N - 1) {
      const int slot = e & 1;
      const uint32_t limit = (e + 1 == a.n_emit) ? a.last_limit : uint32_t(N - 1);
      // one pass of emission e (emit_pass: its last).  The consumer instantiates
      // the body twice so that discard_every = 1 runs it with emit_pass folded.
      auto pass_body = [&](auto emit_tag, bool emit_rt) __attribute__((always_inline)) {
        const bool emit_pass = decltype(emit_tag)::value ? true : emit_rt;
        const bool renorm_now = pc == 0;
        const bool fast = FAST && emit_pass && !renorm_now && limit == uint32_t(N - 1);
        // the emission scale is final before this pass (published behind at
        // least one barrier); load it up front so its latency hides
        const double scd = WB_PREFETCH ? s.scale[slot] : 0.0;
        if (!WB_PREFETCH || ROT) plan = s_plans[p * PW];
        const uint32_t plan_p = plan;
        const uint32_t plan_q = ROT ? s_plans[p * PW + 1] : 0u;  // rotation: sweep-1 word
        if (WB_PREFETCH && !ROT) plan = s_plans[p + 1 < a.n_passes ? p + 1 : p];  // next pass's plan
        const bool do_emit = fast && WB_ABLATE != 1;
        T sc = T(0);
        uint32_t delta = 0;
        if (do_emit) {
          sc = from_double<T>(WB_PREFETCH ? scd : s.scale[slot]);
          delta = (G::VEC - (uint32_t)((reinterpret_cast<uintptr_t>(gbase) / sizeof(T)) & (G::VEC - 1))) &
                  (G::VEC - 1);
#if WB_ABLATE == 5
          delta = 0;  // timing-only: every emission aligned (stores at an aligned-down base)
#endif
        }
        // the emission is the pool itself: shifted shared write + bulk copy
        const bool bulk = RAWB && do_emit;
        // element shift of the layout this pass writes (bulk) so that slot
        // and global address of every emitted element agree mod 16 bytes
        const uint32_t sigma = (G::VEC - delta) & (G::VEC - 1);
        uint32_t zf = 0;
        double dsum = 0.0;  // defect suite: this thread's sum of squares / mark
        bool dmark = false;
        T prev[4] = {T(0), T(0), T(0), T(0)};  // lane 31's pending block (emission)
        T x_last = T(0);
        if (G::CHAINW && do_emit && compute) {
          // S/r/scale of emission e come from the chain warp: one lane per
          // warp polls (acquire), __syncwarp orders the other lanes' reads
          if (lane == 0)
            while (ld_acquire_cta(&s.ready) < e) {
              if (WB_CHAIN_SLEEP) __nanosleep(WB_CHAIN_SLEEP);
            }
          __syncwarp();
          sc = from_double<T>(*static_cast<volatile double*>(&s.scale[slot]));
        }
        // chunk of 4-blocks held in registers at a time (half chunks for the
        // consumer remove its spills but cost a second permutation dispatch
        // per pass: measured slower)
        constexpr int JCL = G::JC;
        const bool staged = STAGED_OK && do_emit;
        T Xo[STAGED_OK ? JCL : 1][4];  // staged: the pass's values stay live after the barrier
        for (int c0 = 0; c0 < J && compute; c0 += JCL) {
          T Xi[STAGED_OK ? 1 : JCL][4];
          T (&X)[JCL][4] = *reinterpret_cast<T(*)[JCL][4]>(STAGED_OK ? &Xo[0][0] : &Xi[0][0]);
          if constexpr (ROT)
            run_pass_rot<T, LOG2N, JCL, PT & 1>(cbase, cur_off, cur_off ^ FLIP, plan_p, plan_q, b0 + 32 * c0, X,
                                                a.rot_c, a.rot_s);
          else
            run_pass<T, LOG2N, JCL, PT>(cbase, cur_off + sh, cur_off ^ FLIP, plan_p, b0 + 32 * c0, X, s_hs,
                                        !bulk, STAGED_OK && stage_pending);
          if (do_emit) {
            if constexpr (MODE == kModeDefect) {
              defect_chunk<T, LOG2N, JCL>(X, dsum, dmark, sc, mean_t, mean_zero, b0 + 32 * c0, a.def_threshold);
            } else if constexpr (MODE != kModeConsume) {
              if constexpr (RAWB) {
                T* sb = reinterpret_cast<T*>(pbase + (cur_off ^ FLIP)) + sigma;
                shift_chunk_any<T, LOG2N>(delta, X, c0, prev, sb, lane, warp, &zf);
              } else if constexpr (STAGED_OK) {
                // written after the barrier (below)
              } else {
#if WB_ABLATE == 5
                emit_chunk_any<T, LOG2N>(delta, mean_zero, X, c0, prev,
                                         reinterpret_cast<T*>(reinterpret_cast<uintptr_t>(gbase) & ~uintptr_t(15)),
                                         sc, mean_t, lane, warp);
#else
                emit_chunk_any<T, LOG2N>(delta, mean_zero, X, c0, prev, gbase, sc, mean_t, lane, warp);
#endif
              }
            } else {
              consume_chunk<T, LOG2N, JCL>(X, cons, sc, mean_t, mean_zero, b0 + 32 * c0);
            }
          }
          x_last = X[JCL - 1][3];
        }
        if constexpr (STAGED_OK) stage_pending = false;  // waited for in run_pass
        if constexpr (ROT && G::CHAINW)
          if (!compute) __syncthreads();  // the chain warp joins the rotation pass's inner barrier
        if constexpr (MODE == kModeConsume)
          if (do_emit) cons.flush();
        if constexpr (MODE == kModeDefect) {
          if (do_emit) {
            const double ws = warp_sum_f64(dsum);
            const bool wm = __any_sync(0xffffffffu, dmark);
            if (lane == 0) {
              s_def[slot][warp] = ws;
              s_defm[slot][warp] = wm;
            }
          }
        }
        if (bulk) {
          fence_proxy_async_smem();  // this thread's shared stores -> visible to the bulk copy
          if (BULK_OK && zf) s.zero_seen = 1;
        }
        if (!G::CHAINW && do_emit && tid == G::OWNER && WB_ABLATE != 3 && !DEFER) {
          if constexpr (BULK_OK) {
            // bulk kernels run with disable_chi2: S = sum_sq, r and scale are
            // functions of the current sum_sq alone, nothing in the launch
            // reads them, and only the last emission's values persist
            // (reserved_prev, last_*): the chain runs once, after the loop
            if (e + 1 == a.n_emit) {
              s.x_last_bulk = static_cast<double>(x_last);
              s.x_last_bulk_set = 1;
            }
          } else {
            owner_chain(s, slot, static_cast<double>(x_last), e + 1 < a.n_emit, a.chi2, a.sigma);
          }
        }
        // the bulk copy of the previous emission must have read its source
        // before this barrier releases that buffer for overwriting
        if (bulk_pending && tid == 0) bulk_wait_read();
        bulk_pending = false;
        __syncthreads();
        cur_off ^= PFLIP;
        sh = bulk ? sigma * uint32_t(sizeof(T)) : 0u;
        T* const cur = reinterpret_cast<T*>(pbase + cur_off + sh);
        if constexpr (STAGED_OK) {
          if (staged) {
            // the pass's source buffer is dead: the scaled values go there in
            // the shifted layout, and each warp sends its segment (one bulk
            // copy, issued by lane 0) while the next pass runs; that pass
            // waits for the copy's read before its stores (run_pass)
            // (the scale is read here: for d = 1 the owner publishes it
            // behind the barrier that ends this pass, see below)
            const T scs = DEFER ? from_double<T>(s.scale[slot]) : sc;
            T* const sb = reinterpret_cast<T*>(pbase + (cur_off ^ FLIP)) + sigma;
            T (&X)[JCL][4] = *reinterpret_cast<T(*)[JCL][4]>(&Xo[0][0]);
            if (WB_ABLATE != 8)
              stage_chunk_any<T, LOG2N>(delta, mean_zero, X, 0, prev, sb, gbase, scs, mean_t, lane, warp);
            if (WB_ABLATE != 9) fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
              uint32_t lo, hi;
              staged_range<T, LOG2N>(sigma, warp, lo, hi);
              bulk_s2g(gbase + (lo - sigma), static_cast<uint32_t>(__cvta_generic_to_shared(sb - sigma + lo)),
                       (hi - lo) * uint32_t(sizeof(T)));
              bulk_commit();
            }
            stage_pending = WB_ABLATE != 7;
            // generator.cpp:373-375 for this emission and S/r/scale of the
            // next one, off the barrier's critical path: the next reader is
            // the next emission, behind at least one more barrier
            if (DEFER && tid == G::OWNER && WB_ABLATE != 3)
              owner_chain(s, slot, static_cast<double>(x_last), e + 1 < a.n_emit, a.chi2, a.sigma);
          }
        }
        if (G::CHAINW && fast && tid == G::CT) {
          // generator.cpp:373-375 for emission e, then S/r/scale of e+1; the
          // compute warps pick them up at emission e+1 (acquire on s.ready)
          chain_close(s, slot, static_cast<double>(cur[N - 1]));
          if (e + 1 < a.n_emit) chain_draw(s, slot ^ 1, a.chi2, a.sigma);
          st_release_cta(&s.ready, e + 1);
        }
        if constexpr (MODE == kModeDefect) {
          // the emission's total: reserved^2 (chain_close ran before the
          // barrier) plus the warp partials in warp order; its mark
          if (do_emit && tid == 0) {
            double t = __dmul_rn(s.reserved_prev, s.reserved_prev);
            uint32_t m = 0;
            for (int w = 0; w < G::NW; ++w) {
              t = __dadd_rn(t, s_def[slot][w]);
              m |= s_defm[slot][w];
            }
            a.def_totals[pool * a.def_stride + a.def_e0 + e] = t;
            a.def_marks[pool * a.def_stride + a.def_e0 + e] = m ? 1 : 0;
          }
        }
        if (RAWB && bulk) {
          // the aligned middle [delta, delta + L) in one copy; the <= VEC-1
          // head values [0, delta) and tail values [delta + L, N-1) as
          // scalar stores of x*1 + 0
          constexpr uint32_t NE = N - 1;
          const uint32_t L = ((NE - delta) / G::VEC) * G::VEC;
          if (tid == 0) {
            bulk_s2g(gbase + delta, static_cast<uint32_t>(__cvta_generic_to_shared(cur + delta)),
                     L * uint32_t(sizeof(T)));
            bulk_commit();
          } else if (uint32_t(tid) <= NE - L) {
            const uint32_t t = tid - 1;
            const uint32_t i = t < delta ? t : L + t;
            stg1(gbase + i, fma_rn(cur[i], T(1), T(0)));
          }
          bulk_pending = true;
          if (BULK_OK && s.zero_seen) {  // rare: rewrite -0 as +0 once the bulk copy landed
            if (tid == 0) {
              bulk_wait_all();
              fence_proxy_async_global();
            }
            __syncthreads();
            for (uint32_t i = delta + tid; i < delta + L; i += THREADS)
              if (is_neg_zero(cur[i])) stg1(gbase + i, T(0));
            __syncthreads();
            if (tid == 0) s.zero_seen = 0;
            __syncthreads();
          }
        }
        if (renorm_now) {
          if (G::CHAINW) __syncthreads();  // the chain warp's draw precedes the rescale
          // the consumer (one warp per pool): the warp-parallel sums, inline
          constexpr bool INL = MODE == kModeConsume && WB_CONS_NEUM && THREADS == 32;
          renormalize<T, N, THREADS, G::LAT, false, INL>(
              cur, s, tid, G::INPLACE ? nullptr : reinterpret_cast<double*>(pbase + (cur_off ^ FLIP)));
          // refill_ reads sum_sq after step_pass renormalised (generator.cpp:342, 363)
          if (tid == 0) chain_rescale(s, slot, a.chi2, a.sigma);
          __syncthreads();
        }
        if (emit_pass && !fast) {
          // slow emission from shared memory: the partial last emission, an
          // emission right after a renormalisation, pools below 128 values
          if constexpr (BULK_OK) {
            // the fast emissions skipped the chain: this emission's scale on
            // demand (after a renormalisation chain_rescale already has it)
            if (!renorm_now) {
              if (tid == 0) chain_draw(s, slot, a.chi2, a.sigma);
              __syncthreads();
            }
          }
          const T sc = from_double<T>(s.scale[slot]);
          double ds = 0.0;
          bool dm = false;
          for (uint32_t i = tid; i < limit; i += THREADS) {
            const T v = emit_value(cur[i], sc, mean_t, mean_zero);
            if constexpr (MODE == kModeConsume) {
              cons.add(v);
            } else if constexpr (MODE == kModeDefect) {
              const double dv = static_cast<double>(v);
              ds = __dadd_rn(ds, __dmul_rn(dv, dv));
              dm |= fabs(dv) > a.def_threshold;
            } else {
              stg1(gbase + i, v);
            }
          }
          if constexpr (MODE == kModeConsume) cons.flush();
          if constexpr (MODE == kModeDefect) {
            const double ws = warp_sum_f64(ds);
            const bool wm = __any_sync(0xffffffffu, dm);
            if (lane == 0) {
              s_def[slot][warp] = ws;
              s_defm[slot][warp] = wm;
            }
            __syncthreads();
          }
          if (tid == 0) {
            chain_close(s, slot, static_cast<double>(cur[N - 1]));
            if (e + 1 < a.n_emit) chain_draw(s, slot ^ 1, a.chi2, a.sigma);
            s.ready = e + 1;
            if constexpr (MODE == kModeDefect) {
              double t = __dmul_rn(s.reserved_prev, s.reserved_prev);
              uint32_t m = 0;
              for (int w = 0; w < G::NW; ++w) {
                t = __dadd_rn(t, s_def[slot][w]);
                m |= s_defm[slot][w];
              }
              a.def_totals[pool * a.def_stride + a.def_e0 + e] = t;
              a.def_marks[pool * a.def_stride + a.def_e0 + e] = m ? 1 : 0;
            }
          }
          __syncthreads();
        }
        pc = (pc + 1) & 255u;
      };
      if (MODE == kModeConsume && a.d == 1) {
        pass_body(std::true_type{}, true);
        ++p;
      } else {
        for (uint32_t q = 1; q <= a.d; ++q, ++p) pass_body(std::false_type{}, q == a.d);
      }
    }
    if constexpr (BULK_OK) {
      // the last emission's chain (see above); a slow last emission closed it already
      __syncthreads();
      if (tid == G::OWNER && s.x_last_bulk_set) {
        const int slot = (a.n_emit - 1) & 1;
        chain_draw(s, slot, a.chi2, a.sigma);
        chain_close(s, slot, s.x_last_bulk);
      }
    }
    if (bulk_pending && tid == 0) bulk_wait_all();  // smem must outlive the copies
    if (STAGED_OK && lane == 0) bulk_wait_all();
    __syncthreads();  // the owner's last chain precedes the epilogue
  }
  T* const cur = reinterpret_cast<T*>(pbase + cur_off + sh);

  // ---- epilogue: pool and state back to HBM ---------------------------------
  if (sh == 0) {
    float4* dst = reinterpret_cast<float4*>(static_cast<T*>(a.pools_out) + pool * N);
    const float4* src = reinterpret_cast<const float4*>(cur);
    constexpr int NV = N * sizeof(T) / 16;
    for (int i = tid; i < NV; i += THREADS) dst[i] = src[i];
  } else {  // the last pass was a bulk emission: shifted layout
    T* dst = static_cast<T*>(a.pools_out) + pool * N;
    for (int i = tid; i < N; i += THREADS) dst[i] = cur[i];
  }
  if constexpr (MODE == kModeConsume) {
    // fixed-order block reduction of the moment sums
    __shared__ double s_red[4][32];
    double v[4] = {cons.s1, cons.s2, cons.s3, cons.s4};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v[k] = __dadd_rn(v[k], __shfl_down_sync(0xffffffffu, v[k], o));
    }
    if (lane == 0)
      for (int k = 0; k < 4; ++k) s_red[k][warp] = v[k];
    __syncthreads();
    if (tid < 4) {
      double acc = 0.0;
      for (int w = 0; w < G::NW; ++w) acc = __dadd_rn(acc, s_red[tid][w]);
      a.part_sums[pool * 4 + tid] = acc;
    }
    for (int i = tid; i < 258; i += THREADS) a.part_hist[pool * 258 + i] = s_hist[i];
  }
  if (tid == 0) {
    PoolState& so = a.st_out[pool];
    so.reserved_prev = s.reserved_prev;
    so.sum_sq = s.sum_sq;
    so.pass_count = pass0 + a.n_passes;
    so.clamp_count = a.st_in[pool].clamp_count + s.clamp;
    uint32_t flags = s.flags;
    // chi2_sample threw in the reference (chi2.cpp:29-31): report it to the
    // host; the non-finite reserved value re-raises at every later emission
    if (flags & kFlagChi2NonFinite) atomicOr(a.err_word, 1u);
    flags &= ~kFlagChi2NonFinite;
    so.scale = s.closed >= 0 ? s.scale[s.closed] : s.last_scale;
    so.r = s.last_r;
    so.last_chi2 = s.closed >= 0 ? s.S[s.closed] : s.last_chi2;
    if (MODE != kModePasses && a.n_emit > 0) {
      so.cursor = a.last_limit;
      flags &= ~kFlagLeftover;
    } else {
      so.cursor = cursor0 + (MODE != kModePasses ? a.lead : 0);
    }
    so.flags = flags;
    so.seed = a.st_in[pool].seed;
    if (a.n_passes == 0 && &so != &a.st_in[pool]) {  // no plan launch copied the stream
      for (int k = 0; k < 4; ++k) so.s[k] = a.st_in[pool].s[k];
      so.draws = a.st_in[pool].draws;
    }
  }
}

// ---------------------------------------------------------------------------
// host-callable launch table
// ---------------------------------------------------------------------------
template <typename T, int LOG2N, int MODE, int PT>
cudaError_t launch_pool_mode(const FillArgs& a, uint64_t n_pools, cudaStream_t stream) {
  using SM = Smem<T, LOG2N>;
  constexpr size_t PW = PT >= 2 ? 2 : 1;
  const size_t plans = (a.n_passes * 4 * PW + 15) & ~size_t(15);
  const size_t ring = MODE == kModeFillLat ? 16 * size_t(a.n_emit) + 8 * (size_t(a.n_emit) / WB_LAT_CBATCH + 1) : 0;
  if (MODE == kModeFillLat && a.n_emit > kLatRingMax) return cudaErrorInvalidValue;
  size_t smem = (SM::STATIC ? 0 : size_t(SM::TOTAL)) + plans + ring;
  // latency fills with a chain CTA: more than half an SM's shared memory per
  // CTA, so the two CTAs of a cluster run on different SMs
  constexpr bool CLU = MODE == kModeFillLat && WB_LAT_CLUSTER;
  constexpr size_t kCluSmem = WB_LAT_CLU_SMEM_KB * 1024;
  if (CLU && smem < kCluSmem) smem = kCluSmem;
  auto fn = pool_kernel<T, LOG2N, MODE, PT>;
  // attributes are set once per instantiation and device; concurrent first
  // launches from several host threads set them twice, which is harmless
  static std::atomic<uint64_t> configured{0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return cudaGetLastError();
  const uint64_t dev_bit = uint64_t(1) << (dev & 63);
  if (!(configured.load(std::memory_order_acquire) & dev_bit)) {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout,
                                         cudaSharedmemCarveoutMaxShared);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               int(std::max<size_t>(CLU ? kCluSmem : 0,
                                                    (SM::STATIC ? 16 * 1024 : SM::TOTAL + 16 * 1024) +
                                                        (MODE == kModeFillLat ? 16 * kLatRingMax : 0))));
    if (e != cudaSuccess) return e;
    configured.fetch_or(dev_bit, std::memory_order_release);
  }
  if constexpr (CLU) {
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3(unsigned(2 * n_pools));
    lc.blockDim = dim3(kernel_threads<T, LOG2N, MODE>());
    lc.dynamicSmemBytes = smem;
    lc.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    lc.attrs = attr;
    lc.numAttrs = 1;
    return cudaLaunchKernelEx(&lc, fn, a);
  } else {
    fn<<<dim3(unsigned(n_pools)), dim3(kernel_threads<T, LOG2N, MODE>()), smem, stream>>>(a);
    return cudaGetLastError();
  }
}

template <typename T, int LOG2N, int PT>
cudaError_t launch_pool(const FillArgs& a, uint64_t n_pools, cudaStream_t stream) {
  switch (a.mode) {
    case kModeFill: return launch_pool_mode<T, LOG2N, kModeFill, PT>(a, n_pools, stream);
    case kModeFillBulk:
      // the host selects it for the throughput geometry and wallace4 only
      if constexpr (LOG2N < 16 && LOG2N >= 7 && PT < 2 && !Geo<T, LOG2N>::INPLACE)
        return launch_pool_mode<T, LOG2N, kModeFillBulk, PT>(a, n_pools, stream);
      else
        return cudaErrorInvalidValue;
    case kModeFillLat:
      if constexpr (LOG2N >= 16 + 7 && PT < 2 && Geo<T, LOG2N>::CT <= 512 && !Geo<T, LOG2N>::CHAINW)
        return launch_pool_mode<T, LOG2N, kModeFillLat, PT>(a, n_pools, stream);
      else
        return cudaErrorInvalidValue;
    case kModeFillStaged:
      if constexpr (LOG2N < 16 && LOG2N >= 7 && PT < 2 && !Geo<T, LOG2N>::INPLACE)
        return launch_pool_mode<T, LOG2N, kModeFillStaged, PT>(a, n_pools, stream);
      else
        return cudaErrorInvalidValue;
    case kModePasses: return launch_pool_mode<T, LOG2N, kModePasses, PT>(a, n_pools, stream);
    case kModeDefect: return launch_pool_mode<T, LOG2N, kModeDefect, PT>(a, n_pools, stream);
    default: return launch_pool_mode<T, LOG2N, kModeConsume, PT>(a, n_pools, stream);
  }
}

// WB_QUICK (measurement builds only): the BASELINE configs' sizes, nothing else
#ifndef WB_QUICK
#define WB_QUICK 0
#endif
template <typename T, int PT>
cudaError_t launch_pool_dispatch(int log2n, const FillArgs& a, uint64_t n_pools, cudaStream_t s) {
#if WB_QUICK
  if constexpr (PT != 0) {
    return cudaErrorInvalidValue;
  } else {
    switch (log2n) {
      case 16 + 10: return launch_pool<T, 16 + 10, PT>(a, n_pools, s);
      case 16 + 11: return launch_pool<T, 16 + 11, PT>(a, n_pools, s);
      case 16 + 12: return launch_pool<T, 16 + 12, PT>(a, n_pools, s);
      case 10: return launch_pool<T, 10, PT>(a, n_pools, s);
      case 11: return launch_pool<T, 11, PT>(a, n_pools, s);
      case 12: return launch_pool<T, 12, PT>(a, n_pools, s);
      default: return cudaErrorInvalidValue;
    }
  }
#else
  switch (log2n) {
    // latency kernels (key log2(N) + 16)
    case 16 + 8: return launch_pool<T, 16 + 8, PT>(a, n_pools, s);
    case 16 + 9: return launch_pool<T, 16 + 9, PT>(a, n_pools, s);
    case 16 + 10: return launch_pool<T, 16 + 10, PT>(a, n_pools, s);
    case 16 + 11: return launch_pool<T, 16 + 11, PT>(a, n_pools, s);
    case 16 + 12: return launch_pool<T, 16 + 12, PT>(a, n_pools, s);
    case 16 + 13: return launch_pool<T, 16 + 13, PT>(a, n_pools, s);
    case 16 + 14:
      if constexpr (sizeof(T) == 4) return launch_pool<T, 16 + 14, PT>(a, n_pools, s);
      else return cudaErrorInvalidValue;
    case 5: return launch_pool<T, 5, PT>(a, n_pools, s);
    case 6: return launch_pool<T, 6, PT>(a, n_pools, s);
    case 7: return launch_pool<T, 7, PT>(a, n_pools, s);
    case 8: return launch_pool<T, 8, PT>(a, n_pools, s);
    case 9: return launch_pool<T, 9, PT>(a, n_pools, s);
    case 10: return launch_pool<T, 10, PT>(a, n_pools, s);
    case 11: return launch_pool<T, 11, PT>(a, n_pools, s);
    case 12: return launch_pool<T, 12, PT>(a, n_pools, s);
    case 13: return launch_pool<T, 13, PT>(a, n_pools, s);
    case 14:
      if constexpr (sizeof(T) == 4) return launch_pool<T, 14, PT>(a, n_pools, s);
      else return cudaErrorInvalidValue;
    default: return cudaErrorInvalidValue;
  }
#endif
}

// one translation unit per pass type (pool_pt<PT>.cu) defines this
template <int PT>
cudaError_t launch_pool_pt(int dtype, int log2n, const FillArgs& a, uint64_t n_pools, cudaStream_t s);

}  // namespace wb
