// pair_kernel: fp32 pools of N = 4096, wallace4 passes with stride mixing,
// discard_every = 2 (BASELINE configs 2 and 3) -- two passes per shared-memory
// round trip.
//
// One pass (generator.cpp:64-85) gathers row r = (off + b*STRIDE) mod ROWS of
// the four columns and writes 4-block b.  The NEXT pass's butterfly for row
// r2 reads element c*ROWS + r2 = slot r2 & 3 of 4-block c*ROWS/4 + (r2 >> 2):
// the four 4-blocks q, q + 256, q + 512, q + 768 of one pass are exactly the
// inputs of the next pass's rows 4q .. 4q+3 (a 4x4 transpose in registers).
// A thread that owns those four 4-blocks runs both passes without the pool
// going through shared memory in between: per pass pair the L1TEX data path
// carries 4 B of gathers and 4 B of stores per value instead of 16 B.
//
// A pair is (pA, pB) = (emission e's second pass, emission e+1's first pass):
// the emission sits between the two, in registers, as natural 4-blocks.
//
// Layout L of the pool between pairs (written by pB, gathered by the next
// pA).  pB's outputs are the 4-blocks b' = ((4q + i - offB) * SINV) mod ROWS,
// i = 0..3 (SINV = STRIDE^-1 mod ROWS), scattered; the next pA reads rows
// rho = (offA + (q + 256c')*STRIDE) mod ROWS.  With
//   - rows rotated by R = offA & ~3 inside each column (rho~ = rho - R; the
//     plan of the next pass is known when pB stores), and
//   - 16-byte slot P of rotated 4-block b~: P = (b~ >> 2) + 256 * (b~ & 3),
// the word of element (column c, rho~) is
//   256c + 1024*((rho~ >> 2) & 3) + 4*(rho~ >> 4) + (rho~ & 3)
// and with the thread -> q map  q = SINV * (d - eps) mod 128 (+ 128 g),
// eps = offA & 3, d = 16a + 4((a + warp) & 3) + k for lane = 4a + k:
//   - gathers: rho~ mod 128 = d is static per lane, the bank is 4a + k:
//     32 lanes, 32 banks;
//   - stores: slot P mod 8 = (SINV*q + const) mod 8, and q mod 8 is distinct
//     over each 8-lane phase of a 128-bit store;
//   - the emission's 128-bit stores of natural 4-blocks q + 256c' into the
//     staging row: q mod 8 distinct over each phase.
// All three are bank-conflict-free for every plan offset.
//
// The emission (N-1 values, so row e of the output starts at an address that
// is misaligned by sigma = e mod 4 elements) is staged as y = x*scale + mean
// with value i at slot i + sigma of a staging row, so the row's 16-byte
// pieces line up with global memory, and leaves by one cp.async.bulk (the
// <= 3 head / tail values by scalar stores).  The blocks of a misaligned row
// go out as 32- or 64-bit stores; lane class j = (lane >> 3) & 3 writes
// element (i + j) & 3 in store i so that the 32 lanes hit 32 banks
// (stage_rows).  (TMA tensor stores would take element coordinates, but
// their global address must be 16-byte aligned: tools/probes/tma_probe.cu.)
//
// pB keeps no 24-way dispatch over the row permutation: its blocks go to
// shared memory in butterfly order (bfly_raw) and the next pA -- one slot per
// lane -- gathers position src[slot]; only pA, whose blocks are emitted,
// needs the natural slot order.  The add stages of both butterflies and the
// emission scaling run on f32x2 pairs (FADD2 / FFMA2, bit-identical).
//
// A service warp (warp THREADS/32) runs the per-emission chi2 chain
// (generator.cpp:358-364, 373-375), precomputes the next pair's pB
// constants (make_passb) and issues the bulk copies.  Compute -> service
// hand-offs are named barriers (the service warp sleeps in hardware),
// service -> compute hand-offs are mbarriers that are normally complete when
// waited for.
//
// The host (run_emit) selects this kernel per launch when the launch starts
// at an emission boundary, no pass of it ends on a renormalisation
// (pass_count % 256 == 0, generator.cpp:342) and the output rows are
// 16-byte aligned; everything else runs pool_kernel.
#include "wallace_pool.cuh"

namespace wb {
namespace pairk {

constexpr int LOG2N = 12;
constexpr int N = 1 << LOG2N, ROWS = N / 4, NQ = ROWS / 4;
constexpr uint32_t S = default_stride_c(ROWS) % ROWS;
constexpr uint32_t inv_pow2(uint32_t a) {  // a^-1 mod 2^32, a odd
  uint32_t x = a;
  for (int i = 0; i < 5; ++i) x *= 2u - a * x;
  return x;
}
constexpr uint32_t SINV = inv_pow2(S) & (ROWS - 1);
static_assert(((S * SINV) & (ROWS - 1)) == 1, "stride inverse");
static_assert(NQ == 256, "thread -> q map is written for 256 block quads");
constexpr uint32_t CSTEP = (NQ * S) & (ROWS - 1);  // row step between a quad's 4-blocks
static_assert((CSTEP & 127) == 0, "quad rows agree mod 128");

constexpr uint32_t BUF = N * 4;  // bytes per buffer
// staging rows: 1 (the row is free again once its bulk copy has read it,
// most of a pair before the next emission is staged) or 2
#ifndef WB_PAIR_NSG
#define WB_PAIR_NSG 1
#endif
constexpr int NSG = WB_PAIR_NSG;
constexpr uint32_t SGS = BUF + 16;  // a row holds its emission shifted by up to 3 values
constexpr uint32_t OFF_L0 = 0, OFF_SG0 = 2 * BUF, OFF_PLANS = OFF_SG0 + NSG * SGS;
constexpr uint32_t MAX_PLAN_BYTES = 8 * 1024;

// groups (block quads) per thread: 2 -> 128 threads, 1 -> 256 threads
#ifndef WB_PAIR_G
#define WB_PAIR_G 2
#endif
constexpr int G = WB_PAIR_G;
constexpr int THREADS = 256 / G;
constexpr int JB = 4 * G;  // 4-blocks per thread
#ifndef WB_PAIR_DEBUGKNOBS
#define WB_PAIR_DEBUGKNOBS 0  // 1: WALLACE_B200_PAIR_DEBUG (FillArgs::pad_ab) selects a timing-only ablation
#endif
#ifndef WB_PAIR_NOCHAIN
#define WB_PAIR_NOCHAIN 0  // timing only
#endif
#ifndef WB_PAIR_MINB
#define WB_PAIR_MINB 4
#endif

__device__ __forceinline__ float4 lds128(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr));
  return v;
}
__device__ __forceinline__ float lds32(uint32_t addr) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ void sts32(uint32_t addr, float a) {
  asm volatile("st.shared.f32 [%0], %1;" ::"r"(addr), "f"(a) : "memory");
}
__device__ __forceinline__ void sts64(uint32_t addr, float a, float b) {
  asm volatile("st.shared.v2.f32 [%0], {%1, %2};" ::"r"(addr), "f"(a), "f"(b) : "memory");
}
__device__ __forceinline__ void sts128(uint32_t addr, float a, float b, float c, float d) {
  asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "f"(a), "f"(b), "f"(c), "f"(d) : "memory");
}

// Packed f32x2 butterfly stages (FADD2 on sm_100: two independently rounded
// lanes per instruction, bit-identical to the scalar adds; the negations fold
// into operand modifiers).  lo / hi = two 4-blocks; z as in apply_wallace4
// (transforms.hpp:89-103): z0 = a - d, z1 = b + c, z2 = b - c, z3 = -a - d.
#ifndef WB_PAIR_PACKED
#define WB_PAIR_PACKED 1
#endif
__device__ __forceinline__ uint64_t neg2(uint64_t a) {
  float lo, hi;
  upk2(a, lo, hi);
  return pk2(-lo, -hi);
}
__device__ __forceinline__ void bfly_z2(const float (&vl)[4], const float (&vh)[4], float (&zl)[4], float (&zh)[4]) {
  const uint64_t v0 = pk2(vl[0], vh[0]), v1 = pk2(vl[1], vh[1]), v2 = pk2(vl[2], vh[2]), v3 = pk2(vl[3], vh[3]);
  const uint64_t aa = add2_rn(v0, v1), bb = add2_rn(v0, neg2(v1)), cc = add2_rn(v2, v3), dd = add2_rn(v2, neg2(v3));
  upk2(add2_rn(aa, neg2(dd)), zl[0], zh[0]);
  upk2(add2_rn(bb, cc), zl[1], zh[1]);
  upk2(add2_rn(bb, neg2(cc)), zl[2], zh[2]);
  upk2(add2_rn(neg2(aa), neg2(dd)), zl[3], zh[3]);
}
__device__ __forceinline__ void bfly_z1(const float (&v)[4], float (&z)[4]) {
  const float aa = add_rn(v[0], v[1]);
  const float bb = sub_rn(v[0], v[1]);
  const float cc = add_rn(v[2], v[3]);
  const float dd = sub_rn(v[2], v[3]);
  z[0] = sub_rn(aa, dd);
  z[1] = add_rn(bb, cc);
  z[2] = sub_rn(bb, cc);
  z[3] = sub_rn(-aa, dd);
}
template <int J>
__device__ __forceinline__ void bfly_z(const float (&v)[J][4], float (&z)[J][4]) {
  static_assert(J % 2 == 0, "blocks in pairs");
  if (WB_PAIR_PACKED) {
#pragma unroll
    for (int j = 0; j < J; j += 2) bfly_z2(v[j], v[j + 1], z[j], z[j + 1]);
  } else {
#pragma unroll
    for (int j = 0; j < J; ++j) bfly_z1(v[j], z[j]);
  }
}

// butterfly + signed row permutation of J 4-blocks (apply_wallace4 op order,
// transforms.hpp:89-103; generator.cpp:70-81)
template <int J>
__device__ __forceinline__ void bfly(const float (&v)[J][4], uint32_t plan, const float* hs_lut, float (&X)[J][4]) {
  const uint32_t variant = plan >> 16;
  const uint32_t perm = variant >> 4;
  const float4 h = reinterpret_cast<const float4*>(hs_lut)[variant & 15u];
  const float hs[4] = {h.x, h.y, h.z, h.w};
  float z[J][4];
  bfly_z<J>(v, z);
  switch (perm) {
#define WB_PERM_CASE(P)                                   \
  case P:                                                 \
    _Pragma("unroll") for (int j = 0; j < J; ++j) {       \
      X[j][0] = mul_rn(hs[0], z[j][PermAt<P, 0>::v]);     \
      X[j][1] = mul_rn(hs[1], z[j][PermAt<P, 1>::v]);     \
      X[j][2] = mul_rn(hs[2], z[j][PermAt<P, 2>::v]);     \
      X[j][3] = mul_rn(hs[3], z[j][PermAt<P, 3>::v]);     \
    }                                                     \
    break;
    WB_PERM_CASE(0) WB_PERM_CASE(1) WB_PERM_CASE(2) WB_PERM_CASE(3) WB_PERM_CASE(4)
    WB_PERM_CASE(5) WB_PERM_CASE(6) WB_PERM_CASE(7) WB_PERM_CASE(8) WB_PERM_CASE(9)
    WB_PERM_CASE(10) WB_PERM_CASE(11) WB_PERM_CASE(12) WB_PERM_CASE(13) WB_PERM_CASE(14)
    WB_PERM_CASE(15) WB_PERM_CASE(16) WB_PERM_CASE(17) WB_PERM_CASE(18) WB_PERM_CASE(19)
    WB_PERM_CASE(20) WB_PERM_CASE(21) WB_PERM_CASE(22) WB_PERM_CASE(23)
    default: __builtin_unreachable();  // perm = variant >> 4 < 24 (variant = w0 % 384)
#undef WB_PERM_CASE
  }
}

// Row permutation p as packed 2-bit fields: bits 2k+1:2k = src[k] (slot k of
// an output block is z[src[k]], transforms.cpp:24-35), bits 8+2m+1:8+2m =
// the slot that z[m] goes to.
constexpr uint32_t perm_pack(int p) {
  uint32_t w = 0;
  for (int k = 0; k < 4; ++k) {
    const uint32_t m = uint32_t(perm_at(p, k));
    w |= m << (2 * k);
    w |= uint32_t(k) << (8 + 2 * m);
  }
  return w;
}
#define WB_PP4(a) perm_pack(a), perm_pack(a + 1), perm_pack(a + 2), perm_pack(a + 3)
__constant__ uint32_t c_perm_pack[24] = {WB_PP4(0), WB_PP4(4), WB_PP4(8), WB_PP4(12), WB_PP4(16), WB_PP4(20)};
#undef WB_PP4

// butterfly whose output blocks keep z's order: Y[j][m] = (0.5*sign_k) * z[m]
// with k the slot z[m] belongs to -- the same products as bfly, slot k of the
// block held in position src[k].  No dispatch over the permutation: pB's
// blocks go to shared memory like this and the next pA's gathers (one slot
// per lane) read position src[slot] instead.
template <int J>
__device__ __forceinline__ void bfly_raw(const float (&v)[J][4], uint32_t plan, const float* hs_lut,
                                         float (&Y)[J][4]) {
  const uint32_t variant = plan >> 16;
  const uint32_t pk = c_perm_pack[variant >> 4] >> 8;
  const float* hsv = hs_lut + 4u * (variant & 15u);
  const float hm[4] = {hsv[pk & 3u], hsv[(pk >> 2) & 3u], hsv[(pk >> 4) & 3u], hsv[(pk >> 6) & 3u]};
  float z[J][4];
  bfly_z<J>(v, z);
#pragma unroll
  for (int j = 0; j < J; ++j)
#pragma unroll
    for (int m = 0; m < 4; ++m) Y[j][m] = mul_rn(hm[m], z[j][m]);
}
// position of slot k in a block stored by bfly_raw under `plan`
__device__ __forceinline__ uint32_t raw_slot(uint32_t plan, uint32_t k) {
  return (c_perm_pack[plan >> 20] >> (2u * k)) & 3u;
}

// pB: the pass over rows 4q .. 4q+3 of each group (inputs: slot i of the
// group's four 4-blocks), stored in layout L rotated for the next pass.
// X[g*4 + c][k]: 4-block q_g + 256c of the pool before the pass.
__device__ __forceinline__ void pass_b(const float (&X)[JB][4], uint32_t plan, uint32_t off_next,
                                       const uint32_t (&tq)[G], uint32_t lbuf, const float* hs_lut) {
  float v[JB][4], Y[JB][4];
#pragma unroll
  for (int g = 0; g < G; ++g)
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int c = 0; c < 4; ++c) v[g * 4 + i][c] = X[g * 4 + c][i];
  bfly_raw<JB>(v, plan, hs_lut, Y);
  const uint32_t off = plan & 0xffffu;
  const uint32_t rot = off_next >> 2;  // rotation of the next pass, in 4-blocks
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    // output 4-block of row 4q + i: b' = ((4q + i - off) * SINV) mod ROWS
    //   = 4*((q*SINV + m) mod 256) + n with (i - off)*SINV = 4m + n mod ROWS
    const uint32_t ci = ((uint32_t(i) - off) * SINV) & (ROWS - 1);
    const uint32_t cr = (ci - rot) & (ROWS - 1);  // low 8 bits: rotated inside the column
    const uint32_t m1 = (ci >> 2) << 4;
    const uint32_t m2 = (((cr >> 2) & 63u) << 4) + ((cr & 3u) << 12);
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const uint32_t a1 = (tq[g] << 4) + m1;          // bits 11:10: the column
      const uint32_t a2 = ((tq[g] & 63u) << 4) + m2;  // bits 9:4: slot in the plane
      const uint32_t addr = ((a1 & 0xC00u) | (a2 & ~0xC00u)) + lbuf;  // (lbuf is not 4 KiB aligned)
      sts128(addr, Y[g * 4 + i][0], Y[g * 4 + i][1], Y[g * 4 + i][2], Y[g * 4 + i][3]);
    }
  }
}

// The plan-dependent constants of pass_b, one set per row i of a quad:
// m1 / m2 as in pass_b and hm = bfly_raw's factors.  Uniform over the CTA,
// so the service warp's lanes 0..3 compute them one pair ahead (make_passb)
// and the compute warps read them with three broadcast loads (pass_b_desc).
struct PassB {
  uint32_t m1[4], m2[4];
  float hm[4];
};
__device__ __forceinline__ void make_passb(uint32_t plan, uint32_t off_next, uint32_t i, const float* hs_lut,
                                           uint32_t& m1, uint32_t& m2, float& hm) {
  const uint32_t off = plan & 0xffffu, rot = off_next >> 2;
  const uint32_t ci = ((i - off) * SINV) & (ROWS - 1);
  const uint32_t cr = (ci - rot) & (ROWS - 1);
  m1 = (ci >> 2) << 4;
  m2 = (((cr >> 2) & 63u) << 4) + ((cr & 3u) << 12);
  const uint32_t variant = plan >> 16;
  const uint32_t pk = c_perm_pack[variant >> 4] >> 8;
  hm = hs_lut[4u * (variant & 15u) + ((pk >> (2u * i)) & 3u)];
}
// pB in two parts: the add stages (X -> z) and the factors + stores.  With
// WB_PAIR_LATE_STAGE the emission is staged between the two, so the wait for
// the staging row comes one add stage later.
#ifndef WB_PAIR_LATE_STAGE
#define WB_PAIR_LATE_STAGE 0  // measured slower (3.14 vs 2.85 ms: register pressure, 40 bytes of spills)
#endif
__device__ __forceinline__ void pass_b_adds(const float (&X)[JB][4], float (&z)[JB][4]) {
  float v[JB][4];
#pragma unroll
  for (int g = 0; g < G; ++g)
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int c = 0; c < 4; ++c) v[g * 4 + i][c] = X[g * 4 + c][i];
  bfly_z<JB>(v, z);
}
__device__ __forceinline__ void pass_b_stores(const float (&z)[JB][4], const PassB& d, const uint32_t (&tq)[G],
                                              uint32_t lbuf) {
  uint32_t t16[G], t6[G];
#pragma unroll
  for (int g = 0; g < G; ++g) {
    t16[g] = tq[g] << 4;
    t6[g] = (tq[g] & 63u) << 4;
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const uint32_t a1 = t16[g] + d.m1[i], a2 = t6[g] + d.m2[i];
      const uint32_t addr = ((a1 & 0xC00u) | (a2 & ~0xC00u)) + lbuf;
      const float(&zz)[4] = z[g * 4 + i];
      sts128(addr, mul_rn(d.hm[0], zz[0]), mul_rn(d.hm[1], zz[1]), mul_rn(d.hm[2], zz[2]), mul_rn(d.hm[3], zz[3]));
    }
}

// named barriers: 1 = the compute warps' pair barrier; 2, 3 = "staging row of
// an even / odd emission complete", 4, 5 = "pool element N-1 of an even / odd
// emission published" (compute warps arrive, the service warp waits; two
// ids each: an arrival for emission e + 2 follows the service warp's wait
// for emission e through the staging row's hand-back)
template <int ID, int NT>
__device__ __forceinline__ void nbar_sync() {
  asm volatile("bar.sync %0, %1;" ::"n"(ID), "n"(NT) : "memory");
}
template <int ID, int NT>
__device__ __forceinline__ void nbar_arrive() {
  asm volatile("bar.arrive %0, %1;" ::"n"(ID), "n"(NT) : "memory");
}
// The compute warps' pair barrier, split: a warp arrives when its pB stores
// are done and waits just before the next pair's first gather, so the next
// pair's address arithmetic runs while the other warps finish.
#ifndef WB_PAIR_SPLITBAR
#define WB_PAIR_SPLITBAR 0  // measured equal (2.849 vs 2.847 ms): the named barrier stays
#endif
// service warp -> compute warps through mbarriers (count 1; arrive =
// release, try_wait = acquire; normally complete when waited for): emission
// e uses slot e & 1 of xl / scale and waits for completion e >> 1 of the
// slot's barrier; staging row e % NSG is free again at completion e / NSG
// (+1: pre-arrived in the prologue).  Compute -> service: named barriers.
struct PairSync {
  double xl[2];                       // pool element N-1 of the emission in each slot (generator.cpp:373)
  float scf[2];                       // (float)scale of the emission in each slot
  // pB of the pair in each slot, precomputed by the service warp (PassB)
  __align__(16) uint32_t d_m1[2][4];
  __align__(16) uint32_t d_m2[2][4];
  __align__(16) float d_hm[2][4];
  __align__(8) uint64_t mb_scale[2];  // S / r / scale of the slot final (service warp; slot 0 pre-arrived)
  __align__(8) uint64_t mb_copied[2]; // staging row read by its bulk copy (service warp; pre-arrived)
  __align__(8) uint64_t mb_pair;      // WB_PAIR_SPLITBAR: the compute warps' pair barrier (one arrival per warp)
};
__device__ __forceinline__ void mbar_arrive(uint64_t* m) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(m)))
               : "memory");
}

// The same on shared-window addresses: the compute loop keeps PairSync's
// address in a register (ptxas otherwise rebuilds it from SR_CgaCtaId, a
// long-latency read, in every pair).
__device__ __forceinline__ void mbar_wait_parity_sa(uint32_t addr, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WB_MBAR_WAITSA_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WB_MBAR_WAITSA_%=;\n}" ::"r"(addr),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ float lds32_volatile(uint32_t addr) {
  float v;
  asm volatile("ld.volatile.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr) : "memory");
  return v;
}
__device__ __forceinline__ void sts_f64(uint32_t addr, double v) {
  asm volatile("st.shared.f64 [%0], %1;" ::"r"(addr), "d"(v) : "memory");
}

// the emission's values y = x*scale + mean of one thread's JB natural
// 4-blocks into the staging row: value i at slot i + sigma (sigma = the
// output row's misalignment in values), so the row's 16-byte pieces line up
// with global memory for the bulk copy.  SG = sigma class: 0 aligned (one
// 128-bit store per block), 2 even (two 64-bit stores), 1 odd (four 32-bit
// stores).
//
// Bank conflicts: the lanes of a warp that share q mod 8 (same lk, same
// parity of la) are la = la0 + 2j, j = cls = (lane >> 3) & 3.  A narrow store
// of the same element by all lanes would hit each bank group four (32-bit)
// or two (64-bit, per half-warp) times, so in store i lane class j writes
// element (i + j) & 3 (pair (i + j) & 1): bank (4q + sigma + k) mod 32 is
// then distinct over the 32 lanes, and every store is one wavefront per 128
// bytes.  The per-lane rotation of the four values costs two select stages.
#ifndef WB_PAIR_ROT
#define WB_PAIR_ROT 1  // 0: every lane stores the same element (4-way / 2-way conflicts)
#endif
template <bool MZ, int SG>
__device__ __forceinline__ void stage_rows(const float (&X)[JB][4], const uint32_t (&q)[G], uint32_t sgs, float sc,
                                           float mean_t, uint32_t cls) {
  const bool r1 = WB_PAIR_ROT && (cls & 1u), r2 = WB_PAIR_ROT && (cls & 2u);
#pragma unroll
  for (int g = 0; g < G; ++g) {
    const uint32_t aq = sgs + 16u * q[g];
    // byte address of store i of this lane (block c1 = 0)
    uint32_t ai[4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
      ai[i] = SG == 1 ? aq + 4u * ((uint32_t(i) + (WB_PAIR_ROT ? cls : 0u)) & 3u)
                      : aq + 8u * ((uint32_t(i) + (WB_PAIR_ROT ? cls : 0u)) & 1u);
#pragma unroll
    for (int c1 = 0; c1 < 4; ++c1) {
      const float(&x)[4] = X[g * 4 + c1];
      float y0, y1, y2, y3;
      if (MZ && WB_PAIR_PACKED) {
        // fma(x, scale, +0) on slot pairs (emit_value's mean-zero form)
        const uint64_t sc2 = pk2(sc, sc), z2 = pk2(0.f, 0.f);
        upk2(fma2_rn(pk2(x[0], x[1]), sc2, z2), y0, y1);
        upk2(fma2_rn(pk2(x[2], x[3]), sc2, z2), y2, y3);
      } else {
        y0 = emit_value(x[0], sc, mean_t, MZ), y1 = emit_value(x[1], sc, mean_t, MZ);
        y2 = emit_value(x[2], sc, mean_t, MZ), y3 = emit_value(x[3], sc, mean_t, MZ);
      }
      if (SG == 0) {
        sts128(aq + 4096u * c1, y0, y1, y2, y3);
      } else if (SG == 2) {
        // pairs (y0, y1) and (y2, y3); odd classes store the upper pair first
        const float p0 = r1 ? y2 : y0, p1 = r1 ? y3 : y1, p2 = r1 ? y0 : y2, p3 = r1 ? y1 : y3;
        sts64(ai[0] + 4096u * c1, p0, p1);
        sts64(ai[1] + 4096u * c1, p2, p3);
      } else {
        const float t0 = r1 ? y1 : y0, t1 = r1 ? y2 : y1, t2 = r1 ? y3 : y2, t3 = r1 ? y0 : y3;
        const float u0 = r2 ? t2 : t0, u1 = r2 ? t3 : t1, u2 = r2 ? t0 : t2, u3 = r2 ? t1 : t3;
        sts32(ai[0] + 4096u * c1, u0);
        sts32(ai[1] + 4096u * c1, u1);
        sts32(ai[2] + 4096u * c1, u2);
        sts32(ai[3] + 4096u * c1, u3);
      }
    }
  }
}
template <bool MZ>
__device__ __forceinline__ void stage_emission(const float (&X)[JB][4], const uint32_t (&q)[G], uint32_t sgs,
                                               uint32_t sigma, float sc, float mean_t, uint32_t cls) {
  if (sigma == 0) stage_rows<MZ, 0>(X, q, sgs, sc, mean_t, cls);
  else if (sigma == 2) stage_rows<MZ, 2>(X, q, sgs, sc, mean_t, cls);
  else stage_rows<MZ, 1>(X, q, sgs, sc, mean_t, cls);
}

__global__ void __launch_bounds__(THREADS + 32, WB_PAIR_MINB) pair_kernel(const __grid_constant__ FillArgs a) {
  extern __shared__ __align__(1024) unsigned char dsm[];
  uint32_t* const s_plans = reinterpret_cast<uint32_t*>(dsm + OFF_PLANS);
  __shared__ SState s;
  __shared__ PairSync ps;
  __shared__ __align__(16) float s_hs[64];  // sign mask -> (0.5*sign_k)_k (transforms.cpp:88)

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NTHR = THREADS + 32;   // compute warps + the service warp
  constexpr int SERVICE = THREADS / 32;
  const uint64_t pool = blockIdx.x;
  const uint32_t sbase = static_cast<uint32_t>(__cvta_generic_to_shared(dsm));
  const bool mean_zero = a.mean_is_zero != 0;
  // timing-only ablations (tools/dbg/pair_abl.sh): compiled in with
  // -DWB_PAIR_DEBUGKNOBS=1 only, so the product kernel carries no checks
  const int pad_ab = WB_PAIR_DEBUGKNOBS ? a.pad_ab : 0;
  const float mean_t = __double2float_rn(a.mean);

  // ---- prologue: state, pool (natural order, into L1), plans ----
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
    s.flags = st.flags & ~kFlagChi2NonFinite;
    chain_draw(s, 0, a.chi2, a.sigma);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&ps.mb_scale[i], 1);
      mbar_init(&ps.mb_copied[i], 1);
    }
    mbar_init(&ps.mb_pair, THREADS / 32);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    ps.scf[0] = __double2float_rn(s.scale[0]);
    mbar_arrive(&ps.mb_scale[0]);  // emission 0's scale: chain_draw above
    for (int i = 0; i < NSG; ++i) mbar_arrive(&ps.mb_copied[i]);  // the rows start free
  }
  for (int i = tid; i < 64; i += NTHR) s_hs[i] = ((i >> 2) >> (i & 3)) & 1 ? -0.5f : 0.5f;
  {
    const float4* src = reinterpret_cast<const float4*>(static_cast<const float*>(a.pools_in) + pool * N);
    float4* dst = reinterpret_cast<float4*>(dsm + OFF_L0 + BUF);
    for (int i = tid; i < N / 4; i += NTHR) dst[i] = __ldcs(src + i);
  }
  for (uint32_t i = tid; i < a.n_passes; i += NTHR) s_plans[i] = a.plans[pool * a.plan_stride + i];
  const uint64_t pass0 = a.st_in[pool].pass_count;
  __syncthreads();
  if (tid < 4 && a.n_emit > 1)
    make_passb(s_plans[2], s_plans[3] & 0xffffu, tid, s_hs, ps.d_m1[0][tid], ps.d_m2[0][tid], ps.d_hm[0][tid]);
  __syncthreads();

  float* const out_pool = static_cast<float*>(a.out) + pool * a.out_stride + a.out_offset + a.lead;
  const uint32_t n_emit = a.n_emit;
  const bool last_full = a.last_limit == uint32_t(N - 1);
  const uint32_t n_full = last_full ? n_emit : n_emit - 1;  // emissions that go through the staging rows

  if (warp == SERVICE) {
    // ---- service warp: the per-emission chain (generator.cpp:358-364,
    // 373-375; chi2.cpp:27-59) off the compute warps' critical path, and the
    // staging rows to global memory.  Row e of the output starts e mod 4
    // values off a 16-byte boundary, so the rows leave as 128-byte lines of
    // 32-bit stores (lane l writes value l of a line) rather than by bulk copies.
    for (uint32_t e = 0; e < n_full; ++e) {
      const int slot = e & 1;
      // xl[slot] is published: a hardware barrier, so the service warp
      // takes no issue slots while it waits
      if (e & 1u) nbar_sync<5, NTHR>();
      else nbar_sync<4, NTHR>();
      if (lane == 0) {
        if (!WB_PAIR_NOCHAIN) owner_chain(s, slot, ps.xl[slot], e + 1 < n_emit, a.chi2, a.sigma);
        ps.scf[slot ^ 1] = __double2float_rn(s.scale[slot ^ 1]);
      }
      // pB of pair e + 1 (plans 2e + 4, 2e + 5), handed over with the scale
      if (lane < 4 && e + 2 < n_emit)
        make_passb(s_plans[2 * e + 4], s_plans[2 * e + 5] & 0xffffu, lane, s_hs, ps.d_m1[slot ^ 1][lane],
                   ps.d_m2[slot ^ 1][lane], ps.d_hm[slot ^ 1][lane]);
      __syncwarp();
      if (lane == 0) mbar_arrive(&ps.mb_scale[slot ^ 1]);
      __syncwarp();
      // every compute thread staged its values of emission e
      if (e & 1u) nbar_sync<3, NTHR>();
      else nbar_sync<2, NTHR>();
      if (pad_ab < 2 || pad_ab >= 4) {
        // the row holds value i at slot i + sigma, so slot and global address
        // agree mod 16 bytes: the aligned middle [delta, delta + L) leaves by
        // one bulk copy, the <= 3 head and <= 3 tail values by scalar stores
        const float* row = reinterpret_cast<const float*>(dsm + OFF_SG0 + (NSG == 2 ? (e & 1u) : 0u) * SGS);
        // (5, timing only: four output rows per pool, resident in L2)
        float* const gp = out_pool + size_t(pad_ab == 5 ? (e & 3u) : e) * (N - 1);
        float* gpa = gp;
        if (pad_ab == 4) gpa = reinterpret_cast<float*>(reinterpret_cast<uintptr_t>(gp) & ~uintptr_t(15));
        const uint32_t sigma = uint32_t(reinterpret_cast<uintptr_t>(gpa) >> 2) & 3u;
        const uint32_t delta = (4u - sigma) & 3u;
        const uint32_t L = ((uint32_t(N - 1) - delta) / 4u) * 4u;
#ifndef WB_PAIR_L2HINT
#define WB_PAIR_L2HINT 0  // 1 evict_first, 2 evict_last on the output copies (measurement knob)
#endif
#ifndef WB_PAIR_SPLIT
#define WB_PAIR_SPLIT 1  // bulk copies per row (measurement knob)
#endif
        if (lane == 0) {
          const uint32_t src0 = static_cast<uint32_t>(__cvta_generic_to_shared(row + delta + sigma));
          constexpr uint32_t PIECE = (uint32_t(N) / WB_PAIR_SPLIT) * 4u;  // bytes, a multiple of 16
#pragma unroll
          for (int k = 0; k < WB_PAIR_SPLIT; ++k) {
            const uint32_t o = uint32_t(k) * PIECE;
            const uint32_t bytes = k + 1 < WB_PAIR_SPLIT ? PIECE : L * 4u - o;
#if WB_PAIR_L2HINT
            {
              uint64_t pol;
              if (WB_PAIR_L2HINT == 1) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
              else asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
              asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(
                               reinterpret_cast<char*>(gpa + delta) + o),
                           "r"(src0 + o), "r"(bytes), "l"(pol)
                           : "memory");
            }
#else
            bulk_s2g(reinterpret_cast<char*>(gpa + delta) + o, src0 + o, bytes);
#endif
          }
          bulk_commit();
        } else if (uint32_t(lane) <= uint32_t(N - 1) - L) {
          const uint32_t t = lane - 1;
          const uint32_t i = t < delta ? t : L + t;
          stg1(gp + i, row[i + sigma]);
        }
        __syncwarp();
        if (lane == 0 && pad_ab != 6) bulk_wait_read();  // (6, timing only: the row is handed back at once)
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&ps.mb_copied[NSG == 2 ? (e & 1u) : 0u]);
    }
    if (lane == 0) bulk_wait_all();  // shared memory outlives the copies
  } else {
    // lane -> d = 16a + 4e + k (see the header): static part of every gather
    const uint32_t la = uint32_t(lane) >> 2, lk = uint32_t(lane) & 3u, le = (la + uint32_t(warp)) & 3u;
    const uint32_t d = 16u * la + 4u * le + lk;
    const uint32_t lbase = 4u * (1024u * le + 4u * la);  // + the lane's slot position (raw_slot)
    const uint32_t g0 = G == 2 ? 0u : (uint32_t(warp) >> 2);  // G == 1: warps 4..7 take the upper quads
    uint32_t ps_sa;  // PairSync's shared-window address, kept in a register
    asm volatile("mov.u32 %0, %1;" : "=r"(ps_sa) : "r"(static_cast<uint32_t>(__cvta_generic_to_shared(&ps))));

    // first pass of emission 0 (pB only): natural 4-blocks in, layout L out
    {
      uint32_t tq[G];
      float X[JB][4];
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const uint32_t q = ((SINV * d) & 127u) + 128u * (g0 + g);
        tq[g] = (q * SINV) & 255u;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const float4 t = lds128(sbase + OFF_L0 + BUF + 16u * q + 4096u * c);
          X[g * 4 + c][0] = t.x;
          X[g * 4 + c][1] = t.y;
          X[g * 4 + c][2] = t.z;
          X[g * 4 + c][3] = t.w;
        }
      }
      pass_b(X, s_plans[0], s_plans[1] & 0xffffu, tq, sbase + OFF_L0, s_hs);
    }
    if (WB_PAIR_SPLITBAR) {
      __syncwarp();
      if (lane == 0) mbar_arrive(&ps.mb_pair);
    } else {
      nbar_sync<1, THREADS>();
    }

    // (a single loop over the passes with one butterfly site -- a third of
    // the code -- measured slower: 4.00 vs 3.67 ms per 2^32 values)
    for (uint32_t e = 0; e < n_emit; ++e) {
      const int slot = e & 1;
      const bool more = e + 1 < n_emit;
      const bool full = more || last_full;
      const uint32_t plan_a = s_plans[2 * e + 1];
      const uint32_t eps = plan_a & 3u;
      // the blocks in shared memory were stored by bfly_raw under the previous pass's plan
      const uint32_t lcur = sbase + OFF_L0 + (e & 1u) * BUF + 4u * raw_slot(s_plans[2 * e], lk);
      const uint32_t lnxt = sbase + OFF_L0 + ((e + 1) & 1u) * BUF;

      // ---- pA: gather from layout L, butterfly ----
      uint32_t q[G], tq[G];
      float v[JB][4], X[JB][4];
      uint32_t ga[G][4];
#pragma unroll
      for (int g = 0; g < G; ++g) {
        q[g] = ((SINV * (d - eps)) & 127u) + 128u * (g0 + g);
        tq[g] = (q[g] * SINV) & 255u;
        const uint32_t u = eps + S * q[g];
#pragma unroll
        for (int c1 = 0; c1 < 4; ++c1) ga[g][c1] = lcur + lbase + ((u + CSTEP * c1) & 896u);
      }
      // every warp's pB stores of the previous pair (completion e of mb_pair)
      if (WB_PAIR_SPLITBAR) mbar_wait_parity(&ps.mb_pair, e & 1u);
#pragma unroll
      for (int g = 0; g < G; ++g)
#pragma unroll
        for (int c1 = 0; c1 < 4; ++c1)
#pragma unroll
          for (int c = 0; c < 4; ++c) v[g * 4 + c1][c] = lds32(ga[g][c1] + 1024u * c);
      bfly<JB>(v, plan_a, s_hs, X);

      // pool element N-1 (4-block ROWS-1 = quad 255, column 3, slot 3) to the chain
      if (full) {
        if (q[G - 1] == uint32_t(NQ - 1))
          sts_f64(ps_sa + uint32_t(offsetof(PairSync, xl)) + 8u * uint32_t(slot), static_cast<double>(X[(G - 1) * 4 + 3][3]));
        __syncwarp();
        if (e & 1u) nbar_arrive<5, NTHR>();
        else nbar_arrive<4, NTHR>();
      }

      // pB's add stages ahead of the staging (WB_PAIR_LATE_STAGE)
      float zb[JB][4];
      if (WB_PAIR_LATE_STAGE && more) pass_b_adds(X, zb);

      // ---- the emission: y = x*scale + mean into the staging row ----
      // this emission's scale (and the pair's pB constants) are final
      if (full) mbar_wait_parity_sa(ps_sa + uint32_t(offsetof(PairSync, mb_scale)) + 8u * uint32_t(slot), (e >> 1) & 1u);
      if (full && pad_ab != 3) {
        // the staging row's previous contents have left
        mbar_wait_parity_sa(ps_sa + uint32_t(offsetof(PairSync, mb_copied)) + 8u * (NSG == 2 ? (e & 1u) : 0u),
                            (NSG == 2 ? (e >> 1) : e) & 1u);
        const float sc = lds32_volatile(ps_sa + uint32_t(offsetof(PairSync, scf)) + 4u * uint32_t(slot));
        uint32_t sigma = uint32_t(reinterpret_cast<uintptr_t>(out_pool + size_t(e) * (N - 1)) >> 2) & 3u;
        if (pad_ab == 4) sigma = 0;  // (timing only: every row aligned)
        const uint32_t sgs = sbase + OFF_SG0 + (NSG == 2 ? (e & 1u) : 0u) * SGS + 4u * sigma;
        if (mean_zero) stage_emission<true>(X, q, sgs, sigma, sc, mean_t, la >> 1);
        else stage_emission<false>(X, q, sgs, sigma, sc, mean_t, la >> 1);
        fence_proxy_async_smem();  // the staged values -> visible to the bulk copy
      }
      if (full) {
        if (e & 1u) nbar_arrive<3, NTHR>();
        else nbar_arrive<2, NTHR>();
      }

      // ---- pB (the next emission's first pass) or the final pool in natural order ----
      if (more) {
        PassB d;
        {
          const float4 m1 = lds128(ps_sa + uint32_t(offsetof(PairSync, d_m1)) + 16u * uint32_t(slot));
          const float4 m2 = lds128(ps_sa + uint32_t(offsetof(PairSync, d_m2)) + 16u * uint32_t(slot));
          const float4 hm = lds128(ps_sa + uint32_t(offsetof(PairSync, d_hm)) + 16u * uint32_t(slot));
          d.m1[0] = __float_as_uint(m1.x), d.m1[1] = __float_as_uint(m1.y);
          d.m1[2] = __float_as_uint(m1.z), d.m1[3] = __float_as_uint(m1.w);
          d.m2[0] = __float_as_uint(m2.x), d.m2[1] = __float_as_uint(m2.y);
          d.m2[2] = __float_as_uint(m2.z), d.m2[3] = __float_as_uint(m2.w);
          d.hm[0] = hm.x, d.hm[1] = hm.y, d.hm[2] = hm.z, d.hm[3] = hm.w;
        }
        if (!WB_PAIR_LATE_STAGE) pass_b_adds(X, zb);
        pass_b_stores(zb, d, tq, lnxt);
      } else {
#pragma unroll
        for (int g = 0; g < G; ++g)
#pragma unroll
          for (int c1 = 0; c1 < 4; ++c1) {
            const float(&x)[4] = X[g * 4 + c1];
            sts128(lnxt + 16u * q[g] + 4096u * c1, x[0], x[1], x[2], x[3]);
          }
      }
      if (WB_PAIR_SPLITBAR) {
        __syncwarp();
        if (lane == 0) mbar_arrive(&ps.mb_pair);
      } else {
        nbar_sync<1, THREADS>();
      }

      if (!full) {
        if (WB_PAIR_SPLITBAR) mbar_wait_parity(&ps.mb_pair, (e + 1) & 1u);
        // the partial last emission, from the natural-order pool
        mbar_wait_parity(&ps.mb_scale[slot], (e >> 1) & 1u);
        const float* nat = reinterpret_cast<const float*>(dsm + OFF_L0 + ((e + 1) & 1u) * BUF);
        const float scp = *static_cast<volatile float*>(&ps.scf[slot]);
        float* const gb = out_pool + size_t(e) * (N - 1);
        for (uint32_t i = tid; i < a.last_limit; i += THREADS) stg1(gb + i, emit_value(nat[i], scp, mean_t, mean_zero));
        if (tid == 0) chain_close(s, slot, static_cast<double>(nat[N - 1]));
      }
    }
  }
  __syncthreads();  // the service warp's last chain and the final pool precede the epilogue

  // ---- epilogue: pool (natural order) and state back to HBM ----
  {
    const float4* src = reinterpret_cast<const float4*>(dsm + OFF_L0 + (n_emit & 1u) * BUF);
    float4* dst = reinterpret_cast<float4*>(static_cast<float*>(a.pools_out) + pool * N);
    for (int i = tid; i < N / 4; i += NTHR) dst[i] = src[i];
  }
  if (tid == 0) {
    PoolState& so = a.st_out[pool];
    so.reserved_prev = s.reserved_prev;
    so.sum_sq = s.sum_sq;
    so.pass_count = pass0 + a.n_passes;
    so.clamp_count = a.st_in[pool].clamp_count + s.clamp;
    uint32_t flags = s.flags;
    // chi2_sample threw in the reference (chi2.cpp:29-31)
    if (flags & kFlagChi2NonFinite) atomicOr(a.err_word, 1u);
    flags &= ~(kFlagChi2NonFinite | kFlagLeftover);
    so.scale = s.closed >= 0 ? s.scale[s.closed] : s.last_scale;
    so.r = s.last_r;
    so.last_chi2 = s.closed >= 0 ? s.S[s.closed] : s.last_chi2;
    so.cursor = a.last_limit;
    so.flags = flags;
    so.seed = a.st_in[pool].seed;
  }
}

}  // namespace pairk

// a: mode kModeFillPair launch: lead == 0, d == 2, n_passes == 2 * n_emit >= 2
cudaError_t launch_pair_kernel(const FillArgs& a, uint64_t n_pools, cudaStream_t stream) {
  static std::atomic<uint64_t> configured{0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return cudaGetLastError();
  const uint64_t dev_bit = uint64_t(1) << (dev & 63);
  if (!(configured.load(std::memory_order_acquire) & dev_bit)) {
    cudaError_t e = cudaFuncSetAttribute(pairk::pair_kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                                         cudaSharedmemCarveoutMaxShared);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(pairk::pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               int(pairk::OFF_PLANS + pairk::MAX_PLAN_BYTES));
    if (e != cudaSuccess) return e;
    configured.fetch_or(dev_bit, std::memory_order_release);
  }
  if (size_t(a.n_passes) * 4 > pairk::MAX_PLAN_BYTES || a.n_emit < 1 || a.n_passes != 2 * a.n_emit)
    return cudaErrorInvalidValue;
  const size_t smem = pairk::OFF_PLANS + ((size_t(a.n_passes) * 4 + 15) & ~size_t(15));
  pairk::pair_kernel<<<dim3(unsigned(n_pools)), dim3(pairk::THREADS + 32), smem, stream>>>(a);
  return cudaGetLastError();
}

}  // namespace wb
