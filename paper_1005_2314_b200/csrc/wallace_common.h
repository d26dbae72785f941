// Shared host/device definitions for the B200 Wallace pool generator.
//
// Terminology follows the reference (arXiv 1005.2314 / maxent-rng):
//   pool      — N raw normal variates (NormalPool::raw, generator.hpp:81-87)
//   pass      — one regeneration y = Qx over the whole pool (step_pass,
//               generator.cpp:333-343)
//   emission  — one refill_: discard_every passes, then N-1 scaled outputs
//               (generator.cpp:353-376)
//   plan      — the (variant, offset) decoded from two xoshiro words
//               (decode_pass_plan, generator.cpp:238-257)
#pragma once


#include <cstdint>

namespace wb {

// Persistent per-pool state, resident in HBM between launches (the
// checkpoint).  Mirrors the private members of maxent::Generator
// (generator.hpp:140-148) plus the emission bookkeeping needed to resume a
// partially consumed emission without storing it.
struct alignas(16) PoolState {
  double reserved_prev;  // NormalPool::reserved_prev
  double sum_sq;         // NormalPool::sum_sq (cached, updated at renorm/inject)
  double scale;          // out_sigma * r of the current emission
  double r;              // sqrt(S / sum_sq) of the current emission
  double last_chi2;      // S of the current emission (PoolOutput::chi2_draw)
  uint64_t pass_count;   // NormalPool::pass_count
  uint64_t s[4];         // xoshiro256** state (UniformState::s)
  uint64_t draws;        // UniformState::draws
  uint64_t clamp_count;  // chi2 clamp counter
  uint32_t cursor;       // consumed values of the current emission, N-1 = empty
  uint32_t flags;        // kFlagLeftover | kFlagChi2NonFinite
  uint64_t seed;
  uint64_t pad_[2];
};
static_assert(sizeof(PoolState) == 128, "PoolState layout");

constexpr uint32_t kFlagLeftover = 1u;      // leftover emission materialized
constexpr uint32_t kFlagChi2NonFinite = 2u; // chi2_sample saw non-finite x (this launch only;
                                            // reported through FillArgs::err_word)

// Precomputed chi2 constants (chi2.cpp:27-59).  Every entry is computed on
// the host with the same double expression the reference evaluates per call,
// so hoisting them is bit-identical.
struct Chi2Consts {
  double nu;
  double a;            // compute_a(nu)            (cubic_a)
  double cubic_c;      // sqrt(2 * (nu - a * a))   (cubic_a)
  double shift_c;      // sqrt(2 * nu - 1)         (sqrt_shift)
  double wh_sqrt_d;    // sqrt(d), d = 2/(9 nu)    (wilson_hilferty)
  double wh_one_m_d;   // 1 - d                    (wilson_hilferty)
  double floor_v;      // 1e-6 * nu
  int32_t method;      // 0 sqrt_shift, 1 wilson_hilferty, 2 cubic_a
  int32_t disable;     // diag.disable_chi2
};

enum Mode : int32_t {
  kModeFill = 0,     // emit into the caller's buffer
  kModePasses = 1,   // passes only (warm-up / step_pass)
  kModeConsume = 2,  // emit into fused moment/histogram consumer
  kModeFillBulk = 3, // emit into the caller's buffer, every emission the pool
                     // itself (scale 1, mean +0): bulk copies from shared memory
  kModeDefect = 4,   // emit into the defect-suite consumer: per-emission sum
                     // of squares (+ reserved^2) and rare-event mark
  kModeFillStaged = 5, // emit into the caller's buffer, any scale: after the
                     // emission pass's barrier the scaled values are staged
                     // in the dead source buffer and each warp sends its
                     // segment with one bulk copy
  kModeFillLat = 6,  // emit into the caller's buffer, latency geometry: each
                     // emission's raw pool goes to a pitched row by one bulk
                     // copy, a chain warp runs the per-emission chi2/scale
                     // recurrence off the passes' critical path, and
                     // rescale_kernel writes x*scale+mean to the output
  kModeFillPair = 7, // pair_kernel (pool_pair.cu): fp32 N = 4096, wallace4 +
                     // stride mixing, discard_every 2: two passes per
                     // shared-memory round trip, TMA tensor-store emission
};

struct FillArgs {
  const void* pools_in;  // T[n_pools * N]
  void* pools_out;
  const PoolState* st_in;
  PoolState* st_out;
  const uint32_t* plans;  // [n_pools][plan_stride] words: wallace4 offset | variant << 16;
                          // rotation two per pass, offset | t << 16 | negate << 20
  uint32_t plan_stride;
  uint32_t n_passes;      // passes in this launch
  uint32_t d;             // discard_every
  uint32_t lead;          // leftover values emitted before the first pass
  uint32_t n_emit;        // emissions in this launch
  uint32_t last_limit;    // values taken from the last emission (<= N-1)
  int32_t mode;
  int32_t mean_is_zero;   // out_mean == +0.0: x*scale+0 fused (bit-identical)
  int32_t pad_ab;
  void* out;              // T, pool-major
  uint64_t out_stride;    // elements per pool slice
  uint64_t out_offset;    // element offset inside each slice
  void* leftover;         // T[n_pools * (N-1)] materialized leftovers
  double mean;
  double sigma;
  Chi2Consts chi2;
  // pass type (pass_type_of: 2*family + mixing) and, for the rotation
  // family, the 16 table coefficients c, s (transforms.cpp:39-70)
  int32_t pass_type;
  int32_t pad_pt;
  double rot_c[16];
  double rot_s[16];
  // defect suite: kModeDefect per-emission outputs, kModePasses probes
  double* def_totals;     // [n_pools][def_stride]: reserved^2 + sum v^2 per emission
  uint8_t* def_marks;     // [n_pools][def_stride]: any |v| > def_threshold
  uint64_t def_stride;
  uint64_t def_e0;        // emission index of this launch's first emission
  double def_threshold;
  double* probe_acc;      // [n_pools][n_probes][6]: sx, sxx, sy, syy, sxy, sxy2
  uint32_t n_probes;      // 0 = no probes
  uint32_t probe_out[32];
  uint32_t probe_in[32];
  // HBM-resident large pools (wallace_large.cu): second pool buffer, per-pool
  // chain state, the pass constants and the pass count before this launch
  void* lg_pool2;
  void* lg_state;
  uint64_t lg_stride;     // default_stride(rows) % rows
  uint64_t lg_stride_inv; // its inverse mod rows (rows a power of two, stride odd)
  int32_t lg_row_major;   // wallace4 stride passes: a thread per gathered row (coalesced)
  int32_t pad_rm;
  uint64_t lg_alpha;      // default_multipliers(N)
  uint64_t lg_beta;
  uint64_t lg_pass0;
  int32_t lg_log2n;
  int32_t pad_lg;
  double* lg_aux;         // per pool: consumer totals, defect mark, probe x, block partials
  uint64_t lg_aux_stride; // doubles per pool
  uint64_t lg_npools;     // pools of the launch (pool index = blockIdx.y + 65535 * blockIdx.z)
  // kModeFillLat: per-emission scale of each pool, [n_pools][scale_stride],
  // and the raw emissions, one pitched row of N values per emission:
  // [n_pools][lat_rows][N]
  double* scales;
  uint64_t scale_stride;
  void* lat_raw;
  uint64_t lat_rows;
  // consumer (kModeConsume)
  double* part_sums;      // [n_pools][4]
  uint32_t* part_hist;    // [n_pools][258]
  // set (atomicOr 1) when some pool's chi2 draw saw a non-finite reserved
  // value: the reference's chi2_sample throws there (chi2.cpp:29-31)
  uint32_t* err_word;
};

struct PlanArgs {
  const PoolState* st_in;
  PoolState* st_out;
  uint32_t* plans;
  uint32_t plan_stride;
  uint32_t n_passes;
  uint32_t n_pools;
  uint32_t off_mask;       // rows-1 (stride_transpose) or N-1 (affine)
  int32_t fixed_transform;
  int32_t rotation;        // family: two plan words per pass
  int32_t large;           // HBM-resident pools: 31-bit offsets, 2 (wallace4) / 3 (rotation) words
};

}  // namespace wb
