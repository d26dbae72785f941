// wallace_b200.hpp — C++ drop-in for maxent::Generator on a B200.
//
// Header-only layer over the C-ABI (wallace_b200.h).  The reference API
// (/root/reference/proj/core/include/maxent/generator.hpp:18-149) is kept:
// same class and member names, same argument meaning, same exceptions
// (ConfigError naming the field, InvalidParameterError), same stream.
//
//   maxent::Generator           -> wallace_b200::Generator  (one pool, fp64,
//                                  bit-identical to the reference)
//   (many Generators in parallel) -> wallace_b200::PoolBatch (n pools, f32/f64,
//                                  device buffers, the throughput path)
//
// Generator keeps the reference's next_normal() buffer semantics on the host:
// it never reads past the current emission, so step_pass()/inject_pool()
// between calls behave exactly as in the reference (generator.cpp:387-413).
#pragma once

#include <algorithm>
#include <array>
#include <cmath>
#include <cstddef>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <limits>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <string_view>
#include <utility>
#include <vector>

#include "wallace_b200.h"

namespace wallace_b200 {

// maxent/errors.hpp:12-21
class InvalidParameterError : public std::invalid_argument {
 public:
  using std::invalid_argument::invalid_argument;
};
class ConfigError : public std::invalid_argument {
 public:
  using std::invalid_argument::invalid_argument;
};
// a reference option this build does not implement (rotation, affine)
class UnsupportedError : public std::logic_error {
 public:
  using std::logic_error::logic_error;
};
class DeviceError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};

inline void check(wallace_status st) {
  if (st == WALLACE_OK) return;
  const std::string msg = wallace_last_error();
  switch (st) {
    case WALLACE_ERR_CONFIG: throw ConfigError(msg);
    case WALLACE_ERR_INVALID_PARAM: throw InvalidParameterError(msg);
    case WALLACE_ERR_UNSUPPORTED: throw UnsupportedError(msg);
    default: throw DeviceError(msg);
  }
}

// maxent::TransformFamily / MixingScheme / Chi2Method (generator.hpp:19-20, chi2.hpp:21)
enum class TransformFamily { wallace4, rotation };
enum class MixingScheme { stride_transpose, affine };
enum class Chi2Method { sqrt_shift, wilson_hilferty, cubic_a };

// ---- baselines.hpp:27-72: the uniform helper and the conventional normal
// generators (host, bit-identical to the reference through the C-ABI) -------
struct UniformState {
  std::array<std::uint64_t, 4> s{1, 2, 3, 4};
  std::uint64_t draws = 0;
  UniformState() = default;
  explicit UniformState(std::uint64_t seed) {
    wallace_uniform_state c{};
    wallace_uniform_seed(seed, &c);
    from_c(c);
  }
  wallace_uniform_state to_c() const {
    wallace_uniform_state c{};
    for (int k = 0; k < 4; ++k) c.s[k] = s[static_cast<std::size_t>(k)];
    c.draws = draws;
    return c;
  }
  void from_c(const wallace_uniform_state& c) {
    for (int k = 0; k < 4; ++k) s[static_cast<std::size_t>(k)] = c.s[k];
    draws = c.draws;
  }
};
inline std::uint64_t splitmix64(std::uint64_t& state) { return wallace_splitmix64(&state); }
inline std::uint64_t uniform_bits(UniformState& u) {
  wallace_uniform_state c = u.to_c();
  const std::uint64_t w = wallace_uniform_bits(&c);
  u.from_c(c);
  return w;
}
inline double uniform_next(UniformState& u) {
  wallace_uniform_state c = u.to_c();
  const double v = wallace_uniform_next(&c);
  u.from_c(c);
  return v;
}

struct BaselineState {
  UniformState uniform;
  std::optional<double> cached;
  BaselineState() = default;
  explicit BaselineState(std::uint64_t seed) : uniform(seed) {}
  wallace_baseline_state to_c() const {
    wallace_baseline_state c{};
    c.uniform = uniform.to_c();
    c.has_cached = cached ? 1 : 0;
    c.cached = cached ? *cached : 0.0;
    return c;
  }
  void from_c(const wallace_baseline_state& c) {
    uniform.from_c(c.uniform);
    if (c.has_cached) cached = c.cached;
    else cached.reset();
  }
};
inline double polar_next(BaselineState& s) {
  wallace_baseline_state c = s.to_c();
  const double v = wallace_polar_next(&c);
  s.from_c(c);
  return v;
}
inline std::pair<double, double> boxmuller_pair(double u1, double u2) {
  double z1 = 0.0, z2 = 0.0;
  check(wallace_boxmuller_pair(u1, u2, &z1, &z2));
  return {z1, z2};
}
inline double boxmuller_next(BaselineState& s) {
  wallace_baseline_state c = s.to_c();
  const double v = wallace_boxmuller_next(&c);
  s.from_c(c);
  return v;
}
inline double exact_chi2_oracle(std::uint64_t nu, BaselineState& s) {
  wallace_baseline_state c = s.to_c();
  double v = 0.0;
  check(wallace_exact_chi2_oracle(nu, &c, &v));
  s.from_c(c);
  return v;
}

// ---- chi2.hpp:21-41 ----------------------------------------------------------
inline double compute_a(std::uint64_t nu) {
  double a = 0.0;
  check(wallace_compute_a(nu, &a));
  return a;
}
struct Chi2Params {
  std::uint64_t nu = 0;
  double a_value = 0.0;
  static Chi2Params for_nu(std::uint64_t nu) {
    Chi2Params p;
    p.nu = nu;
    check(wallace_chi2_params(nu, &p.a_value));
    return p;
  }
};
inline double chi2_sample(double x, const Chi2Params& params, Chi2Method method, bool* clamped = nullptr) {
  double s = 0.0;
  std::int32_t c = 0;
  check(wallace_chi2_sample(x, params.nu, params.a_value, static_cast<std::int32_t>(method), &c, &s));
  if (clamped != nullptr) *clamped = c != 0;
  return s;
}

// ---- transforms.hpp:21-137 ---------------------------------------------------
struct RotationCoeffs {
  double c;
  double s;
  double t;
};
inline RotationCoeffs rotation_from_t(double t) {
  RotationCoeffs r{0.0, 0.0, t};
  check(wallace_rotation_from_t(t, &r.c, &r.s));
  return r;
}
inline std::pair<double, double> apply_rotation(double x1, double x2, const RotationCoeffs& r) {
  return {r.c * x1 + r.s * x2, -r.s * x1 + r.c * x2};
}
inline std::span<const double> rotation_t_table() {
  static const std::array<double, 16> table = [] {
    std::array<double, 16> t{};
    wallace_rotation_table(t.data(), nullptr, nullptr);
    return t;
  }();
  return table;
}

inline constexpr std::size_t wallace_variant_count = 384;
struct WallaceMatrix {
  std::array<std::array<double, 4>, 4> entries;
  int variant_id = 0;
  std::array<std::uint8_t, 4> source_row{0, 1, 2, 3};
  std::array<double, 4> row_sign{1.0, 1.0, 1.0, 1.0};
};
inline WallaceMatrix wallace_variant(int variant_id) {
  WallaceMatrix m{};
  double e[16];
  check(::wallace_variant(variant_id, e, m.source_row.data(), m.row_sign.data()));
  m.variant_id = variant_id;
  for (int k = 0; k < 4; ++k)
    for (int j = 0; j < 4; ++j) m.entries[static_cast<std::size_t>(k)][static_cast<std::size_t>(j)] = e[4 * k + j];
  return m;
}
inline WallaceMatrix wallace_a1() { return wallace_variant(0); }
inline std::vector<WallaceMatrix> wallace_variants(std::size_t count) {
  if (count < 1 || count > wallace_variant_count)
    throw InvalidParameterError("wallace_variants: count must be in [1, 384], got " + std::to_string(count));
  std::vector<WallaceMatrix> out;
  out.reserve(count);
  for (std::size_t id = 0; id < count; ++id) out.push_back(wallace_variant(static_cast<int>(id)));
  return out;
}
// transforms.hpp:89-103: the signed butterfly (eight additions, one halving
// per output), the op order of the pass kernels
inline std::array<double, 4> apply_wallace4(const std::array<double, 4>& v, const WallaceMatrix& m) {
  const double a = v[0] + v[1], b = v[0] - v[1], c = v[2] + v[3], d = v[2] - v[3];
  const std::array<double, 4> z{a - d, b + c, b - c, -a - d};
  std::array<double, 4> out{};
  for (std::size_t k = 0; k < 4; ++k) out[k] = (0.5 * m.row_sign[k]) * z[m.source_row[k]];
  return out;
}
inline std::uint64_t default_stride(std::uint64_t rows) { return wallace_default_stride(rows); }

// maxent::GeneratorConfig (generator.hpp:21-45)
struct GeneratorConfig {
  std::size_t pool_size = 1024;
  TransformFamily transform_family = TransformFamily::wallace4;
  MixingScheme mixing = MixingScheme::stride_transpose;
  Chi2Method chi2_method = Chi2Method::cubic_a;
  std::size_t discard_every = 1;
  double out_mean = 0.0;
  double out_sigma = 1.0;
  std::uint64_t seed = 0;
  struct Diagnostics {
    bool fixed_transform = false;
    bool disable_chi2 = false;
  } diag;

  wallace_config to_c() const {
    wallace_config c{};
    c.pool_size = pool_size;
    c.transform_family = static_cast<int32_t>(transform_family);
    c.mixing = static_cast<int32_t>(mixing);
    c.chi2_method = static_cast<int32_t>(chi2_method);
    c.fixed_transform = diag.fixed_transform ? 1 : 0;
    c.disable_chi2 = diag.disable_chi2 ? 1 : 0;
    c.discard_every = discard_every;
    c.out_mean = out_mean;
    c.out_sigma = out_sigma;
    c.seed = seed;
    return c;
  }
  // Throws ConfigError naming the offending field (generator.cpp:221-236).
  void validate() const {
    const wallace_config c = to_c();
    check(wallace_validate_config(&c));
  }
};

// maxent::NormalPool (generator.hpp:81-87)
struct NormalPool {
  std::vector<double> raw;
  double reserved_prev = 0.0;
  std::uint64_t pass_count = 0;
  double sum_sq = 0.0;
};

// maxent::PassPlan (generator.hpp:50-55)
struct PassPlan {
  int wallace_variant = 0;
  std::array<int, 2> t_index{0, 0};
  std::array<bool, 2> negate{false, false};
  std::array<std::uint64_t, 2> offset{0, 0};
  wallace_pass_plan to_c() const {
    wallace_pass_plan p{};
    p.wallace_variant = wallace_variant;
    for (int s = 0; s < 2; ++s) {
      p.t_index[s] = t_index[static_cast<std::size_t>(s)];
      p.negate[s] = negate[static_cast<std::size_t>(s)] ? 1 : 0;
      p.offset[s] = offset[static_cast<std::size_t>(s)];
    }
    return p;
  }
};

// maxent::decode_pass_plan / run_pass / pass_coefficient / default_multipliers
// (generator.hpp:56-77); run_pass executes on the device.
inline PassPlan decode_pass_plan(const GeneratorConfig& cfg, std::uint64_t transform_word,
                                 std::uint64_t offset_word) {
  const wallace_config c = cfg.to_c();
  wallace_pass_plan p{};
  check(wallace_decode_pass_plan_ex(&c, transform_word, offset_word, &p));
  PassPlan out;
  out.wallace_variant = p.wallace_variant;
  for (int s = 0; s < 2; ++s) {
    out.t_index[static_cast<std::size_t>(s)] = p.t_index[s];
    out.negate[static_cast<std::size_t>(s)] = p.negate[s] != 0;
    out.offset[static_cast<std::size_t>(s)] = p.offset[s];
  }
  return out;
}
inline void run_pass(const GeneratorConfig& cfg, const PassPlan& plan, std::span<const double> in,
                     std::span<double> out) {
  if (in.size() != cfg.pool_size || out.size() != cfg.pool_size)
    throw InvalidParameterError("run_pass: buffers must match pool_size");
  const wallace_config c = cfg.to_c();
  const wallace_pass_plan p = plan.to_c();
  check(wallace_run_pass(&c, &p, in.data(), out.data()));
}
inline double pass_coefficient(const GeneratorConfig& cfg, const PassPlan& plan, std::size_t out_i,
                               std::size_t in_j) {
  const wallace_config c = cfg.to_c();
  const wallace_pass_plan p = plan.to_c();
  double v = 0.0;
  check(wallace_pass_coefficient(&c, &p, out_i, in_j, &v));
  return v;
}
inline std::pair<std::uint64_t, std::uint64_t> default_multipliers(std::size_t n) {
  std::uint64_t a = 0, b = 0;
  wallace_default_multipliers(n, &a, &b);
  return {a, b};
}

// maxent::ProbePair (stats.hpp:78-81)
struct ProbePair {
  std::size_t out_i;
  std::size_t in_j;
};

// Many independent pools on the device (one reference Generator per pool).
class PoolBatch {
 public:
  PoolBatch(const GeneratorConfig& cfg, std::uint64_t n_pools, const std::uint64_t* seeds = nullptr,
            wallace_dtype dtype = WALLACE_F32, void* stream = nullptr)
      : cfg_(cfg), n_pools_(n_pools), dtype_(dtype) {
    const wallace_config c = cfg.to_c();
    check(wallace_create(&c, n_pools, seeds, dtype, stream, &h_));
  }
  ~PoolBatch() {
    if (h_) wallace_destroy(h_);
  }
  PoolBatch(const PoolBatch&) = delete;
  PoolBatch& operator=(const PoolBatch&) = delete;
  PoolBatch(PoolBatch&& o) noexcept { *this = std::move(o); }
  PoolBatch& operator=(PoolBatch&& o) noexcept {
    std::swap(h_, o.h_);
    cfg_ = o.cfg_;
    n_pools_ = o.n_pools_;
    dtype_ = o.dtype_;
    return *this;
  }

  // fill(count) for every pool into a DEVICE buffer of n_pools*count values
  // (asynchronous: chi2_sample's error is raised by the next synchronising
  // call, e.g. synchronize()).
  void fill_device(void* dev_out, std::uint64_t count_per_pool) {
    check(wallace_fill(h_, dev_out, count_per_pool));
  }
  void synchronize() { check(wallace_synchronize(h_)); }
  // fill(count) for every pool into HOST memory (end to end).
  void fill_host(void* host_out, std::uint64_t count_per_pool) {
    check(wallace_fill_host(h_, host_out, count_per_pool));
  }
  void step_pass(std::uint64_t n = 1) { check(wallace_step_pass(h_, n)); }
  void inject_pool(std::uint64_t pool, std::span<const double> values) {
    check(wallace_inject_pool(h_, pool, values.data(), values.size()));
  }
  wallace_pool_info info(std::uint64_t pool) const {
    wallace_pool_info i{};
    check(wallace_get_pool_info(h_, pool, &i));
    return i;
  }
  std::vector<double> raw(std::uint64_t pool) const {
    std::vector<double> r(cfg_.pool_size);
    check(wallace_get_pool(h_, pool, r.data(), r.size()));
    return r;
  }
  // The gen wire format (cmd_gen.cpp:39-57): `count_per_pool` further
  // values of every pool to fd, pool-major (see wallace_write_stream).
  void write_stream(int fd, std::uint64_t count_per_pool, wallace_format fmt = WALLACE_FMT_F64LE) {
    check(wallace_write_stream(h_, count_per_pool, fmt, fd));
  }
  // Defect-suite accumulators (stats.cpp): `passes` step_pass() with the
  // ProbeAccumulator sums [n_pools][probes][6]; `emissions` next_pool()
  // with the per-emission totals and rare-event marks [n_pools][emissions].
  std::vector<double> cross_pool_probes(std::uint64_t passes, std::span<const ProbePair> probes) {
    std::vector<std::uint64_t> oi, ij;
    for (const auto& p : probes) {
      oi.push_back(p.out_i);
      ij.push_back(p.in_j);
    }
    std::vector<double> acc(n_pools_ * probes.size() * 6);
    check(wallace_cross_pool_probes(h_, passes, static_cast<std::uint32_t>(probes.size()), oi.data(), ij.data(),
                                    acc.data()));
    return acc;
  }
  void pool_defect_stats(std::uint64_t emissions, double threshold, std::vector<double>& totals,
                         std::vector<std::uint8_t>& marks) {
    totals.resize(n_pools_ * emissions);
    marks.resize(n_pools_ * emissions);
    check(wallace_pool_defect_stats(h_, emissions, threshold, totals.data(), marks.data()));
  }
  wallace_handle* handle() const { return h_; }
  const GeneratorConfig& config() const { return cfg_; }
  std::uint64_t n_pools() const { return n_pools_; }

 private:
  GeneratorConfig cfg_;
  std::uint64_t n_pools_ = 0;
  wallace_dtype dtype_ = WALLACE_F32;
  wallace_handle* h_ = nullptr;
};

// maxent::Generator (generator.hpp:98-149): one pool, fp64, bit-identical.
//
// The device generates the stream ahead of the caller, in blocks of kBlock
// values double-buffered in page-locked host memory: while the caller
// consumes block k, block k+1 is generated and copied
// (wallace_fill_host_async).  next_normal() is then an inline cursor as in
// the reference (generator.hpp:102-105) and fill() a copy.  Each block
// starts with a device snapshot (slot = its buffer), so every call that
// observes or changes the pool (step_pass, inject_pool, next_pool, pool()
// and the counters) first rolls the device back to the consumed position
// (restore the current block's snapshot, replay the values consumed from
// it: sync_device_) and sees the reference's state.  A chi2_sample error
// inside a look-ahead block is raised only when the values that need it are
// requested: that part is regenerated exactly, up to the request.
class Generator {
 public:
  static constexpr std::size_t kDefaultBlock = std::size_t(1) << 20;

  explicit Generator(GeneratorConfig cfg, void* stream = nullptr)
      : batch_(cfg, 1, &cfg.seed, WALLACE_F64, stream) {
    if (const char* e = std::getenv("WALLACE_B200_LOOKAHEAD")) kBlock = std::max<std::size_t>(1, std::strtoull(e, nullptr, 10));
    void* p = nullptr;
    check(wallace_host_alloc(2 * kBlock * sizeof(double), &p));
    blk_[0] = static_cast<double*>(p);
    blk_[1] = blk_[0] + kBlock;
  }
  ~Generator() {
    if (inflight_) (void)wallace_synchronize(batch_.handle());
    wallace_host_free(blk_[0]);
  }
  Generator(const Generator&) = delete;
  Generator& operator=(const Generator&) = delete;

  double next_normal() {
    if (cur_ == end_) advance_(1);
    return *cur_++;
  }

  // Exactly equivalent to `count` next_normal() calls. count >= 1.
  std::vector<double> fill(std::size_t count) {
    if (count < 1) throw InvalidParameterError("fill: count must be >= 1");
    std::vector<double> out(count);
    fill(std::span<double>{out});
    return out;
  }
  void fill(std::span<double> out) {
    if (out.empty()) throw InvalidParameterError("fill: count must be >= 1");
    double* dst = out.data();
    std::size_t rest = out.size();
    while (rest > 0) {
      if (cur_ == end_) {
        if (rest >= kBlock) {
          // large requests go straight to the caller's memory from the
          // consumed position
          sync_device_();
          batch_.fill_host(dst, rest);
          return;
        }
        advance_(rest);
      }
      const std::size_t k = std::min<std::size_t>(rest, static_cast<std::size_t>(end_ - cur_));
      std::copy_n(cur_, k, dst);
      cur_ += k;
      dst += k;
      rest -= k;
    }
  }

  struct PoolOutput {
    std::span<const double> values;
    double reserved;
    double chi2_draw;
  };
  // generator.cpp:401-405: refill, discard any partially consumed buffer.
  PoolOutput next_pool() {
    sync_device_();
    last_pool_.resize(batch_.config().pool_size - 1);
    double reserved = 0.0, chi2 = 0.0;
    check(wallace_next_pool_host(batch_.handle(), last_pool_.data(), &reserved, &chi2));
    return {std::span<const double>{last_pool_}, reserved, chi2};
  }

  const GeneratorConfig& config() const { return batch_.config(); }
  const NormalPool& pool() const {
    sync_device_();
    const wallace_pool_info i = batch_.info(0);
    pool_cache_.raw = batch_.raw(0);
    pool_cache_.reserved_prev = i.reserved_prev;
    pool_cache_.pass_count = i.pass_count;
    pool_cache_.sum_sq = i.sum_sq;
    return pool_cache_;
  }
  std::uint64_t pass_count() const { return info_().pass_count; }
  std::uint64_t uniform_draws() const { return info_().uniform_draws; }
  std::uint64_t chi2_clamp_count() const { return info_().chi2_clamp_count; }

  // One regeneration pass, no emission (generator.cpp:333-343).
  void step_pass() {
    sync_device_();
    batch_.step_pass(1);
  }
  // Replace the raw pool; sum of squares recomputed (generator.cpp:407-413).
  void inject_pool(std::span<const double> values) {
    if (values.size() != batch_.config().pool_size)
      throw InvalidParameterError("inject_pool: size must equal pool_size");
    sync_device_();
    batch_.inject_pool(0, values);
  }

  PoolBatch& batch() {
    sync_device_();
    return batch_;
  }

 private:
  // queue block generation into buffer q (snapshot slot q = its start)
  void queue_(int q) const {
    wallace_handle* h = batch_.handle();
    check(wallace_snapshot_ex(h, q));
    check(wallace_fill_host_async(h, blk_[q], kBlock));
    inflight_ = true;
    q_ = q;
  }
  // The current block is used up: make the next one current (at least
  // `want` values) and queue the one after it.
  void advance_(std::size_t want) {
    wallace_handle* h = batch_.handle();
    if (!inflight_) queue_(c_ < 0 ? 0 : c_ ^ 1);
    const wallace_status st = wallace_synchronize(h);
    inflight_ = false;
    if (st == WALLACE_OK) {
      c_ = q_;
      cur_ = blk_[c_];
      end_ = cur_ + kBlock;
      queue_(c_ ^ 1);
      return;
    }
    cur_ = end_ = nullptr;
    c_ = -1;
    if (st != WALLACE_ERR_INVALID_PARAM) check(st);
    // chi2_sample threw inside the look-ahead block: regenerate only what
    // was asked for, so that the error surfaces at the reference's call
    check(wallace_restore_snapshot_ex(h, q_));
    exact_.resize(want);
    check(wallace_fill_host(h, exact_.data(), want));
    cur_ = exact_.data();
    end_ = cur_ + want;
  }
  // Make the device state the consumed position (roll back the look-ahead).
  void sync_device_() const {
    wallace_handle* h = batch_.handle();
    if (inflight_) {
      (void)wallace_synchronize(h);  // an error there is in values not handed out
      inflight_ = false;
      if (c_ < 0 || cur_ == end_) check(wallace_restore_snapshot_ex(h, q_));  // = the current block's end
    }
    if (c_ >= 0 && cur_ != end_) {
      check(wallace_restore_snapshot_ex(h, c_));
      const std::size_t used = static_cast<std::size_t>(cur_ - blk_[c_]);
      if (used > 0) check(wallace_discard(h, used));
    }
    cur_ = end_ = nullptr;
    c_ = -1;
  }
  wallace_pool_info info_() const {
    sync_device_();
    return batch_.info(0);
  }
  PoolBatch batch_;
  std::size_t kBlock = kDefaultBlock;    // values per look-ahead block
  double* blk_[2] = {nullptr, nullptr};  // page-locked look-ahead buffers
  mutable double* cur_ = nullptr;        // [cur_, end_): values not yet handed out
  mutable double* end_ = nullptr;
  mutable int c_ = -1;                   // buffer of the current look-ahead block (-1: none)
  mutable int q_ = 0;                    // buffer being generated
  mutable bool inflight_ = false;
  std::vector<double> exact_;            // exact regeneration after a look-ahead error
  std::vector<double> last_pool_;
  mutable NormalPool pool_cache_;
};

// ---- defect suite (stats.hpp / stats.cpp), accumulated on the device -------

// maxent::TestReport (stats.hpp:37-49, stats.cpp:58-75)
struct TestReport {
  std::string name;
  double statistic = 0.0;
  double expected = 0.0;
  double std_error = 0.0;
  double z_score = 0.0;
  bool pass = true;
  static TestReport make(std::string name, double statistic, double expected, double std_error) {
    TestReport r;
    r.name = std::move(name);
    r.statistic = statistic;
    r.expected = expected;
    r.std_error = std_error;
    if (std_error > 0.0) {
      r.z_score = (statistic - expected) / std_error;
    } else {
      r.z_score = statistic == expected ? 0.0
                                        : std::copysign(std::numeric_limits<double>::infinity(),
                                                        statistic - expected);
    }
    r.pass = std::abs(r.z_score) <= 5.0;
    return r;
  }
  // stats.cpp:77-96: the CLI's report lines (byte-equal to the reference's)
  std::string text() const {
    char buf[256];
    std::snprintf(buf, sizeof(buf), "[%s] %-40s statistic=%- 14.6g expected=%- 14.6g se=%- 12.4g z=%- .3f",
                  pass ? "PASS" : "FAIL", name.c_str(), statistic, expected, std_error, z_score);
    return buf;
  }
  std::string machine() const {
    auto g17 = [](double v) {
      char b[40];
      std::snprintf(b, sizeof(b), "%.17g", v);
      return std::string(b);
    };
    return "name=" + name + ",statistic=" + g17(statistic) + ",expected=" + g17(expected) +
           ",se=" + g17(std_error) + ",z=" + g17(z_score) + ",verdict=" + (pass ? "PASS" : "FAIL");
  }
};

// maxent::MomentSummary / moments (stats.hpp:23-35, stats.cpp:25-56)
struct MomentSummary {
  std::size_t count = 0;
  double mean = 0.0;
  double variance = 0.0;
  double skewness = 0.0;
  double excess_kurtosis = 0.0;
};
inline MomentSummary moments(std::span<const double> samples) {
  if (samples.size() < 2) throw InvalidParameterError("moments: need at least 2 samples");
  double mean = 0.0, m2 = 0.0, m3 = 0.0, m4 = 0.0;
  std::size_t n = 0;
  for (const double x : samples) {
    const double n1 = static_cast<double>(n);
    ++n;
    const double nn = static_cast<double>(n);
    const double delta = x - mean;
    const double delta_n = delta / nn;
    const double delta_n2 = delta_n * delta_n;
    const double term1 = delta * delta_n * n1;
    mean += delta_n;
    m4 += term1 * delta_n2 * (nn * nn - 3.0 * nn + 3.0) + 6.0 * delta_n2 * m2 - 4.0 * delta_n * m3;
    m3 += term1 * delta_n * (nn - 2.0) - 3.0 * delta_n * m2;
    m2 += term1;
  }
  MomentSummary out;
  out.count = n;
  out.mean = mean;
  out.variance = m2 / static_cast<double>(n - 1);
  if (m2 > 0.0) {
    const double nn = static_cast<double>(n);
    out.skewness = std::sqrt(nn) * m3 / std::pow(m2, 1.5);
    out.excess_kurtosis = nn * m4 / (m2 * m2) - 3.0;
  }
  return out;
}

// maxent::moment_reports (stats.cpp:98-109): mean / variance / skewness /
// excess kurtosis against N(0, 1), standard errors 1/sqrt(N), sqrt(2/N),
// sqrt(6/N), sqrt(24/N)
inline std::vector<TestReport> moment_reports(const MomentSummary& m, std::string_view prefix) {
  const double n = static_cast<double>(m.count);
  const std::string p{prefix};
  return {TestReport::make(p + ".mean", m.mean, 0.0, 1.0 / std::sqrt(n)),
          TestReport::make(p + ".variance", m.variance, 1.0, std::sqrt(2.0 / n)),
          TestReport::make(p + ".skewness", m.skewness, 0.0, std::sqrt(6.0 / n)),
          TestReport::make(p + ".excess_kurtosis", m.excess_kurtosis, 0.0, std::sqrt(24.0 / n))};
}

// maxent::CrossPoolOptions (stats.hpp:83-95), streaming variant
struct CrossPoolOptions {
  std::size_t pool_pairs = 100000;  // >= 1e3
  std::vector<ProbePair> probes;    // empty -> default spread of 8 probes
  bool fixed_transform = false;     // fresh Polar pool per pair, one pinned pass
  bool expect_composed_q = false;   // report against q_{i,j} instead of 0
};

// stats.cpp:310-338 on a streaming generator: the probe sums are accumulated
// on the device in pass order (bit-identical), finalized here as
// ProbeAccumulator::finalize (stats.cpp:202-234).
inline std::vector<TestReport> cross_pool_correlation(Generator& gen, const CrossPoolOptions& opts) {
  if (opts.pool_pairs < 1000) throw InvalidParameterError("cross_pool_correlation: pool_pairs must be >= 1000");
  const std::size_t n = gen.config().pool_size;
  std::vector<ProbePair> probes = opts.probes;
  if (probes.empty())
    for (std::size_t k = 0; k < 8; ++k) probes.push_back({(5 * k) % n, (11 * k + 3) % n});
  for (const auto& p : probes)
    if (p.out_i >= n || p.in_j >= n) throw InvalidParameterError("cross_pool_correlation: probe index out of range");
  const std::vector<double> acc = gen.batch().cross_pool_probes(opts.pool_pairs, probes);
  std::vector<TestReport> reports;
  const double nn = static_cast<double>(opts.pool_pairs);
  for (std::size_t k = 0; k < probes.size(); ++k) {
    const double* a = acc.data() + k * 6;
    const std::string name =
        "cross_pool_corr.i" + std::to_string(probes[k].out_i) + ".j" + std::to_string(probes[k].in_j);
    const double mx = a[0] / nn, my = a[2] / nn;
    const double vx = a[1] / nn - mx * mx, vy = a[3] / nn - my * my;
    if (!(vx > 0.0) || !(vy > 0.0))
      throw InvalidParameterError("cross_pool_correlation: zero-variance pool values at probe " + name);
    const double denom = std::sqrt(vx * vy);
    const double cov = a[4] / nn - mx * my;
    const double mean_xy = a[4] / nn;
    const double var_xy = a[5] / nn - mean_xy * mean_xy;
    const double se = std::sqrt(var_xy / nn) / denom;
    reports.push_back(TestReport::make(name, cov / denom, 0.0, se));
  }
  return reports;
}

// stats.cpp:260-307 cross_pool_correlation(cfg, opts): the streaming
// generator, or with fixed_transform fresh Polar pools pushed through one
// pinned pass each (device batch), reported against 0 or q_{i,j}.
inline std::vector<TestReport> cross_pool_correlation(const GeneratorConfig& cfg, const CrossPoolOptions& opts) {
  cfg.validate();
  if (opts.pool_pairs < 1000) throw InvalidParameterError("cross_pool_correlation: pool_pairs must be >= 1000");
  if (!opts.fixed_transform) {
    GeneratorConfig streaming = cfg;
    streaming.diag.fixed_transform = false;
    Generator gen(streaming);
    return cross_pool_correlation(gen, opts);
  }
  const std::size_t n = cfg.pool_size;
  std::vector<ProbePair> probes = opts.probes;
  if (probes.empty())
    for (std::size_t k = 0; k < 8; ++k) probes.push_back({(5 * k) % n, (11 * k + 3) % n});
  std::vector<std::uint64_t> oi, ij;
  for (const auto& p : probes) {
    if (p.out_i >= n || p.in_j >= n) throw InvalidParameterError("cross_pool_correlation: probe index out of range");
    oi.push_back(p.out_i);
    ij.push_back(p.in_j);
  }
  const wallace_config c = cfg.to_c();
  std::vector<double> acc(probes.size() * 6);
  check(wallace_cross_pool_fixed(&c, opts.pool_pairs, static_cast<std::uint32_t>(probes.size()), oi.data(),
                                 ij.data(), acc.data()));
  std::vector<TestReport> reports;
  const double nn = static_cast<double>(opts.pool_pairs);
  const PassPlan plan{};
  for (std::size_t k = 0; k < probes.size(); ++k) {
    const double* a = acc.data() + k * 6;
    const std::string name =
        "cross_pool_corr.i" + std::to_string(probes[k].out_i) + ".j" + std::to_string(probes[k].in_j);
    const double mx = a[0] / nn, my = a[2] / nn;
    const double vx = a[1] / nn - mx * mx, vy = a[3] / nn - my * my;
    if (!(vx > 0.0) || !(vy > 0.0))
      throw InvalidParameterError("cross_pool_correlation: zero-variance pool values at probe " + name);
    const double denom = std::sqrt(vx * vy);
    const double cov = a[4] / nn - mx * my;
    const double mean_xy = a[4] / nn;
    const double var_xy = a[5] / nn - mean_xy * mean_xy;
    const double se = std::sqrt(var_xy / nn) / denom;
    const double expected =
        opts.expect_composed_q ? pass_coefficient(cfg, plan, probes[k].out_i, probes[k].in_j) : 0.0;
    reports.push_back(TestReport::make(name, cov / denom, expected, se));
  }
  return reports;
}

// maxent::PoolSumSquares / pool_sum_squares_test (stats.cpp:340-369); the
// per-pool sums are tree-ordered on the device (equal to rounding).
struct PoolSumSquares {
  TestReport mean_report;
  TestReport variance_report;
};
inline PoolSumSquares pool_sum_squares_test(const GeneratorConfig& cfg, std::size_t pools) {
  if (pools < 1000) throw InvalidParameterError("pool_sum_squares_test: pools must be >= 1000");
  GeneratorConfig standardized = cfg;
  standardized.out_mean = 0.0;
  standardized.out_sigma = 1.0;
  PoolBatch b(standardized, 1, &standardized.seed, WALLACE_F64);
  std::vector<double> sums;
  std::vector<std::uint8_t> marks;
  b.pool_defect_stats(pools, std::numeric_limits<double>::infinity(), sums, marks);
  const MomentSummary m = moments(sums);
  const double nu = static_cast<double>(cfg.pool_size);
  const double pp = static_cast<double>(pools);
  const double se_mean = std::sqrt(m.variance / pp);
  const double se_var = m.variance * std::sqrt(std::max(m.excess_kurtosis + 2.0, 0.0) / pp);
  return {TestReport::make("pool_sum_squares.mean", m.mean, nu, se_mean),
          TestReport::make("pool_sum_squares.variance", m.variance, 2.0 * nu, se_var)};
}

// maxent::rare_event_adjacency (stats.cpp:375-403, 424-447): marks from the
// device, AdjacencyCounter over the consecutive emissions.
inline TestReport rare_event_adjacency(const GeneratorConfig& cfg, std::size_t samples, double threshold) {
  if (threshold < 3.0) throw InvalidParameterError("rare_event_adjacency: threshold must be >= 3");
  if (samples < 100000) throw InvalidParameterError("rare_event_adjacency: samples must be >= 1e5");
  GeneratorConfig standardized = cfg;
  standardized.out_mean = 0.0;
  standardized.out_sigma = 1.0;
  const std::size_t pools = samples / (cfg.pool_size - 1);
  PoolBatch b(standardized, 1, &standardized.seed, WALLACE_F64);
  std::vector<double> sums;
  std::vector<std::uint8_t> marks;
  b.pool_defect_stats(pools, threshold, sums, marks);
  std::uint64_t successors = 0, base = 0, cond_pop = 0, cond = 0;
  for (std::size_t p = 1; p < pools; ++p) {
    ++successors;
    if (marks[p]) ++base;
    if (marks[p - 1]) {
      ++cond_pop;
      if (marks[p]) ++cond;
    }
  }
  std::string name = "rare_event_adjacency.pool" + std::to_string(cfg.pool_size);
  if (cond_pop == 0 || base == 0) return TestReport::make(name + "[no-marks]", 1.0, 1.0, 0.0);
  const double b_rate = static_cast<double>(base) / static_cast<double>(successors);
  const double c_rate = static_cast<double>(cond) / static_cast<double>(cond_pop);
  const double se_cond = std::sqrt(b_rate * (1.0 - b_rate) / static_cast<double>(cond_pop));
  return TestReport::make(name, c_rate / b_rate, 1.0, se_cond / b_rate);
}

}  // namespace wallace_b200
