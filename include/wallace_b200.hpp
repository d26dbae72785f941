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

#include <cstddef>
#include <cstdint>
#include <span>
#include <stdexcept>
#include <string>
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

  // fill(count) for every pool into a DEVICE buffer of n_pools*count values.
  void fill_device(void* dev_out, std::uint64_t count_per_pool) {
    check(wallace_fill(h_, dev_out, count_per_pool));
  }
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
class Generator {
 public:
  explicit Generator(GeneratorConfig cfg, void* stream = nullptr)
      : batch_(cfg, 1, &cfg.seed, WALLACE_F64, stream) {}

  double next_normal() {
    if (cursor_ == buf_.size()) refill_buffer_();
    return buf_[cursor_++];
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
    std::size_t i = 0;
    // values already handed to the host by next_normal come first
    while (i < out.size() && cursor_ < buf_.size()) out[i++] = buf_[cursor_++];
    if (i < out.size()) batch_.fill_host(out.data() + i, out.size() - i);
  }

  struct PoolOutput {
    std::span<const double> values;
    double reserved;
    double chi2_draw;
  };
  // generator.cpp:401-405: refill, discard any partially consumed buffer.
  PoolOutput next_pool() {
    last_pool_.resize(batch_.config().pool_size - 1);
    double reserved = 0.0, chi2 = 0.0;
    check(wallace_next_pool_host(batch_.handle(), last_pool_.data(), &reserved, &chi2));
    buf_.clear();
    cursor_ = 0;
    return {std::span<const double>{last_pool_}, reserved, chi2};
  }

  const GeneratorConfig& config() const { return batch_.config(); }
  const NormalPool& pool() const {
    const wallace_pool_info i = batch_.info(0);
    pool_cache_.raw = batch_.raw(0);
    pool_cache_.reserved_prev = i.reserved_prev;
    pool_cache_.pass_count = i.pass_count;
    pool_cache_.sum_sq = i.sum_sq;
    return pool_cache_;
  }
  std::uint64_t pass_count() const { return batch_.info(0).pass_count; }
  std::uint64_t uniform_draws() const { return batch_.info(0).uniform_draws; }
  std::uint64_t chi2_clamp_count() const { return batch_.info(0).chi2_clamp_count; }

  // One regeneration pass, no emission (generator.cpp:333-343).
  void step_pass() { batch_.step_pass(1); }
  // Replace the raw pool; sum of squares recomputed (generator.cpp:407-413).
  void inject_pool(std::span<const double> values) {
    if (values.size() != batch_.config().pool_size)
      throw InvalidParameterError("inject_pool: size must equal pool_size");
    batch_.inject_pool(0, values);
  }

  PoolBatch& batch() { return batch_; }

 private:
  // Take the rest of the current emission (never more: the reference's out_
  // buffer never holds values of a later emission).
  void refill_buffer_() {
    const wallace_pool_info i = batch_.info(0);
    const std::size_t k = i.buffered > 0 ? i.buffered : batch_.config().pool_size - 1;
    buf_.resize(k);
    batch_.fill_host(buf_.data(), k);
    cursor_ = 0;
  }
  PoolBatch batch_;
  std::vector<double> buf_;
  std::size_t cursor_ = 0;
  std::vector<double> last_pool_;
  mutable NormalPool pool_cache_;
};

}  // namespace wallace_b200
