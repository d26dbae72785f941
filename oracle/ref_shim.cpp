// TEST INFRASTRUCTURE ONLY — extern "C" shim over the UNMODIFIED reference
// library (maxent::Generator and friends).  oracle/Makefile compiles this file
// together with the reference sources where they lie under
// /root/reference/proj/core/src into oracle/_ref/libmaxent_ref.so.  It is used
// to pin the C oracle (tests/test_oracle_pin.py), to generate golden fixtures
// (tests/golden/make_golden.py) and as the CPU arm of bench.py
// (`--impl reference`, `cpu_baseline.kind = "reference"`).
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <span>
#include <string>
#include <thread>
#include <vector>

#include "maxent/baselines.hpp"
#include "maxent/chi2.hpp"
#include "maxent/generator.hpp"
#include "maxent/stats.hpp"
#include "maxent/transforms.hpp"

namespace {
thread_local std::string g_err;

maxent::GeneratorConfig to_cfg(uint64_t pool_size, int chi2_method,
                               uint64_t discard_every, double mean,
                               double sigma, uint64_t seed, int fixed,
                               int disable_chi2, int family = 0,
                               int mixing = 0) {
  maxent::GeneratorConfig c;
  c.pool_size = pool_size;
  c.transform_family = static_cast<maxent::TransformFamily>(family);
  c.mixing = static_cast<maxent::MixingScheme>(mixing);
  c.chi2_method = static_cast<maxent::Chi2Method>(chi2_method);
  c.discard_every = discard_every;
  c.out_mean = mean;
  c.out_sigma = sigma;
  c.seed = seed;
  c.diag.fixed_transform = fixed != 0;
  c.diag.disable_chi2 = disable_chi2 != 0;
  return c;
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

void* ref_create(uint64_t pool_size, int chi2_method, uint64_t discard_every,
                 double mean, double sigma, uint64_t seed, int fixed,
                 int disable_chi2) {
  try {
    return new maxent::Generator(to_cfg(pool_size, chi2_method, discard_every,
                                        mean, sigma, seed, fixed,
                                        disable_chi2));
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

void* ref_create_ex(uint64_t pool_size, int chi2_method, uint64_t discard_every,
                    double mean, double sigma, uint64_t seed, int fixed,
                    int disable_chi2, int family, int mixing) {
  try {
    return new maxent::Generator(to_cfg(pool_size, chi2_method, discard_every,
                                        mean, sigma, seed, fixed, disable_chi2,
                                        family, mixing));
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

void ref_rotation_table(double* t16, double* c16, double* s16) {
  const auto tab = maxent::rotation_t_table();
  for (size_t k = 0; k < tab.size() && k < 16; ++k) {
    const auto rc = maxent::rotation_from_t(tab[k]);
    t16[k] = rc.t;
    c16[k] = rc.c;
    s16[k] = rc.s;
  }
}

void ref_default_multipliers(uint64_t n, uint64_t* alpha, uint64_t* beta) {
  const auto ab = maxent::default_multipliers(n);
  *alpha = ab.first;
  *beta = ab.second;
}

void ref_destroy(void* g) { delete static_cast<maxent::Generator*>(g); }

int ref_fill(void* g, double* out, uint64_t count) {
  try {
    static_cast<maxent::Generator*>(g)->fill(std::span<double>(out, count));
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// next_normal / next_pool can throw (chi2_sample on a non-finite reserved
// value, chi2.cpp:29-31): *err / the return value report it
double ref_next_normal_ex(void* g, int* err) {
  try {
    *err = 0;
    return static_cast<maxent::Generator*>(g)->next_normal();
  } catch (const std::exception& e) {
    g_err = e.what();
    *err = 1;
    return 0.0;
  }
}

double ref_next_normal(void* g) {
  int err = 0;
  return ref_next_normal_ex(g, &err);
}

int ref_next_pool(void* g, double* values, double* reserved, double* chi2) {
  try {
    auto po = static_cast<maxent::Generator*>(g)->next_pool();
    if (values) std::memcpy(values, po.values.data(), po.values.size() * 8);
    *reserved = po.reserved;
    *chi2 = po.chi2_draw;
    return static_cast<int>(po.values.size());
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

void ref_step_pass(void* g) { static_cast<maxent::Generator*>(g)->step_pass(); }

int ref_inject_pool(void* g, const double* v, uint64_t n) {
  try {
    static_cast<maxent::Generator*>(g)->inject_pool(
        std::span<const double>(v, n));
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

void ref_get_pool(void* g, double* raw) {
  const auto& p = static_cast<maxent::Generator*>(g)->pool();
  std::memcpy(raw, p.raw.data(), p.raw.size() * 8);
}

void ref_get_stats(void* g, uint64_t* pass_count, uint64_t* draws,
                   uint64_t* clamp, double* sum_sq, double* reserved_prev) {
  auto* gen = static_cast<maxent::Generator*>(g);
  *pass_count = gen->pass_count();
  *draws = gen->uniform_draws();
  *clamp = gen->chi2_clamp_count();
  *sum_sq = gen->pool().sum_sq;
  *reserved_prev = gen->pool().reserved_prev;
}

void ref_uniform_bits(uint64_t seed, uint64_t n, uint64_t* out) {
  maxent::UniformState u(seed);
  for (uint64_t i = 0; i < n; ++i) out[i] = maxent::uniform_bits(u);
}

uint64_t ref_default_stride(uint64_t rows) { return maxent::default_stride(rows); }

double ref_compute_a(uint64_t nu) { return maxent::compute_a(nu); }

double ref_chi2_sample(double x, uint64_t nu, int method, int* clamped) {
  bool c = false;
  const double s = maxent::chi2_sample(x, maxent::Chi2Params::for_nu(nu),
                                       static_cast<maxent::Chi2Method>(method),
                                       &c);
  *clamped = c ? 1 : 0;
  return s;
}

void ref_wallace_variant(int id, int src[4], double sign[4], double entries[16]) {
  const auto m = maxent::wallace_variant(id);
  for (int k = 0; k < 4; ++k) {
    src[k] = m.source_row[k];
    sign[k] = m.row_sign[k];
    for (int j = 0; j < 4; ++j) entries[4 * k + j] = m.entries[k][j];
  }
}

int ref_decode_pass_plan(uint64_t pool_size, uint64_t w0, uint64_t w1,
                         uint64_t* offset0) {
  maxent::GeneratorConfig c;
  c.pool_size = pool_size;
  const auto plan = maxent::decode_pass_plan(c, w0, w1);
  *offset0 = plan.offset[0];
  return plan.wallace_variant;
}

// decode_pass_plan for any family/mixing: ints = {variant, t0, t1, neg0, neg1}
void ref_decode_pass_plan_ex(uint64_t pool_size, int family, int mixing, uint64_t w0,
                             uint64_t w1, int32_t* ints, uint64_t* offsets) {
  maxent::GeneratorConfig c;
  c.pool_size = pool_size;
  c.transform_family = static_cast<maxent::TransformFamily>(family);
  c.mixing = static_cast<maxent::MixingScheme>(mixing);
  const auto plan = maxent::decode_pass_plan(c, w0, w1);
  ints[0] = plan.wallace_variant;
  ints[1] = plan.t_index[0];
  ints[2] = plan.t_index[1];
  ints[3] = plan.negate[0] ? 1 : 0;
  ints[4] = plan.negate[1] ? 1 : 0;
  offsets[0] = plan.offset[0];
  offsets[1] = plan.offset[1];
}

// The reference's defect-suite reports (stats.cpp), for pinning the GPU
// accumulators: out[k*4 + {0..3}] = statistic, expected, se, z of report k.
int ref_cross_pool_correlation(void* g, uint64_t pool_pairs, uint32_t n_probes,
                               const uint64_t* out_i, const uint64_t* in_j, double* out) {
  try {
    maxent::CrossPoolOptions o;
    o.pool_pairs = pool_pairs;
    for (uint32_t k = 0; k < n_probes; ++k) o.probes.push_back({out_i[k], in_j[k]});
    const auto reps = maxent::cross_pool_correlation(*static_cast<maxent::Generator*>(g), o);
    for (size_t k = 0; k < reps.size(); ++k) {
      out[k * 4 + 0] = reps[k].statistic;
      out[k * 4 + 1] = reps[k].expected;
      out[k * 4 + 2] = reps[k].std_error;
      out[k * 4 + 3] = reps[k].z_score;
    }
    return static_cast<int>(reps.size());
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

int ref_pool_sum_squares(uint64_t pool_size, int chi2_method, uint64_t discard_every, uint64_t seed,
                         int disable_chi2, int family, int mixing, uint64_t pools, double* out) {
  try {
    const auto r = maxent::pool_sum_squares_test(
        to_cfg(pool_size, chi2_method, discard_every, 0.0, 1.0, seed, 0, disable_chi2, family, mixing),
        pools);
    const maxent::TestReport* rs[2] = {&r.mean_report, &r.variance_report};
    for (int k = 0; k < 2; ++k) {
      out[k * 4 + 0] = rs[k]->statistic;
      out[k * 4 + 1] = rs[k]->expected;
      out[k * 4 + 2] = rs[k]->std_error;
      out[k * 4 + 3] = rs[k]->z_score;
    }
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

int ref_rare_event_adjacency(uint64_t pool_size, int chi2_method, uint64_t discard_every,
                             uint64_t seed, int disable_chi2, uint64_t samples, double threshold,
                             double* out) {
  try {
    const auto r = maxent::rare_event_adjacency(
        to_cfg(pool_size, chi2_method, discard_every, 0.0, 1.0, seed, 0, disable_chi2), samples,
        threshold);
    out[0] = r.statistic;
    out[1] = r.expected;
    out[2] = r.std_error;
    out[3] = r.z_score;
    return r.name.find("[no-marks]") != std::string::npos ? 1 : 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// run_pass / pass_coefficient with an explicit plan {variant, t0, t1, neg0, neg1}, {off0, off1}
static maxent::PassPlan plan_of(const int32_t* ints, const uint64_t* offs) {
  maxent::PassPlan p;
  p.wallace_variant = ints[0];
  p.t_index = {ints[1], ints[2]};
  p.negate = {ints[3] != 0, ints[4] != 0};
  p.offset = {offs[0], offs[1]};
  return p;
}
int ref_run_pass(uint64_t n, int family, int mixing, const int32_t* ints, const uint64_t* offs, const double* in,
                 double* out) {
  try {
    maxent::run_pass(to_cfg(n, 2, 1, 0.0, 1.0, 0, 0, 0, family, mixing), plan_of(ints, offs),
                     std::span<const double>(in, n), std::span<double>(out, n));
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}
double ref_pass_coefficient(uint64_t n, int family, int mixing, const int32_t* ints, const uint64_t* offs,
                            uint64_t i, uint64_t j) {
  return maxent::pass_coefficient(to_cfg(n, 2, 1, 0.0, 1.0, 0, 0, 0, family, mixing), plan_of(ints, offs), i, j);
}
// cross_pool_correlation(cfg, opts) with fixed_transform (and expect_composed_q)
int ref_cross_pool_fixed(uint64_t n, int family, int mixing, uint64_t seed, uint64_t pairs, uint32_t n_probes,
                         const uint64_t* out_i, const uint64_t* in_j, int expect_q, double* out) {
  try {
    maxent::CrossPoolOptions o;
    o.pool_pairs = pairs;
    o.fixed_transform = true;
    o.expect_composed_q = expect_q != 0;
    for (uint32_t k = 0; k < n_probes; ++k) o.probes.push_back({out_i[k], in_j[k]});
    const auto reps =
        maxent::cross_pool_correlation(to_cfg(n, 2, 1, 0.0, 1.0, seed, 0, 0, family, mixing), o);
    for (size_t k = 0; k < reps.size(); ++k) {
      out[k * 4 + 0] = reps[k].statistic;
      out[k * 4 + 1] = reps[k].expected;
      out[k * 4 + 2] = reps[k].std_error;
      out[k * 4 + 3] = reps[k].z_score;
    }
    return static_cast<int>(reps.size());
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// tools/cmd_test.cpp:40-60 run_moments_suite: the report lines (machine()
// or text()) of the reference, joined by '\n'; returns the length or -1
int ref_moments_suite(uint64_t seed, uint64_t n, int machine, char* out, uint64_t cap) {
  try {
    std::string all;
    auto print = [&](const std::vector<maxent::TestReport>& rs) {
      for (const auto& r : rs) all += (machine ? r.machine() : r.text()) + "\n";
    };
    {
      maxent::GeneratorConfig cfg;
      cfg.seed = seed;
      maxent::Generator gen(cfg);
      print(maxent::moment_reports(maxent::moments(gen.fill(n)), "wallace4"));
    }
    {
      maxent::BaselineState s(seed);
      std::vector<double> buf(n);
      for (auto& v : buf) v = maxent::polar_next(s);
      print(maxent::moment_reports(maxent::moments(buf), "polar"));
    }
    {
      maxent::BaselineState s(seed);
      std::vector<double> buf(n);
      for (auto& v : buf) v = maxent::boxmuller_next(s);
      print(maxent::moment_reports(maxent::moments(buf), "boxmuller"));
    }
    if (all.size() + 1 > cap) return -1;
    std::memcpy(out, all.c_str(), all.size() + 1);
    return static_cast<int>(all.size());
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// one-core rates of the reference's own call patterns on a Generator
// (bench.cpp:43-59 fill chunks, cmd_gen.cpp:127-134, next_normal loop):
// values per second, pattern 0 = next_normal, else fill in `chunk` pieces
double ref_pattern_rate(uint64_t pool_size, uint64_t seed, int pattern, uint64_t chunk, uint64_t total) {
  maxent::GeneratorConfig cfg;
  cfg.pool_size = pool_size;
  cfg.seed = seed;
  maxent::Generator gen(cfg);
  std::vector<double> buf(chunk > 0 ? chunk : 1);
  double sink = 0.0;
  const auto t0 = std::chrono::steady_clock::now();
  if (pattern == 0) {
    for (uint64_t i = 0; i < total; ++i) sink += gen.next_normal();
  } else {
    for (uint64_t i = 0; i < total; i += chunk) {
      gen.fill(std::span<double>(buf));
      sink += buf[0];
    }
  }
  const double dt = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  if (sink == 12345.678) std::puts("");
  return static_cast<double>(total) / dt;
}

void ref_polar(uint64_t seed, uint64_t n, double* out) {
  maxent::BaselineState s(seed);
  for (uint64_t i = 0; i < n; ++i) out[i] = maxent::polar_next(s);
}

void ref_boxmuller(uint64_t seed, uint64_t n, double* out) {
  maxent::BaselineState s(seed);
  for (uint64_t i = 0; i < n; ++i) out[i] = maxent::boxmuller_next(s);
}

void ref_moments(const double* x, uint64_t n, double out[4]) {
  const auto m = maxent::moments(std::span<const double>(x, n));
  out[0] = m.mean;
  out[1] = m.variance;
  out[2] = m.skewness;
  out[3] = m.excess_kurtosis;
}

// Whole-job runner for the CPU baseline: pools [0, n_pools) with seeds
// seed_base + p, one Generator per pool claimed from an atomic counter by
// `threads` std::threads.  Pools are processed in batches of
// at most 1024 so memory stays bounded: for each batch, phase 1 constructs
// every Generator (Polar init + 16 warm-up passes) and phase 2 fill()s
// count_per_pool values per pool in 65536-value chunks, the reference's own
// bench chunking (bench.cpp:43-59), folded into a sink so no work is elided.
// Each phase is timed by wall clock across all threads and summed over
// batches.  Returns the sink.
double ref_run_job_ex(uint64_t pool_size, int chi2_method, uint64_t discard_every,
                      int disable_chi2, int family, int mixing, uint64_t seed_base,
                      uint64_t n_pools, uint64_t count_per_pool, int threads,
                      double* init_seconds, double* fill_seconds);

double ref_run_job(uint64_t pool_size, int chi2_method, uint64_t discard_every,
                   int disable_chi2, uint64_t seed_base, uint64_t n_pools,
                   uint64_t count_per_pool, int threads, double* init_seconds,
                   double* fill_seconds) {
  return ref_run_job_ex(pool_size, chi2_method, discard_every, disable_chi2, 0, 0, seed_base,
                        n_pools, count_per_pool, threads, init_seconds, fill_seconds);
}

double ref_run_job_ex(uint64_t pool_size, int chi2_method, uint64_t discard_every,
                      int disable_chi2, int family, int mixing, uint64_t seed_base,
                      uint64_t n_pools, uint64_t count_per_pool, int threads,
                      double* init_seconds, double* fill_seconds) {
  std::vector<double> sinks(static_cast<size_t>(threads), 0.0);
  double t_init = 0.0, t_fill = 0.0;
  const uint64_t batch = 1024;
  for (uint64_t b0 = 0; b0 < n_pools; b0 += batch) {
    const uint64_t nb = std::min(batch, n_pools - b0);
    std::vector<maxent::Generator*> gens(nb, nullptr);
    auto run = [&](auto&& body) {
      std::atomic<uint64_t> next{0};
      std::vector<std::thread> pool;
      for (int t = 0; t < threads; ++t) {
        pool.emplace_back([&, t] {
          for (;;) {
            const uint64_t p = next.fetch_add(1);
            if (p >= nb) break;
            body(t, p);
          }
        });
      }
      for (auto& th : pool) th.join();
    };
    const auto c0 = std::chrono::steady_clock::now();
    run([&](int, uint64_t p) {
      gens[p] = new maxent::Generator(to_cfg(pool_size, chi2_method, discard_every, 0.0, 1.0,
                                             seed_base + b0 + p, 0, disable_chi2, family, mixing));
    });
    const auto c1 = std::chrono::steady_clock::now();
    run([&](int t, uint64_t p) {
      thread_local std::vector<double> buf(65536);
      double sink = 0.0;
      uint64_t left = count_per_pool;
      while (left) {
        const uint64_t take = std::min<uint64_t>(left, buf.size());
        gens[p]->fill(std::span<double>(buf.data(), take));
        sink += buf[0] + buf[take - 1];
        left -= take;
      }
      sinks[static_cast<size_t>(t)] += sink;
    });
    const auto c2 = std::chrono::steady_clock::now();
    for (auto* g : gens) delete g;
    t_init += std::chrono::duration<double>(c1 - c0).count();
    t_fill += std::chrono::duration<double>(c2 - c1).count();
  }
  *init_seconds = t_init;
  *fill_seconds = t_fill;
  double s = 0.0;
  for (const double v : sinks) s += v;
  return s;
}

}  // extern "C"
