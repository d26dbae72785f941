// Drop-in test: the reference's hot-path test cases
// (/root/reference/proj/tests/test_generator.cpp) replayed against
// wallace_b200::Generator (include/wallace_b200.hpp -> C-ABI -> sm_100a),
// plus bit-for-bit stream comparison with the UNMODIFIED reference library
// (oracle/_ref/libmaxent_ref.so, extern "C" shim in oracle/ref_shim.cpp).
// Needs a GPU.  Exit code 0 = all checks passed.
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <limits>
#include <string>
#include <vector>

#include "wallace_b200.hpp"

// ---- the reference library, through the test shim (oracle/ref_shim.cpp) ----
extern "C" {
void* ref_create_ex(uint64_t pool_size, int chi2_method, uint64_t discard_every, double mean,
                    double sigma, uint64_t seed, int fixed, int disable_chi2, int family, int mixing);
void ref_destroy(void* g);
int ref_fill(void* g, double* out, uint64_t count);
double ref_next_normal(void* g);
int ref_next_pool(void* g, double* values, double* reserved, double* chi2);
void ref_step_pass(void* g);
int ref_inject_pool(void* g, const double* v, uint64_t n);
void ref_get_pool(void* g, double* raw);
void ref_get_stats(void* g, uint64_t* pass_count, uint64_t* draws, uint64_t* clamp,
                   double* sum_sq, double* reserved_prev);
double ref_chi2_sample(double x, uint64_t nu, int method, int* clamped);
int ref_cross_pool_correlation(void* g, uint64_t pool_pairs, uint32_t n_probes, const uint64_t* out_i,
                               const uint64_t* in_j, double* out);
int ref_pool_sum_squares(uint64_t pool_size, int chi2_method, uint64_t discard_every, uint64_t seed,
                         int disable_chi2, int family, int mixing, uint64_t pools, double* out);
int ref_rare_event_adjacency(uint64_t pool_size, int chi2_method, uint64_t discard_every, uint64_t seed,
                             int disable_chi2, uint64_t samples, double threshold, double* out);
int ref_run_pass(uint64_t n, int family, int mixing, const int32_t* ints, const uint64_t* offs, const double* in,
                 double* out);
double ref_pass_coefficient(uint64_t n, int family, int mixing, const int32_t* ints, const uint64_t* offs,
                            uint64_t i, uint64_t j);
int ref_cross_pool_fixed(uint64_t n, int family, int mixing, uint64_t seed, uint64_t pairs, uint32_t n_probes,
                         const uint64_t* out_i, const uint64_t* in_j, int expect_q, double* out);
double ref_next_normal_ex(void* g, int* err);
int ref_moments_suite(uint64_t seed, uint64_t n, int machine, char* out, uint64_t cap);
double ref_pattern_rate(uint64_t pool_size, uint64_t seed, int pattern, uint64_t chunk, uint64_t total);
void ref_uniform_bits(uint64_t seed, uint64_t n, uint64_t* out);
void ref_polar(uint64_t seed, uint64_t n, double* out);
void ref_boxmuller(uint64_t seed, uint64_t n, double* out);
double ref_compute_a(uint64_t nu);
void ref_wallace_variant(int id, int src[4], double sign[4], double entries[16]);
}

// ---- tools/cmd_test.cpp:40-60 compiled against the drop-in namespace -------
// (the reference's statistic caller, unchanged but for the namespace alias)
namespace maxent = wallace_b200;
namespace wallace_b200::cli {  // tools/cmd_test.cpp's `namespace maxent::cli`
static std::string run_moments_suite(uint64_t seed, std::size_t n, bool machine) {
  std::string all;
  auto print = [&](const std::vector<maxent::TestReport>& rs) {
    for (const auto& r : rs) all += (machine ? r.machine() : r.text()) + "\n";
  };
  {
    maxent::GeneratorConfig cfg;
    cfg.seed = seed;
    maxent::Generator gen(cfg);
    print(moment_reports(moments(gen.fill(n)), "wallace4"));
  }
  {
    maxent::BaselineState s(seed);
    std::vector<double> buf(n);
    for (auto& v : buf) v = polar_next(s);
    print(moment_reports(moments(buf), "polar"));
  }
  {
    maxent::BaselineState s(seed);
    std::vector<double> buf(n);
    for (auto& v : buf) v = boxmuller_next(s);
    print(moment_reports(moments(buf), "boxmuller"));
  }
  return all;
}
}  // namespace wallace_b200::cli

namespace wb = wallace_b200;

static int g_checks = 0, g_fail = 0;
#define CHECK(cond)                                                          \
  do {                                                                       \
    ++g_checks;                                                              \
    if (!(cond)) {                                                           \
      ++g_fail;                                                              \
      std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);   \
    }                                                                        \
  } while (0)
#define CHECK_THROWS_AS(expr, type)                                          \
  do {                                                                       \
    bool caught_ = false;                                                    \
    try {                                                                    \
      (void)(expr);                                                          \
    } catch (const type&) {                                                  \
      caught_ = true;                                                        \
    } catch (...) {                                                          \
    }                                                                        \
    CHECK(caught_ && #type);                                                 \
  } while (0)
#define CHECK_THROWS_WITH(expr, type, needle)                                \
  do {                                                                       \
    bool ok_ = false;                                                        \
    try {                                                                    \
      (void)(expr);                                                          \
    } catch (const type& e_) {                                               \
      ok_ = std::string(e_.what()).find(needle) != std::string::npos;        \
    } catch (...) {                                                          \
    }                                                                        \
    CHECK(ok_ && needle);                                                    \
  } while (0)

struct Ref {
  void* g;
  explicit Ref(const wb::GeneratorConfig& c)
      : g(ref_create_ex(c.pool_size, static_cast<int>(c.chi2_method), c.discard_every, c.out_mean,
                        c.out_sigma, c.seed, c.diag.fixed_transform, c.diag.disable_chi2,
                        static_cast<int>(c.transform_family), static_cast<int>(c.mixing))) {}
  ~Ref() { ref_destroy(g); }
  std::vector<double> fill(size_t n) {
    std::vector<double> v(n);
    ref_fill(g, v.data(), n);
    return v;
  }
};

static bool same_bits(const std::vector<double>& a, const std::vector<double>& b) {
  return a.size() == b.size() && std::memcmp(a.data(), b.data(), a.size() * 8) == 0;
}

static double pool_sum_sq(const std::vector<double>& v) {
  double s = 0.0;
  for (double x : v) s += x * x;
  return s;
}

static wb::GeneratorConfig cfg_of(size_t n, uint64_t seed) {
  wb::GeneratorConfig c;
  c.pool_size = n;
  c.seed = seed;
  return c;
}

int main() {
  // test_generator.cpp:42-72 config validation names the offending field
  {
    wb::GeneratorConfig cfg;
    cfg.pool_size = 48;
    CHECK_THROWS_WITH(cfg.validate(), wb::ConfigError, "pool_size");
    cfg.pool_size = 16;
    CHECK_THROWS_AS(cfg.validate(), wb::ConfigError);
    cfg.pool_size = 1024;
    cfg.discard_every = 0;
    CHECK_THROWS_WITH(cfg.validate(), wb::ConfigError, "discard_every");
    cfg.discard_every = 1;
    cfg.out_sigma = 0.0;
    CHECK_THROWS_WITH(cfg.validate(), wb::ConfigError, "out_sigma");
    cfg.out_sigma = 1.0;
    cfg.out_mean = std::numeric_limits<double>::infinity();
    CHECK_THROWS_WITH(cfg.validate(), wb::ConfigError, "out_mean");
    cfg.out_mean = 0.0;
    cfg.validate();
    CHECK_THROWS_AS(wb::Generator(cfg_of(48, 0)), wb::ConfigError);
  }
  // a pool above the on-chip limit (fp64 N = 2^14) runs HBM-resident: the
  // same stream as the reference, across a renormalisation
  {
    wb::Generator g(cfg_of(1u << 14, 1));
    Ref r(cfg_of(1u << 14, 1));
    CHECK(same_bits(g.fill(250000), r.fill(250000)));
    for (int i = 0; i < 260; ++i) {
      g.step_pass();
      ref_step_pass(r.g);
    }
    CHECK(same_bits(g.fill(70000), r.fill(70000)));
  }
  // rotation family and affine mixing (generator.cpp:86-172): the same
  // stream as the reference, through next_normal / fill / step_pass
  for (int fm = 1; fm < 4; ++fm) {
    wb::GeneratorConfig c = cfg_of(256, 7 + fm);
    c.transform_family = fm >= 2 ? wb::TransformFamily::rotation : wb::TransformFamily::wallace4;
    c.mixing = (fm & 1) ? wb::MixingScheme::affine : wb::MixingScheme::stride_transpose;
    c.discard_every = 2;
    wb::Generator g(c);
    Ref r(c);
    CHECK(same_bits(g.fill(5000), r.fill(5000)));
    bool nn = true;
    std::vector<double> rn = r.fill(300);
    for (int i = 0; i < 300; ++i) nn = nn && g.next_normal() == rn[i];
    CHECK(nn);
    g.step_pass();
    ref_step_pass(r.g);
    CHECK(same_bits(g.fill(1000), r.fill(1000)));
  }
  // :74-82 identical config gives a bit-identical stream (and == reference)
  {
    wb::Generator a(cfg_of(128, 42)), b(cfg_of(128, 42));
    Ref r(cfg_of(128, 42));
    bool same = true, ref_same = true;
    for (int i = 0; i < 10000; ++i) {
      const double x = a.next_normal();
      same = same && x == b.next_normal();
      ref_same = ref_same && x == ref_next_normal(r.g);
    }
    CHECK(same);
    CHECK(ref_same);
  }
  // :84-91 construction normalizes the pool and warms up
  {
    wb::Generator gen(cfg_of(1024, 7));
    CHECK(gen.pass_count() == 16);
    CHECK(std::abs(pool_sum_sq(gen.pool().raw) - 1024.0) <= 1e-12 * 1024.0);
    CHECK(std::abs(gen.pool().sum_sq - 1024.0) <= 1e-12 * 1024.0);
  }
  // :93-101 a pool of zeros stays zero under any pass
  {
    wb::Generator gen(cfg_of(64, 3));
    gen.inject_pool(std::vector<double>(64, 0.0));
    gen.step_pass();
    bool zero = true;
    for (double v : gen.pool().raw) zero = zero && v == 0.0;
    CHECK(zero);
  }
  // :143-154 conservation through the 256-pass renormalization
  {
    wb::Generator gen(cfg_of(256, 17));
    bool ok = true;
    for (int p = 0; p < 300; ++p) {
      gen.step_pass();
      const auto& pool = gen.pool();
      const double actual = pool_sum_sq(pool.raw);
      ok = ok && std::abs(actual - pool.sum_sq) <= 1e-9 * 256.0 &&
           std::abs(actual - 256.0) <= 1e-6 * 256.0;
    }
    CHECK(ok);
  }
  // :218-231 chi-squared scaling disabled reproduces the raw pool
  {
    wb::GeneratorConfig cfg = cfg_of(128, 5);
    cfg.diag.disable_chi2 = true;
    wb::Generator gen(cfg);
    const auto po = gen.next_pool();
    CHECK(po.values.size() == 127);
    const auto raw = gen.pool().raw;
    bool eq = true;
    for (size_t i = 0; i < po.values.size(); ++i) eq = eq && po.values[i] == raw[i];
    CHECK(eq);
    CHECK(po.reserved == raw[127]);
    CHECK(po.chi2_draw == gen.pool().sum_sq);
  }
  // :233-244 mean and sigma are an exact affine map of the unit stream
  {
    wb::GeneratorConfig unit = cfg_of(256, 99), scaled = cfg_of(256, 99);
    scaled.out_mean = 5.0;
    scaled.out_sigma = 2.0;
    wb::Generator a(unit), b(scaled);
    bool ok = true;
    for (int i = 0; i < 10000; ++i) ok = ok && 2.0 * a.next_normal() + 5.0 == b.next_normal();
    CHECK(ok);
  }
  // :246-260 emission scales to the chi-squared draw
  {
    wb::Generator gen(cfg_of(1024, 31));
    bool ok = true;
    for (int rep = 0; rep < 50; ++rep) {
      const auto po = gen.next_pool();
      std::vector<double> vals(po.values.begin(), po.values.end());
      const double total = pool_sum_sq(vals) + po.reserved * po.reserved;
      ok = ok && std::abs(total - po.chi2_draw) <= 1e-9 * 1024.0;
      const auto pool = gen.pool();
      const double r = std::sqrt(po.chi2_draw / pool.sum_sq);
      ok = ok && po.reserved == pool.raw[1023] * r;
    }
    CHECK(ok);
  }
  // :280-291 reserved variate is sourced from the previous pool
  {
    wb::Generator gen(cfg_of(64, 77));
    const auto p0 = gen.next_pool();
    int clamped = 0;
    const double expect_s = ref_chi2_sample(p0.reserved, 64, 2, &clamped);
    const auto p1 = gen.next_pool();
    CHECK(p1.chi2_draw == expect_s);
  }
  // :293-310 fill is equivalent to repeated next_normal; fill(0) throws
  {
    wb::Generator a(cfg_of(64, 21)), b(cfg_of(64, 21));
    const auto first = a.fill(5);
    const auto second = a.fill(5);
    bool ok = true;
    for (int i = 0; i < 5; ++i) ok = ok && first[i] == b.next_normal();
    for (int i = 0; i < 5; ++i) ok = ok && second[i] == b.next_normal();
    CHECK(ok);
    CHECK_THROWS_AS(a.fill(0), wb::InvalidParameterError);
    wb::Generator c(cfg_of(64, 21));
    const auto before = c.pass_count();
    c.fill(3 * 64);
    CHECK(c.pass_count() - before >= 3);
  }
  // :312-335 discard policy emits every k-th pool
  {
    wb::GeneratorConfig third = cfg_of(64, 9);
    third.discard_every = 3;
    wb::Generator b(third);
    bool ok = true;
    for (int i = 0; i < 10; ++i) {
      b.next_pool();
      ok = ok && b.pass_count() == uint64_t(16 + 3 * (i + 1));
    }
    CHECK(ok);
  }
  // :337-351 at least one uniform draw per pool
  {
    for (size_t discard : {size_t(1), size_t(3)}) {
      wb::GeneratorConfig cfg = cfg_of(64, 2);
      cfg.discard_every = discard;
      wb::Generator gen(cfg);
      uint64_t prev = gen.uniform_draws();
      bool ok = true;
      for (int i = 0; i < 20; ++i) {
        gen.next_pool();
        const uint64_t d = gen.uniform_draws();
        ok = ok && d - prev >= discard;
        prev = d;
      }
      CHECK(ok);
    }
  }
  // :353-358 inject_pool validates the size
  {
    wb::Generator gen(cfg_of(64, 2));
    CHECK_THROWS_AS(gen.inject_pool(std::vector<double>(63, 1.0)), wb::InvalidParameterError);
  }
  // :360-376 stream moments are sane at a million draws
  {
    wb::Generator gen(cfg_of(1024, 4242));
    const auto v = gen.fill(1000000);
    double sum = 0.0, sum2 = 0.0;
    for (double z : v) {
      sum += z;
      sum2 += z * z;
    }
    const double nn = 1e6, mean = sum / nn, var = sum2 / nn - mean * mean;
    CHECK(std::abs(mean) <= 5.0 / std::sqrt(nn));
    CHECK(std::abs(var - 1.0) <= 5.0 * std::sqrt(2.0 / nn));
  }
  // bit-for-bit against the reference library on every BASELINE shape, and
  // through an interleaved API sequence
  {
    struct Case {
      size_t n, d;
      int chi2;
      bool dis;
      uint64_t seed;
      size_t count;
    };
    const Case cases[] = {{4096, 2, 2, true, 1, 1 << 18},  {4096, 2, 2, false, 1, 1 << 18},
                          {2048, 3, 2, false, 7, 1 << 17}, {1024, 1, 2, false, 1, 1 << 20},
                          {64, 1, 0, false, 5, 100000},     {128, 3, 1, false, 9, 50000}};
    for (const auto& k : cases) {
      wb::GeneratorConfig c = cfg_of(k.n, k.seed);
      c.discard_every = k.d;
      c.chi2_method = static_cast<wb::Chi2Method>(k.chi2);
      c.diag.disable_chi2 = k.dis;
      wb::Generator g(c);
      Ref r(c);
      CHECK(same_bits(g.fill(k.count), r.fill(k.count)));
    }
    wb::GeneratorConfig c = cfg_of(64, 21);
    c.out_mean = 5.0;
    c.out_sigma = 2.0;
    c.discard_every = 2;
    wb::Generator g(c);
    Ref r(c);
    bool ok = true;
    for (size_t k : {5, 5, 200, 63, 1}) ok = ok && same_bits(g.fill(k), r.fill(k));
    g.step_pass();
    ref_step_pass(r.g);
    for (int i = 0; i < 100; ++i) ok = ok && g.next_normal() == ref_next_normal(r.g);
    const auto po = g.next_pool();
    std::vector<double> rv(63);
    double rres, rchi;
    ref_next_pool(r.g, rv.data(), &rres, &rchi);
    ok = ok && std::memcmp(po.values.data(), rv.data(), 63 * 8) == 0 && po.reserved == rres &&
         po.chi2_draw == rchi;
    std::vector<double> inj(64);
    for (int i = 0; i < 64; ++i) inj[i] = -2.0 + 4.0 * i / 63.0;
    g.inject_pool(inj);
    ref_inject_pool(r.g, inj.data(), 64);
    ok = ok && same_bits(g.fill(300), r.fill(300));
    std::vector<double> rp(64);
    ref_get_pool(r.g, rp.data());
    ok = ok && same_bits(g.pool().raw, rp);
    uint64_t pc, dr, cl;
    double ss, rpv;
    ref_get_stats(r.g, &pc, &dr, &cl, &ss, &rpv);
    ok = ok && g.pass_count() == pc && g.uniform_draws() == dr && g.chi2_clamp_count() == cl &&
         g.pool().sum_sq == ss && g.pool().reserved_prev == rpv;
    CHECK(ok);
  }
  // stats.cpp defect suite through the drop-in (device accumulators)
  {
    wb::GeneratorConfig c = cfg_of(256, 9);
    wb::Generator g(c);
    Ref r(c);
    wb::CrossPoolOptions o;
    o.pool_pairs = 1500;
    const auto mine = wb::cross_pool_correlation(g, o);
    std::vector<uint64_t> oi, ij;
    for (std::size_t k = 0; k < 8; ++k) {
      oi.push_back((5 * k) % 256);
      ij.push_back((11 * k + 3) % 256);
    }
    double out[32];
    CHECK(ref_cross_pool_correlation(r.g, 1500, 8, oi.data(), ij.data(), out) == 8);
    bool same = mine.size() == 8;
    for (std::size_t k = 0; k < mine.size() && same; ++k)
      same = mine[k].statistic == out[4 * k] && mine[k].expected == out[4 * k + 1] &&
             mine[k].std_error == out[4 * k + 2] && mine[k].z_score == out[4 * k + 3];
    CHECK(same);  // bit-identical probe sums -> identical reports
    CHECK(same_bits(g.fill(1000), r.fill(1000)));  // the stream continues identically
    CHECK_THROWS_AS(wb::cross_pool_correlation(g, wb::CrossPoolOptions{10, {}}), wb::InvalidParameterError);

    wb::GeneratorConfig c2 = cfg_of(64, 3);
    const wb::TestReport ra = wb::rare_event_adjacency(c2, 200000, 3.0);
    double ro[4];
    CHECK(ref_rare_event_adjacency(64, 2, 1, 3, 0, 200000, 3.0, ro) == 0);
    CHECK(ra.statistic == ro[0] && ra.std_error == ro[2] && ra.z_score == ro[3]);
    CHECK_THROWS_AS(wb::rare_event_adjacency(c2, 200000, 2.0), wb::InvalidParameterError);

    wb::GeneratorConfig c3 = cfg_of(128, 5);
    c3.discard_every = 2;
    const wb::PoolSumSquares ps = wb::pool_sum_squares_test(c3, 1200);
    double po[8];
    CHECK(ref_pool_sum_squares(128, 2, 2, 5, 0, 0, 0, 1200, po) == 0);
    CHECK(std::abs(ps.mean_report.statistic - po[0]) <= 1e-9 * po[0]);
    CHECK(std::abs(ps.variance_report.statistic - po[4]) <= 1e-9 * po[4]);
    CHECK(ps.mean_report.pass && ps.variance_report.pass);
  }
  // generator.hpp free functions: run_pass / pass_coefficient, and the
  // fixed-transform cross-pool test (criterion 4's second half)
  {
    wb::GeneratorConfig c = cfg_of(64, 20260808);
    c.transform_family = wb::TransformFamily::rotation;
    c.mixing = wb::MixingScheme::affine;
    wb::PassPlan plan;
    plan.t_index = {3, 11};
    plan.negate = {true, false};
    plan.offset = {17, 40};
    const int32_t ints[5] = {0, 3, 11, 1, 0};
    const uint64_t offs[2] = {17, 40};
    std::vector<double> in(64), out(64), ref_out(64);
    for (int k = 0; k < 64; ++k) in[static_cast<std::size_t>(k)] = std::sin(0.37 * k + 1.0);
    wb::run_pass(c, plan, in, out);
    CHECK(ref_run_pass(64, 1, 1, ints, offs, in.data(), ref_out.data()) == 0);
    CHECK(same_bits(out, ref_out));
    bool q_same = true;
    for (std::size_t i = 0; i < 64 && q_same; ++i)
      for (std::size_t j = 0; j < 64; ++j)
        q_same = q_same && wb::pass_coefficient(c, plan, i, j) == ref_pass_coefficient(64, 1, 1, ints, offs, i, j);
    CHECK(q_same);
    wb::GeneratorConfig c4 = cfg_of(64, 20260808);
    wb::CrossPoolOptions fixed;
    fixed.pool_pairs = 20000;
    fixed.fixed_transform = true;
    fixed.expect_composed_q = true;
    for (std::size_t i = 0; i < 64 && fixed.probes.size() < 4; ++i)
      for (std::size_t j = 0; j < 64; ++j)
        if (std::abs(wb::pass_coefficient(c4, wb::PassPlan{}, i, j)) == 0.5) {
          fixed.probes.push_back({i, j});
          break;
        }
    const auto mine = wb::cross_pool_correlation(c4, fixed);
    std::vector<uint64_t> oi, ij;
    for (const auto& p : fixed.probes) {
      oi.push_back(p.out_i);
      ij.push_back(p.in_j);
    }
    double out4[16];
    CHECK(ref_cross_pool_fixed(64, 0, 0, 20260808, 20000, 4, oi.data(), ij.data(), 1, out4) == 4);
    bool same = mine.size() == 4;
    for (std::size_t k = 0; k < mine.size() && same; ++k)
      same = mine[k].statistic == out4[4 * k] && mine[k].expected == out4[4 * k + 1] &&
             mine[k].std_error == out4[4 * k + 2] && mine[k].z_score == out4[4 * k + 3];
    CHECK(same);
  }
  // cmd_test's moments suite through `namespace maxent = wallace_b200`: the
  // report lines are byte-equal to the reference's (machine and text forms)
  for (uint64_t seed : {uint64_t(1), uint64_t(42)}) {
    std::vector<char> buf(1 << 16);
    for (int machine = 0; machine < 2; ++machine) {
      const int len = ref_moments_suite(seed, 100000, machine, buf.data(), buf.size());
      CHECK(len > 0);
      const std::string mine = maxent::cli::run_moments_suite(seed, 100000, machine != 0);
      CHECK(mine == std::string(buf.data()));
      if (seed == 1 && machine) std::printf("%s", mine.c_str());
    }
  }
  // the L1a free functions of the namespace (baselines / chi2 / transforms)
  {
    maxent::UniformState u(42);
    std::vector<uint64_t> w(100);
    ref_uniform_bits(42, 100, w.data());
    bool ok = true;
    for (int i = 0; i < 100; ++i) ok = ok && maxent::uniform_bits(u) == w[static_cast<std::size_t>(i)];
    CHECK(ok && u.draws == 100);
    std::vector<double> rp(1001), rb(1001);
    ref_polar(7, 1001, rp.data());
    ref_boxmuller(7, 1001, rb.data());
    maxent::BaselineState sp(7), sb(7);
    for (int i = 0; i < 1001; ++i) {
      ok = ok && maxent::polar_next(sp) == rp[static_cast<std::size_t>(i)];
      ok = ok && maxent::boxmuller_next(sb) == rb[static_cast<std::size_t>(i)];
    }
    CHECK(ok);
    const auto params = maxent::Chi2Params::for_nu(1024);
    CHECK(params.a_value == ref_compute_a(1024));
    int rc = 0;
    bool cl = false;
    CHECK(maxent::chi2_sample(-0.3, params, maxent::Chi2Method::cubic_a, &cl) ==
          ref_chi2_sample(-0.3, 1024, 2, &rc));
    CHECK_THROWS_WITH(maxent::chi2_sample(std::numeric_limits<double>::quiet_NaN(), params,
                                          maxent::Chi2Method::cubic_a),
                      maxent::InvalidParameterError, "x must be finite");
    CHECK_THROWS_AS(maxent::Chi2Params::for_nu(7), maxent::InvalidParameterError);
    bool vok = true;
    for (int id = 0; id < 384; ++id) {
      const auto m = maxent::wallace_variant(id);
      int src[4];
      double sg[4], e[16];
      ref_wallace_variant(id, src, sg, e);
      for (int k = 0; k < 4; ++k) {
        vok = vok && m.source_row[static_cast<std::size_t>(k)] == src[k] && m.row_sign[static_cast<std::size_t>(k)] == sg[k];
        for (int j = 0; j < 4; ++j) vok = vok && m.entries[static_cast<std::size_t>(k)][static_cast<std::size_t>(j)] == e[4 * k + j];
      }
    }
    CHECK(vok);
    const auto col = maxent::apply_wallace4({1, 0, 0, 0}, maxent::wallace_a1());
    CHECK(col[0] == 0.5 && col[1] == 0.5 && col[2] == 0.5 && col[3] == -0.5);
    CHECK(maxent::default_stride(256) == 87 && maxent::default_stride(16) == 7);
    const auto half = maxent::rotation_from_t(0.5);
    CHECK(half.c == 0.6 && half.s == 0.8 && maxent::rotation_t_table().size() == 16);
  }
  // chi2_sample's throw reaches the drop-in where the reference throws:
  // inject a non-finite pool, then next_normal / fill until the reference's
  // next_normal throws; the drop-in throws on the same value
  for (int how = 0; how < 2; ++how) {
    wb::GeneratorConfig c = cfg_of(1024, 11);
    wb::Generator g(c);
    Ref r(c);
    CHECK(same_bits(g.fill(3000), r.fill(3000)));
    std::vector<double> inj(1024);
    for (int i = 0; i < 1024; ++i) inj[static_cast<std::size_t>(i)] = std::cos(0.1 * i);
    inj[1023] = std::numeric_limits<double>::infinity();
    g.inject_pool(inj);
    ref_inject_pool(r.g, inj.data(), 1024);
    long ref_at = -1, mine_at = -1;
    for (long i = 0; i < 200000 && ref_at < 0; ++i) {
      int err = 0;
      ref_next_normal_ex(r.g, &err);
      if (err) ref_at = i;
    }
    try {
      if (how == 0) {
        for (long i = 0; i < 200000; ++i, mine_at = i) g.next_normal();
      } else {
        for (long i = 0; i < 200000; i += 100, mine_at = i) g.fill(100);
      }
      mine_at = -1;
    } catch (const wb::InvalidParameterError& e) {
      CHECK(std::string(e.what()) == "chi2_sample: x must be finite");
    }
    CHECK(ref_at > 0);
    if (how == 0) CHECK(mine_at == ref_at);
    else CHECK(mine_at == (ref_at / 100) * 100);
    CHECK_THROWS_AS(g.next_normal(), wb::InvalidParameterError);  // and again, as the reference
  }
  // the look-ahead rolls back exactly: deep inside a block, every
  // state-observing call sees the reference's state
  {
    wb::GeneratorConfig c = cfg_of(512, 123);
    c.discard_every = 2;
    wb::Generator g(c);
    Ref r(c);
    bool ok = true;
    for (int round = 0; round < 3; ++round) {
      for (int i = 0; i < 70001; ++i) ok = ok && g.next_normal() == ref_next_normal(r.g);
      uint64_t pc, dr, cl;
      double ss, rpv;
      ref_get_stats(r.g, &pc, &dr, &cl, &ss, &rpv);
      ok = ok && g.pass_count() == pc && g.uniform_draws() == dr && g.chi2_clamp_count() == cl;
      g.step_pass();
      ref_step_pass(r.g);
      ok = ok && same_bits(g.fill(33333), r.fill(33333));
    }
    CHECK(ok);
  }
  // the reference's own call patterns (bench.cpp:43-59 fill(65536),
  // cmd_gen.cpp:127-134 fill(16384), next_normal) are at least as fast as
  // the reference on one core
  {
    const uint64_t total = 1 << 24;
    const struct {
      int pattern;
      uint64_t chunk;
      const char* name;
    } pats[] = {{0, 0, "next_normal"}, {1, 16384, "fill(16384)"}, {1, 65536, "fill(65536)"}};
    for (const auto& p : pats) {
      const double ref_rate = ref_pattern_rate(1024, 1, p.pattern, p.chunk, total);
      wb::Generator g(cfg_of(1024, 1));
      std::vector<double> buf(p.chunk > 0 ? p.chunk : 1);
      double sink = 0.0;
      g.fill(1);  // first block
      const auto t0 = std::chrono::steady_clock::now();
      if (p.pattern == 0) {
        for (uint64_t i = 0; i < total; ++i) sink += g.next_normal();
      } else {
        for (uint64_t i = 0; i < total; i += p.chunk) {
          g.fill(std::span<double>(buf));
          sink += buf[0];
        }
      }
      const double dt = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      const double rate = static_cast<double>(total) / dt;
      std::printf("drop-in %-12s %.3e values/s  (reference 1 core %.3e, x%.2f)%s\n", p.name, rate, ref_rate,
                  rate / ref_rate, sink == 1.5 ? " " : "");
      CHECK(rate >= ref_rate);
    }
  }
  std::printf("%d checks, %d failed\n", g_checks, g_fail);
  return g_fail == 0 ? 0 : 1;
}
