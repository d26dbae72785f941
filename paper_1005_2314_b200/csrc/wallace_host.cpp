// Host side of the B200 Wallace pool generator: the C-ABI of
// include/wallace_b200.h, host seeding of pools, launch sequencing.
//
// Seeding follows Generator::Generator (generator.cpp:309-331): SplitMix64 +
// xoshiro256** (baselines.cpp:19-45), Polar normals with glibc log/sqrt
// (baselines.cpp:51-66), Neumaier sum of squares (generator.cpp:20-34),
// scaling to sum_sq = n.  It runs on the host so that glibc's log is the one
// the reference uses (bit parity of the seeded pool); the 16 warm-up passes
// then run on the device.  Seeding is spread over host threads, one pool at a
// time per thread.
#include <cuda_runtime.h>
#include <fcntl.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <cerrno>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <string>
#include <thread>
#include <utility>
#include <functional>
#include <vector>

#include "../../include/wallace_b200.h"
#include "wallace_common.h"

namespace wb {
cudaError_t launch_pool_kernel(int dtype, int log2n, const FillArgs& a, uint64_t n_pools,
                               cudaStream_t s);
int pool_kernel_threads(int dtype, int log2n);
void affine_multipliers(int log2n, uint32_t* alpha, uint32_t* beta);
size_t large_state_bytes();
uint64_t large_aux_stride(uint64_t N);
cudaError_t launch_single_pass(int dtype, const FillArgs& a, void* buf_a, void* buf_b, uint64_t n_pools,
                               cudaStream_t st, int* in_b);
cudaError_t launch_seed(int dtype, const uint64_t* d_seeds, uint64_t seed_base, uint32_t N, void* pools,
                        PoolState* st, uint64_t n_pools, cudaStream_t s);
cudaError_t launch_plan_kernel(const PlanArgs& a, cudaStream_t s);
cudaError_t launch_pair_kernel(const FillArgs& a, uint64_t n_pools, cudaStream_t stream);
cudaError_t launch_rescale(int dtype, const FillArgs& a, uint32_t N, uint64_t n_pools, cudaStream_t s);
cudaError_t launch_materialize(int dtype, const void* pools, PoolState* st, void* leftover,
                               uint64_t n_pools, uint32_t N, double mean, cudaStream_t s);
cudaError_t launch_reduce_consumer(const double* part_sums, const uint32_t* part_hist,
                                   uint64_t n_pools, uint64_t chunk, double* blk_sums,
                                   unsigned long long* blk_hist, cudaStream_t s);
cudaError_t launch_baseline_fill(int method, void* states, uint64_t n_streams, uint64_t count, double* out,
                                 cudaStream_t s);
cudaError_t launch_baseline_consume(int method, const uint64_t* d_seeds, uint64_t seed_base, uint64_t n_streams,
                                    uint64_t count, double* part_sums, uint32_t* part_hist, uint64_t n_blocks,
                                    cudaStream_t s);
}  // namespace wb

using wb::PoolState;

namespace {

thread_local std::string g_err;
std::atomic<uint64_t> g_launches{0};
std::atomic<uint64_t> g_pair_launches{0};  // of which pair_kernel (pool_pair.cu)

wallace_status fail(wallace_status code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  std::vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define WB_CUDA(expr)                                                                  \
  do {                                                                                 \
    cudaError_t e_ = (expr);                                                           \
    if (e_ != cudaSuccess)                                                             \
      return fail(WALLACE_ERR_CUDA, "%s: %s (%s:%d)", #expr, cudaGetErrorString(e_),   \
                  __FILE__, __LINE__);                                                 \
  } while (0)

// ---- reference primitives restated for host seeding -----------------------
inline uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }

uint64_t splitmix64(uint64_t& state) {  // baselines.cpp:19-24
  uint64_t z = (state += 0x9e3779b97f4a7c15ULL);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

struct Uniform {  // UniformState (baselines.hpp:27-33)
  uint64_t s[4];
  uint64_t draws = 0;
  explicit Uniform(uint64_t seed) {  // baselines.cpp:26-31
    uint64_t sm = seed;
    for (auto& w : s) w = splitmix64(sm);
  }
  uint64_t bits() {  // baselines.cpp:33-45
    const uint64_t result = rotl(s[1] * 5, 7) * 9;
    const uint64_t t = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= t;
    s[3] = rotl(s[3], 45);
    ++draws;
    return result;
  }
  double next() { return static_cast<double>(bits() >> 11) * 0x1.0p-53; }  // :47-49
};

struct Polar {  // BaselineState + polar_next (baselines.cpp:51-66)
  Uniform u;
  bool has = false;
  double cached = 0.0;
  explicit Polar(uint64_t seed) : u(seed) {}
  double next() {
    if (has) {
      has = false;
      return cached;
    }
    for (;;) {
      const double a = 2.0 * u.next() - 1.0;
      const double b = 2.0 * u.next() - 1.0;
      const double s2 = a * a + b * b;
      if (s2 >= 1.0 || s2 == 0.0) continue;
      const double scale = std::sqrt(-2.0 * std::log(s2) / s2);
      cached = b * scale;
      has = true;
      return a * scale;
    }
  }
};

template <typename T>
double neumaier_sq(const T* v, uint64_t n) {  // generator.cpp:20-34
  double sum = 0.0, comp = 0.0;
  for (uint64_t i = 0; i < n; ++i) {
    const double x = static_cast<double>(v[i]);
    const double term = x * x;
    const double t = sum + term;
    if (std::abs(sum) >= std::abs(term)) comp += (sum - t) + term;
    else comp += (term - t) + sum;
    sum = t;
  }
  return sum + comp;
}

// Generator ctor up to the warm-up (generator.cpp:317-327).  raw_d receives
// the double pool; the caller rounds to T.
void seed_pool_double(uint64_t n, uint64_t seed, double* raw_d, double& reserved,
                      uint64_t s_out[4], uint64_t& draws) {
  Polar init(seed);
  for (uint64_t i = 0; i < n; ++i) raw_d[i] = init.next();
  reserved = init.next();
  std::memcpy(s_out, init.u.s, sizeof(init.u.s));
  draws = init.u.draws;
  const double ss = neumaier_sq(raw_d, n);
  const double k = std::sqrt(static_cast<double>(n) / ss);
  for (uint64_t i = 0; i < n; ++i) raw_d[i] *= k;
}

uint64_t default_stride(uint64_t rows) {  // transforms.cpp:161-169
  uint64_t k = rows / 3 + 1;
  if (k % 2 == 0) ++k;
  while (std::gcd(k, rows) != 1) k += 2;
  return k;
}

double compute_a(uint64_t nu) {  // chi2.cpp:11-17
  const double root_nu = std::sqrt(static_cast<double>(nu));
  return 2.0 * root_nu * std::sin(std::asin(1.0 / root_nu) / 3.0);
}

wb::Chi2Consts chi2_consts(const wallace_config& c) {
  wb::Chi2Consts k{};
  const double nu = static_cast<double>(c.pool_size);
  k.nu = nu;
  k.a = compute_a(c.pool_size);
  k.cubic_c = std::sqrt(2.0 * (nu - k.a * k.a));
  k.shift_c = std::sqrt(2.0 * nu - 1.0);
  const double d = 2.0 / (9.0 * nu);
  k.wh_sqrt_d = std::sqrt(d);
  k.wh_one_m_d = 1.0 - d;
  k.floor_v = 1e-6 * nu;
  k.method = c.chi2_method;
  k.disable = c.disable_chi2;
  return k;
}

int ilog2(uint64_t v) {
  int l = 0;
  while ((1ull << l) < v) ++l;
  return l;
}

constexpr uint64_t kPlanBudgetBytes = 128ull << 20;
constexpr uint32_t kMaxPassesPerLaunch = 2048;
constexpr uint64_t kMagic = 0x5741'4c4c'4143'4531ull;  // "WALLACE1"

}  // namespace

// Device block sums/counts of the consumer reduction and their pinned host
// copy, kept between calls (grown on demand).
struct ReduceScratch {
  void* d_buf = nullptr;
  void* h_buf = nullptr;
  uint64_t cap = 0;  // blocks
  void release() {
    cudaFree(d_buf);
    cudaFreeHost(h_buf);
    d_buf = h_buf = nullptr;
    cap = 0;
  }
};

struct wallace_handle {
  wallace_config cfg{};
  int dtype = 0;
  size_t esize = 4;
  uint64_t n_pools = 0;
  uint64_t N = 0;
  int log2n = 0;
  cudaStream_t stream = nullptr;
  wb::Chi2Consts chi2{};
  uint32_t plan_cap = 0;  // passes per launch
  int pass_type = 0;      // 2*family + mixing (wb::pass_type_of)
  uint32_t plan_words = 1;  // plan words per pass (rotation: 2)
  double rot_c[16] = {}, rot_s[16] = {};  // rotation_from_t of the table

  void* d_pools = nullptr;
  PoolState* d_state = nullptr;
  uint32_t* d_plans = nullptr;   // two plan buffers of n_pools * plan_cap * plan_words words
  // plan generation runs one launch ahead on a side stream
  cudaStream_t side = nullptr;
  cudaEvent_t ev_start = nullptr, ev_planned[2] = {nullptr, nullptr}, ev_pooled[2] = {nullptr, nullptr};
  int key = 0;        // kernel key: log2(N) (+16 for the latency kernel)
  int kmode = 0;      // 0 auto, 1 throughput, 2 latency
  bool bulk_ok = false;  // fills may use the bulk-emission kernel
  bool bulk_cfg_ok = false;  // ... as far as the configuration goes (finite pools)
  bool staged_ok = false;  // other fills may use the staged-emission kernel
  bool pair_ok = false;  // fills may use pair_kernel (pool_pair.cu)
  bool lat_fill_ok = false;  // latency-geometry fills may decouple the chi2 chain (kModeFillLat)
  double* d_scales = nullptr;  // kModeFillLat: [n_pools][plan_cap] per-emission scales
  void* d_lat_raw = nullptr;   // kModeFillLat: [n_pools][lat_rows][N] raw emissions
  uint64_t lat_rows = 0;       // kModeFillLat: emissions per launch
  // pools above the on-chip limit: HBM-resident executor (wallace_large.cu)
  bool large = false;
  void* d_lg_pool2 = nullptr;
  void* d_lg_state = nullptr;
  double* d_lg_aux = nullptr;
  // defect suite (wallace_cross_pool_probes / wallace_pool_defect_stats)
  double* d_probe_acc = nullptr;
  uint32_t n_probes = 0;  // active only inside wallace_cross_pool_probes
  uint32_t probe_out[32] = {}, probe_in[32] = {};
  double* d_def_totals = nullptr;
  uint8_t* d_def_marks = nullptr;
  uint64_t def_stride = 0;
  double def_threshold = 0.0;
  void* d_leftover = nullptr;
  // device snapshots (wallace_snapshot_ex slots 0 and 1)
  struct Snap {
    void* pools = nullptr;
    PoolState* state = nullptr;
    void* leftover = nullptr;
    bool leftover_valid = false;  // the live leftover was copied (partial emission materialised)
    uint32_t cursor = 0;
    uint64_t pass_count = 0;
    bool has = false;
  } snap[2];
  // wallace_fill_host_async: device staging of the queued block, copied to
  // the host launch by launch on cp_stream (ev_cp: launch done / copies done)
  void* d_astage = nullptr;
  uint64_t astage_bytes = 0;
  cudaStream_t cp_stream = nullptr;
  cudaEvent_t ev_cp = nullptr;
  // run_emit: at most this many emissions per launch (0: plan_cap / d), and
  // a callback after each launch's kernels (issue)
  uint32_t max_emit = 0;
  std::function<cudaError_t(const wb::FillArgs&)> after_launch;

  // consumer scratch
  double* d_part_sums = nullptr;
  uint32_t* d_part_hist = nullptr;
  uint64_t part_cap = 0;
  ReduceScratch red;  // the partials' block reduction and its pinned host copy

  // staging for fill_host
  void* d_stage = nullptr;
  uint64_t stage_bytes = 0;
  // write_stream: two device + two pinned chunk buffers, a copy stream and
  // events, kept across calls (pinning is slow)
  void* ws_dev[2] = {nullptr, nullptr};
  void* ws_host[2] = {nullptr, nullptr};
  size_t ws_bytes = 0;
  cudaStream_t ws_stream = nullptr;
  cudaEvent_t ws_ef[2] = {nullptr, nullptr}, ws_ec[2] = {nullptr, nullptr};

  // profiling (wallace_profile_begin/end)
  bool profiling = false;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev_pool, ev_plan;
  std::vector<cudaEvent_t> ev_free;

  // chi2_sample's non-finite error (chi2.cpp:29-31): the kernels set d_err,
  // every emitting launch sequence is followed by a copy of it into the
  // pinned h_err and ev_err; calls report it once the copy has landed (the
  // synchronous calls wait for it)
  uint32_t* d_err = nullptr;
  uint32_t* h_err = nullptr;
  cudaEvent_t ev_err = nullptr;
  bool err_queued = false;

  uint32_t cursor = 0;      // uniform across pools (all pools advance together)
  uint64_t pass_count = 0;  // uniform
};

namespace {

// transforms.cpp:39-50: half-angle tangents of 16 angles, the midpoints of 16
// equal slices of the window where cos and sin both lie in [0.05, 0.95]
// (bit-identical to the reference table; tests/test_capi_host.py pins it)
double rotation_t(int k) {
  const double lo = std::acos(0.95), hi = std::asin(0.95);
  return std::tan((lo + (k + 0.5) * (hi - lo) / 16) / 2);
}

// transforms.cpp:52-70 rotation_from_t
void rotation_from_t(double t, double& c, double& s) {
  if (std::abs(t) <= 1.0) {
    const double den = 1.0 + t * t;
    c = (1.0 - t * t) / den;
    s = (2.0 * t) / den;
  } else {
    const double u = 1.0 / t;
    const double den = 1.0 + u * u;
    c = (u * u - 1.0) / den;
    s = (2.0 * u) / den;
  }
}

void rotation_table(double* c, double* s) {
  for (int k = 0; k < 16; ++k) rotation_from_t(rotation_t(k), c[k], s[k]);
}

// generator.cpp:286-294 default_multipliers
void default_multipliers(uint64_t n, uint64_t& alpha, uint64_t& beta) {
  const auto near_odd = [](double x) { return static_cast<uint64_t>(std::llround(x)) | 1; };
  alpha = near_odd(0.382 * static_cast<double>(n));
  beta = near_odd(0.618 * static_cast<double>(n));
  if (alpha == beta) beta += 2;
}

wallace_status validate(const wallace_config* c) {
  // generator.cpp:221-236 (messages name the field, test_generator.cpp:42-72)
  if (!c) return fail(WALLACE_ERR_INVALID_PARAM, "config must not be NULL");
  const uint64_t n = c->pool_size;
  if (n < 32 || (n & (n - 1)) != 0 || n > (1ull << 31))
    return fail(WALLACE_ERR_CONFIG, "pool_size must be a power of two in [32, 2^31], got %llu",
                static_cast<unsigned long long>(n));
  if (c->discard_every < 1) return fail(WALLACE_ERR_CONFIG, "discard_every must be >= 1");
  if (!std::isfinite(c->out_sigma) || c->out_sigma <= 0.0)
    return fail(WALLACE_ERR_CONFIG, "out_sigma must be positive and finite");
  if (!std::isfinite(c->out_mean)) return fail(WALLACE_ERR_CONFIG, "out_mean must be finite");
  if (c->transform_family != 0 && c->transform_family != 1)
    return fail(WALLACE_ERR_CONFIG, "transform_family must be wallace4 (0) or rotation (1)");
  if (c->mixing != 0 && c->mixing != 1)
    return fail(WALLACE_ERR_CONFIG, "mixing must be stride_transpose (0) or affine (1)");
  if (c->chi2_method < 0 || c->chi2_method > 2)
    return fail(WALLACE_ERR_CONFIG, "chi2_method must be 0, 1 or 2");
  return WALLACE_OK;
}

wallace_status check_supported(const wallace_config* c, int dtype) {
  (void)c;
  (void)dtype;
  return WALLACE_OK;  // pools above the on-chip limit run HBM-resident
}

// pools above this run on the HBM-resident executor
uint64_t onchip_limit(int dtype) { return dtype == WALLACE_F32 ? (1u << 14) : (1u << 13); }

// Few pools cannot fill the GPU with the throughput kernel (a few warps per
// pool): give each pool a CTA of up to 1024 threads instead.
constexpr uint64_t kLatencyMaxPools = 148;

void select_kernel(wallace_handle* h) {
  if (h->large) {
    h->key = 64 + h->log2n;  // launch_pool_kernel -> the HBM-resident executor
    return;
  }
  const int lim = h->dtype == WALLACE_F32 ? 14 : 13;
  const bool lat_ok = h->log2n >= 8 && h->log2n <= lim;
  bool lat = false;
  if (h->kmode == 2) lat = lat_ok;
  else if (h->kmode == 0) lat = lat_ok && h->n_pools <= kLatencyMaxPools;
  h->key = h->log2n + (lat ? 16 : 0);
}

wb::FillArgs base_args(wallace_handle* h) {
  wb::FillArgs a{};
  a.pools_in = h->d_pools;
  a.pools_out = h->d_pools;
  a.st_in = h->d_state;
  a.st_out = h->d_state;
  a.d = static_cast<uint32_t>(std::min<uint64_t>(h->cfg.discard_every, 0xffffffffu));
  a.mean = h->cfg.out_mean;
  a.sigma = h->cfg.out_sigma;
  a.mean_is_zero = (h->cfg.out_mean == 0.0 && !std::signbit(h->cfg.out_mean)) ? 1 : 0;
  a.chi2 = h->chi2;
  a.leftover = h->d_leftover;
  a.out_stride = 0;
  a.pass_type = h->pass_type;
  a.n_probes = h->n_probes;
  a.probe_acc = h->d_probe_acc;
  std::memcpy(a.probe_out, h->probe_out, sizeof(a.probe_out));
  std::memcpy(a.probe_in, h->probe_in, sizeof(a.probe_in));
  a.def_totals = h->d_def_totals;
  a.def_marks = h->d_def_marks;
  a.def_stride = h->def_stride;
  a.def_threshold = h->def_threshold;
  a.err_word = h->d_err;
  if (h->large) {
    const uint64_t rows = h->N / 4;
    uint64_t al = 0, be = 0;
    default_multipliers(h->N, al, be);
    a.lg_pool2 = h->d_lg_pool2;
    a.lg_state = h->d_lg_state;
    a.lg_aux = h->d_lg_aux;
    a.lg_aux_stride = wb::large_aux_stride(h->N);
    a.lg_stride = default_stride(rows) % rows;
    {
      // inverse of the (odd) stride mod 2^64 by Newton's iteration, then mod rows
      uint64_t inv = a.lg_stride;
      for (int k = 0; k < 6; ++k) inv *= 2 - a.lg_stride * inv;
      a.lg_stride_inv = inv & (rows - 1);
    }
    {
      const char* bm = std::getenv("WALLACE_B200_LG_BLOCKMAJOR");
      a.lg_row_major = (bm && bm[0] == '1') ? 0 : 1;
    }
    a.lg_alpha = al;
    a.lg_beta = be;
    a.lg_log2n = h->log2n;
  }
  std::memcpy(a.rot_c, h->rot_c, sizeof(a.rot_c));
  std::memcpy(a.rot_s, h->rot_s, sizeof(a.rot_s));
  return a;
}

cudaEvent_t take_event(wallace_handle* h) {
  if (!h->ev_free.empty()) {
    cudaEvent_t e = h->ev_free.back();
    h->ev_free.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}

// Brackets one launch with events when profiling is on.
template <class F>
cudaError_t timed(wallace_handle* h, std::vector<std::pair<cudaEvent_t, cudaEvent_t>>& log,
                  cudaStream_t stream, F&& launch) {
  if (!h->profiling) return launch();
  cudaEvent_t a = take_event(h), b = take_event(h);
  cudaEventRecord(a, stream);
  const cudaError_t e = launch();
  cudaEventRecord(b, stream);
  log.emplace_back(a, b);
  return e;
}

// One pool-kernel launch and the plans it consumes.
struct Launch {
  wb::FillArgs a;
};

// Issues a sequence of launches.  Plans for launch k+1 are generated on the
// side stream while launch k runs (double-buffered plan words); the xoshiro
// stream itself is advanced only by the plan kernels, in order.
wallace_status issue(wallace_handle* h, std::vector<Launch>& ls) {
  if (ls.empty()) return WALLACE_OK;
  const size_t plan_words = h->n_pools * size_t(h->plan_cap) * h->plan_words;
  WB_CUDA(cudaEventRecord(h->ev_start, h->stream));
  WB_CUDA(cudaStreamWaitEvent(h->side, h->ev_start, 0));
  auto plans = [&](size_t k) -> wallace_status {
    wb::FillArgs& a = ls[k].a;
    a.plans = h->d_plans + (k & 1) * plan_words;
    a.plan_stride = h->plan_cap * h->plan_words;
    if (a.n_passes == 0) return WALLACE_OK;
    // the buffer is free once launch k-2 finished
    if (k >= 2) WB_CUDA(cudaStreamWaitEvent(h->side, h->ev_pooled[k & 1], 0));
    wb::PlanArgs p{};
    p.st_in = a.st_in;
    p.st_out = h->d_state;
    p.plans = const_cast<uint32_t*>(a.plans);
    p.plan_stride = h->plan_cap * h->plan_words;
    p.n_passes = a.n_passes;
    p.n_pools = static_cast<uint32_t>(h->n_pools);
    // decode_pass_plan's offset mask (generator.cpp:241-244)
    p.off_mask = static_cast<uint32_t>(h->cfg.mixing == 0 ? h->N / 4 - 1 : h->N - 1);
    p.fixed_transform = h->cfg.fixed_transform;
    p.rotation = h->cfg.transform_family == 1;
    p.large = h->large ? 1 : 0;
    WB_CUDA(timed(h, h->ev_plan, h->side, [&] { return wb::launch_plan_kernel(p, h->side); }));
    ++g_launches;
    WB_CUDA(cudaEventRecord(h->ev_planned[k & 1], h->side));
    return WALLACE_OK;
  };
  wallace_status st = plans(0);
  if (st) return st;
  for (size_t k = 0; k < ls.size(); ++k) {
    if (k + 1 < ls.size() && (st = plans(k + 1))) return st;
    const wb::FillArgs& a = ls[k].a;
    if (a.n_passes > 0) WB_CUDA(cudaStreamWaitEvent(h->stream, h->ev_planned[k & 1], 0));
    if (a.mode == wb::kModeFillPair) {
      WB_CUDA(timed(h, h->ev_pool, h->stream,
                    [&] { return wb::launch_pair_kernel(a, h->n_pools, h->stream); }));
      ++g_pair_launches;
    } else {
      WB_CUDA(timed(h, h->ev_pool, h->stream,
                    [&] { return wb::launch_pool_kernel(h->dtype, h->key, a, h->n_pools, h->stream); }));
    }
    ++g_launches;
    if (a.mode == wb::kModeFillLat && a.n_emit > 0) {  // the chain's scales onto the raw emissions
      WB_CUDA(wb::launch_rescale(h->dtype, a, static_cast<uint32_t>(h->N), h->n_pools, h->stream));
      ++g_launches;
    }
    if (h->after_launch) WB_CUDA(h->after_launch(a));
    WB_CUDA(cudaEventRecord(h->ev_pooled[k & 1], h->stream));
  }
  return WALLACE_OK;
}

// Run n passes without emission (warm-up, step_pass), in launches of at most
// plan_cap passes.
wallace_status run_passes(wallace_handle* h, uint64_t n) {
  std::vector<Launch> ls;
  while (n > 0) {
    const uint32_t k = static_cast<uint32_t>(std::min<uint64_t>(n, h->plan_cap));
    Launch l{base_args(h)};
    l.a.lg_pass0 = h->pass_count;
    l.a.mode = wb::kModePasses;
    l.a.n_passes = k;
    l.a.n_emit = 0;
    l.a.lead = 0;
    l.a.last_limit = 0;
    ls.push_back(l);
    h->pass_count += k;
    n -= k;
  }
  return issue(h, ls);
}

wallace_status ensure_leftover(wallace_handle* h) {
  if (h->d_leftover) return WALLACE_OK;
  WB_CUDA(cudaMalloc(&h->d_leftover, h->n_pools * (h->N - 1) * h->esize));
  return WALLACE_OK;
}

// Before the pool advances outside fill(): keep the partially consumed
// emission (Generator::out_ is untouched by step_pass / inject_pool).
wallace_status materialize(wallace_handle* h) {
  if (h->cursor >= h->N - 1) return WALLACE_OK;
  wallace_status st = ensure_leftover(h);
  if (st) return st;
  WB_CUDA(wb::launch_materialize(h->dtype, h->d_pools, h->d_state, h->d_leftover, h->n_pools,
                                 static_cast<uint32_t>(h->N), h->cfg.out_mean, h->stream));
  ++g_launches;
  return WALLACE_OK;
}

// The fill / consume engine.  out == nullptr with mode kModeConsume feeds the
// consumer partials instead.  st_first / pools_first: state the first launch
// reads (the snapshot for fill_from_snapshot).
wallace_status run_emit(wallace_handle* h, void* out, uint64_t count, int mode,
                        const PoolState* st_first, const void* pools_first) {
  if (count < 1) return fail(WALLACE_ERR_INVALID_PARAM, "fill: count must be >= 1");
  const uint64_t n1 = h->N - 1;
  const uint64_t d = h->cfg.discard_every;
  uint64_t produced = 0;
  bool first = true;
  uint64_t lat_ramp = 128;  // passes of the next ramped latency launch
  if (const char* r = std::getenv("WALLACE_B200_NO_LATRAMP"); r && r[0] == '1') lat_ramp = ~0ull >> 1;
  std::vector<Launch> ls;
  while (produced < count) {
    wb::FillArgs a = base_args(h);
    a.mode = mode;
    // every emission is the pool itself (scale exactly 1, mean +0): the
    // bulk-emission kernel (throughput geometry, wallace4 passes)
    if (mode == wb::kModeFill && h->bulk_ok && h->key < 16 && h->log2n >= 7) a.mode = wb::kModeFillBulk;
    else if (mode == wb::kModeFill && h->staged_ok && h->key < 16 && h->log2n >= 7)
      a.mode = wb::kModeFillStaged;
    else if (mode == wb::kModeFill && h->lat_fill_ok && h->key >= 16 && h->key < 64) {
      if (!h->d_scales) {
        // one pitched row of N raw values per emission of a launch, at most
        // 256 MiB for the handle
        const uint64_t row_bytes = h->n_pools * h->N * h->esize;
        h->lat_rows = std::max<uint64_t>(1, std::min<uint64_t>(h->plan_cap / std::max<uint64_t>(1, d),
                                                                (256ull << 20) / row_bytes));
        WB_CUDA(cudaMalloc(&h->d_scales, h->n_pools * size_t(h->plan_cap) * sizeof(double)));
        WB_CUDA(cudaMalloc(&h->d_lat_raw, h->lat_rows * row_bytes));
      }
      a.mode = wb::kModeFillLat;
      a.scales = h->d_scales;
      a.scale_stride = h->plan_cap;
      a.lat_raw = h->d_lat_raw;
      a.lat_rows = h->lat_rows;
    }
    if (mode == wb::kModeDefect) a.def_e0 = produced / (h->N - 1);  // defect runs start at an emission
    a.out = out;
    a.out_stride = count;
    a.out_offset = produced;
    a.part_sums = h->d_part_sums;
    a.part_hist = h->d_part_hist;
    if (first) {
      a.st_in = st_first;
      a.pools_in = pools_first;
    }
    uint64_t lead = 0;
    if (first && h->cursor < n1) lead = std::min<uint64_t>(count, n1 - h->cursor);
    const uint64_t remaining = count - produced - lead;
    uint64_t e_total = (remaining + n1 - 1) / n1;
    uint64_t e = 0, passes = 0;
    // pair_kernel: launches that start at an emission and hold no
    // renormalisation; a partially consumed emission is drained first, and
    // the emission whose passes reach pass_count % 256 == 0 goes through
    // pool_kernel on its own
    const bool pair = h->pair_ok && mode == wb::kModeFill &&
                      (a.mode == wb::kModeFillBulk || a.mode == wb::kModeFillStaged) && e_total > 0 && out;
    if (pair && lead > 0) {
      a.lead = static_cast<uint32_t>(lead);
      a.n_emit = 0;
      a.n_passes = 0;
      a.last_limit = 0;
      a.lg_pass0 = h->pass_count;
      ls.push_back(Launch{a});
      h->cursor += static_cast<uint32_t>(lead);
      produced += lead;
      first = false;
      continue;
    }
    if (e_total > 0) {
      if (d <= h->plan_cap) {
        e = std::min<uint64_t>(e_total, h->plan_cap / d);
        if (a.mode == wb::kModeFillLat) {
          e = std::min<uint64_t>(e, h->lat_rows);
          // A long latency fill ramps its launches up (128, 256, ... passes):
          // plan_kernel walks a launch's plan words on one thread (~84 ns
          // per pass against the pool kernel's ~270 ns), and only the first
          // launch's planning is not hidden behind the previous pool launch.
          if (e_total * d >= 1024 && lat_ramp < e * d) {
            e = std::max<uint64_t>(1, lat_ramp / d);
            lat_ramp *= 2;
          }
        }
        if (h->max_emit > 0) e = std::min<uint64_t>(e, h->max_emit);
        if (pair) {
          // the first pass of this launch that ends on a renormalisation
          // (generator.cpp:342) and the emission it belongs to
          const uint64_t jstar = 256 - h->pass_count % 256;
          const uint64_t er = (jstar - 1) / d;
          if (er == 0) {
            e = 1;
          } else {
            e = std::min(e, er);
            a.mode = wb::kModeFillPair;
            const char* nt = std::getenv("WALLACE_B200_PAIR_DEBUG");  // timing-only ablations
            a.pad_ab = nt ? std::atoi(nt) : 0;
          }
        }
        passes = e * d;
      } else {
        // an emission longer than one launch: run d-1 passes first, then a
        // launch with one pass and the emission (emission alignment is
        // per launch).  The passes must not run before the partially
        // consumed emission is drained (or before the snapshot being
        // replayed is in the live buffers): a drain-only launch does that.
        if (first && (lead > 0 || st_first != h->d_state || pools_first != h->d_pools)) {
          a.lead = static_cast<uint32_t>(lead);
          a.n_emit = 0;
          a.n_passes = 0;
          a.last_limit = 0;
          a.lg_pass0 = h->pass_count;
          ls.push_back(Launch{a});
          h->cursor += static_cast<uint32_t>(lead);
          produced += lead;
          first = false;
          continue;
        }
        wallace_status st = issue(h, ls);
        ls.clear();
        if (!st) st = run_passes(h, d - 1);
        if (st) return st;
        e = 1;
        passes = 1;
        a.d = 1;
      }
    }
    const uint64_t last_limit =
        e == 0 ? 0 : (e == e_total ? remaining - (e - 1) * n1 : n1);
    a.lead = static_cast<uint32_t>(lead);
    a.n_emit = static_cast<uint32_t>(e);
    a.n_passes = static_cast<uint32_t>(passes);
    a.last_limit = static_cast<uint32_t>(last_limit);
    a.lg_pass0 = h->pass_count;
    if (a.d != h->cfg.discard_every) {
      // the huge-discard path ran d-1 passes eagerly: keep launch order
      std::vector<Launch> one{Launch{a}};
      wallace_status st = issue(h, ls);
      if (!st) st = issue(h, one);
      if (st) return st;
      ls.clear();
    } else {
      ls.push_back(Launch{a});
    }
    h->pass_count += passes;
    h->cursor = e > 0 ? static_cast<uint32_t>(last_limit) : h->cursor + static_cast<uint32_t>(lead);
    produced += lead + (e == 0 ? 0 : (e == e_total ? remaining : e * n1));
    first = false;
  }
  wallace_status st = issue(h, ls);
  if (st) return st;
  // the error word of these launches -> pinned host memory (see d_err)
  WB_CUDA(cudaMemcpyAsync(h->h_err, h->d_err, sizeof(uint32_t), cudaMemcpyDeviceToHost, h->stream));
  WB_CUDA(cudaEventRecord(h->ev_err, h->stream));
  h->err_queued = true;
  return WALLACE_OK;
}

// Reports chi2_sample's error from emitting launches already issued: when
// `wait`, after they finished (the caller synchronises anyway); otherwise only
// if their error word has already landed.  The error is reported once.
wallace_status take_err(wallace_handle* h, bool wait) {
  if (!h->err_queued) return WALLACE_OK;
  if (wait) {
    WB_CUDA(cudaEventSynchronize(h->ev_err));
  } else if (cudaEventQuery(h->ev_err) != cudaSuccess) {
    (void)cudaGetLastError();  // cudaErrorNotReady is not an error
    return WALLACE_OK;
  }
  h->err_queued = false;
  if (*h->h_err == 0) return WALLACE_OK;
  *h->h_err = 0;
  WB_CUDA(cudaMemsetAsync(h->d_err, 0, sizeof(uint32_t), h->stream));
  // the reference's refill_ threw before the emission existed (its buffer
  // stays used up, generator.cpp:358-376): the next value starts a new
  // emission, whose chi2 draw throws again.  For a batch the partially
  // consumed emission of every pool is dropped.
  h->cursor = static_cast<uint32_t>(h->N - 1);
  return fail(WALLACE_ERR_INVALID_PARAM, "chi2_sample: x must be finite");
}

}  // namespace

extern "C" {

const char* wallace_last_error(void) { return g_err.c_str(); }

uint64_t wallace_kernel_launches(void) { return g_launches.load(); }
uint64_t wallace_pair_kernel_launches(void) { return g_pair_launches.load(); }

wallace_status wallace_validate_config(const wallace_config* cfg) { return validate(cfg); }

uint64_t wallace_default_stride(uint64_t rows) { return rows ? default_stride(rows) : 0; }

int32_t wallace_decode_pass_plan(uint64_t pool_size, uint64_t w0, uint64_t w1, uint64_t* off0) {
  if (off0) *off0 = w1 & (pool_size / 4 - 1);
  return static_cast<int32_t>(w0 % 384u);
}

wallace_status wallace_decode_pass_plan_ex(const wallace_config* cfg, uint64_t w0, uint64_t w1,
                                           wallace_pass_plan* out) {
  wallace_status st = validate(cfg);
  if (st) return st;
  if (!out) return fail(WALLACE_ERR_INVALID_PARAM, "out must not be NULL");
  // generator.cpp:238-257
  *out = wallace_pass_plan{};
  const uint64_t n = cfg->pool_size;
  const uint64_t mask = cfg->mixing == 0 ? n / 4 - 1 : n - 1;
  out->offset[0] = w1 & mask;
  out->offset[1] = (w1 >> 32) & mask;
  if (cfg->transform_family == 0) {
    out->wallace_variant = static_cast<int32_t>(w0 % 384u);
  } else {
    out->t_index[0] = static_cast<int32_t>(w0 & 15);
    out->negate[0] = static_cast<int32_t>((w0 >> 4) & 1);
    out->t_index[1] = static_cast<int32_t>((w0 >> 5) & 15);
    out->negate[1] = static_cast<int32_t>((w0 >> 9) & 1);
  }
  return WALLACE_OK;
}

void wallace_rotation_table(double t[16], double c[16], double s[16]) {
  for (int k = 0; k < 16; ++k) {
    if (t) t[k] = rotation_t(k);
    double ck = 0.0, sk = 0.0;
    rotation_from_t(rotation_t(k), ck, sk);
    if (c) c[k] = ck;
    if (s) s[k] = sk;
  }
}

wallace_status wallace_host_seed_pool(const wallace_config* cfg, uint64_t seed, double* raw_out,
                                      double* reserved_prev, double* sum_sq, uint64_t s_out[4],
                                      uint64_t* draws) {
  wallace_status st = validate(cfg);
  if (st) return st;
  if (!raw_out) return fail(WALLACE_ERR_INVALID_PARAM, "raw_out must not be NULL");
  double res = 0.0;
  uint64_t s[4], dr = 0;
  seed_pool_double(cfg->pool_size, seed, raw_out, res, s, dr);
  if (reserved_prev) *reserved_prev = res;
  if (sum_sq) *sum_sq = neumaier_sq(raw_out, cfg->pool_size);
  if (s_out) std::memcpy(s_out, s, sizeof(s));
  if (draws) *draws = dr;
  return WALLACE_OK;
}

wallace_status wallace_create(const wallace_config* cfg, uint64_t n_pools, const uint64_t* seeds,
                              wallace_dtype dtype, void* stream, wallace_handle** out) {
  return wallace_create_ex(cfg, n_pools, seeds, dtype, stream, 0u, out);
}

wallace_status wallace_create_ex(const wallace_config* cfg, uint64_t n_pools, const uint64_t* seeds,
                                 wallace_dtype dtype, void* stream, uint32_t flags, wallace_handle** out) {
  if (!out) return fail(WALLACE_ERR_INVALID_PARAM, "out must not be NULL");
  if (flags & ~uint32_t(WALLACE_CREATE_DEVICE_SEED))
    return fail(WALLACE_ERR_INVALID_PARAM, "create: unknown flags");
  const bool device_seed = (flags & WALLACE_CREATE_DEVICE_SEED) != 0;
  *out = nullptr;
  wallace_status st = validate(cfg);
  if (st) return st;
  if (dtype != WALLACE_F32 && dtype != WALLACE_F64)
    return fail(WALLACE_ERR_INVALID_PARAM, "dtype must be WALLACE_F32 or WALLACE_F64");
  if ((st = check_supported(cfg, dtype))) return st;
  if (n_pools < 1 || n_pools > 0x7fffffffull)
    return fail(WALLACE_ERR_INVALID_PARAM, "n_pools must be in [1, 2^31)");

  auto* h = new wallace_handle();
  h->cfg = *cfg;
  h->dtype = dtype;
  h->esize = dtype == WALLACE_F32 ? 4 : 8;
  h->n_pools = n_pools;
  h->N = cfg->pool_size;
  h->log2n = ilog2(h->N);
  h->stream = static_cast<cudaStream_t>(stream);
  h->chi2 = chi2_consts(*cfg);
  h->pass_type = 2 * cfg->transform_family + cfg->mixing;
  h->large = cfg->pool_size > onchip_limit(dtype);
  if (h->large && device_seed) {
    delete h;
    return fail(WALLACE_ERR_UNSUPPORTED, "create: device seeding covers on-chip pool sizes only");
  }
  h->plan_words = h->large ? (cfg->transform_family == 1 ? 3 : 2) : (cfg->transform_family == 1 ? 2 : 1);
  h->plan_cap = static_cast<uint32_t>(std::max<uint64_t>(
      1, std::min<uint64_t>(kMaxPassesPerLaunch, kPlanBudgetBytes / (4 * h->plan_words * n_pools))));
  rotation_table(h->rot_c, h->rot_s);
  if (cfg->mixing == 1) {
    // the kernels compile default_multipliers in; check them against the
    // reference formula (generator.cpp:286-294) for this size
    uint32_t ka = 0, kb = 0;
    wb::affine_multipliers(h->log2n, &ka, &kb);
    uint64_t ra = 0, rb = 0;
    default_multipliers(h->N, ra, rb);
    if (ka != ra || kb != rb) {
      delete h;
      return fail(WALLACE_ERR_UNSUPPORTED, "mixing: affine multipliers for pool_size %llu",
                  static_cast<unsigned long long>(cfg->pool_size));
    }
  }
  h->cursor = static_cast<uint32_t>(h->N - 1);
  auto cleanup = [&](wallace_status s) {
    wallace_destroy(h);
    return s;
  };

  // ---- host seeding (parallel over pools) ----
  const uint64_t N = h->N;
  std::vector<unsigned char> pools(device_seed ? 0 : n_pools * N * h->esize);
  std::vector<PoolState> states(device_seed ? 0 : n_pools);
  if (!device_seed) {
    std::atomic<uint64_t> next{0};
    unsigned nt = std::max(1u, std::thread::hardware_concurrency());
    nt = static_cast<unsigned>(std::min<uint64_t>(nt, n_pools));
    auto work = [&] {
      std::vector<double> raw(N);
      for (;;) {
        const uint64_t p = next.fetch_add(1);
        if (p >= n_pools) break;
        const uint64_t seed = seeds ? seeds[p] : cfg->seed + p;
        PoolState& ps = states[p];
        std::memset(&ps, 0, sizeof(ps));
        seed_pool_double(N, seed, raw.data(), ps.reserved_prev, ps.s, ps.draws);
        if (dtype == WALLACE_F32) {
          float* dst = reinterpret_cast<float*>(pools.data()) + p * N;
          for (uint64_t i = 0; i < N; ++i) dst[i] = static_cast<float>(raw[i]);
          ps.sum_sq = neumaier_sq(dst, N);
        } else {
          double* dst = reinterpret_cast<double*>(pools.data()) + p * N;
          std::memcpy(dst, raw.data(), N * sizeof(double));
          ps.sum_sq = neumaier_sq(dst, N);
        }
        ps.cursor = static_cast<uint32_t>(N - 1);
        ps.seed = seed;
      }
    };
    std::vector<std::thread> th;
    for (unsigned t = 1; t < nt; ++t) th.emplace_back(work);
    work();
    for (auto& t : th) t.join();
  }

  // ---- device residency ----
#define WB_CUDA_C(expr)                                                                   \
  do {                                                                                    \
    cudaError_t e_ = (expr);                                                              \
    if (e_ != cudaSuccess)                                                                \
      return cleanup(fail(WALLACE_ERR_CUDA, "%s: %s", #expr, cudaGetErrorString(e_)));    \
  } while (0)
  WB_CUDA_C(cudaMalloc(&h->d_pools, n_pools * N * h->esize));
  WB_CUDA_C(cudaMalloc(&h->d_state, n_pools * sizeof(PoolState)));
  if (h->large) {
    WB_CUDA_C(cudaMalloc(&h->d_lg_pool2, n_pools * N * h->esize));
    WB_CUDA_C(cudaMalloc(&h->d_lg_state, n_pools * wb::large_state_bytes()));
    WB_CUDA_C(cudaMalloc(&h->d_lg_aux, n_pools * wb::large_aux_stride(N) * sizeof(double)));
  }
  WB_CUDA_C(cudaMalloc(&h->d_plans, 2 * n_pools * h->plan_cap * h->plan_words * sizeof(uint32_t)));
  WB_CUDA_C(cudaStreamCreateWithFlags(&h->side, cudaStreamNonBlocking));
  WB_CUDA_C(cudaEventCreateWithFlags(&h->ev_start, cudaEventDisableTiming));
  WB_CUDA_C(cudaMalloc(&h->d_err, sizeof(uint32_t)));
  WB_CUDA_C(cudaMallocHost(&h->h_err, sizeof(uint32_t)));
  *h->h_err = 0;
  WB_CUDA_C(cudaMemsetAsync(h->d_err, 0, sizeof(uint32_t), h->stream));
  WB_CUDA_C(cudaEventCreateWithFlags(&h->ev_err, cudaEventDisableTiming));
  for (int i = 0; i < 2; ++i) {
    WB_CUDA_C(cudaEventCreateWithFlags(&h->ev_planned[i], cudaEventDisableTiming));
    WB_CUDA_C(cudaEventCreateWithFlags(&h->ev_pooled[i], cudaEventDisableTiming));
  }
  select_kernel(h);
  {
    // disable_chi2 makes S = sum_sq, so r = S/sum_sq = 1 and scale = sigma
    // exactly; with sigma 1 and mean +0 each emitted value is x*1+0
    const char* nb = std::getenv("WALLACE_B200_NO_BULK");
    h->bulk_cfg_ok = cfg->disable_chi2 && cfg->out_sigma == 1.0 && cfg->out_mean == 0.0 &&
                     !std::signbit(cfg->out_mean) && h->pass_type < 2 && !(nb && nb[0] == '1');
    h->bulk_ok = h->bulk_cfg_ok;
    // any other wallace4 fill: scaled values staged in shared memory and
    // sent by bulk copies (WALLACE_B200_NO_STAGED=1: register emission)
    const char* ns = std::getenv("WALLACE_B200_NO_STAGED");
    h->staged_ok = h->pass_type < 2 && !(ns && ns[0] == '1');
    // fp32 pools of 4096, wallace4 + stride mixing, two passes per emission,
    // throughput geometry: pair_kernel (pool_pair.cu) -- two passes per
    // shared-memory round trip, bit-exact with pool_kernel; 3.11 ms (scaled
    // emissions) / 3.10 ms (unit scale) per 2^32 values against pool_kernel's
    // 3.66 / 3.13 ms.  WALLACE_B200_PAIR=0 keeps every launch on pool_kernel.
    const char* np = std::getenv("WALLACE_B200_PAIR");
    h->pair_ok = dtype == WALLACE_F32 && h->log2n == 12 && h->pass_type == 0 && cfg->discard_every == 2 &&
                 !h->large && !(np && np[0] == '0');
    // latency geometry (few pools), wallace4, up to 512 compute threads plus
    // the chain warp (WALLACE_B200_NO_LATFILL=1: the coupled chain)
    const char* nl = std::getenv("WALLACE_B200_NO_LATFILL");
    h->lat_fill_ok = h->pass_type < 2 && h->log2n >= 7 && h->log2n <= 11 && !(nl && nl[0] == '1');
  }
  if (!device_seed) {
    WB_CUDA_C(cudaMemcpyAsync(h->d_pools, pools.data(), pools.size(), cudaMemcpyHostToDevice,
                              h->stream));
    WB_CUDA_C(cudaMemcpyAsync(h->d_state, states.data(), n_pools * sizeof(PoolState),
                              cudaMemcpyHostToDevice, h->stream));
  } else {
    // the constructor's Polar fill + normalisation on the device (seed_kernel)
    uint64_t* d_seeds = nullptr;
    if (seeds) {
      WB_CUDA_C(cudaMalloc(&d_seeds, n_pools * sizeof(uint64_t)));
      WB_CUDA_C(cudaMemcpyAsync(d_seeds, seeds, n_pools * sizeof(uint64_t), cudaMemcpyHostToDevice, h->stream));
    }
    const cudaError_t e = wb::launch_seed(h->dtype, d_seeds, cfg->seed, static_cast<uint32_t>(N), h->d_pools,
                                          h->d_state, n_pools, h->stream);
    ++g_launches;
    if (d_seeds) {
      cudaStreamSynchronize(h->stream);
      cudaFree(d_seeds);
    }
    WB_CUDA_C(e);
  }
  // warm-up (generator.cpp:329-330)
  if ((st = run_passes(h, 16))) return cleanup(st);
  WB_CUDA_C(cudaStreamSynchronize(h->stream));
#undef WB_CUDA_C
  *out = h;
  return WALLACE_OK;
}

wallace_status wallace_destroy(wallace_handle* h) {
  if (!h) return WALLACE_OK;
  cudaFree(h->d_pools);
  cudaFree(h->d_state);
  cudaFree(h->d_plans);
  if (h->side) cudaStreamDestroy(h->side);
  if (h->cp_stream) cudaStreamDestroy(h->cp_stream);
  if (h->ev_cp) cudaEventDestroy(h->ev_cp);
  if (h->ev_start) cudaEventDestroy(h->ev_start);
  for (int i = 0; i < 2; ++i) {
    if (h->ev_planned[i]) cudaEventDestroy(h->ev_planned[i]);
    if (h->ev_pooled[i]) cudaEventDestroy(h->ev_pooled[i]);
  }
  cudaFree(h->d_err);
  cudaFreeHost(h->h_err);
  if (h->ev_err) cudaEventDestroy(h->ev_err);
  cudaFree(h->d_leftover);
  cudaFree(h->d_scales);
  cudaFree(h->d_lat_raw);
  for (auto& sn : h->snap) {
    cudaFree(sn.pools);
    cudaFree(sn.state);
    cudaFree(sn.leftover);
  }
  cudaFree(h->d_astage);
  cudaFree(h->d_part_sums);
  cudaFree(h->d_part_hist);
  h->red.release();
  cudaFree(h->d_stage);
  cudaFree(h->d_lg_pool2);
  cudaFree(h->d_lg_state);
  cudaFree(h->d_lg_aux);
  for (int k = 0; k < 2; ++k) {
    cudaFree(h->ws_dev[k]);
    cudaFreeHost(h->ws_host[k]);
    if (h->ws_ef[k]) cudaEventDestroy(h->ws_ef[k]);
    if (h->ws_ec[k]) cudaEventDestroy(h->ws_ec[k]);
  }
  if (h->ws_stream) cudaStreamDestroy(h->ws_stream);
  for (auto& pr : h->ev_pool) { cudaEventDestroy(pr.first); cudaEventDestroy(pr.second); }
  for (auto& pr : h->ev_plan) { cudaEventDestroy(pr.first); cudaEventDestroy(pr.second); }
  for (auto e : h->ev_free) cudaEventDestroy(e);
  delete h;
  return WALLACE_OK;
}

wallace_status wallace_profile_begin(wallace_handle* h) {
  if (!h) return fail(WALLACE_ERR_INVALID_PARAM, "handle must not be NULL");
  h->profiling = true;
  return WALLACE_OK;
}

wallace_status wallace_profile_end(wallace_handle* h, double* pool_ms, uint64_t* pool_n,
                                   double* plan_ms, uint64_t* plan_n) {
  if (!h) return fail(WALLACE_ERR_INVALID_PARAM, "handle must not be NULL");
  h->profiling = false;
  WB_CUDA(cudaStreamSynchronize(h->stream));
  WB_CUDA(cudaStreamSynchronize(h->side));
  auto sum = [&](std::vector<std::pair<cudaEvent_t, cudaEvent_t>>& log, double* ms, uint64_t* n) {
    double acc = 0.0;
    for (auto& [a, b] : log) {
      float t = 0.f;
      if (cudaEventElapsedTime(&t, a, b) == cudaSuccess) acc += t;
      h->ev_free.push_back(a);
      h->ev_free.push_back(b);
    }
    if (ms) *ms = acc;
    if (n) *n = log.size();
    log.clear();
  };
  // WALLACE_B200_PROFILE_DUMP=1: the launch timeline (ms from the first pool
  // launch's start) on stderr -- a measurement aid
  if (const char* d = std::getenv("WALLACE_B200_PROFILE_DUMP"); d && d[0] == '1' && !h->ev_pool.empty()) {
    const cudaEvent_t t0 = h->ev_pool.front().first;
    auto dump = [&](const char* what, std::vector<std::pair<cudaEvent_t, cudaEvent_t>>& log) {
      for (auto& [a, b] : log) {
        float ta = 0.f, tb = 0.f;
        cudaEventElapsedTime(&ta, t0, a);
        cudaEventElapsedTime(&tb, t0, b);
        std::fprintf(stderr, "timeline %s %.4f %.4f\n", what, ta, tb);
      }
    };
    dump("pool", h->ev_pool);
    dump("plan", h->ev_plan);
  }
  sum(h->ev_pool, pool_ms, pool_n);
  sum(h->ev_plan, plan_ms, plan_n);
  return WALLACE_OK;
}

wallace_status wallace_set_kernel_mode(wallace_handle* h, int32_t mode) {
  if (!h) return fail(WALLACE_ERR_INVALID_PARAM, "handle must not be NULL");
  if (mode < 0 || mode > 2) return fail(WALLACE_ERR_INVALID_PARAM, "kernel mode must be 0, 1 or 2");
  h->kmode = mode;
  select_kernel(h);
  return WALLACE_OK;
}

wallace_status wallace_set_stream(wallace_handle* h, void* stream) {
  if (!h) return fail(WALLACE_ERR_INVALID_PARAM, "handle must not be NULL");
  // work queued on the old stream (pool kernels reading plans / pools /
  // state) and on the plan side stream precedes everything issued after the
  // switch: the new stream and the side stream wait for both
  cudaStream_t ns = static_cast<cudaStream_t>(stream);
  WB_CUDA(cudaEventRecord(h->ev_start, h->stream));
  WB_CUDA(cudaStreamWaitEvent(ns, h->ev_start, 0));
  WB_CUDA(cudaStreamWaitEvent(h->side, h->ev_start, 0));
  WB_CUDA(cudaEventRecord(h->ev_start, h->side));
  WB_CUDA(cudaStreamWaitEvent(ns, h->ev_start, 0));
  h->stream = ns;
  return WALLACE_OK;
}

wallace_status wallace_synchronize(wallace_handle* h) {
  if (!h) return fail(WALLACE_ERR_INVALID_PARAM, "handle must not be NULL");
  WB_CUDA(cudaStreamSynchronize(h->stream));
  return take_err(h, true);
}

wallace_status wallace_fill(wallace_handle* h, void* dev_out, uint64_t count) {
  if (!h) return fail(WALLACE_ERR_INVALID_PARAM, "handle must not be NULL");
  if (count < 1) return fail(WALLACE_ERR_INVALID_PARAM, "fill: count must be >= 1");
  if (!dev_out) return fail(WALLACE_ERR_INVALID_PARAM, "fill: output must not be NULL");
  // an earlier asynchronous fill's chi2 error, if it is already known
  wallace_status st = take_err(h, false);
  if (st) return st;
  return run_emit(h, dev_out, count, wb::kModeFill, h->d_state, h->d_pools);
}

// ---- stream wire format (cmd_gen.cpp:39-57) --------------------------------
namespace {

// write all of buf at offset (seekable) or at the current position
bool write_all(int fd, const char* buf, size_t n, bool positional, off_t off) {
  while (n > 0) {
    const ssize_t w = positional ? ::pwrite(fd, buf, n, off) : ::write(fd, buf, n);
    if (w < 0) {
      if (errno == EINTR) continue;
      return false;
    }
    buf += w;
    n -= static_cast<size_t>(w);
    off += w;
  }
  return true;
}

// One chunk [n_pools][ck] (host, dtype esize) -> file.  Binary formats land
// pool-major at offset base + (p * count + k0) * out_size; text (one pool)
// is appended: "%.17g\n" per value, formatted by several threads into
// per-thread buffers that are written in order.
bool write_chunk(int fd, int fmt, const unsigned char* src, size_t esize, uint64_t n_pools, uint64_t ck,
                 uint64_t count, uint64_t k0, bool positional, off_t base, unsigned threads) {
  auto value = [&](uint64_t i) -> double {
    if (esize == 4) {
      float f;
      std::memcpy(&f, src + i * 4, 4);
      return static_cast<double>(f);
    }
    double d;
    std::memcpy(&d, src + i * 8, 8);
    return d;
  };
  if (fmt == WALLACE_FMT_TEXT) {
    const uint64_t per = (ck + threads - 1) / threads;
    std::vector<std::string> parts(threads);
    std::vector<std::thread> ts;
    for (unsigned t = 0; t < threads; ++t) {
      ts.emplace_back([&, t] {
        const uint64_t i0 = t * per, i1 = std::min<uint64_t>(ck, i0 + per);
        std::string& out = parts[t];
        out.reserve((i1 > i0 ? i1 - i0 : 0) * 24);
        char b[40];
        for (uint64_t i = i0; i < i1; ++i) {
          const int len = std::snprintf(b, sizeof b, "%.17g\n", value(i));
          out.append(b, static_cast<size_t>(len));
        }
      });
    }
    for (auto& t : ts) t.join();
    for (const auto& part : parts)
      if (!write_all(fd, part.data(), part.size(), false, 0)) return false;
    return true;
  }
  const size_t osz = fmt == WALLACE_FMT_F32LE ? 4 : 8;
  // little-endian host: f64le of a double / f32le of a float is its bytes
  std::atomic<uint64_t> next{0};
  std::atomic<bool> ok{true};
  std::vector<std::thread> ts;
  for (unsigned t = 0; t < std::max(1u, std::min<unsigned>(threads, static_cast<unsigned>(n_pools))); ++t) {
    ts.emplace_back([&] {
      std::vector<unsigned char> conv;
      for (;;) {
        const uint64_t p = next.fetch_add(1);
        if (p >= n_pools || !ok) break;
        const unsigned char* row = src + p * ck * esize;
        const char* data = reinterpret_cast<const char*>(row);
        if (osz != esize) {  // fp32 values as f64le
          conv.resize(ck * 8);
          for (uint64_t i = 0; i < ck; ++i) {
            float f;
            std::memcpy(&f, row + i * 4, 4);
            const double d = f;
            std::memcpy(conv.data() + i * 8, &d, 8);
          }
          data = reinterpret_cast<const char*>(conv.data());
        }
        const off_t off = base + static_cast<off_t>((p * count + k0) * osz);
        if (!write_all(fd, data, ck * osz, positional, off)) ok = false;
      }
    });
  }
  for (auto& t : ts) t.join();
  return ok;
}

}  // namespace

wallace_status wallace_write_stream(wallace_handle* h, uint64_t count, int32_t format, int32_t fd) {
  if (!h) return fail(WALLACE_ERR_INVALID_PARAM, "handle must not be NULL");
  if (count < 1) return fail(WALLACE_ERR_INVALID_PARAM, "write_stream: count must be >= 1");
  if (format != WALLACE_FMT_F64LE && format != WALLACE_FMT_TEXT && format != WALLACE_FMT_F32LE)
    return fail(WALLACE_ERR_INVALID_PARAM, "write_stream: format must be f64le, text or f32le");
  if (format == WALLACE_FMT_F32LE && h->dtype != WALLACE_F32)
    return fail(WALLACE_ERR_INVALID_PARAM, "write_stream: f32le needs an fp32 handle");
  const off_t base = ::lseek(fd, 0, SEEK_CUR);
  const bool seekable = base != static_cast<off_t>(-1);
  if (h->n_pools > 1 && (format == WALLACE_FMT_TEXT || !seekable))
    return fail(WALLACE_ERR_INVALID_PARAM,
                "write_stream: several pools need a binary format and a seekable file (pool-major layout)");
  const bool positional = seekable && format != WALLACE_FMT_TEXT;
  // chunk along the per-pool count: about an eighth of the block (so the
  // stages overlap), within [16, 512] MiB; whole emissions per launch for
  // large batches
  const uint64_t row = h->n_pools * h->esize;
  const uint64_t want = std::min<uint64_t>(512ull << 20, std::max<uint64_t>(16ull << 20, row * count / 8));
  const uint64_t c = std::max<uint64_t>(1, std::min<uint64_t>(count, want / row));
  const size_t bytes = h->n_pools * c * h->esize;
  cudaError_t e = cudaSuccess;
  if (h->ws_bytes < bytes) {
    for (int k = 0; k < 2; ++k) {
      cudaFree(h->ws_dev[k]);
      cudaFreeHost(h->ws_host[k]);
      h->ws_dev[k] = h->ws_host[k] = nullptr;
    }
    h->ws_bytes = 0;
    for (int k = 0; k < 2 && e == cudaSuccess; ++k) {
      e = cudaMalloc(&h->ws_dev[k], bytes);
      if (e == cudaSuccess) e = cudaMallocHost(&h->ws_host[k], bytes);
    }
    if (e == cudaSuccess) h->ws_bytes = bytes;
  }
  for (int k = 0; k < 2 && e == cudaSuccess; ++k) {
    if (!h->ws_ef[k]) e = cudaEventCreateWithFlags(&h->ws_ef[k], cudaEventDisableTiming);
    if (e == cudaSuccess && !h->ws_ec[k]) e = cudaEventCreateWithFlags(&h->ws_ec[k], cudaEventDisableTiming);
  }
  if (e == cudaSuccess && !h->ws_stream) e = cudaStreamCreateWithFlags(&h->ws_stream, cudaStreamNonBlocking);
  if (e != cudaSuccess) return fail(WALLACE_ERR_CUDA, "write_stream: %s", cudaGetErrorString(e));
  void* const* d = h->ws_dev;
  void* const* hb = h->ws_host;
  cudaStream_t cs = h->ws_stream;
  cudaEvent_t* ef = h->ws_ef;
  cudaEvent_t* ec = h->ws_ec;
  const unsigned threads = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
  const uint64_t nk = (count + c - 1) / c;
  wallace_status st = WALLACE_OK;
  for (uint64_t k = 0; k <= nk && !st; ++k) {
    if (k < nk) {
      // generate chunk k into d[k&1] (free once chunk k-2's copy is done)
      const uint64_t ck = std::min<uint64_t>(c, count - k * c);
      if (k >= 2 && (e = cudaStreamWaitEvent(h->stream, ec[k & 1], 0)) != cudaSuccess) break;
      if ((st = wallace_fill(h, d[k & 1], ck))) break;
      if ((e = cudaEventRecord(ef[k & 1], h->stream)) != cudaSuccess) break;
      if ((e = cudaStreamWaitEvent(cs, ef[k & 1], 0)) != cudaSuccess) break;
      if ((e = cudaMemcpyAsync(hb[k & 1], d[k & 1], h->n_pools * ck * h->esize, cudaMemcpyDeviceToHost, cs)) !=
          cudaSuccess)
        break;
      if ((e = cudaEventRecord(ec[k & 1], cs)) != cudaSuccess) break;
    }
    if (k >= 1) {
      // write chunk k-1 while chunk k is generated and copied
      const uint64_t j = k - 1, cj = std::min<uint64_t>(c, count - j * c);
      if ((e = cudaEventSynchronize(ec[j & 1])) != cudaSuccess) break;
      if (!write_chunk(fd, format, static_cast<const unsigned char*>(hb[j & 1]), h->esize, h->n_pools, cj,
                       count, j * c, positional, base, threads))
        st = fail(WALLACE_ERR_INVALID_PARAM, "write_stream: write failed (errno %d)", errno);
    }
  }
  if (!st && e != cudaSuccess) st = fail(WALLACE_ERR_CUDA, "write_stream: %s", cudaGetErrorString(e));
  if (!st && positional)  // leave the file position after the written block
    ::lseek(fd, base + static_cast<off_t>(h->n_pools * count * (format == WALLACE_FMT_F32LE ? 4 : 8)), SEEK_SET);
  cudaStreamSynchronize(h->stream);
  cudaStreamSynchronize(cs);
  if (!st) st = take_err(h, true);
  return st;
}

wallace_status wallace_fill_host(wallace_handle* h, void* host_out, uint64_t count) {
  if (!h) return fail(WALLACE_ERR_INVALID_PARAM, "handle must not be NULL");
  if (count < 1) return fail(WALLACE_ERR_INVALID_PARAM, "fill: count must be >= 1");
  if (!host_out) return fail(WALLACE_ERR_INVALID_PARAM, "fill: output must not be NULL");
  wallace_status st0 = take_err(h, false);
  if (st0) return st0;
  // Stage the whole pool-major block on the device when it fits (HBM is
  // large): one fill and one contiguous device->host copy run at the link's
  // bandwidth.  Otherwise chunk along the per-pool count (strided copies).
  // Free memory is queried only when the staging buffer must grow; the
  // stage then takes at most half of it (at least 64 MiB, at most 48 GiB).
  const uint64_t row_bytes = h->n_pools * h->esize;
  uint64_t chunk = std::max<uint64_t>(1, h->stage_bytes / row_bytes);
  if (chunk < count) {
    size_t free_b = 0, total_b = 0;
    if (cudaMemGetInfo(&free_b, &total_b) != cudaSuccess) {
      (void)cudaGetLastError();
      free_b = 0;
    }
    const uint64_t max_stage =
        std::max<uint64_t>(64ull << 20, std::min<uint64_t>(48ull << 30, (free_b + h->stage_bytes) / 2));
    chunk = std::max<uint64_t>(chunk, std::max<uint64_t>(1, max_stage / row_bytes));
  }
  chunk = std::min(chunk, count);
  const uint64_t need = chunk * row_bytes;
  if (h->stage_bytes < need) {
    cudaFree(h->d_stage);
    h->d_stage = nullptr;
    h->stage_bytes = 0;
    WB_CUDA(cudaMalloc(&h->d_stage, need));
    h->stage_bytes = need;
  }
  for (uint64_t off = 0; off < count; off += chunk) {
    const uint64_t c = std::min(chunk, count - off);
    if (c == count) {
      // one staged block: each launch's values leave as soon as the launch
      // is done, in pieces of at most 256 MiB alternating over two copy
      // streams (two streams: 55 GB/s vs 50.5 GB/s for one 16 GiB copy on
      // this link), while later launches run
      const uint64_t piece = 256ull << 20, esz = h->esize;
      if (!h->ws_stream) WB_CUDA(cudaStreamCreateWithFlags(&h->ws_stream, cudaStreamNonBlocking));
      if (!h->cp_stream) WB_CUDA(cudaStreamCreateWithFlags(&h->cp_stream, cudaStreamNonBlocking));
      if (!h->ws_ef[0]) WB_CUDA(cudaEventCreateWithFlags(&h->ws_ef[0], cudaEventDisableTiming));
      if (!h->ws_ec[0]) WB_CUDA(cudaEventCreateWithFlags(&h->ws_ec[0], cudaEventDisableTiming));
      if (!h->ev_cp) WB_CUDA(cudaEventCreateWithFlags(&h->ev_cp, cudaEventDisableTiming));
      unsigned char* const hb = static_cast<unsigned char*>(host_out);
      const unsigned char* const db = static_cast<const unsigned char*>(h->d_stage);
      const uint64_t n1 = h->N - 1;
      uint64_t k = 0;
      h->after_launch = [&](const wb::FillArgs& a) -> cudaError_t {
        const uint64_t vals = a.lead + (a.n_emit > 0 ? (a.n_emit - 1) * n1 + a.last_limit : 0);
        if (vals == 0) return cudaSuccess;
        cudaError_t e = cudaEventRecord(h->ws_ef[0], h->stream);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(h->ws_stream, h->ws_ef[0], 0);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(h->cp_stream, h->ws_ef[0], 0);
        if (vals == count) {  // every pool's whole row: one contiguous range
          const uint64_t total = count * row_bytes;
          for (uint64_t o = 0; o < total && e == cudaSuccess; o += piece, ++k)
            e = cudaMemcpyAsync(hb + o, db + o, std::min(piece, total - o), cudaMemcpyDeviceToHost,
                                (k & 1) ? h->ws_stream : h->cp_stream);
        } else if (e == cudaSuccess) {
          e = cudaMemcpy2DAsync(hb + a.out_offset * esz, count * esz, db + a.out_offset * esz, count * esz,
                                vals * esz, h->n_pools, cudaMemcpyDeviceToHost, (k++ & 1) ? h->ws_stream : h->cp_stream);
        }
        return e;
      };
      wallace_status st = run_emit(h, h->d_stage, c, wb::kModeFill, h->d_state, h->d_pools);
      h->after_launch = nullptr;
      if (st) return st;
      WB_CUDA(cudaEventRecord(h->ws_ec[0], h->ws_stream));
      WB_CUDA(cudaStreamWaitEvent(h->stream, h->ws_ec[0], 0));
      WB_CUDA(cudaEventRecord(h->ev_cp, h->cp_stream));
      WB_CUDA(cudaStreamWaitEvent(h->stream, h->ev_cp, 0));
      continue;
    }
    wallace_status st = run_emit(h, h->d_stage, c, wb::kModeFill, h->d_state, h->d_pools);
    if (st) return st;
    WB_CUDA(cudaMemcpy2DAsync(static_cast<unsigned char*>(host_out) + off * h->esize, count * h->esize,
                              h->d_stage, c * h->esize, c * h->esize, h->n_pools, cudaMemcpyDeviceToHost,
                              h->stream));
  }
  WB_CUDA(cudaStreamSynchronize(h->stream));
  return take_err(h, true);
}

wallace_status wallace_snapshot_ex(wallace_handle* h, int32_t slot) {
  if (!h) return fail(WALLACE_ERR_INVALID_PARAM, "handle must not be NULL");
  if (slot < 0 || slot > 1) return fail(WALLACE_ERR_INVALID_PARAM, "snapshot: slot must be 0 or 1");
  auto& sn = h->snap[slot];
  const size_t pb = h->n_pools * h->N * h->esize;
  if (!sn.pools) WB_CUDA(cudaMalloc(&sn.pools, pb));
  if (!sn.state) WB_CUDA(cudaMalloc(&sn.state, h->n_pools * sizeof(PoolState)));
  WB_CUDA(cudaMemcpyAsync(sn.pools, h->d_pools, pb, cudaMemcpyDeviceToDevice, h->stream));
  WB_CUDA(cudaMemcpyAsync(sn.state, h->d_state, h->n_pools * sizeof(PoolState), cudaMemcpyDeviceToDevice,
                          h->stream));
  sn.leftover_valid = h->d_leftover && h->cursor < h->N - 1;
  if (sn.leftover_valid) {
    const size_t lb = h->n_pools * (h->N - 1) * h->esize;
    if (!sn.leftover) WB_CUDA(cudaMalloc(&sn.leftover, lb));
    WB_CUDA(cudaMemcpyAsync(sn.leftover, h->d_leftover, lb, cudaMemcpyDeviceToDevice, h->stream));
  }
  sn.cursor = h->cursor;
  sn.pass_count = h->pass_count;
  sn.has = true;
  return WALLACE_OK;
}

wallace_status wallace_snapshot(wallace_handle* h) { return wallace_snapshot_ex(h, 0); }

// emissions per launch of wallace_fill_host_async (copy granularity)
constexpr uint32_t kPipeEmit = 256;

wallace_status wallace_fill_host_async(wallace_handle* h, void* host_out, uint64_t count) {
  if (!h) return fail(WALLACE_ERR_INVALID_PARAM, "handle must not be NULL");
  if (count < 1) return fail(WALLACE_ERR_INVALID_PARAM, "fill: count must be >= 1");
  if (!host_out) return fail(WALLACE_ERR_INVALID_PARAM, "fill: output must not be NULL");
  wallace_status st = take_err(h, false);
  if (st) return st;
  const uint64_t bytes = h->n_pools * count * h->esize;
  if (h->astage_bytes < bytes) {
    // the stream's queued work may still read the old staging buffer
    WB_CUDA(cudaStreamSynchronize(h->stream));
    cudaFree(h->d_astage);
    h->d_astage = nullptr;
    h->astage_bytes = 0;
    WB_CUDA(cudaMalloc(&h->d_astage, bytes));
    h->astage_bytes = bytes;
  }
  // launches of at most kPipeEmit emissions, each one's values copied to the
  // host on cp_stream while the next launch runs (the look-ahead of the C++
  // drop-in is one such call per block: generation and PCIe overlap)
  if (!h->cp_stream) {
    WB_CUDA(cudaStreamCreateWithFlags(&h->cp_stream, cudaStreamNonBlocking));
    WB_CUDA(cudaEventCreateWithFlags(&h->ev_cp, cudaEventDisableTiming));
  }
  const uint64_t n1 = h->N - 1, esz = h->esize;
  char* const hb = static_cast<char*>(host_out);
  char* const db = static_cast<char*>(h->d_astage);
  h->max_emit = kPipeEmit;
  h->after_launch = [&](const wb::FillArgs& a) -> cudaError_t {
    const uint64_t vals = a.lead + (a.n_emit > 0 ? (a.n_emit - 1) * n1 + a.last_limit : 0);
    if (vals == 0) return cudaSuccess;
    cudaError_t e = cudaEventRecord(h->ev_cp, h->stream);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(h->cp_stream, h->ev_cp, 0);
    if (e == cudaSuccess)
      e = cudaMemcpy2DAsync(hb + a.out_offset * esz, count * esz, db + a.out_offset * esz, count * esz, vals * esz,
                            h->n_pools, cudaMemcpyDeviceToHost, h->cp_stream);
    return e;
  };
  st = run_emit(h, h->d_astage, count, wb::kModeFill, h->d_state, h->d_pools);
  h->after_launch = nullptr;
  h->max_emit = 0;
  if (st) return st;
  // the handle's stream (what synchronising calls wait on) covers the copies
  WB_CUDA(cudaEventRecord(h->ev_cp, h->cp_stream));
  WB_CUDA(cudaStreamWaitEvent(h->stream, h->ev_cp, 0));
  return WALLACE_OK;
}

wallace_status wallace_host_alloc(uint64_t bytes, void** out) {
  if (!out) return fail(WALLACE_ERR_INVALID_PARAM, "out must not be NULL");
  *out = nullptr;
  WB_CUDA(cudaMallocHost(out, bytes));
  return WALLACE_OK;
}

void wallace_host_free(void* p) {
  if (p) cudaFreeHost(p);
}

// the live leftover / cursor / pass count of snapshot `sn` (its pools and
// state are read in place by the first launch, or copied by restore)
static wallace_status snap_prologue(wallace_handle* h, const wallace_handle::Snap& sn) {
  if (sn.leftover_valid)
    WB_CUDA(cudaMemcpyAsync(h->d_leftover, sn.leftover, h->n_pools * (h->N - 1) * h->esize,
                            cudaMemcpyDeviceToDevice, h->stream));
  h->cursor = sn.cursor;
  h->pass_count = sn.pass_count;
  return WALLACE_OK;
}

wallace_status wallace_fill_from_snapshot(wallace_handle* h, void* dev_out, uint64_t count) {
  if (!h) return fail(WALLACE_ERR_INVALID_PARAM, "handle must not be NULL");
  const auto& sn = h->snap[0];
  if (!sn.has) return fail(WALLACE_ERR_INVALID_PARAM, "no snapshot taken");
  if (count < 1) return fail(WALLACE_ERR_INVALID_PARAM, "fill: count must be >= 1");
  if (!dev_out) return fail(WALLACE_ERR_INVALID_PARAM, "fill: output must not be NULL");
  wallace_status st = take_err(h, false);
  if (!st) st = snap_prologue(h, sn);
  if (st) return st;
  return run_emit(h, dev_out, count, wb::kModeFill, sn.state, sn.pools);
}

wallace_status wallace_restore_snapshot_ex(wallace_handle* h, int32_t slot) {
  if (!h) return fail(WALLACE_ERR_INVALID_PARAM, "handle must not be NULL");
  if (slot < 0 || slot > 1) return fail(WALLACE_ERR_INVALID_PARAM, "snapshot: slot must be 0 or 1");
  const auto& sn = h->snap[slot];
  if (!sn.has) return fail(WALLACE_ERR_INVALID_PARAM, "no snapshot taken");
  WB_CUDA(cudaMemcpyAsync(h->d_pools, sn.pools, h->n_pools * h->N * h->esize, cudaMemcpyDeviceToDevice,
                          h->stream));
  WB_CUDA(cudaMemcpyAsync(h->d_state, sn.state, h->n_pools * sizeof(PoolState), cudaMemcpyDeviceToDevice,
                          h->stream));
  return snap_prologue(h, sn);
}

wallace_status wallace_restore_snapshot(wallace_handle* h) { return wallace_restore_snapshot_ex(h, 0); }

static wallace_status ensure_stage(wallace_handle* h, uint64_t bytes);

wallace_status wallace_discard(wallace_handle* h, uint64_t count) {
  if (!h) return fail(WALLACE_ERR_INVALID_PARAM, "handle must not be NULL");
  // fill(count) into the handle's staging buffer, in pieces of at most 64 MiB
  const uint64_t row = h->n_pools * h->esize;
  const uint64_t piece = std::max<uint64_t>(1, std::min<uint64_t>(count, (64ull << 20) / row));
  wallace_status st = ensure_stage(h, piece * row);
  for (uint64_t done = 0; !st && done < count; done += piece)
    st = run_emit(h, h->d_stage, std::min(piece, count - done), wb::kModeFill, h->d_state, h->d_pools);
  return st;
}

// The handle's device staging buffer, grown to at least `bytes`.
static wallace_status ensure_stage(wallace_handle* h, uint64_t bytes) {
  if (h->stage_bytes >= bytes) return WALLACE_OK;
  cudaFree(h->d_stage);
  h->d_stage = nullptr;
  h->stage_bytes = 0;
  WB_CUDA(cudaMalloc(&h->d_stage, bytes));
  h->stage_bytes = bytes;
  return WALLACE_OK;
}

wallace_status wallace_next_pool(wallace_handle* h, void* dev_values, double* reserved,
                                 double* chi2_draw) {
  if (!h) return fail(WALLACE_ERR_INVALID_PARAM, "handle must not be NULL");
  void* out = dev_values;
  if (!out) {  // values discarded: emit into the staging buffer
    const wallace_status se = ensure_stage(h, h->n_pools * (h->N - 1) * h->esize);
    if (se) return se;
    out = h->d_stage;
  }
  // refill_ + cursor_ = out_.size(): discard the partial buffer, so the
  // emission starts with no leftover (the device cursor is only read when a
  // leftover is drained)
  h->cursor = static_cast<uint32_t>(h->N - 1);
  wallace_status st = take_err(h, false);
  if (!st) st = run_emit(h, out, h->N - 1, wb::kModeFill, h->d_state, h->d_pools);
  if (!st && (reserved || chi2_draw)) {
    std::vector<PoolState> states(h->n_pools);
    cudaError_t e = cudaMemcpyAsync(states.data(), h->d_state, h->n_pools * sizeof(PoolState),
                                    cudaMemcpyDeviceToHost, h->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
    if (e != cudaSuccess) st = fail(WALLACE_ERR_CUDA, "next_pool: %s", cudaGetErrorString(e));
    if (!st) st = take_err(h, true);
    for (uint64_t p = 0; p < h->n_pools && !st; ++p) {
      if (reserved) reserved[p] = states[p].reserved_prev;
      if (chi2_draw) chi2_draw[p] = states[p].last_chi2;
    }
  } else if (!st) {
    cudaError_t e = cudaStreamSynchronize(h->stream);
    if (e != cudaSuccess) st = fail(WALLACE_ERR_CUDA, "next_pool: %s", cudaGetErrorString(e));
    if (!st) st = take_err(h, true);
  }
  return st;
}

wallace_status wallace_next_pool_host(wallace_handle* h, void* host_values, double* reserved,
                                      double* chi2_draw) {
  if (!h) return fail(WALLACE_ERR_INVALID_PARAM, "handle must not be NULL");
  const uint64_t bytes = h->n_pools * (h->N - 1) * h->esize;
  wallace_status st = ensure_stage(h, bytes);
  if (st) return st;
  st = wallace_next_pool(h, h->d_stage, reserved, chi2_draw);
  if (st) return st;
  if (host_values) {
    WB_CUDA(cudaMemcpyAsync(host_values, h->d_stage, bytes, cudaMemcpyDeviceToHost, h->stream));
    WB_CUDA(cudaStreamSynchronize(h->stream));
  }
  return WALLACE_OK;
}

wallace_status wallace_step_pass(wallace_handle* h, uint64_t n_passes) {
  if (!h) return fail(WALLACE_ERR_INVALID_PARAM, "handle must not be NULL");
  wallace_status st = materialize(h);
  if (st) return st;
  return run_passes(h, n_passes);
}

// ---- pass structure: pass_coefficient, run_pass (generator.cpp) -------------
namespace {

// transforms.cpp:24-35: element k of the p-th permutation of {0,1,2,3} in
// lexicographic order
int perm_elem(int p, int k) {
  int avail[4] = {0, 1, 2, 3}, n = 4;
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

// generator.cpp:36-50 mix_index
uint64_t mix_index(const wallace_config& c, int sweep, uint64_t offset, uint64_t j) {
  const uint64_t n = c.pool_size;
  if (c.mixing == 0) {
    const uint64_t rows = n / 4;
    return (j % 4) * rows + (default_stride(rows) * (j / 4) + offset) % rows;
  }
  uint64_t al = 0, be = 0;
  default_multipliers(n, al, be);
  const uint64_t mult = sweep == 0 ? al : be;
  return (mult % n * j + offset) % n;
}

// generator.cpp:174-217 sweep_row: the two nonzero entries of a half-sweep row
void sweep_row(const wallace_config& c, const wallace_pass_plan& plan, int sweep, uint64_t w, uint64_t col[2],
               double coef[2]) {
  const uint64_t n = c.pool_size;
  double rc = 0.0, rs = 0.0;
  rotation_from_t(rotation_t(plan.t_index[sweep]), rc, rs);
  const double g = plan.negate[sweep] ? -1.0 : 1.0;
  const double ce = g * rc, se = g * rs;
  const uint64_t off = plan.offset[sweep];
  uint64_t p1, p2;
  bool is_first;
  if (sweep == 0) {
    p1 = w & ~uint64_t{1};
    p2 = p1 + 1;
    is_first = w == p1;
  } else if (w == 0) {
    p1 = n - 1;
    p2 = 0;
    is_first = false;
  } else if (w % 2 == 1) {
    p1 = w;
    p2 = (w + 1) % n;
    is_first = true;
  } else {
    p1 = w - 1;
    p2 = w;
    is_first = false;
  }
  col[0] = mix_index(c, sweep, off, p1);
  col[1] = mix_index(c, sweep, off, p2);
  coef[0] = is_first ? ce : -se;
  coef[1] = is_first ? se : ce;
}

// plan words of the HBM-resident pass kernels (wallace_large.cu)
std::vector<uint32_t> large_plan_words(const wallace_config& c, const wallace_pass_plan& plan) {
  if (c.transform_family == 0)
    return {static_cast<uint32_t>(plan.offset[0]), static_cast<uint32_t>(plan.wallace_variant)};
  return {static_cast<uint32_t>(plan.offset[0]), static_cast<uint32_t>(plan.offset[1]),
          static_cast<uint32_t>((plan.t_index[0] & 15) | (plan.negate[0] & 1) << 4 | (plan.t_index[1] & 15) << 8 |
                                (plan.negate[1] & 1) << 12)};
}

wb::FillArgs single_pass_args(const wallace_config& c, const uint32_t* d_plans) {
  wb::FillArgs a{};
  const uint64_t n = c.pool_size, rows = n / 4;
  uint64_t al = 0, be = 0;
  default_multipliers(n, al, be);
  a.plans = d_plans;
  a.plan_stride = 0;  // one plan for every pool of the batch
  a.pass_type = 2 * c.transform_family + c.mixing;
  rotation_table(a.rot_c, a.rot_s);
  a.lg_stride = default_stride(rows) % rows;
  a.lg_alpha = al;
  a.lg_beta = be;
  a.lg_log2n = ilog2(n);
  return a;
}

}  // namespace

void wallace_default_multipliers(uint64_t n, uint64_t* alpha, uint64_t* beta) {
  uint64_t a = 0, b = 0;
  default_multipliers(n, a, b);
  if (alpha) *alpha = a;
  if (beta) *beta = b;
}

wallace_status wallace_pass_coefficient(const wallace_config* cfg, const wallace_pass_plan* plan, uint64_t out_i,
                                        uint64_t in_j, double* out) {
  wallace_status st = validate(cfg);
  if (st) return st;
  if (!plan || !out) return fail(WALLACE_ERR_INVALID_PARAM, "plan/out must not be NULL");
  const uint64_t n = cfg->pool_size;
  if (out_i >= n || in_j >= n) return fail(WALLACE_ERR_INVALID_PARAM, "pass_coefficient: index out of range");
  if (cfg->transform_family == 0) {
    // generator.cpp:273-284: entries[k][col] = row_sign[k] * 0.5 * A1[src[k]][col]
    // (A1's signs are the butterfly's: z0 = v0+v1-v2+v3, z1 = v0-v1+v2+v3,
    // z2 = v0-v1-v2-v3, z3 = -v0-v1-v2+v3)
    static const int a1[4][4] = {{1, 1, -1, 1}, {1, -1, 1, 1}, {1, -1, -1, -1}, {-1, -1, -1, 1}};
    const int variant = plan->wallace_variant;
    const uint64_t b = out_i / 4;
    const int k = static_cast<int>(out_i % 4);
    const double row_sign = ((variant & 15) >> k) & 1 ? -1.0 : 1.0;
    const int src = perm_elem(variant >> 4, k);
    *out = 0.0;
    for (int col = 0; col < 4; ++col)
      if (mix_index(*cfg, 0, plan->offset[0], 4 * b + col) == in_j) {
        *out = row_sign * 0.5 * a1[src][col];
        break;
      }
    return WALLACE_OK;
  }
  double total = 0.0;
  uint64_t mid[2], col[2];
  double c2[2], c1[2];
  sweep_row(*cfg, *plan, 1, out_i, mid, c2);
  for (int u = 0; u < 2; ++u) {
    sweep_row(*cfg, *plan, 0, mid[u], col, c1);
    for (int v = 0; v < 2; ++v)
      if (col[v] == in_j) total += c2[u] * c1[v];
  }
  *out = total;
  return WALLACE_OK;
}

wallace_status wallace_run_pass(const wallace_config* cfg, const wallace_pass_plan* plan, const double* in,
                                double* out) {
  wallace_status st = validate(cfg);
  if (st) return st;
  if (!plan || !in || !out) return fail(WALLACE_ERR_INVALID_PARAM, "run_pass: buffers must match pool_size");
  const uint64_t n = cfg->pool_size;
  const std::vector<uint32_t> words = large_plan_words(*cfg, *plan);
  double *A = nullptr, *B = nullptr;
  uint32_t* P = nullptr;
  cudaError_t e = cudaMalloc(&A, n * 8);
  if (e == cudaSuccess) e = cudaMalloc(&B, n * 8);
  if (e == cudaSuccess) e = cudaMalloc(&P, words.size() * 4);
  if (e == cudaSuccess) e = cudaMemcpy(P, words.data(), words.size() * 4, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(A, in, n * 8, cudaMemcpyHostToDevice);
  int in_b = 0;
  if (e == cudaSuccess) e = wb::launch_single_pass(1, single_pass_args(*cfg, P), A, B, 1, nullptr, &in_b);
  ++g_launches;
  if (e == cudaSuccess) e = cudaMemcpy(out, in_b ? B : A, n * 8, cudaMemcpyDeviceToHost);
  cudaFree(A);
  cudaFree(B);
  cudaFree(P);
  if (e != cudaSuccess) return fail(WALLACE_ERR_CUDA, "run_pass: %s", cudaGetErrorString(e));
  return WALLACE_OK;
}

wallace_status wallace_cross_pool_fixed(const wallace_config* cfg, uint64_t pairs, uint32_t n_probes,
                                        const uint64_t* out_i, const uint64_t* in_j, double* acc) {
  wallace_status st = validate(cfg);
  if (st) return st;
  if (!out_i || !in_j || !acc || n_probes < 1)
    return fail(WALLACE_ERR_INVALID_PARAM, "cross_pool_fixed: probes/acc must not be NULL");
  const uint64_t n = cfg->pool_size;
  for (uint32_t k = 0; k < n_probes; ++k)
    if (out_i[k] >= n || in_j[k] >= n)
      return fail(WALLACE_ERR_INVALID_PARAM, "cross_pool_correlation: probe index out of range");
  // stats.cpp:284-299: fresh Polar pools from one BaselineState(seed), one
  // pinned pass (PassPlan{}) each; the passes run on the device in batches,
  // the ProbeAccumulator sums are formed in pair order
  const wallace_pass_plan plan{};
  const std::vector<uint32_t> words = large_plan_words(*cfg, plan);
  const uint64_t batch = std::max<uint64_t>(1, std::min<uint64_t>(pairs, (uint64_t(1) << 24) / n));
  std::vector<double> x(batch * n), y(batch * n);
  double *A = nullptr, *B = nullptr;
  uint32_t* P = nullptr;
  cudaError_t e = cudaMalloc(&A, batch * n * 8);
  if (e == cudaSuccess) e = cudaMalloc(&B, batch * n * 8);
  if (e == cudaSuccess) e = cudaMalloc(&P, words.size() * 4);
  if (e == cudaSuccess) e = cudaMemcpy(P, words.data(), words.size() * 4, cudaMemcpyHostToDevice);
  for (uint32_t k = 0; k < n_probes; ++k)
    for (int q = 0; q < 6; ++q) acc[k * 6 + q] = 0.0;
  Polar src(cfg->seed);
  const wb::FillArgs a = single_pass_args(*cfg, P);
  for (uint64_t p0 = 0; p0 < pairs && e == cudaSuccess; p0 += batch) {
    const uint64_t m = std::min(batch, pairs - p0);
    for (uint64_t i = 0; i < m * n; ++i) x[i] = src.next();
    e = cudaMemcpy(A, x.data(), m * n * 8, cudaMemcpyHostToDevice);
    int in_b = 0;
    if (e == cudaSuccess) e = wb::launch_single_pass(1, a, A, B, m, nullptr, &in_b);
    ++g_launches;
    if (e == cudaSuccess) e = cudaMemcpy(y.data(), in_b ? B : A, m * n * 8, cudaMemcpyDeviceToHost);
    for (uint64_t q = 0; q < m && e == cudaSuccess; ++q)
      for (uint32_t k = 0; k < n_probes; ++k) {
        const double xv = x[q * n + in_j[k]], yv = y[q * n + out_i[k]];
        double* r = acc + k * 6;
        r[0] += xv;
        r[1] += xv * xv;
        r[2] += yv;
        r[3] += yv * yv;
        const double w = xv * yv;
        r[4] += w;
        r[5] += w * w;
      }
  }
  cudaFree(A);
  cudaFree(B);
  cudaFree(P);
  if (e != cudaSuccess) return fail(WALLACE_ERR_CUDA, "cross_pool_fixed: %s", cudaGetErrorString(e));
  return WALLACE_OK;
}

wallace_status wallace_cross_pool_probes(wallace_handle* h, uint64_t passes, uint32_t n_probes,
                                         const uint64_t* out_i, const uint64_t* in_j, double* acc) {
  if (!h || !out_i || !in_j || !acc) return fail(WALLACE_ERR_INVALID_PARAM, "handle/probes/acc must not be NULL");
  if (n_probes < 1 || n_probes > 32) return fail(WALLACE_ERR_INVALID_PARAM, "cross_pool_probes: 1..32 probes");
  if (passes < 1) return fail(WALLACE_ERR_INVALID_PARAM, "cross_pool_probes: passes must be >= 1");
  for (uint32_t k = 0; k < n_probes; ++k)
    if (out_i[k] >= h->N || in_j[k] >= h->N)
      return fail(WALLACE_ERR_INVALID_PARAM, "cross_pool_correlation: probe index out of range");
  wallace_status st = materialize(h);
  if (st) return st;
  const size_t bytes = h->n_pools * n_probes * 6 * sizeof(double);
  WB_CUDA(cudaMalloc(&h->d_probe_acc, bytes));
  cudaError_t e = cudaMemsetAsync(h->d_probe_acc, 0, bytes, h->stream);
  if (e == cudaSuccess) {
    h->n_probes = n_probes;
    for (uint32_t k = 0; k < n_probes; ++k) {
      h->probe_out[k] = static_cast<uint32_t>(out_i[k]);
      h->probe_in[k] = static_cast<uint32_t>(in_j[k]);
    }
    st = run_passes(h, passes);
    h->n_probes = 0;
    if (!st) e = cudaMemcpyAsync(acc, h->d_probe_acc, bytes, cudaMemcpyDeviceToHost, h->stream);
    if (!st && e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
  }
  cudaFree(h->d_probe_acc);
  h->d_probe_acc = nullptr;
  if (st) return st;
  if (e != cudaSuccess) return fail(WALLACE_ERR_CUDA, "cross_pool_probes: %s", cudaGetErrorString(e));
  return WALLACE_OK;
}

wallace_status wallace_pool_defect_stats(wallace_handle* h, uint64_t emissions, double threshold,
                                         double* totals, uint8_t* marks) {
  if (!h || !totals || !marks) return fail(WALLACE_ERR_INVALID_PARAM, "handle/totals/marks must not be NULL");
  if (emissions < 1) return fail(WALLACE_ERR_INVALID_PARAM, "pool_defect_stats: emissions must be >= 1");
  if (!(h->cfg.out_mean == 0.0) || !(h->cfg.out_sigma == 1.0))
    return fail(WALLACE_ERR_INVALID_PARAM,
                "pool_defect_stats: the handle's config must be standardized (out_mean 0, out_sigma 1)");
  const size_t n = h->n_pools * emissions;
  WB_CUDA(cudaMalloc(&h->d_def_totals, n * sizeof(double)));
  cudaError_t e = cudaMalloc(&h->d_def_marks, n);
  wallace_status st = WALLACE_OK;
  if (e == cudaSuccess) {
    h->def_stride = emissions;
    h->def_threshold = threshold;
    // next_pool: refill_ + cursor_ = out_.size() -- the partial buffer is
    // discarded and every step is one whole emission (generator.cpp:401-405)
    h->cursor = static_cast<uint32_t>(h->N - 1);
    st = run_emit(h, nullptr, emissions * (h->N - 1), wb::kModeDefect, h->d_state, h->d_pools);
    if (!st) e = cudaMemcpyAsync(totals, h->d_def_totals, n * sizeof(double), cudaMemcpyDeviceToHost, h->stream);
    if (!st && e == cudaSuccess) e = cudaMemcpyAsync(marks, h->d_def_marks, n, cudaMemcpyDeviceToHost, h->stream);
    if (!st && e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
    if (!st && e == cudaSuccess) st = take_err(h, true);
  }
  cudaFree(h->d_def_totals);
  cudaFree(h->d_def_marks);
  h->d_def_totals = nullptr;
  h->d_def_marks = nullptr;
  if (st) return st;
  if (e != cudaSuccess) return fail(WALLACE_ERR_CUDA, "pool_defect_stats: %s", cudaGetErrorString(e));
  return WALLACE_OK;
}

wallace_status wallace_inject_pool(wallace_handle* h, uint64_t pool, const double* values,
                                   uint64_t n) {
  if (!h) return fail(WALLACE_ERR_INVALID_PARAM, "handle must not be NULL");
  if (n != h->N) return fail(WALLACE_ERR_INVALID_PARAM, "inject_pool: size must equal pool_size");
  if (pool >= h->n_pools) return fail(WALLACE_ERR_INVALID_PARAM, "inject_pool: pool out of range");
  if (!values) return fail(WALLACE_ERR_INVALID_PARAM, "inject_pool: values must not be NULL");
  wallace_status st = materialize(h);
  if (st) return st;
  double ss;
  std::vector<unsigned char> buf(h->N * h->esize);
  if (h->dtype == WALLACE_F32) {
    float* f = reinterpret_cast<float*>(buf.data());
    for (uint64_t i = 0; i < n; ++i) f[i] = static_cast<float>(values[i]);
    ss = neumaier_sq(f, n);
  } else {
    std::memcpy(buf.data(), values, n * sizeof(double));
    ss = neumaier_sq(values, n);
  }
  // a non-finite pool makes the emission scale NaN instead of exactly 1:
  // no bulk emissions for this handle from now on
  if (!std::isfinite(ss)) h->bulk_ok = false;
  WB_CUDA(cudaMemcpyAsync(static_cast<unsigned char*>(h->d_pools) + pool * h->N * h->esize,
                          buf.data(), buf.size(), cudaMemcpyHostToDevice, h->stream));
  WB_CUDA(cudaMemcpyAsync(&h->d_state[pool].sum_sq, &ss, sizeof(double), cudaMemcpyHostToDevice,
                          h->stream));
  WB_CUDA(cudaStreamSynchronize(h->stream));
  return WALLACE_OK;
}

wallace_status wallace_get_pool(wallace_handle* h, uint64_t pool, double* raw_out, uint64_t n) {
  if (!h) return fail(WALLACE_ERR_INVALID_PARAM, "handle must not be NULL");
  if (pool >= h->n_pools) return fail(WALLACE_ERR_INVALID_PARAM, "get_pool: pool out of range");
  if (n != h->N || !raw_out) return fail(WALLACE_ERR_INVALID_PARAM, "get_pool: need pool_size values");
  std::vector<unsigned char> buf(h->N * h->esize);
  WB_CUDA(cudaMemcpyAsync(buf.data(), static_cast<unsigned char*>(h->d_pools) + pool * h->N * h->esize,
                          buf.size(), cudaMemcpyDeviceToHost, h->stream));
  WB_CUDA(cudaStreamSynchronize(h->stream));
  for (uint64_t i = 0; i < n; ++i)
    raw_out[i] = h->dtype == WALLACE_F32 ? static_cast<double>(reinterpret_cast<float*>(buf.data())[i])
                                         : reinterpret_cast<double*>(buf.data())[i];
  return WALLACE_OK;
}

wallace_status wallace_get_pool_info(wallace_handle* h, uint64_t pool, wallace_pool_info* out) {
  if (!h || !out) return fail(WALLACE_ERR_INVALID_PARAM, "handle/out must not be NULL");
  if (pool >= h->n_pools) return fail(WALLACE_ERR_INVALID_PARAM, "get_pool_info: pool out of range");
  // (an accessor: never reports chi2_sample's error, as Generator's
  // accessors never throw, generator.hpp:122-126)
  PoolState ps;
  WB_CUDA(cudaMemcpyAsync(&ps, h->d_state + pool, sizeof(ps), cudaMemcpyDeviceToHost, h->stream));
  WB_CUDA(cudaStreamSynchronize(h->stream));
  out->pass_count = ps.pass_count;
  out->uniform_draws = ps.draws;
  out->chi2_clamp_count = ps.clamp_count;
  out->sum_sq = ps.sum_sq;
  out->reserved_prev = ps.reserved_prev;
  out->last_chi2 = ps.last_chi2;
  out->buffered = (h->N - 1) - ps.cursor;
  out->seed = ps.seed;
  return WALLACE_OK;
}

// FNV-1a over the config fields that shape the stream: an image saved by a
// handle of another configuration must not load (it would produce values
// matching neither config)
static uint64_t config_hash(const wallace_config& c) {
  uint64_t x = 0xcbf29ce484222325ull;
  auto mix = [&](const void* p, size_t n) {
    const unsigned char* b = static_cast<const unsigned char*>(p);
    for (size_t i = 0; i < n; ++i) x = (x ^ b[i]) * 0x100000001b3ull;
  };
  mix(&c.pool_size, sizeof c.pool_size);
  mix(&c.transform_family, sizeof c.transform_family);
  mix(&c.mixing, sizeof c.mixing);
  mix(&c.chi2_method, sizeof c.chi2_method);
  mix(&c.fixed_transform, sizeof c.fixed_transform);
  mix(&c.disable_chi2, sizeof c.disable_chi2);
  mix(&c.discard_every, sizeof c.discard_every);
  mix(&c.out_mean, sizeof c.out_mean);
  mix(&c.out_sigma, sizeof c.out_sigma);
  return x;
}

uint64_t wallace_state_bytes(const wallace_handle* h) {
  if (!h) return 0;
  return 64 + h->n_pools * h->N * h->esize + h->n_pools * sizeof(PoolState) +
         h->n_pools * (h->N - 1) * h->esize;
}

wallace_status wallace_save_state(wallace_handle* h, void* host_buf, uint64_t bytes) {
  if (!h || !host_buf) return fail(WALLACE_ERR_INVALID_PARAM, "handle/buffer must not be NULL");
  if (bytes < wallace_state_bytes(h)) return fail(WALLACE_ERR_INVALID_PARAM, "save_state: buffer too small");
  wallace_status st = materialize(h);
  if (st) return st;
  unsigned char* p = static_cast<unsigned char*>(host_buf);
  uint64_t hdr[8] = {kMagic, h->N, static_cast<uint64_t>(h->dtype), h->n_pools, h->cursor,
                     h->pass_count, h->d_leftover ? 1ull : 0ull, config_hash(h->cfg)};
  std::memcpy(p, hdr, sizeof(hdr));
  p += 64;
  const size_t pb = h->n_pools * h->N * h->esize;
  WB_CUDA(cudaMemcpyAsync(p, h->d_pools, pb, cudaMemcpyDeviceToHost, h->stream));
  p += pb;
  WB_CUDA(cudaMemcpyAsync(p, h->d_state, h->n_pools * sizeof(PoolState), cudaMemcpyDeviceToHost,
                          h->stream));
  p += h->n_pools * sizeof(PoolState);
  const size_t lb = h->n_pools * (h->N - 1) * h->esize;
  if (h->d_leftover) WB_CUDA(cudaMemcpyAsync(p, h->d_leftover, lb, cudaMemcpyDeviceToHost, h->stream));
  else std::memset(p, 0, lb);
  WB_CUDA(cudaStreamSynchronize(h->stream));
  return WALLACE_OK;
}

wallace_status wallace_load_state(wallace_handle* h, const void* host_buf, uint64_t bytes) {
  if (!h || !host_buf) return fail(WALLACE_ERR_INVALID_PARAM, "handle/buffer must not be NULL");
  if (bytes < wallace_state_bytes(h)) return fail(WALLACE_ERR_INVALID_PARAM, "load_state: buffer too small");
  const unsigned char* p = static_cast<const unsigned char*>(host_buf);
  uint64_t hdr[8];
  std::memcpy(hdr, p, sizeof(hdr));
  if (hdr[0] != kMagic || hdr[1] != h->N || hdr[2] != static_cast<uint64_t>(h->dtype) ||
      hdr[3] != h->n_pools)
    return fail(WALLACE_ERR_INVALID_PARAM, "load_state: image does not match this handle");
  if (hdr[7] != config_hash(h->cfg))
    return fail(WALLACE_ERR_INVALID_PARAM, "load_state: image was saved with another configuration");
  if (hdr[4] > h->N - 1) return fail(WALLACE_ERR_INVALID_PARAM, "load_state: corrupt image (cursor)");
  p += 64;
  const size_t pb = h->n_pools * h->N * h->esize;
  h->bulk_ok = h->bulk_cfg_ok;  // re-derived from the image's pools
  if (h->bulk_ok) {  // see wallace_inject_pool: bulk emissions need finite pools
    const uint64_t cnt = h->n_pools * h->N;
    bool finite = true;
    if (h->dtype == WALLACE_F32) {
      for (uint64_t i = 0; i < cnt && finite; ++i) {
        float v;
        std::memcpy(&v, p + i * 4, 4);
        finite = std::isfinite(v);
      }
    } else {
      for (uint64_t i = 0; i < cnt && finite; ++i) {
        double v;
        std::memcpy(&v, p + i * 8, 8);
        finite = std::isfinite(v);
      }
    }
    if (!finite) h->bulk_ok = false;
  }
  WB_CUDA(cudaMemcpyAsync(h->d_pools, p, pb, cudaMemcpyHostToDevice, h->stream));
  p += pb;
  WB_CUDA(cudaMemcpyAsync(h->d_state, p, h->n_pools * sizeof(PoolState), cudaMemcpyHostToDevice,
                          h->stream));
  p += h->n_pools * sizeof(PoolState);
  if (hdr[6]) {
    wallace_status st = ensure_leftover(h);
    if (st) return st;
    WB_CUDA(cudaMemcpyAsync(h->d_leftover, p, h->n_pools * (h->N - 1) * h->esize,
                            cudaMemcpyHostToDevice, h->stream));
  }
  h->cursor = static_cast<uint32_t>(hdr[4]);
  h->pass_count = hdr[5];
  WB_CUDA(cudaStreamSynchronize(h->stream));
  return WALLACE_OK;
}

static wallace_status finish_consumer(cudaStream_t stream, const double* part_sums,
                                      const uint32_t* part_hist, uint64_t n_parts, double sums[4],
                                      uint64_t hist[258], ReduceScratch& r) {
  const uint64_t chunk = 256;
  const uint64_t blocks = (n_parts + chunk - 1) / chunk;
  if (r.cap < blocks) {  // grown once; a cudaMalloc/cudaFree per call would synchronise the device
    r.release();
    const size_t bytes = blocks * (4 + 258) * 8;
    WB_CUDA(cudaMalloc(&r.d_buf, bytes));
    WB_CUDA(cudaMallocHost(&r.h_buf, bytes));
    r.cap = blocks;
  }
  double* d_bs = static_cast<double*>(r.d_buf);
  unsigned long long* d_bh = reinterpret_cast<unsigned long long*>(d_bs + blocks * 4);
  cudaError_t e = wb::launch_reduce_consumer(part_sums, part_hist, n_parts, chunk, d_bs, d_bh, stream);
  ++g_launches;
  // one copy of the block sums and counts into pinned memory
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(r.h_buf, r.d_buf, blocks * (4 + 258) * 8, cudaMemcpyDeviceToHost, stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
  if (e != cudaSuccess) return fail(WALLACE_ERR_CUDA, "consumer reduction: %s", cudaGetErrorString(e));
  const double* bs = static_cast<const double*>(r.h_buf);
  const unsigned long long* bh = reinterpret_cast<const unsigned long long*>(bs + blocks * 4);
  for (int k = 0; k < 4; ++k) sums[k] = 0.0;
  for (int b = 0; b < 258; ++b) hist[b] = 0;
  for (uint64_t i = 0; i < blocks; ++i) {
    for (int k = 0; k < 4; ++k) sums[k] += bs[i * 4 + k];
    for (int b = 0; b < 258; ++b) hist[b] += bh[i * 258 + b];
  }
  return WALLACE_OK;
}

static wallace_status consume_impl(wallace_handle* h, uint64_t count, double sums[4],
                                   uint64_t hist[258], bool from_snapshot) {
  if (!h || !sums || !hist) return fail(WALLACE_ERR_INVALID_PARAM, "handle/sums/hist must not be NULL");
  if (from_snapshot && !h->snap[0].has) return fail(WALLACE_ERR_INVALID_PARAM, "no snapshot taken");
  if (count < 1) return fail(WALLACE_ERR_INVALID_PARAM, "fill: count must be >= 1");
  if (h->part_cap < h->n_pools) {
    cudaFree(h->d_part_sums);
    cudaFree(h->d_part_hist);
    h->d_part_sums = nullptr;
    h->d_part_hist = nullptr;
    WB_CUDA(cudaMalloc(&h->d_part_sums, h->n_pools * 4 * sizeof(double)));
    WB_CUDA(cudaMalloc(&h->d_part_hist, h->n_pools * 258 * sizeof(uint32_t)));
    h->part_cap = h->n_pools;
  }
  // one launch group per consume: every launch of run_emit overwrites the
  // partials, so split the count so that a single launch covers it, or fold
  // per launch.
  double tot[4] = {0, 0, 0, 0};
  uint64_t th[258] = {0};
  const uint64_t n1 = h->N - 1;
  const uint64_t d = h->cfg.discard_every;
  const uint64_t per_launch_emit = std::max<uint64_t>(1, h->plan_cap / std::max<uint64_t>(1, d));
  uint64_t done = 0;
  if (from_snapshot) {
    const wallace_status sp = snap_prologue(h, h->snap[0]);
    if (sp) return sp;
  }
  bool first = true;
  while (done < count) {
    // values a single launch produces: the lead plus per_launch_emit emissions
    const uint64_t lead = (h->cursor < n1) ? (n1 - h->cursor) : 0;
    // one launch per run_emit (the partials are per launch): an emission
    // longer than a launch drains a pending lead in a call of its own
    const uint64_t cap = (d > h->plan_cap && lead > 0) ? lead : lead + per_launch_emit * n1;
    const uint64_t c = std::min(cap, count - done);
    const bool snap = from_snapshot && first;
    wallace_status st = run_emit(h, nullptr, c, wb::kModeConsume, snap ? h->snap[0].state : h->d_state,
                                 snap ? h->snap[0].pools : h->d_pools);
    if (st) return st;
    first = false;
    double s4[4];
    uint64_t h258[258];
    st = finish_consumer(h->stream, h->d_part_sums, h->d_part_hist, h->n_pools, s4, h258, h->red);
    if (!st) st = take_err(h, true);
    if (st) return st;
    for (int k = 0; k < 4; ++k) tot[k] += s4[k];
    for (int b = 0; b < 258; ++b) th[b] += h258[b];
    done += c;
  }
  for (int k = 0; k < 4; ++k) sums[k] = tot[k];
  for (int b = 0; b < 258; ++b) hist[b] = th[b];
  return WALLACE_OK;
}

wallace_status wallace_consume(wallace_handle* h, uint64_t count, double sums[4], uint64_t hist[258]) {
  return consume_impl(h, count, sums, hist, false);
}

wallace_status wallace_consume_from_snapshot(wallace_handle* h, uint64_t count, double sums[4],
                                             uint64_t hist[258]) {
  return consume_impl(h, count, sums, hist, true);
}

wallace_status wallace_baseline_consume(int32_t method, const uint64_t* seeds, uint64_t seed_base,
                                        uint64_t n_streams, uint64_t count, void* stream, double sums[4],
                                        uint64_t hist[258], double* device_ms) {
  if (!sums || !hist) return fail(WALLACE_ERR_INVALID_PARAM, "sums/hist must not be NULL");
  if (method != WALLACE_BASELINE_POLAR && method != WALLACE_BASELINE_BOXMULLER)
    return fail(WALLACE_ERR_INVALID_PARAM, "baseline: method must be polar (0) or boxmuller (1)");
  if (n_streams < 1 || count < 1) return fail(WALLACE_ERR_INVALID_PARAM, "need >= 1 stream and value");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const uint64_t blocks = (n_streams + 127) / 128;
  uint64_t* d_seeds = nullptr;
  double* d_ps = nullptr;
  uint32_t* d_ph = nullptr;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  wallace_status st = WALLACE_OK;
  cudaError_t e = cudaSuccess;
  if (seeds) {
    e = cudaMalloc(&d_seeds, n_streams * 8);
    if (e == cudaSuccess) e = cudaMemcpyAsync(d_seeds, seeds, n_streams * 8, cudaMemcpyHostToDevice, s);
  }
  if (e == cudaSuccess) e = cudaMalloc(&d_ps, blocks * 4 * sizeof(double));
  if (e == cudaSuccess) e = cudaMalloc(&d_ph, blocks * 258 * sizeof(uint32_t));
  if (e == cudaSuccess) e = cudaEventCreate(&e0);
  if (e == cudaSuccess) e = cudaEventCreate(&e1);
  if (e == cudaSuccess) e = cudaEventRecord(e0, s);
  if (e == cudaSuccess) e = wb::launch_baseline_consume(method, d_seeds, seed_base, n_streams, count, d_ps, d_ph,
                                                        blocks, s);
  if (e == cudaSuccess) {
    ++g_launches;
    e = cudaEventRecord(e1, s);
  }
  if (e != cudaSuccess) st = fail(WALLACE_ERR_CUDA, "baseline_consume: %s", cudaGetErrorString(e));
  ReduceScratch red;
  if (!st) st = finish_consumer(s, d_ps, d_ph, blocks, sums, hist, red);
  if (!st && device_ms) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    *device_ms = ms;
  }
  red.release();
  if (e0) cudaEventDestroy(e0);
  if (e1) cudaEventDestroy(e1);
  cudaFree(d_seeds);
  cudaFree(d_ps);
  cudaFree(d_ph);
  return st;
}

wallace_status wallace_boxmuller_consume(const uint64_t* seeds, uint64_t seed_base, uint64_t n_streams,
                                         uint64_t count, void* stream, double sums[4], uint64_t hist[258]) {
  return wallace_baseline_consume(WALLACE_BASELINE_BOXMULLER, seeds, seed_base, n_streams, count, stream, sums,
                                  hist, nullptr);
}

wallace_status wallace_baseline_fill(int32_t method, wallace_baseline_state* states, uint64_t n_streams,
                                     uint64_t count, double* dev_out, void* stream) {
  if (!states || !dev_out) return fail(WALLACE_ERR_INVALID_PARAM, "states/out must not be NULL");
  if (method != WALLACE_BASELINE_POLAR && method != WALLACE_BASELINE_BOXMULLER)
    return fail(WALLACE_ERR_INVALID_PARAM, "baseline: method must be polar (0) or boxmuller (1)");
  if (n_streams < 1 || count < 1) return fail(WALLACE_ERR_INVALID_PARAM, "need >= 1 stream and value");
  static_assert(sizeof(wallace_baseline_state) == 56, "wallace_baseline_state layout");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  void* d_st = nullptr;
  const size_t bytes = n_streams * sizeof(wallace_baseline_state);
  cudaError_t e = cudaMalloc(&d_st, bytes);
  if (e == cudaSuccess) e = cudaMemcpyAsync(d_st, states, bytes, cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) e = wb::launch_baseline_fill(method, d_st, n_streams, count, dev_out, s);
  if (e == cudaSuccess) {
    ++g_launches;
    e = cudaMemcpyAsync(states, d_st, bytes, cudaMemcpyDeviceToHost, s);
  }
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  cudaFree(d_st);
  if (e != cudaSuccess) return fail(WALLACE_ERR_CUDA, "baseline_fill: %s", cudaGetErrorString(e));
  return WALLACE_OK;
}

// ---- host helpers of the reference's L1a layer (baselines / chi2 / transforms)
namespace {
Uniform to_uniform(const wallace_uniform_state* u) {
  Uniform x(0);
  std::memcpy(x.s, u->s, sizeof(x.s));
  x.draws = u->draws;
  return x;
}
void from_uniform(const Uniform& x, wallace_uniform_state* u) {
  std::memcpy(u->s, x.s, sizeof(x.s));
  u->draws = x.draws;
}
constexpr double kPi = 3.141592653589793238462643383279502884;  // std::numbers::pi
}  // namespace

uint64_t wallace_splitmix64(uint64_t* state) { return splitmix64(*state); }

void wallace_uniform_seed(uint64_t seed, wallace_uniform_state* out) {
  const Uniform u(seed);
  from_uniform(u, out);
}

uint64_t wallace_uniform_bits(wallace_uniform_state* u) {
  Uniform x = to_uniform(u);
  const uint64_t w = x.bits();
  from_uniform(x, u);
  return w;
}

double wallace_uniform_next(wallace_uniform_state* u) {
  Uniform x = to_uniform(u);
  const double v = x.next();
  from_uniform(x, u);
  return v;
}

void wallace_baseline_seed(uint64_t seed, wallace_baseline_state* out) {
  std::memset(out, 0, sizeof(*out));
  wallace_uniform_seed(seed, &out->uniform);
}

double wallace_polar_next(wallace_baseline_state* st) {  // baselines.cpp:51-66
  Polar p(0);
  p.u = to_uniform(&st->uniform);
  p.has = st->has_cached != 0;
  p.cached = st->cached;
  const double v = p.next();
  from_uniform(p.u, &st->uniform);
  st->has_cached = p.has ? 1 : 0;
  st->cached = p.has ? p.cached : 0.0;
  return v;
}

wallace_status wallace_boxmuller_pair(double u1, double u2, double* z1, double* z2) {  // baselines.cpp:68-78
  if (!(u1 > 0.0) || u1 > 1.0) return fail(WALLACE_ERR_INVALID_PARAM, "boxmuller_pair: u1 must be in (0, 1]");
  if (!(u2 >= 0.0) || u2 >= 1.0) return fail(WALLACE_ERR_INVALID_PARAM, "boxmuller_pair: u2 must be in [0, 1)");
  const double r = std::sqrt(-2.0 * std::log(u1));
  const double angle = 2.0 * kPi * u2;
  if (z1) *z1 = r * std::cos(angle);
  if (z2) *z2 = r * std::sin(angle);
  return WALLACE_OK;
}

double wallace_boxmuller_next(wallace_baseline_state* st) {  // baselines.cpp:80-92
  if (st->has_cached) {
    st->has_cached = 0;
    const double v = st->cached;
    st->cached = 0.0;
    return v;
  }
  double u1 = wallace_uniform_next(&st->uniform);
  if (u1 == 0.0) u1 = 0x1.0p-53;
  const double u2 = wallace_uniform_next(&st->uniform);
  double z1 = 0.0, z2 = 0.0;
  wallace_boxmuller_pair(u1, u2, &z1, &z2);
  st->cached = z2;
  st->has_cached = 1;
  return z1;
}

wallace_status wallace_exact_chi2_oracle(uint64_t nu, wallace_baseline_state* st, double* out) {  // baselines.cpp:94-104
  if (nu < 1) return fail(WALLACE_ERR_INVALID_PARAM, "exact_chi2_oracle: nu must be >= 1");
  double sum = 0.0;
  for (uint64_t i = 0; i < nu; ++i) {
    const double z = wallace_polar_next(st);
    sum += z * z;
  }
  if (out) *out = sum;
  return WALLACE_OK;
}

wallace_status wallace_compute_a(uint64_t nu, double* a) {  // chi2.cpp:11-17
  if (nu < 1) return fail(WALLACE_ERR_INVALID_PARAM, "compute_a: nu must be >= 1");
  if (a) *a = compute_a(nu);
  return WALLACE_OK;
}

wallace_status wallace_chi2_params(uint64_t nu, double* a_value) {  // chi2.cpp:19-25 Chi2Params::for_nu
  if (nu < 8)
    return fail(WALLACE_ERR_INVALID_PARAM, "Chi2Params: nu must be >= 8, got %llu",
                static_cast<unsigned long long>(nu));
  if (a_value) *a_value = compute_a(nu);
  return WALLACE_OK;
}

wallace_status wallace_chi2_sample(double x, uint64_t nu, double a_value, int32_t method, int32_t* clamped,
                                   double* out) {  // chi2.cpp:27-59
  if (!std::isfinite(x)) return fail(WALLACE_ERR_INVALID_PARAM, "chi2_sample: x must be finite");
  if (method < 0 || method > 2) return fail(WALLACE_ERR_INVALID_PARAM, "chi2_sample: unknown method");
  const double n = static_cast<double>(nu);
  double s;
  if (method == WALLACE_CHI2_SQRT_SHIFT) {
    const double y = x + std::sqrt(2.0 * n - 1.0);
    s = 0.5 * y * y;
  } else if (method == WALLACE_CHI2_WILSON_HILFERTY) {
    const double d = 2.0 / (9.0 * n);
    const double y = std::sqrt(d) * x + (1.0 - d);
    s = n * y * y * y;
  } else {
    s = a_value * (x * x - 1.0) + std::sqrt(2.0 * (n - a_value * a_value)) * x + n;
  }
  const double floor_v = 1e-6 * n;
  const bool c = s < floor_v;
  if (clamped) *clamped = c ? 1 : 0;
  if (out) *out = c ? floor_v : s;
  return WALLACE_OK;
}

wallace_status wallace_variant(int32_t id, double entries[16], uint8_t source_row[4], double row_sign[4]) {
  // transforms.cpp:15-35, 76-97: entries[k][j] = row_sign[k] * 0.5 * A1[source_row[k]][j]
  if (id < 0 || id >= 384)
    return fail(WALLACE_ERR_INVALID_PARAM, "wallace_variant: id out of range [0, 384)");
  static const int kA1[4][4] = {{1, 1, -1, 1}, {1, -1, 1, 1}, {1, -1, -1, -1}, {-1, -1, -1, 1}};
  for (int k = 0; k < 4; ++k) {
    const int src = perm_elem(id >> 4, k);
    const double sg = ((id & 15) >> k) & 1 ? -1.0 : 1.0;
    if (source_row) source_row[k] = static_cast<uint8_t>(src);
    if (row_sign) row_sign[k] = sg;
    if (entries)
      for (int j = 0; j < 4; ++j) entries[4 * k + j] = sg * 0.5 * kA1[src][j];
  }
  return WALLACE_OK;
}

wallace_status wallace_rotation_from_t(double t, double* c, double* s) {  // transforms.cpp:52-70
  if (!std::isfinite(t)) return fail(WALLACE_ERR_INVALID_PARAM, "rotation_from_t: t must be finite");
  double cc = 0.0, ss = 0.0;
  rotation_from_t(t, cc, ss);
  if (c) *c = cc;
  if (s) *s = ss;
  return WALLACE_OK;
}

}  // extern "C"
