/*
 * TEST INFRASTRUCTURE ONLY — CPU oracle for the Wallace pool generator.
 * See wallace_oracle.h for the contract.  Compiled with -ffp-contract=off
 * (the reference pins the same flag, /root/reference/proj/CMakeLists.txt:10-14)
 * so that every multiply-add rounds twice, as in the reference.
 */
#include "wallace_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

struct wo_gen {
  wo_config cfg;
  int dtype; /* 0 f32, 1 f64 */
  double a;  /* Chi2Params::a_value (chi2.cpp:19-25) */
  void* raw;
  void* scratch;
  void* out;
  void* tmp; /* rotation: the sweep-0 result */
  uint64_t alpha, beta; /* affine multipliers (generator.cpp:286-294) */
  double rot_c[16], rot_s[16]; /* rotation_from_t of the 16 table entries */
  uint64_t out_len;
  uint64_t cursor;
  uint64_t u[4];
  uint64_t draws;
  uint64_t pass_count;
  uint64_t clamp_count;
  double reserved_prev;
  double sum_sq;
  double last_chi2;
};

/* baselines.cpp:13-15 */
static inline uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }

/* baselines.cpp:19-24 */
uint64_t wo_splitmix64(uint64_t* state) {
  uint64_t z = (*state += 0x9e3779b97f4a7c15ULL);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

/* baselines.cpp:26-31 */
void wo_uniform_seed(uint64_t seed, uint64_t s[4]) {
  uint64_t sm = seed;
  for (int i = 0; i < 4; ++i) s[i] = wo_splitmix64(&sm);
}

/* baselines.cpp:33-45 (draw counting is done by the callers) */
uint64_t wo_uniform_bits(uint64_t s[4]) {
  const uint64_t result = rotl(s[1] * 5, 7) * 9;
  const uint64_t t = s[1] << 17;
  s[2] ^= s[0];
  s[3] ^= s[1];
  s[1] ^= s[2];
  s[0] ^= s[3];
  s[2] ^= t;
  s[3] = rotl(s[3], 45);
  return result;
}

/* baselines.cpp:47-49 */
double wo_uniform_next(uint64_t s[4]) {
  return (double)(wo_uniform_bits(s) >> 11) * 0x1.0p-53;
}

void wo_baseline_seed(wo_baseline* b, uint64_t seed) {
  wo_uniform_seed(seed, b->s);
  b->draws = 0;
  b->has_cached = 0;
  b->cached = 0.0;
}

/* baselines.cpp:51-66 */
double wo_polar_next(wo_baseline* b) {
  if (b->has_cached) {
    b->has_cached = 0;
    return b->cached;
  }
  for (;;) {
    const double u = 2.0 * wo_uniform_next(b->s) - 1.0;
    const double v = 2.0 * wo_uniform_next(b->s) - 1.0;
    b->draws += 2;
    const double s2 = u * u + v * v;
    if (s2 >= 1.0 || s2 == 0.0) continue;
    const double scale = sqrt(-2.0 * log(s2) / s2);
    b->cached = v * scale;
    b->has_cached = 1;
    return u * scale;
  }
}

/* baselines.cpp:68-92 (boxmuller_pair's argument checks cannot fire here:
 * u1 is in (0,1] after the zero remap and u2 in [0,1)). */
double wo_boxmuller_next(wo_baseline* b) {
  if (b->has_cached) {
    b->has_cached = 0;
    return b->cached;
  }
  double u1 = wo_uniform_next(b->s);
  if (u1 == 0.0) u1 = 0x1.0p-53;
  const double u2 = wo_uniform_next(b->s);
  b->draws += 2;
  const double r = sqrt(-2.0 * log(u1));
  const double angle = 2.0 * 3.141592653589793 * u2; /* std::numbers::pi */
  b->cached = r * sin(angle);
  b->has_cached = 1;
  return r * cos(angle);
}

static uint64_t gcd_u64(uint64_t a, uint64_t b) {
  while (b) {
    const uint64_t t = a % b;
    a = b;
    b = t;
  }
  return a;
}

/* transforms.cpp:161-169 */
uint64_t wo_default_stride(uint64_t rows) {
  uint64_t k = rows / 3 + 1;
  if (k % 2 == 0) ++k;
  while (gcd_u64(k, rows) != 1) k += 2;
  return k;
}

/* transforms.cpp:24-35: the 24 permutations of {0,1,2,3} in lexicographic
 * (std::next_permutation) order. */
static void perm_of_index(int idx, int out[4]) {
  int avail[4] = {0, 1, 2, 3};
  int navail = 4;
  int fact[4] = {6, 2, 1, 1};
  for (int pos = 0; pos < 4; ++pos) {
    const int q = idx / fact[pos];
    idx %= fact[pos];
    out[pos] = avail[q];
    for (int j = q; j + 1 < navail; ++j) avail[j] = avail[j + 1];
    --navail;
  }
}

/* transforms.cpp:76-97 */
void wo_wallace_variant(int id, int source_row[4], double row_sign[4]) {
  const unsigned sign_mask = (unsigned)id & 15u;
  const int perm_index = id >> 4;
  perm_of_index(perm_index, source_row);
  for (int k = 0; k < 4; ++k) row_sign[k] = ((sign_mask >> k) & 1u) ? -1.0 : 1.0;
}

/* chi2.cpp:11-17 */
double wo_compute_a(uint64_t nu) {
  const double root_nu = sqrt((double)nu);
  return 2.0 * root_nu * sin(asin(1.0 / root_nu) / 3.0);
}

/* chi2.cpp:27-59 (the non-finite-x check is the caller's) */
double wo_chi2_sample(double x, uint64_t nu_i, double a, int method, int* clamped) {
  const double nu = (double)nu_i;
  double s;
  if (method == 0) {
    const double y = x + sqrt(2.0 * nu - 1.0);
    s = 0.5 * y * y;
  } else if (method == 1) {
    const double d = 2.0 / (9.0 * nu);
    const double y = sqrt(d) * x + (1.0 - d);
    s = nu * y * y * y;
  } else {
    s = a * (x * x - 1.0) + sqrt(2.0 * (nu - a * a)) * x + nu;
  }
  const double floor_v = 1e-6 * nu;
  if (s < floor_v) {
    if (clamped) *clamped = 1;
    return floor_v;
  }
  if (clamped) *clamped = 0;
  return s;
}

/* generator.cpp:286-294 default_multipliers */
void wo_default_multipliers(uint64_t n, uint64_t* alpha, uint64_t* beta) {
  uint64_t a = (uint64_t)llround(0.382 * (double)n) | 1;
  uint64_t b = (uint64_t)llround(0.618 * (double)n) | 1;
  if (a == b) b += 2;
  *alpha = a;
  *beta = b;
}

/* transforms.cpp:39-50: half-angle tangents of 16 angles evenly spaced over
 * the window where cos and sin both lie in [0.05, 0.95] -- the midpoints of
 * 16 equal slices of [acos(0.95), asin(0.95)] (bit-identical to the
 * reference's table; pinned by tests/test_oracle_pin.py). */
double wo_rotation_t(int k) {
  const double lo = acos(0.95), hi = asin(0.95);
  return tan((lo + (k + 0.5) * (hi - lo) / 16) / 2);
}

/* transforms.cpp:52-70 rotation_from_t (t finite) */
void wo_rotation_from_t(double t, double* c, double* s) {
  if (fabs(t) <= 1.0) {
    const double den = 1.0 + t * t;
    *c = (1.0 - t * t) / den;
    *s = (2.0 * t) / den;
  } else {
    const double u = 1.0 / t;
    const double den = 1.0 + u * u;
    *c = (u * u - 1.0) / den;
    *s = (2.0 * u) / den;
  }
}

#define T double
#define SFX _f64
#include "oracle_gen.inc"
#undef T
#undef SFX
#define T float
#define SFX _f32
#include "oracle_gen.inc"
#undef T
#undef SFX

/* generator.cpp:221-236 (the caller reports which field failed). */
static int validate(const wo_config* c) {
  const uint64_t n = c->pool_size;
  if (n < 32 || (n & (n - 1)) != 0 || n > (1ULL << 31)) return -1;
  if (c->discard_every < 1) return -2;
  if (!isfinite(c->out_sigma) || c->out_sigma <= 0.0) return -3;
  if (!isfinite(c->out_mean)) return -4;
  if (c->transform_family < 0 || c->transform_family > 1 || c->mixing < 0 || c->mixing > 1) return -5;
  return 0;
}

int wo_create(const wo_config* cfg, int dtype, wo_gen** out) {
  const int v = validate(cfg);
  if (v) return v;
  wo_gen* g = (wo_gen*)calloc(1, sizeof(wo_gen));
  g->cfg = *cfg;
  g->dtype = dtype;
  g->a = wo_compute_a(cfg->pool_size);
  const size_t es = dtype ? sizeof(double) : sizeof(float);
  g->raw = malloc(cfg->pool_size * es);
  g->scratch = malloc(cfg->pool_size * es);
  g->out = malloc(cfg->pool_size * es);
  g->tmp = malloc(cfg->pool_size * es);
  wo_default_multipliers(cfg->pool_size, &g->alpha, &g->beta);
  for (int k = 0; k < 16; ++k) wo_rotation_from_t(wo_rotation_t(k), &g->rot_c[k], &g->rot_s[k]);
  g->out_len = 0;
  g->cursor = 0;
  if (dtype) init_f64(g);
  else init_f32(g);
  *out = g;
  return 0;
}

void wo_destroy(wo_gen* g) {
  if (!g) return;
  free(g->raw);
  free(g->scratch);
  free(g->out);
  free(g->tmp);
  free(g);
}

int wo_fill(wo_gen* g, void* out, uint64_t count) {
  if (count < 1) return -10;
  return g->dtype ? fill_f64(g, (double*)out, count) : fill_f32(g, (float*)out, count);
}

/* generator.cpp:401-405 */
int wo_next_pool(wo_gen* g, void* values, double* reserved, double* chi2_draw) {
  const int rc = g->dtype ? refill_f64(g) : refill_f32(g);
  if (rc) return rc;
  g->cursor = g->out_len;
  const size_t es = g->dtype ? sizeof(double) : sizeof(float);
  if (values) memcpy(values, g->out, g->out_len * es);
  if (reserved) *reserved = g->reserved_prev;
  if (chi2_draw) *chi2_draw = g->last_chi2;
  return 0;
}

void wo_step_pass(wo_gen* g) {
  if (g->dtype) step_pass_f64(g);
  else step_pass_f32(g);
}

int wo_inject_pool(wo_gen* g, const double* values, uint64_t n) {
  if (n != g->cfg.pool_size) return -10;
  if (g->dtype) inject_f64(g, values);
  else inject_f32(g, values);
  return 0;
}

void wo_get_pool(const wo_gen* g, double* raw) {
  for (uint64_t i = 0; i < g->cfg.pool_size; ++i)
    raw[i] = g->dtype ? ((const double*)g->raw)[i] : (double)((const float*)g->raw)[i];
}

void wo_get_stats(const wo_gen* g, uint64_t* pass_count, uint64_t* draws,
                  uint64_t* clamp_count, double* sum_sq, double* reserved_prev,
                  uint64_t* cursor) {
  if (pass_count) *pass_count = g->pass_count;
  if (draws) *draws = g->draws;
  if (clamp_count) *clamp_count = g->clamp_count;
  if (sum_sq) *sum_sq = g->sum_sq;
  if (reserved_prev) *reserved_prev = g->reserved_prev;
  if (cursor) *cursor = g->out_len - g->cursor;
}

void wo_peek_plan(const wo_gen* g, int* variant, uint64_t* offset0) {
  uint64_t s[4];
  memcpy(s, g->u, sizeof(s));
  const uint64_t w0 = wo_uniform_bits(s);
  const uint64_t w1 = wo_uniform_bits(s);
  *variant = (int)(w0 % 384u);
  *offset0 = w1 & (g->cfg.pool_size / 4 - 1);
}

/* stats.cpp:25-56 */
void wo_moments(const double* x, uint64_t cnt, double* mean_o, double* var_o,
                double* skew_o, double* kurt_o) {
  double mean = 0.0, m2 = 0.0, m3 = 0.0, m4 = 0.0;
  uint64_t n = 0;
  for (uint64_t i = 0; i < cnt; ++i) {
    const double n1 = (double)n;
    ++n;
    const double nn = (double)n;
    const double delta = x[i] - mean;
    const double delta_n = delta / nn;
    const double delta_n2 = delta_n * delta_n;
    const double term1 = delta * delta_n * n1;
    mean += delta_n;
    m4 += term1 * delta_n2 * (nn * nn - 3.0 * nn + 3.0) + 6.0 * delta_n2 * m2 -
          4.0 * delta_n * m3;
    m3 += term1 * delta_n * (nn - 2.0) - 3.0 * delta_n * m2;
    m2 += term1;
  }
  *mean_o = mean;
  *var_o = m2 / (double)(n - 1);
  *skew_o = 0.0;
  *kurt_o = 0.0;
  if (m2 > 0.0) {
    const double nn = (double)n;
    *skew_o = sqrt(nn) * m3 / pow(m2, 1.5);
    *kurt_o = nn * m4 / (m2 * m2) - 3.0;
  }
}

/* ---- config-5 consumer oracle (multi-threaded over pools) ---- */
typedef struct {
  const wo_config* cfg;
  int dtype;
  const uint64_t* seeds;
  uint64_t n_pools, count;
  uint64_t next;
  pthread_mutex_t mu;
  double* pool_sums; /* n_pools x 4 */
  uint64_t* pool_hist; /* n_pools x 258, too big for many pools: per thread */
  uint64_t hist_total[258];
} consume_job;

static void consume_one(consume_job* j, uint64_t p, uint64_t* hist) {
  wo_config c = *j->cfg;
  c.seed = j->seeds[p];
  wo_gen* g = NULL;
  wo_create(&c, j->dtype, &g);
  const uint64_t chunk = 65536;
  void* buf = malloc(chunk * sizeof(double));
  double s1 = 0, s2 = 0, s3 = 0, s4 = 0;
  uint64_t left = j->count;
  while (left) {
    const uint64_t take = left < chunk ? left : chunk;
    wo_fill(g, buf, take);
    for (uint64_t i = 0; i < take; ++i) {
      int bin;
      double x;
      if (j->dtype) {
        const double v = ((double*)buf)[i];
        x = v;
        const double t = (v + 8.0) * 16.0;
        bin = t < 0.0 ? -1 : (t >= 256.0 ? 256 : (int)floor(t));
      } else {
        const float v = ((float*)buf)[i];
        x = (double)v;
        const float t = (v + 8.0f) * 16.0f;
        bin = t < 0.0f ? -1 : (t >= 256.0f ? 256 : (int)floorf(t));
      }
      hist[bin + 1]++;
      const double x2 = x * x;
      s1 += x;
      s2 += x2;
      s3 += x2 * x;
      s4 += x2 * x2;
    }
    left -= take;
  }
  j->pool_sums[4 * p + 0] = s1;
  j->pool_sums[4 * p + 1] = s2;
  j->pool_sums[4 * p + 2] = s3;
  j->pool_sums[4 * p + 3] = s4;
  free(buf);
  wo_destroy(g);
}

static void* consume_worker(void* arg) {
  consume_job* j = (consume_job*)arg;
  uint64_t hist[258];
  memset(hist, 0, sizeof(hist));
  for (;;) {
    pthread_mutex_lock(&j->mu);
    const uint64_t p = j->next++;
    pthread_mutex_unlock(&j->mu);
    if (p >= j->n_pools) break;
    consume_one(j, p, hist);
  }
  pthread_mutex_lock(&j->mu);
  for (int b = 0; b < 258; ++b) j->hist_total[b] += hist[b];
  pthread_mutex_unlock(&j->mu);
  return NULL;
}

int wo_consume_pools(const wo_config* cfg, int dtype, const uint64_t* seeds,
                     uint64_t n_pools, uint64_t count_per_pool, int threads,
                     double sums[4], uint64_t hist[258]) {
  wo_config probe = *cfg;
  const int v = validate(&probe);
  if (v) return v;
  consume_job j;
  memset(&j, 0, sizeof(j));
  j.cfg = cfg;
  j.dtype = dtype;
  j.seeds = seeds;
  j.n_pools = n_pools;
  j.count = count_per_pool;
  pthread_mutex_init(&j.mu, NULL);
  j.pool_sums = (double*)calloc(n_pools * 4, sizeof(double));
  if (threads < 1) threads = 1;
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)threads);
  for (int t = 0; t < threads; ++t) pthread_create(&th[t], NULL, consume_worker, &j);
  for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
  for (int k = 0; k < 4; ++k) sums[k] = 0.0;
  for (uint64_t p = 0; p < n_pools; ++p)
    for (int k = 0; k < 4; ++k) sums[k] += j.pool_sums[4 * p + k];
  memcpy(hist, j.hist_total, sizeof(j.hist_total));
  free(j.pool_sums);
  free(th);
  pthread_mutex_destroy(&j.mu);
  return 0;
}
