/*
 * TEST INFRASTRUCTURE ONLY — CPU oracle for the Wallace pool generator.
 *
 * This is a plain-C restatement of the reference's hot path
 * (/root/reference/proj/core/src/{baselines,transforms,chi2,generator}.cpp),
 * used exclusively as the checker by tests/, __graft_entry__.smoke() and the
 * cpu_baseline leg of bench.py.  The product (paper_1005_2314_b200) never
 * links, loads or calls it.
 *
 * Two instantiations share one source (oracle_gen.inc):
 *   - f64: the reference's own semantics, op for op (parity target: 0 ulp
 *          against the unmodified reference library, oracle/_ref).
 *   - f32: the documented fp32 restatement, the oracle for the
 *          fp32 configurations; the reference has no fp32 mode.
 *
 * Parity is pinned: tests/test_oracle_pin.py checks the f64 instantiation
 * bit-for-bit against oracle/_ref (built from the reference sources by
 * oracle/Makefile) and against the reference's frozen xoshiro vectors.
 */
#ifndef WALLACE_ORACLE_H
#define WALLACE_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Mirrors maxent::GeneratorConfig (generator.hpp:21-45). */
typedef struct wo_config {
  uint64_t pool_size;
  int32_t transform_family; /* 0 = wallace4, 1 = rotation */
  int32_t mixing;           /* 0 = stride_transpose, 1 = affine */
  int32_t chi2_method;      /* 0 sqrt_shift, 1 wilson_hilferty, 2 cubic_a */
  int32_t fixed_transform;  /* diag.fixed_transform */
  int32_t disable_chi2;     /* diag.disable_chi2 */
  int32_t pad_;
  uint64_t discard_every;
  double out_mean;
  double out_sigma;
  uint64_t seed;
} wo_config;

typedef struct wo_gen wo_gen;

/* splitmix64 / xoshiro256** (baselines.cpp:19-45) */
uint64_t wo_splitmix64(uint64_t* state);
void wo_uniform_seed(uint64_t seed, uint64_t s[4]);
uint64_t wo_uniform_bits(uint64_t s[4]);
double wo_uniform_next(uint64_t s[4]);

/* transforms.cpp:161-169 */
uint64_t wo_default_stride(uint64_t rows);
/* transforms.cpp:76-97: source_row[4] and row_sign[4] of a variant */
void wo_wallace_variant(int id, int source_row[4], double row_sign[4]);
/* generator.cpp:286-294; transforms.cpp:39-70 */
void wo_default_multipliers(uint64_t n, uint64_t* alpha, uint64_t* beta);
double wo_rotation_t(int k);
void wo_rotation_from_t(double t, double* c, double* s);
/* chi2.cpp:11-17, 27-59 */
double wo_compute_a(uint64_t nu);
double wo_chi2_sample(double x, uint64_t nu, double a, int method, int* clamped);

/* Generator lifecycle; dtype 0 = f32 restatement, 1 = f64 reference. */
int wo_create(const wo_config* cfg, int dtype, wo_gen** out);
void wo_destroy(wo_gen* g);
/* chi2_sample's InvalidParameterError for a non-finite reserved value
 * (chi2.cpp:29-31), raised from refill_ inside fill / next_pool */
#define WO_ERR_CHI2_NONFINITE (-20)
/* fill(count) — out is float* (f32) or double* (f64); 0 or an error code */
int wo_fill(wo_gen* g, void* out, uint64_t count);
/* next_pool(): writes pool_size-1 values to out */
int wo_next_pool(wo_gen* g, void* values, double* reserved, double* chi2_draw);
void wo_step_pass(wo_gen* g);
int wo_inject_pool(wo_gen* g, const double* values, uint64_t n);
/* raw pool (converted to double), and bookkeeping */
void wo_get_pool(const wo_gen* g, double* raw);
void wo_get_stats(const wo_gen* g, uint64_t* pass_count, uint64_t* draws,
                  uint64_t* clamp_count, double* sum_sq, double* reserved_prev,
                  uint64_t* cursor);
/* Plan words consumed so far are reconstructible; this returns the decoded
 * plan of the next pass without consuming it (test helper). */
void wo_peek_plan(const wo_gen* g, int* variant, uint64_t* offset0);

/* Polar / Box-Muller streams (baselines.cpp:51-92) */
typedef struct wo_baseline {
  uint64_t s[4];
  uint64_t draws;
  int has_cached;
  double cached;
} wo_baseline;
void wo_baseline_seed(wo_baseline* b, uint64_t seed);
double wo_polar_next(wo_baseline* b);
double wo_boxmuller_next(wo_baseline* b);

/* Welford/Pebay one-pass moments (stats.cpp:25-56) */
void wo_moments(const double* x, uint64_t n, double* mean, double* variance,
                double* skewness, double* excess_kurtosis);

/* Multi-pool job with a fused consumer (config 5 oracle): per pool p with
 * seed seeds[p], fill(count_per_pool) and accumulate sum x, x^2, x^3, x^4
 * (fp64, sequential per pool, pools summed in order) and a 256-bin
 * histogram of floor((x+8)*16) over [-8, 8) plus under/over counts. */
int wo_consume_pools(const wo_config* cfg, int dtype, const uint64_t* seeds,
                     uint64_t n_pools, uint64_t count_per_pool, int threads,
                     double sums[4], uint64_t hist[258]);

#ifdef __cplusplus
}
#endif
#endif
