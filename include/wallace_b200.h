/*
 * wallace_b200.h — C-ABI of the B200-native Wallace maximum-entropy normal
 * generator (arXiv 1005.2314, reference: maxent-rng).
 *
 * The reference has no FFI: its boundary is the C++ class maxent::Generator
 * (/root/reference/proj/core/include/maxent/generator.hpp:98-149) and the
 * free functions decode_pass_plan / run_pass (generator.hpp:57-66).  Each
 * entry point below names the reference interface it replaces.  The C++
 * drop-in (include/wallace_b200.hpp) and the Python tests bind only these
 * symbols.  No C++ exception crosses this boundary; every call returns a
 * wallace_status and wallace_last_error() holds the message (which, for
 * WALLACE_ERR_CONFIG, names the offending field exactly as ConfigError does,
 * generator.cpp:221-236).
 *
 * A handle owns a BATCH of independent pools (one reference Generator per
 * pool; "distinct instances with distinct seeds may run in parallel",
 * generator.hpp:96-97).  Pool p is seeded with seeds[p] (or cfg.seed + p).
 * Every pool of a batch advances together; slice p of every output equals
 * what the reference's Generator(seed_p) would produce for the same calls.
 * A handle is single-threaded and bound to one CUDA stream.
 */
#ifndef WALLACE_B200_H
#define WALLACE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum wallace_status {
  WALLACE_OK = 0,
  WALLACE_ERR_CONFIG = 1,        /* maxent::ConfigError (errors.hpp:18-21) */
  WALLACE_ERR_INVALID_PARAM = 2, /* maxent::InvalidParameterError (errors.hpp:12-16) */
  WALLACE_ERR_CUDA = 3,          /* device failure (no reference equivalent) */
  WALLACE_ERR_UNSUPPORTED = 4    /* valid in the reference, not built here */
} wallace_status;

typedef enum wallace_dtype { WALLACE_F32 = 0, WALLACE_F64 = 1 } wallace_dtype;

/* maxent::Chi2Method (chi2.hpp:21) — same numbering */
typedef enum wallace_chi2_method {
  WALLACE_CHI2_SQRT_SHIFT = 0,
  WALLACE_CHI2_WILSON_HILFERTY = 1,
  WALLACE_CHI2_CUBIC_A = 2
} wallace_chi2_method;

/* maxent::GeneratorConfig (generator.hpp:21-45).  transform_family: 0
 * wallace4, 1 rotation (generator.cpp:113-172); mixing: 0 stride_transpose,
 * 1 affine (generator.cpp:86-110).  All four combinations run on the B200. */
typedef struct wallace_config {
  uint64_t pool_size;       /* power of two in [32, 2^31]; on-chip limit 2^14 (f32) / 2^13 (f64) */
  int32_t transform_family; /* TransformFamily */
  int32_t mixing;           /* MixingScheme */
  int32_t chi2_method;      /* wallace_chi2_method */
  int32_t fixed_transform;  /* diag.fixed_transform */
  int32_t disable_chi2;     /* diag.disable_chi2 */
  int32_t reserved_;
  uint64_t discard_every;   /* passes per emission, >= 1 */
  double out_mean;
  double out_sigma;
  uint64_t seed;            /* seed of pool 0 when seeds == NULL */
} wallace_config;

/* Per-pool bookkeeping: Generator::pass_count/uniform_draws/chi2_clamp_count
 * (generator.hpp:124-126), NormalPool::sum_sq/reserved_prev (generator.hpp:81-87),
 * and PoolOutput::chi2_draw (generator.hpp:115-119). */
typedef struct wallace_pool_info {
  uint64_t pass_count;
  uint64_t uniform_draws;
  uint64_t chi2_clamp_count;
  double sum_sq;
  double reserved_prev;
  double last_chi2;
  uint64_t buffered; /* values of the current emission not yet returned */
  uint64_t seed;
} wallace_pool_info;

typedef struct wallace_handle wallace_handle;

/* Generator::Generator(GeneratorConfig) (generator.cpp:309-331), for
 * n_pools pools at once.  Validates (ConfigError semantics), seeds each pool
 * on the host (Polar, Neumaier normalisation — bit-exact with the reference
 * on the same libm), uploads the pools to HBM and runs the 16 warm-up passes
 * on the device.  stream: a cudaStream_t or NULL (legacy default stream). */
wallace_status wallace_create(const wallace_config* cfg, uint64_t n_pools,
                              const uint64_t* seeds, wallace_dtype dtype,
                              void* stream, wallace_handle** out);

wallace_status wallace_destroy(wallace_handle* h);

/* wallace_create with options.  WALLACE_CREATE_DEVICE_SEED runs the
 * constructor's Polar fill and normalisation (generator.cpp:309-327) on the
 * device, one CTA per pool: the xoshiro stream, the Polar acceptance
 * sequence and the draw counts are exact, but the Polar values use CUDA's
 * fp64 log, which can differ from the host glibc log by an ulp, so the
 * seeded pools are within a few ulps of wallace_create's -- a fast start for
 * large batches, NOT a parity path. */
enum { WALLACE_CREATE_DEVICE_SEED = 1 };
wallace_status wallace_create_ex(const wallace_config* cfg, uint64_t n_pools, const uint64_t* seeds,
                                 wallace_dtype dtype, void* stream, uint32_t flags, wallace_handle** out);

/* Generator::fill(std::span<double>) (generator.cpp:387-399) for every pool:
 * dev_out is a DEVICE buffer of n_pools * count_per_pool elements of the
 * handle's dtype, pool-major (pool p at [p*count, (p+1)*count)).  Exactly
 * equivalent to count_per_pool next_normal() calls per pool.  count == 0 is
 * WALLACE_ERR_INVALID_PARAM ("fill: count must be >= 1"). Asynchronous. */
wallace_status wallace_fill(wallace_handle* h, void* dev_out, uint64_t count_per_pool);

/* Same as wallace_fill but writes a HOST buffer (pinned or pageable) of the
 * same layout; device staging and device->host copies are internal.
 * Synchronous. */
wallace_status wallace_fill_host(wallace_handle* h, void* host_out, uint64_t count_per_pool);

/* Generator::next_pool() (generator.cpp:401-405): one emission per pool.
 * dev_values (optional) receives n_pools * (pool_size - 1) values, device
 * memory; reserved / chi2_draw (optional) receive n_pools doubles on the
 * host.  Discards any partially consumed emission. Synchronous. */
wallace_status wallace_next_pool(wallace_handle* h, void* dev_values, double* reserved,
                                 double* chi2_draw);

/* Same as wallace_next_pool but the values land in HOST memory
 * (n_pools * (pool_size - 1) elements of the handle's dtype). */
wallace_status wallace_next_pool_host(wallace_handle* h, void* host_values, double* reserved,
                                      double* chi2_draw);

/* Generator::step_pass() (generator.cpp:333-343), n_passes times. */
wallace_status wallace_step_pass(wallace_handle* h, uint64_t n_passes);

/* Generator::inject_pool(span) (generator.cpp:407-413) for one pool:
 * replaces the raw pool and recomputes sum_sq (not renormalised). */
wallace_status wallace_inject_pool(wallace_handle* h, uint64_t pool, const double* values,
                                   uint64_t n);

/* Generator::pool().raw (generator.hpp:123), converted to double. Synchronous. */
wallace_status wallace_get_pool(wallace_handle* h, uint64_t pool, double* raw_out, uint64_t n);

wallace_status wallace_get_pool_info(wallace_handle* h, uint64_t pool, wallace_pool_info* out);

/* Checkpoint / resume (no reference equivalent: Generator state is private,
 * SURVEY §5).  The state image is pools + per-pool state, host memory; it
 * carries a hash of the configuration and loads only into a handle of the
 * same configuration, pool size, dtype and pool count. */
uint64_t wallace_state_bytes(const wallace_handle* h);
wallace_status wallace_save_state(wallace_handle* h, void* host_buf, uint64_t bytes);
wallace_status wallace_load_state(wallace_handle* h, const void* host_buf, uint64_t bytes);

/* Device-resident snapshot: wallace_snapshot() copies the current state to a
 * device-side checkpoint; wallace_fill_from_snapshot() performs wallace_fill
 * starting from that checkpoint (the live state becomes the result), so a job
 * can be re-run without re-seeding.  Used by bench.py to time the same
 * configured job every step. */
wallace_status wallace_snapshot(wallace_handle* h);
wallace_status wallace_fill_from_snapshot(wallace_handle* h, void* dev_out,
                                          uint64_t count_per_pool);
/* The live state becomes the snapshot again (the snapshot is kept). */
wallace_status wallace_restore_snapshot(wallace_handle* h);
/* Two snapshot slots (slot 0 is the one of wallace_snapshot /
 * wallace_restore_snapshot / wallace_fill_from_snapshot). */
wallace_status wallace_snapshot_ex(wallace_handle* h, int32_t slot);
wallace_status wallace_restore_snapshot_ex(wallace_handle* h, int32_t slot);

/* wallace_fill_host without the wait: the block's generation and its copy to
 * host_out (pinned memory, see wallace_host_alloc) are queued on the
 * handle's stream; wallace_synchronize() waits for them (and reports
 * chi2_sample's error).  host_out must stay valid until then. */
wallace_status wallace_fill_host_async(wallace_handle* h, void* host_out, uint64_t count_per_pool);
/* Page-locked host memory for wallace_fill_host_async / fast host fills. */
wallace_status wallace_host_alloc(uint64_t bytes, void** out);
void wallace_host_free(void* p);
/* count_per_pool further values of every pool, generated and dropped (the
 * stream advances exactly as wallace_fill's would).  Asynchronous. */
wallace_status wallace_discard(wallace_handle* h, uint64_t count_per_pool);

/* Fused consumer (BASELINE config 5): generates count_per_pool values per
 * pool exactly as wallace_fill would, but consumes them in-kernel into
 * sums[4] = {sum x, x^2, x^3, x^4} (fp64, fixed reduction order) and
 * hist[258] = {under, 256 bins of width 1/16 over [-8,8), over}, with bin =
 * floor((x + 8) * 16) computed in the handle's dtype. Synchronous. */
wallace_status wallace_consume(wallace_handle* h, uint64_t count_per_pool, double sums[4],
                               uint64_t hist[258]);

/* wallace_consume starting from the device snapshot (see wallace_snapshot). */
wallace_status wallace_consume_from_snapshot(wallace_handle* h, uint64_t count_per_pool,
                                             double sums[4], uint64_t hist[258]);

/* ---- the reference's conventional generators (baselines.hpp:27-72) ------- */

/* maxent::UniformState (baselines.hpp:27-33) and BaselineState (:49-55). */
typedef struct wallace_uniform_state {
  uint64_t s[4];
  uint64_t draws;
} wallace_uniform_state;
typedef struct wallace_baseline_state {
  wallace_uniform_state uniform;
  int32_t has_cached; /* std::optional<double> cached */
  int32_t reserved_;
  double cached;
} wallace_baseline_state;
enum { WALLACE_BASELINE_POLAR = 0, WALLACE_BASELINE_BOXMULLER = 1 };

/* Host functions, bit-identical to the reference on the same libm:
 * splitmix64 / UniformState(seed) / uniform_bits / uniform_next
 * (baselines.cpp:19-49), polar_next (:51-66), boxmuller_pair (:68-78,
 * InvalidParameterError outside its domain), boxmuller_next (:80-92),
 * exact_chi2_oracle (:94-104). */
uint64_t wallace_splitmix64(uint64_t* state);
void wallace_uniform_seed(uint64_t seed, wallace_uniform_state* out);
uint64_t wallace_uniform_bits(wallace_uniform_state* u);
double wallace_uniform_next(wallace_uniform_state* u);
void wallace_baseline_seed(uint64_t seed, wallace_baseline_state* out);
double wallace_polar_next(wallace_baseline_state* s);
wallace_status wallace_boxmuller_pair(double u1, double u2, double* z1, double* z2);
double wallace_boxmuller_next(wallace_baseline_state* s);
wallace_status wallace_exact_chi2_oracle(uint64_t nu, wallace_baseline_state* s, double* out);

/* chi2.hpp:21-41: compute_a (nu >= 1), Chi2Params::for_nu (nu >= 8, returns
 * a_value), chi2_sample (InvalidParameterError for non-finite x; *clamped
 * set when the draw is clamped to 1e-6 nu). */
wallace_status wallace_compute_a(uint64_t nu, double* a);
wallace_status wallace_chi2_params(uint64_t nu, double* a_value);
wallace_status wallace_chi2_sample(double x, uint64_t nu, double a_value, int32_t method,
                                   int32_t* clamped, double* out);

/* transforms.hpp:64-137: wallace_variant(id) (entries row-major 4x4,
 * source_row, row_sign; any pointer may be NULL; id in [0, 384)) and
 * rotation_from_t (InvalidParameterError for non-finite t). */
wallace_status wallace_variant(int32_t id, double entries[16], uint8_t source_row[4],
                               double row_sign[4]);
wallace_status wallace_rotation_from_t(double t, double* c, double* s);

/* Device streams of polar_next / boxmuller_next (baselines.cpp:51-92), one
 * thread per BaselineState, fp64: states[n_streams] (host) continue where
 * they are and are advanced; stream p's next `count` values land in the
 * DEVICE buffer dev_out[p*count, (p+1)*count).  The uniform words, the
 * Polar acceptance sequence and the draw counts are exact; the values use
 * CUDA's fp64 log/sqrt/sincos (a few ulps from glibc's, see
 * tests/test_gpu_baselines.py).  Synchronous. */
wallace_status wallace_baseline_fill(int32_t method, wallace_baseline_state* states,
                                     uint64_t n_streams, uint64_t count, double* dev_out,
                                     void* stream);

/* Config-5 comparator: stream p = BaselineState(seeds[p] or seed_base+p),
 * `count_per_stream` values of `method` generated as wallace_baseline_fill
 * would, consumed in-kernel into the same sums[4] / hist[258] as
 * wallace_consume (fp64).  *device_ms (optional): the kernel's device time
 * (CUDA events).  Synchronous. */
wallace_status wallace_baseline_consume(int32_t method, const uint64_t* seeds, uint64_t seed_base,
                                        uint64_t n_streams, uint64_t count_per_stream, void* stream,
                                        double sums[4], uint64_t hist[258], double* device_ms);
/* = wallace_baseline_consume(WALLACE_BASELINE_BOXMULLER, ...) */
wallace_status wallace_boxmuller_consume(const uint64_t* seeds, uint64_t seed_base,
                                         uint64_t n_streams, uint64_t count_per_stream,
                                         void* stream, double sums[4], uint64_t hist[258]);

/* Kernel timing for measurement (bench.py): between begin and end, every
 * plan_kernel and pool_kernel launch of this handle is bracketed by CUDA
 * events recorded on the handle's stream.  end synchronizes the stream and
 * returns the summed device milliseconds and launch counts. */
wallace_status wallace_profile_begin(wallace_handle* h);
wallace_status wallace_profile_end(wallace_handle* h, double* pool_kernel_ms,
                                   uint64_t* pool_launches, double* plan_kernel_ms,
                                   uint64_t* plan_launches);

/* Kernel shape: 0 auto (latency kernel for <= 148 pools), 1 throughput
 * kernel (a few warps per pool, many pools per SM), 2 latency kernel (one
 * 4-block per thread, up to 1024 threads per pool).  Results are identical;
 * exposed for tests and tuning. */
wallace_status wallace_set_kernel_mode(wallace_handle* h, int32_t mode);

/* Rebind the handle to another stream.  Work already queued on the old
 * stream is ordered before everything issued after the switch. */
wallace_status wallace_set_stream(wallace_handle* h, void* stream);

/* Waits for the handle's queued work.  chi2_sample's InvalidParameterError
 * (chi2.cpp:29-31: a non-finite reserved value, e.g. after inject_pool of
 * a non-finite pool, reached from refill_ inside fill/next_pool,
 * generator.cpp:358-361) is detected on the device: the synchronous calls
 * (wallace_fill_host, wallace_next_pool(_host), wallace_consume*,
 * wallace_write_stream, wallace_pool_defect_stats, this call) return
 * WALLACE_ERR_INVALID_PARAM "chi2_sample: x must be finite" for every
 * emission they or an earlier asynchronous wallace_fill drew; wallace_fill
 * itself reports an earlier call's error once it is known, at the latest
 * the next synchronous call does.  Each detection is reported once; the
 * non-finite value stays in the pool state, so later emissions raise again,
 * as every later refill_ of the reference throws. */
wallace_status wallace_synchronize(wallace_handle* h);

/* Number of kernels this library has launched (all handles). */
uint64_t wallace_kernel_launches(void);
/* ... of which pair_kernel (fp32 pools of 4096, wallace4 + stride mixing,
 * discard_every = 2: two passes per shared-memory round trip; the other
 * fills run pool_kernel).  WALLACE_B200_PAIR=0 keeps every fill on
 * pool_kernel. */
uint64_t wallace_pair_kernel_launches(void);

/* Message of the last failed call on this thread. */
const char* wallace_last_error(void);

/* Host-only helpers (no device work), exposed for tests and integration:
 * validate a config exactly like GeneratorConfig::validate(); seed one pool
 * on the host like the Generator constructor up to (excluding) the 16
 * warm-up passes: raw_out[pool_size] (double), reserved_prev, sum_sq,
 * xoshiro state s[4] and draws. */
wallace_status wallace_validate_config(const wallace_config* cfg);
wallace_status wallace_host_seed_pool(const wallace_config* cfg, uint64_t seed, double* raw_out,
                                      double* reserved_prev, double* sum_sq, uint64_t s_out[4],
                                      uint64_t* draws);
/* maxent::default_stride (transforms.cpp:161-169) and the plan decode of
 * decode_pass_plan (generator.cpp:238-257) — the integer contract. */
uint64_t wallace_default_stride(uint64_t rows);
int32_t wallace_decode_pass_plan(uint64_t pool_size, uint64_t transform_word,
                                 uint64_t offset_word, uint64_t* offset0);

/* ---- stream wire format (cmd_gen.cpp:39-57) ---------------------------------
 * `count` further values of every pool written to the file descriptor `fd`,
 * pool-major (pool p's values at [p*count, (p+1)*count) in value units, as
 * wallace_fill): WALLACE_FMT_F64LE consecutive 8-byte little-endian IEEE
 * doubles, no header (an fp32 stream widened exactly); WALLACE_FMT_TEXT one
 * "%.17g\n" line per value (round-trips the double; one pool only);
 * WALLACE_FMT_F32LE 4-byte floats (fp32 handles).  For one pool this is the
 * byte stream of the reference's `gen --format f64le|text`.  Several pools
 * need a binary format and a seekable fd.  Generation, the device->host copy
 * and the formatting/writing of consecutive chunks overlap (double-buffered
 * pinned staging).  Synchronous; leaves the file position after the block. */
typedef enum wallace_format {
  WALLACE_FMT_F64LE = 0,
  WALLACE_FMT_TEXT = 1,
  WALLACE_FMT_F32LE = 2
} wallace_format;
wallace_status wallace_write_stream(wallace_handle* h, uint64_t count, int32_t format, int32_t fd);

/* ---- defect suite, GPU-resident (stats.cpp) ---------------------------------
 * cross_pool_correlation(Generator&, opts) (stats.cpp:310-338) for every pool
 * of the batch: `passes` step_pass() calls; for probe k the reference's
 * ProbeAccumulator sums over x = pool_before[in_j[k]] and y =
 * pool_after[out_i[k]], in pass order, fp64 (bit-identical per pool):
 * acc[(pool * n_probes + k) * 6 + {0..5}] = {sx, sxx, sy, syy, sxy, sxy2}.
 * 1 <= n_probes <= 32; the pools advance by `passes`.  Synchronous. */
wallace_status wallace_cross_pool_probes(wallace_handle* h, uint64_t passes, uint32_t n_probes,
                                         const uint64_t* out_i, const uint64_t* in_j, double* acc);
/* pool_sum_squares_test (stats.cpp:340-369) and rare_event_adjacency
 * (:424-447) for every pool: `emissions` next_pool() calls; per emission the
 * total reserved^2 + sum v^2 of the standardized values (fp64; a tree sum,
 * equal to the reference's sequential sum to rounding) and the mark "some
 * |v| > threshold".  totals / marks: [n_pools][emissions].  The handle's
 * config must have out_mean 0 and out_sigma 1 (the reference standardizes
 * the same way).  Synchronous. */
wallace_status wallace_pool_defect_stats(wallace_handle* h, uint64_t emissions, double threshold,
                                         double* totals, uint8_t* marks);

/* maxent::PassPlan (generator.hpp:50-55) and decode_pass_plan(cfg, w0, w1)
 * (generator.cpp:238-257) for every family/mixing combination. */
typedef struct wallace_pass_plan {
  int32_t wallace_variant;
  int32_t t_index[2];
  int32_t negate[2];
  int32_t reserved_;
  uint64_t offset[2];
} wallace_pass_plan;
wallace_status wallace_decode_pass_plan_ex(const wallace_config* cfg, uint64_t transform_word,
                                           uint64_t offset_word, wallace_pass_plan* out);
/* maxent::run_pass (generator.cpp:259-271): one pass of the configured family
 * and mixing with an explicit plan over one fp64 pool (host buffers of
 * pool_size doubles, run on the device). */
wallace_status wallace_run_pass(const wallace_config* cfg, const wallace_pass_plan* plan, const double* in,
                                double* out);
/* maxent::pass_coefficient (generator.cpp:273-284): entry (out_i, in_j) of
 * the composed pass matrix, from the permutation and block structure. */
wallace_status wallace_pass_coefficient(const wallace_config* cfg, const wallace_pass_plan* plan, uint64_t out_i,
                                        uint64_t in_j, double* out);
/* maxent::default_multipliers (generator.cpp:286-294). */
void wallace_default_multipliers(uint64_t n, uint64_t* alpha, uint64_t* beta);
/* cross_pool_correlation's fixed-transform mode (stats.cpp:284-299): `pairs`
 * fresh Polar pools from BaselineState(cfg->seed), one pinned pass
 * (PassPlan{}) each on the device; ProbeAccumulator sums in pair order,
 * acc[k * 6 + {0..5}] = {sx, sxx, sy, syy, sxy, sxy2}. */
wallace_status wallace_cross_pool_fixed(const wallace_config* cfg, uint64_t pairs, uint32_t n_probes,
                                        const uint64_t* out_i, const uint64_t* in_j, double* acc);

/* rotation_t_table() and rotation_from_t (transforms.cpp:39-70): t, c = cos,
 * s = sin of the 16 table entries (any pointer may be NULL). */
void wallace_rotation_table(double t[16], double c[16], double s[16]);

#ifdef __cplusplus
}
#endif
#endif /* WALLACE_B200_H */
