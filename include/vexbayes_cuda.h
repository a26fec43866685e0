/*
 * vexbayes_cuda.h -- C ABI of libvexbayes_cuda.so
 *
 * B200 (sm_100a) implementation of the hot path of the "vexbayes" library
 * (arXiv 1902.09046): batched, independent prior-predictive simulation inside
 * likelihood-free samplers.  Every entry point below replaces one reference
 * interface; the reference location is cited as  file:line  relative to
 * /root/reference/proj/core/.  The reference-side binding a maintainer adds is
 * shown in INTEGRATION.md, the C++ shim that keeps the vexbayes:: signatures is
 * paper_1902_09046_b200/cpp/vexbayes/.
 *
 * Conventions
 *  - plain C types only; return 0 on success, non-zero on failure.  After a
 *    failure vxb_last_error() returns the thread-local text "code: message"
 *    where `code` is one of the reference error codes (errors.hpp:11-28):
 *    invalid-shape, invalid-summary, invalid-range, invalid-scale,
 *    invalid-argument, invalid-horizon, insufficient-data, empty-set,
 *    degenerate-ensemble, plus device-error for CUDA failures.
 *  - the caller owns every buffer it passes in.  A buffer may live in host
 *    memory (pageable or pinned) or in device memory of the context's GPU; the
 *    library detects which (unified virtual addressing) and stages host
 *    buffers through its own device scratch.  Optional outputs may be NULL.
 *  - `precision` selects the element type of every `void*` real buffer:
 *    VXB_F64 -> double, VXB_F32 -> float.  `observed` is always double.
 *  - one vxb_ctx is used by one host thread at a time (the single-owner rule
 *    of rng.hpp:30-31); it owns one CUDA stream and all device scratch.
 *  - there is no CPU fallback: without a CUDA device vxb_init fails.
 */
#ifndef VEXBAYES_CUDA_H
#define VEXBAYES_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define VXB_ABI_VERSION 2

typedef struct vxb_ctx vxb_ctx;

/* ------------------------------------------------------------------ enums */
enum { VXB_MODEL_LOGISTIC_SDE = 1, VXB_MODEL_NORMAL_MEAN = 2, VXB_MODEL_MM_TAULEAP = 3,
       VXB_MODEL_TOGGLE = 4, VXB_MODEL_TB = 5 };
enum { VXB_F64 = 0, VXB_F32 = 1 };
/* VXB_RNG_REF      : Philox2x64-10 + Box-Muller through the reference's own
 *                    polynomials; every variate bit-identical to RngStream
 *                    (rng.cpp:65-78,112-164, fastmath.hpp:23-128).
 * VXB_RNG_FAST     : throughput generator (Philox4x32-10, FMA polynomials /
 *                    MUFU in fp32); statistically validated only.  In fp32 the
 *                    normals are exact in distribution up to 4 sigma, thin beyond 5
 *                    and capped at 5.65 sigma (see vxb_rng_fast_stats).
 * VXB_RNG_EXTERNAL : standard normals are read from a caller buffer. */
enum { VXB_RNG_REF = 0, VXB_RNG_FAST = 1, VXB_RNG_EXTERNAL = 2 };
/* VXB_ARITH_EXACT: separate multiply and add everywhere (the reference builds
 * with -ffp-contract=off, CMakeLists.txt:15-18) => bit parity.
 * VXB_ARITH_FMA  : the simulator update may contract to FMA (<=1e-12 rel.). */
enum { VXB_ARITH_EXACT = 0, VXB_ARITH_FMA = 1 };
/* VXB_KEY_PARTICLE: particle i owns RngStream(seed, stream_id = i), counter 0
 *                   => results independent of sharding / GPU count.
 * VXB_KEY_WORKER  : the reference keying of abc.cpp:43-61: rows are split by
 *                   partition(n, workers, block_width) (blocked.cpp:34-63),
 *                   worker w owns RngStream(seed, w) and its rows consume it
 *                   sequentially => bit-identical to run_prior_predictive for
 *                   the same (seed, workers, block_width). */
enum { VXB_KEY_PARTICLE = 0, VXB_KEY_WORKER = 1 };

/* ------------------------------------------------------------ descriptors */

/* POD replacement for the closures of ModelHooks (model.hpp:19-36).
 *
 * VXB_MODEL_LOGISTIC_SDE  dX = r X (1 - X/K) dt + sigma X dW, theta=(r,K,sigma)
 *   dim = 3, steps Euler-Maruyama steps of size dt from x0, the state is
 *   recorded after every obs_stride-th step: summary_dim = steps / obs_stride.
 *   prior_lo/hi[0..2] = the uniform prior box (map lo + u*(hi-lo), as
 *   toggle_switch.cpp:17-22).  consts[0] = sqrt(dt) (computed by the caller
 *   with the host libm so that host and device agree).
 * VXB_MODEL_NORMAL_MEAN   y_i ~ N(theta,1), i<steps, theta ~ N(0, lambda^2)
 *   steps = n (data per dataset).
 * VXB_MODEL_MM_TAULEAP    S+E->C (k1), C->S+E (k2), C->E+P (k3)
 *   consts[0..3] = initial (S,E,C,P), consts[4..6] = (k1,k2,k3).  precision VXB_F32
 *   (with VXB_RNG_FAST only): propensities and the Poisson inversion in float, exp by one
 *   MUFU; the state stays integer.  Statistically validated, like every throughput mode.
 *   VXB_RNG_REF: reaction r of coupled fine step s owns stream positions 6s+2r, 6s+2r+1
 *   (bit-exact with the oracle).  VXB_RNG_FAST: the six uniforms of a coupled fine step
 *   come from Philox4x32 blocks 2s (leading 21 bits) and 2s+1 (trailing bits; drawn only
 *   when a reaction may fire): 42-bit uniforms in fp64, 23-bit bucket midpoints in fp32.
 * VXB_MODEL_TB            the multi-genotype TB transmission model (tb_model.hpp),
 *   exact Gillespie; theta = (alpha, delta, tau) with the prior of
 *   tb::sample_prior, dim = 3, summaries (G, H), summary_dim = 2;
 *   consts[0] = initial cases, consts[1] = time horizon, consts[2] = case target
 *   (<= 60000 on the device), consts[3] = attempts of vxb_simulate_at (> 1: the
 *   retry-while-extinct loop of bench::tb_observed_summaries, bench.cpp:79-92).
 *   VXB_KEY_PARTICLE only (a row consumes a data-dependent number of variates).
 */
typedef struct vxb_model {
    int32_t model;      /* VXB_MODEL_*            */
    int32_t precision;  /* VXB_F64 | VXB_F32      */
    int32_t rng;        /* VXB_RNG_*              */
    int32_t arith;      /* VXB_ARITH_*            */
    uint32_t dim;
    uint32_t summary_dim;
    uint32_t steps;
    uint32_t obs_stride;
    double dt;
    double x0;
    double prior_lo[8];
    double prior_hi[8];
    double consts[16];
} vxb_model;

typedef struct vxb_keying {
    int32_t mode;         /* VXB_KEY_*                                   */
    uint32_t workers;     /* VXB_KEY_WORKER: P   (abc.cpp:26)            */
    uint32_t block_width; /* VXB_KEY_WORKER: V   (blocked.cpp:10-12)     */
    uint32_t reserved;
    uint64_t seed;
} vxb_keying;

typedef struct vxb_device_props {
    int32_t device;
    int32_t sm_count;
    int32_t cc_major;
    int32_t cc_minor;
    int32_t clock_khz;     /* max SM clock                */
    int32_t reserved;
    uint64_t global_mem;   /* bytes                       */
    char name[128];
} vxb_device_props;

/* kernel families counted by the built-in event profiler */
enum { VXB_K_SIMULATE = 0, VXB_K_SELECT = 1, VXB_K_COMPACT = 2, VXB_K_PPP = 3,
       VXB_K_RESAMPLE = 4, VXB_K_WEIGHTS = 5, VXB_K_PROPOSE = 6, VXB_K_TAULEAP = 7,
       VXB_K_RNGFILL = 8, VXB_K_MISC = 9, VXB_K_COUNT = 10 };
typedef struct vxb_profile {
    uint64_t launches[VXB_K_COUNT];
    double total_ms[VXB_K_COUNT]; /* only while event timing is enabled */
} vxb_profile;

/* ---------------------------------------------------- lifecycle / errors */
int vxb_abi_version(void);
/* Philox4x32 rounds of the throughput generator in this build: 10 (the product
 * library) or 7 (the opt-in build, -DVXB_FAST_ROUNDS=7: the minimum Salmon et al.
 * report as Crush-resistant; +11.6% on the fp64 headline kernel, +16% in fp32;
 * profiles/r2_philox7.json). */
int vxb_fast_generator_rounds(void);
/* device < 0: use the current CUDA device. */
int vxb_init(vxb_ctx** ctx, int device);
void vxb_shutdown(vxb_ctx* ctx);
const char* vxb_last_error(void);
int vxb_device_info(vxb_ctx* ctx, vxb_device_props* out);
/* The context's stream as a cudaStream_t (for event timing by the caller). */
void* vxb_stream(vxb_ctx* ctx);
int vxb_synchronize(vxb_ctx* ctx);
/* Event-time every kernel launch (adds two events per launch). */
/* Context options.  VXB_OPT_EARLY_REJECT (0 / 1, default 0): see vxb_abc_reject. */
enum { VXB_OPT_EARLY_REJECT = 1 };
int vxb_set_option(vxb_ctx* ctx, int option, int64_t value);
int vxb_profile_enable(vxb_ctx* ctx, int on);
int vxb_profile_reset(vxb_ctx* ctx);
int vxb_profile_read(vxb_ctx* ctx, vxb_profile* out); /* synchronises */
/* Device buffers for callers without a CUDA runtime of their own. */
int vxb_device_alloc(vxb_ctx* ctx, size_t bytes, void** out);
int vxb_device_free(vxb_ctx* ctx, void* p);
int vxb_copy(vxb_ctx* ctx, void* dst, const void* src, size_t bytes); /* any direction */

/* glibc ships two builds of its exp on x86-64 (FMA-contracted for CPUs with FMA + AVX2,
 * plain otherwise; they differ in the last ulp of about one result in 10^3).  vxb_init
 * probes the live std::exp of the process and the device reproduces the matching build in
 * vxb_ess / vxb_logsumexp / vxb_resample_multinomial: *variant = 0 FMA build, 1 plain
 * build, -1 neither matched (a different libm: the FMA build is used and those three
 * entry points agree with the host to an ulp instead of bit for bit).  ctx == NULL:
 * probe the calling process now (host only, no GPU needed). */
int vxb_host_exp_variant(vxb_ctx* ctx, int* variant);

/* Guard mode (diagnostics; environment VXB_GUARD=1 when vxb_init runs): every
 * library-owned device allocation (staging, scratch, arenas) is bracketed by 256-byte
 * canary zones that are verified when it is released; a violation prints a line
 * "vxb guard: ..." on stderr and is counted.  *violations = the count so far.
 * selftest != 0: first provoke one violation (a kernel writes one byte past a
 * scratch buffer); *detected = 1 if the guard saw it (it is not counted). */
int vxb_guard_report(vxb_ctx* ctx, int selftest, unsigned long long* violations, int* detected);

/* Roofline denominator: measured throughput (TFLOP/s, FMA = 2 flops) of a
 * dependency-free FMA chain kernel in the given precision on this GPU, timed
 * with events over `iters` iterations per thread.  Diagnostics only. */
int vxb_fma_peak(vxb_ctx* ctx, int precision, uint32_t iters, double* tflops, double* ms);

/* ------------------------------------------------------ substrate (RNG) */
/* splitmix64 (rng.cpp:22-27) and derive_seed (rng.cpp:29-35); host-side. */
uint64_t vxb_splitmix64(uint64_t z);
uint64_t vxb_derive_seed(uint64_t seed, const uint64_t* path, size_t n_path);
/* Device fill of n raw words / uniforms / Gaussians of RngStream(seed,stream_id)
 * starting at counter position `pos`; replaces RngStream::next_u64 (rng.cpp:92-97),
 * fill_uniform (rng.cpp:125-140) and fill_gaussian (rng.cpp:142-164).  Same
 * argument checks: a <= b (invalid-range); sigma >= 0 (invalid-scale). Unlike
 * the reference's fill_gaussian, odd n is allowed: position p always yields the
 * Gaussian of pair p/2 (cos branch even p, sin branch odd p), which is what
 * next_gaussian (rng.cpp:112-123) defines. */
int vxb_rng_fill_u64(vxb_ctx* ctx, uint64_t seed, uint32_t stream_id, uint64_t pos, uint64_t n,
                     uint64_t* out);
int vxb_rng_fill_uniform(vxb_ctx* ctx, uint64_t seed, uint32_t stream_id, uint64_t pos,
                         uint64_t n, double a, double b, double* out);
int vxb_rng_fill_gaussian(vxb_ctx* ctx, uint64_t seed, uint32_t stream_id, uint64_t pos,
                          uint64_t n, double mu, double sigma, double* out);
/* The standard normals of the throughput generator (VXB_RNG_FAST) exactly as the
 * simulation kernels consume them: row r of [first_row, first_row+rows), step j
 * -> out[r*per_row + j]; element type by precision.  For statistical validation. */
int vxb_rng_fill_gaussian_fast(vxb_ctx* ctx, int precision, uint64_t seed, uint64_t first_row,
                               uint64_t rows, uint32_t per_row, void* out);
/* Statistics of the same normals over rows x per_row samples with only counters
 * leaving the GPU (1e10+ samples per call): tail_counts[k] = #{|z| > thresholds[k]}
 * (at most 8 thresholds); moments[0..8] = n, sum z, sum z^2, sum z^3, sum z^4, max |z|,
 * and for VXB_F32 the error of the MUFU evaluation against a double-precision
 * evaluation of the same uniforms: max |z32 - z64|, the same over |z64| > 4, and
 * sum (z32 - z64)^2.
 * FAR TAIL OF THE FP32 GENERATOR: its Box-Muller radius uniform lives on a 2^-23
 * lattice, so |z| <= sqrt(2 * 23 ln 2) = 5.65 sigma (1.6e-8 of the N(0,1) mass lies
 * beyond) and the mass beyond 5 sigma is resolved by ~31 lattice points only: measured
 * over 3 x 1e10 samples it is 4% low at 5 sigma and 35% low at 5.5 sigma, exact (within
 * Poisson error) up to 4 sigma (profiles/r2_fast_generator_stats.json).  The fp64
 * generator's radius uniform has 52 bits: no deficit and no practical cap.
 * csrc/vxb_rng.cuh records why the fp32 tail is left as it is (every in-loop tail test
 * costs the fp32 kernel 8-15%). */
int vxb_rng_fast_stats(vxb_ctx* ctx, int precision, uint64_t seed, uint64_t first_row,
                       uint64_t rows, uint32_t per_row, const double* thresholds,
                       uint32_t n_thresholds, uint64_t* tail_counts, double* moments);
/* Device evaluation of the fastmath functions (fastmath.hpp:23-128), for
 * parity tests: fn 0 log2_pos, 1 ln_pos, 2 exp2_clamped, 3 sinpi, 4 cospi,
 * 5 pow_pos (x = base, y = exponent; y ignored otherwise); and of the
 * throughput-mode functions, for accuracy tests: fn 6 log2 (x > 0 normal),
 * 7 2^x (|x| < 1000), 8 1/x (normal x); fn 9: exp exactly as the host libm
 * evaluates it (glibc >= 2.28) -- what std::exp returns in smc.cpp:214,278,299 and
 * numeric.cpp:16-17, bit for bit: the build of the algorithm this host's libm runs
 * (vxb_host_exp_variant); fn 10 / 11: its FMA / plain build regardless of the host. */
int vxb_fastmath_eval(vxb_ctx* ctx, int fn, const double* x, const double* y, uint64_t n,
                      double* out);
/* partition (blocked.cpp:34-63): writes workers pairs [begin,end). Host-side. */
int vxb_partition(uint64_t total, uint64_t workers, uint64_t block_width, uint64_t* ranges);

/* ------------------------------------------------- ABC rejection (C0/C1) */
/* Drop-in for abc::run_prior_predictive (abc.cpp:26-73) on rows
 * [first, first+count) of an n_total-row job.  Outputs are row-major
 * count x dim, count x summary_dim, count, count; any may be NULL.  A row
 * whose state becomes non-finite is `failed` (summary zeroed, rho NaN),
 * mirroring abc.cpp:54-60.  external_noise (VXB_RNG_EXTERNAL): count x steps
 * standard normals, row-major, element type = precision. */
int vxb_abc_prior_predictive(vxb_ctx* ctx, const vxb_model* model, const vxb_keying* key,
                             uint64_t n_total, uint64_t first, uint64_t count,
                             const double* observed, void* params, void* summaries, void* rho,
                             uint8_t* failed, const void* external_noise);

/* Drop-in for abc::select_epsilon (abc.cpp:75-97) over n discrepancies:
 * epsilon = type-7 q-quantile of the non-failed rho raised to the ceil(q n)-th
 * order statistic, accepted = ascending rows with rho <= epsilon.  At most
 * `cap` indices are written; *n_accepted is the full count.  idx may be NULL. */
int vxb_select_epsilon(vxb_ctx* ctx, int precision, const void* rho, const uint8_t* failed,
                       uint64_t n, double accept_fraction, double* epsilon, uint64_t cap,
                       uint64_t* n_accepted, uint64_t* idx);

/* k-th order statistics (0-based ranks, ascending, NaN/failed rows excluded)
 * of rho; *n_valid receives the number of non-failed rows. */
int vxb_order_statistics(vxb_ctx* ctx, int precision, const void* rho, const uint8_t* failed,
                         uint64_t n, const uint64_t* ranks, uint32_t n_ranks, double* values,
                         uint64_t* n_valid);

/* Ascending compaction of rows with !failed && rho <= epsilon; idx values are
 * row + index_base. */
int vxb_compact_accepted(vxb_ctx* ctx, int precision, const void* rho, const uint8_t* failed,
                         uint64_t n, double epsilon, uint64_t index_base, uint64_t cap,
                         uint64_t* n_accepted, uint64_t* idx);

/* Fused fixed-epsilon rejection (config 1): simulate rows [first,first+count),
 * keep only rows with rho <= epsilon, ascending.  idx holds global row numbers.
 * params: cap x dim, rho: cap.  Trajectories, summaries and rejected rows never
 * leave the GPU.  If n_accepted points to DEVICE memory the call is fully
 * asynchronous: the count is written there, idx/params/rho must be device
 * buffers (or NULL), nothing is copied to the host and the stream is not
 * synchronised -- steps can be queued back to back.
 * With VXB_OPT_EARLY_REJECT (vxb_set_option; off by default) a row stops as soon as its
 * partial squared distance can no longer end below epsilon^2 -- the sum of squares only
 * grows -- and the accepted set, indices, parameters and distances are bit-identical to
 * the full simulation; only the (never returned) distances of rejected rows differ.  It
 * pays when few rows are accepted (3.4x at 0.1 %, 1.4x at 8 %); with nothing to reject it
 * costs 4-8 %. */
int vxb_abc_reject(vxb_ctx* ctx, const vxb_model* model, const vxb_keying* key,
                   uint64_t n_total, uint64_t first, uint64_t count, const double* observed,
                   double epsilon, uint64_t cap, uint64_t* n_accepted, uint64_t* idx,
                   void* params, void* rho);

/* Simulate the model once at theta from RngStream(seed, stream_id) at counter
 * position pos (aligned up to even), the way bench.cpp:69-77 builds observed
 * summaries.  summary: summary_dim reals. */
int vxb_simulate_at(vxb_ctx* ctx, const vxb_model* model, const double* theta, uint64_t seed,
                    uint32_t stream_id, uint64_t pos, void* summary);

/* ------------------------------------- prior-predictive p-values (C2) */
/* For every lambda_k: datasets j in [first, first+count) of m_total, dataset
 * (k,j) drawn from RngStream(derive_seed(seed,{k}), j) in the order of
 * weak_info.cpp:82-106 (align_even; Gaussian prior draw; then the data);
 * counts[k] = #{ j : logm(ybar_kj) <= logm(ybar_obs) } -- the counting rule of
 * estimate_pvalues (weak_info.cpp:108-120, ties count); pvalues[k] =
 * counts[k]/m_total (only meaningful when the shard is the whole job).
 * log_norm[k] = -0.5*log(2 pi v_k), v_k = lambda_k^2 + 1/n, is supplied by the
 * caller (host libm).  ybar_out (optional): n_lambda x count sample means. */
int vxb_ppp_pvalues(vxb_ctx* ctx, const vxb_model* model, const double* lambda,
                    const double* log_norm, uint32_t n_lambda, uint64_t m_total, uint64_t first,
                    uint64_t count, uint64_t seed, double ybar_obs, uint64_t* counts,
                    double* pvalues, double* ybar_out);

/* One rank's accepted set of the fused fixed-epsilon path as ONE block of device
 * memory, so that a single all-gather moves it: [count u64, padded to 16 B]
 * [idx u64 x cap][theta real x cap x dim][rho real x cap], each field 16-byte
 * aligned; `stride` = bytes of a block.  Rows [0, min(count, cap)) are valid. */
typedef struct vxb_accept_layout {
    uint64_t cap;
    uint64_t off_count, off_idx, off_params, off_rho;
    uint64_t stride;
} vxb_accept_layout;
int vxb_accept_layout_of(int precision, uint32_t dim, uint64_t cap, vxb_accept_layout* out);

/* ------------------------------------------- SMC building blocks (C3) */
/* smc::ess (smc.cpp:208-219) and logsumexp (numeric.cpp:11-18): bit-identical to the
 * reference on this host -- every exp is the host libm's (vxb_host_exp_variant), the sums
 * run left to right as the reference's loops do, the final log is the host's. */
int vxb_ess(vxb_ctx* ctx, const double* log_w, uint64_t n, double* ess);
int vxb_logsumexp(vxb_ctx* ctx, const double* x, uint64_t n, double* out);
/* smc::resample_multinomial (smc.cpp:268-300): draw i uses position i of
 * RngStream(seed, stream_id); ancestors[i] = upper_bound(cum, u_i * cum[n-1]),
 * clamped; particles_out row i = particles_in row ancestors[i].  The cumulative
 * weights are the reference's (host-libm exp, sequential running sum), so the
 * ancestors are identical to the reference's, index for index. */
int vxb_resample_multinomial(vxb_ctx* ctx, uint64_t n, uint32_t dim, const double* log_w,
                             const double* particles_in, uint64_t seed, uint32_t stream_id,
                             double* particles_out, uint64_t* ancestors);

typedef struct vxb_abcsmc_cfg {
    uint64_t particles;    /* N                                            */
    uint32_t generations;  /* G (generation 0 = prior)                     */
    uint32_t reserved;
    double quantile;       /* epsilon_g = this quantile of generation g-1  */
    double kernel_scale;   /* covariance multiplier (2.0)                  */
    double jitter;         /* make_kernel jitter (smc.cpp:311-325), 1e-10  */
    uint64_t round_size;   /* proposals per round; 0 => N                  */
    uint64_t max_rounds;   /* safety cap per generation; 0 => 1000         */
    uint64_t seed;
} vxb_abcsmc_cfg;

/* One generation's population and diagnostics.  All arrays caller-owned:
 * theta N x dim, weight N (normalised, linear), rho N; per generation
 * (G entries): epsilon, ess, acceptance rate, proposals used, weighted mean
 * (G x dim) and covariance (G x dim x dim) of the population. */
typedef struct vxb_abcsmc_out {
    double* theta;
    double* weight;
    double* rho;
    double* epsilon;
    double* ess;
    double* accept_rate;
    uint64_t* proposals;
    double* mean;
    double* cov;
} vxb_abcsmc_out;

int vxb_abcsmc_run(vxb_ctx* ctx, const vxb_model* model, const vxb_abcsmc_cfg* cfg,
                   const double* observed, vxb_abcsmc_out* out);

/* The two device stages of a generation, exposed so that a multi-GPU host can
 * shard them (proposals / new particles by global index) and run the
 * collectives itself:
 * propose: for proposals p in [first, first+count) of generation `gen`:
 *   ancestor by inverse CDF over cum (n_prev inclusive cumulative weights),
 *   theta* = theta_a + L z, reject outside the prior box, else simulate and
 *   compare with epsilon.  Outputs per proposal: theta* (count x dim), rho,
 *   flag (1 accepted, 0 rejected by distance, 2 outside the prior, 3 failed).
 *   state (optional, DEVICE uint64[4], see vxb_abcsmc_append_round): the round is
 *   skipped on the device when state[0] >= n_target already -- this is what lets a
 *   multi-GPU host issue rounds ahead of its knowledge of how many are needed.
 *   With device-resident buffers the call does not synchronise.
 * weights: for `count` new particles (theta_new: count x dim): the unnormalised
 *   importance weight 1 / sum_j w_j phi(theta_i; theta_j, Sigma), summed over
 *   j in index order.  rng = the model's generator: VXB_RNG_REF is the bit-exact
 *   kernel, VXB_RNG_FAST the throughput form (whitening + table 2^z) that
 *   vxb_abcsmc_run uses for a VXB_RNG_FAST model -- a sharded run must pass the same
 *   mode to stay identical to the one-GPU run.  count == 0 is allowed (empty shard).
 *   With device-resident buffers the call does not synchronise. */
int vxb_abcsmc_propose(vxb_ctx* ctx, const vxb_model* model, uint64_t seed, uint32_t gen,
                       uint64_t first, uint64_t count, uint64_t n_prev, const double* theta_prev,
                       const double* cum_prev, const double* chol, const double* observed,
                       double epsilon, double* theta_out, double* rho_out, uint8_t* flag_out,
                       const uint64_t* state, uint64_t n_target);
int vxb_abcsmc_weights(vxb_ctx* ctx, int rng, uint32_t dim, uint64_t count, const double* theta_new,
                       uint64_t n_prev, const double* theta_prev,
                       const double* w_prev, const double* chol, double* w_out);

/* Rounds without host round trips (the multi-GPU ABC-SMC host, dist.sharded_abcsmc).
 * state: DEVICE uint64[4] = { rows of the new population filled so far, accepted
 * proposals counted while filling, rounds used, reserved }, zeroed by the caller at
 * the start of a generation.
 * pack_round: the accepted rows (finite rho <= epsilon, !failed) of this rank's
 *   `count` evaluated rows -> one block laid out as vxb_accept_layout_of(VXB_F64, dim,
 *   cap >= count): count | local row numbers | theta | rho; nothing is packed once
 *   state[0] >= n_target.
 * append_round: the gathered blocks of all ranks of a round, in rank order
 *   (= ascending proposal index), are appended behind the filled rows of the new
 *   population up to n rows -- "the first n accepted by proposal index", as the
 *   one-GPU loop of vxb_abcsmc_run takes them -- and the state advances; a round that
 *   arrives after the population is full changes nothing.
 * normalise_by_chunk_totals: w /= (chunk totals added left to right), the divisor
 *   formed on the device; chunk_totals is the all-reduced vector of
 *   vxb_canon_chunk_sums values.
 * Device buffers only; none of the three synchronises. */
int vxb_abcsmc_pack_round(vxb_ctx* ctx, uint32_t dim, const double* theta, const double* rho,
                          const uint8_t* failed, uint64_t count, double epsilon,
                          const vxb_accept_layout* layout, void* block, const uint64_t* state,
                          uint64_t n_target);
int vxb_abcsmc_append_round(vxb_ctx* ctx, uint32_t dim, const void* blocks, uint32_t n_blocks,
                            const vxb_accept_layout* layout, double* pop_theta, double* pop_rho,
                            uint64_t n, uint64_t* state);
int vxb_normalise_by_chunk_totals(vxb_ctx* ctx, double* w, uint64_t n, const double* chunk_totals,
                                  uint64_t n_chunks, double* total_out);

/* Population statistics of a generation in the canonical two-level summation
 * order (chunks of 256 rows left to right, then chunk totals left to right) --
 * the order that makes single- and multi-GPU runs bit-identical.  Exposed for
 * the multi-GPU host (every rank holds the replicated previous population).
 * weighted_moments: mean[dim], cov[dim x dim] = sum w d d^T / (1 - sum w^2)
 *   (sample_covariance's n-1 divisor for equal weights, numeric.cpp:55-79);
 *   *sum_w2 = sum w^2 (ESS = 1/sum_w2, smc.cpp:208-219).  Host outputs.
 * canon_cumsum: inclusive cumulative weights (resample_multinomial's `cum`,
 *   smc.cpp:276-283).  canon_chunk_sums: the ceil(n/256) chunk totals of v, so
 *   that ranks owning chunk-aligned shards can all-reduce them exactly.
 * divide: in-place normalisation of the weights by their canonical sum.
 * quantile: numeric.cpp:20-36 (type 7) of n device- or host-resident values.
 * make_kernel (host only): chol(scale * cov) with the jitter rule of
 *   smc.cpp:311-325. */
int vxb_weighted_moments(vxb_ctx* ctx, const double* theta, const double* w, uint64_t n,
                         uint32_t dim, double* mean, double* cov, double* sum_w2);
int vxb_canon_cumsum(vxb_ctx* ctx, const double* w, uint64_t n, double* cum);
int vxb_canon_chunk_sums(vxb_ctx* ctx, const double* v, uint64_t n, double* chunk_sums);
int vxb_quantile(vxb_ctx* ctx, const double* values, uint64_t n, double level, double* out);
/* v[i] <- v[i] / divisor with IEEE division (the weight normalisation). */
int vxb_divide(vxb_ctx* ctx, double* v, uint64_t n, double divisor);
int vxb_make_kernel(const double* cov, uint32_t dim, double scale, double jitter, double* chol);

/* ------------------ likelihood-annealed SMC / weak-informativity test */
/* The bioassay model (weak_info.cpp:18-160): M dose groups, group sizes n_g,
 * deaths y_g, p_g = 1/(1 + exp(b0 + b1 x_g)), prior (b0, b1) ~ N(0, diag(l1, l2)^2).
 *
 * vxb_bioassay_log_likelihood: bioassay_block_log_likelihood (weak_info.cpp:72-80)
 *   over `lanes` (b0, b1) pairs, row-major.
 * vxb_bioassay_sample: n independent sample_prior_predictive draws
 *   (weak_info.cpp:82-106), draw j from RngStream(seeds[j], 0) under the prior
 *   lambda[2j..2j+1]; theta (optional) n x 2, deaths n x groups.
 * vxb_smc_bioassay: n_runs independent evidence estimates, run r = smc::run_smc
 *   (smc.cpp:352-488; workers = 1, fixed proposal scale, SmcConfig defaults) on
 *   make_bioassay_model(deaths[r], lambda[r]) with seed seeds[r] -- the
 *   evidence_of closure of weak_info.cpp:200-215.  One CTA per run.  status[r]:
 *   0 ok, 1 invalid-model, 2 degenerate-ensemble, 3 non-convergence (the errors
 *   the reference turns into a skipped evidence); log_evidence is NaN then.
 *   trace (optional): n_runs x trace_rows x 6 doubles per iteration: temperature,
 *   ESS after reweighting, move steps R_n, pilot acceptance, log evidence so far,
 *   proposal scale h (the columns of SmcConfig::trace, smc.hpp:125).
 * vxb_smc_bioassay_ensemble: ONE run returning what SmcResult holds: log evidence,
 *   iterations and the final ensemble as 5 x particles doubles (theta0, theta1,
 *   log weights, log likelihoods, log priors); sampler failures are errors
 *   (invalid-model / degenerate-ensemble / non-convergence) as in the reference.
 *   n_scales > 0 (at most 16): SmcConfig::esjd = true with esjd_scales as the grid --
 *   the ESJD scale adaptation (esjd_core, smc.cpp:156-204) replaces the pilot sweep
 *   and the fixed number of move steps; `scale` is then unused.
 *   deaths, lambda, seeds: host arrays.  particles <= 2048. */
int vxb_bioassay_log_likelihood(vxb_ctx* ctx, const double* beta, uint64_t lanes, uint32_t groups,
                                const double* dose, const uint32_t* group_size,
                                const uint32_t* deaths, double* out);
int vxb_bioassay_sample(vxb_ctx* ctx, uint64_t n, uint32_t groups, const double* dose,
                        const uint32_t* group_size, const double* lambda, const uint64_t* seeds,
                        double* theta, uint32_t* deaths);
int vxb_smc_bioassay(vxb_ctx* ctx, uint64_t n_runs, uint32_t groups, const double* dose,
                     const uint32_t* group_size, const uint32_t* deaths, const double* lambda,
                     const uint64_t* seeds, uint64_t particles, uint64_t block_width, double c,
                     double scale, double* log_evidence, uint32_t* iterations, uint8_t* status,
                     double* trace, uint32_t trace_rows);

int vxb_smc_bioassay_ensemble(vxb_ctx* ctx, uint32_t groups, const double* dose,
                              const uint32_t* group_size, const uint32_t* deaths,
                              const double* lambda, uint64_t seed, uint64_t particles,
                              uint64_t block_width, double c, double scale, double* log_evidence,
                              uint32_t* iterations, double* ensemble, double* trace,
                              uint32_t trace_rows, const double* esjd_scales, uint32_t n_scales);

/* WeakInfoConfig (weak_info.hpp:62-75) as a POD; `workers` has no device meaning
 * (all 2 (K+1) N sampler runs are one launch). */
typedef struct vxb_weakinfo_cfg {
    uint64_t hyper_count;  /* K                                   */
    uint64_t datasets;     /* N per prior                         */
    uint64_t particles;    /* N_p                                 */
    uint64_t block_width;  /* validated (blocked.cpp:10-12) only  */
    uint64_t seed;
    double alpha;
    double c;
    double scale;          /* h; <= 0 selects 2.38/sqrt(2)        */
    double base[2];        /* base prior (10, 2.5)                */
    int32_t redraw_base;
    uint32_t groups;
    uint32_t group_size[16];
    double dose[16];
    int32_t arith;         /* VXB_ARITH_EXACT (0, the reference's arithmetic) or VXB_ARITH_FMA:
                              same random numbers and polynomials, multiply-adds contracted */
    int32_t rng;           /* VXB_RNG_REF (0, the reference's streams) or VXB_RNG_FAST: throughput
                              generator (Philox4x32, table-based normals / log / softplus, FMA);
                              statistically validated, not variate-for-variate */
} vxb_weakinfo_cfg;

/* run_weak_info_test (weak_info.cpp:163-277): outputs per row k = 0..K (row 0 is
 * the base prior): lambda (K+1) x 2, gamma, weakly_informative, completed.
 * evidence (optional): (K+1) x N x 2 log evidences, [k][i][0] base data,
 * [k][i][1] data drawn under prior k (NaN where the sampler failed). */
int vxb_weak_info_test(vxb_ctx* ctx, const vxb_weakinfo_cfg* cfg, double* lambda, double* gamma,
                       uint8_t* weakly, uint64_t* completed, double* evidence);
/* The three stages of the test, exposed so that a multi-GPU host can shard the
 * rows (hyperparameters) over ranks -- the reference's own task parallelism
 * (weak_info.cpp:248-262) -- and all-gather the evidences:
 * lambdas:  the K+1 hyperparameter rows (host output, (K+1) x 2).
 * evidence: rows [first_row, first_row+n_rows): n_rows x N x 2 log evidences.
 * cutoffs:  p-values, alpha-cut-offs and flags from the full evidence table
 *           ((K+1) x N x 2, NaN = failed run); host only, no GPU needed. */
int vxb_weak_info_lambdas(vxb_ctx* ctx, const vxb_weakinfo_cfg* cfg, double* lambda);
int vxb_weak_info_evidence(vxb_ctx* ctx, const vxb_weakinfo_cfg* cfg, const double* lambda,
                           uint64_t first_row, uint64_t n_rows, double* evidence);
int vxb_weak_info_cutoffs(const vxb_weakinfo_cfg* cfg, const double* evidence, double* gamma,
                          uint8_t* weakly, uint64_t* completed);

/* ------------------------------------------------ tau-leap MLMC (C4) */
typedef struct vxb_mlmc_cfg {
    uint32_t levels;       /* L+1 levels, l = 0..L              */
    uint32_t refine;       /* M: tau_l = tau0 * M^-l  (4)       */
    double tau0;
    double t_end;
    uint64_t paths;        /* per level                         */
    uint64_t seed;
} vxb_mlmc_cfg;

/* Raw sums of level `level` over paths [first, first+count):
 * sums[0] = sum Y, sums[1] = sum Y^2 (exact integers), sums[2] = sum of the
 * fine path's P(T), sums[3] = Poisson inversion iterations (cost diagnostic).
 * Y = P_fine(T) - P_coarse(T) for level >= 1, P(T) for level 0.
 * y_out (optional): count int32 values of Y. */
int vxb_mlmc_level(vxb_ctx* ctx, const vxb_model* model, const vxb_mlmc_cfg* cfg, uint32_t level,
                   uint64_t first, uint64_t count, int64_t* sums, int32_t* y_out);

typedef struct vxb_mlmc_out {
    double* level_mean;   /* levels                         */
    double* level_var;    /* levels (n-1 divisor)           */
    double* level_cost;   /* levels: fine+coarse steps/path */
    double estimate;
    double std_error;
} vxb_mlmc_out;
int vxb_mlmc_tauleap(vxb_ctx* ctx, const vxb_model* model, const vxb_mlmc_cfg* cfg,
                     vxb_mlmc_out* out);

/* ------------------------------------------------------------ multi-GPU */
/* The path shards by rows with no data-path collective: every variate is keyed by
 * a global row number, so rank r of G simulating partition(n, G, 1)[r]
 * (blocked.cpp:34-63) produces exactly the rows one GPU would.  What the reference
 * does with `workers` std::threads (abc.cpp:43-71, smc.cpp:58-61,
 * weak_info.cpp:258-270) the library does with one vxb_ctx per GPU.  NCCL is used
 * INSIDE the library (loaded with dlopen("libnccl.so.2") on first use, so a
 * single-GPU host needs no NCCL) and only for the exchange of results: the
 * gather of accepted samples below.
 *
 * Two ways to drive several GPUs:
 *  - one PROCESS per GPU (torchrun, MPI): each rank creates its vxb_ctx, rank 0
 *    calls vxb_comm_unique_id and ships the 128 bytes to the others by its own
 *    means, every rank calls vxb_comm_init_rank; the vxb_sharded_* entry points
 *    are then called by all ranks (SPMD);
 *  - one process, several GPUs (the C++ shim): vxb_multi_init creates a context
 *    and a communicator per device; the vxb_multi_* entry points fork one host
 *    thread per device and join, as the reference's drivers do. */
typedef struct vxb_comm vxb_comm;
typedef struct vxb_multi vxb_multi;
#define VXB_COMM_ID_BYTES 128
enum { VXB_DT_U8 = 0, VXB_DT_I64 = 1, VXB_DT_U64 = 2, VXB_DT_F64 = 3, VXB_DT_U32 = 4 };
enum { VXB_OP_SUM = 0, VXB_OP_MAX = 1 };

int vxb_device_count(int* count);
/* NCCL version code (e.g. 22809) of the library that was loaded; fails with
 * device-error when libnccl.so.2 cannot be loaded. */
int vxb_comm_version(int* version);
int vxb_comm_unique_id(void* id /* VXB_COMM_ID_BYTES */);
/* Collective over the n_ranks callers; the communicator runs on ctx's stream. */
int vxb_comm_init_rank(vxb_ctx* ctx, const void* id, int rank, int n_ranks, vxb_comm** comm);
void vxb_comm_destroy(vxb_comm* comm);
int vxb_comm_rank(const vxb_comm* comm);
int vxb_comm_size(const vxb_comm* comm);
/* Stream-ordered collectives on device buffers of the communicator's GPU
 * (asynchronous: they are queued on the context's stream).  allgather: recv holds
 * n_ranks blocks of `bytes` in rank order.  allreduce: in place. */
int vxb_comm_allgather(vxb_comm* comm, const void* send, void* recv, size_t bytes);
int vxb_comm_allreduce(vxb_comm* comm, void* buf, size_t count, int dtype, int op);


/* SPMD form of config 1 (every rank calls it): rank r simulates the rows
 * partition(n_total, n_ranks, 1)[r] with vxb_abc_reject writing into
 * `packed_local` (device, layout->stride bytes), then ONE all-gather places every
 * rank's block into `packed_all` (device, n_ranks * stride bytes, rank order =
 * ascending row order).  Fully asynchronous: nothing returns to the host and the
 * stream is not synchronised.  comm == NULL: one rank, no gather (packed_all may
 * be NULL). */
int vxb_sharded_abc_reject(vxb_ctx* ctx, vxb_comm* comm, const vxb_model* model,
                           const vxb_keying* key, uint64_t n_total, const double* observed,
                           double epsilon, const vxb_accept_layout* layout, void* packed_local,
                           void* packed_all);
/* SPMD form of config 0's selection (select_epsilon, abc.cpp:74-106) over a distance
 * vector that stays sharded: rank r holds rows [first_row, first_row + n_local) (device or
 * host buffers; n_local may be 0).  The valid counts and, in each of the 6 (fp64) / 3
 * (fp32) digit passes of the radix select, the n_ranks x 2048 integer histograms are
 * all-reduced (ncclAllReduce SUM on uint32 -- exact), so every rank walks to the order
 * statistics of the WHOLE vector and returns the same *epsilon, bit-identical to
 * vxb_select_epsilon on the concatenated rows; no distance leaves its device.  Each rank
 * then compacts its accepted rows (global indices, ascending) into `block_local`
 * (device, VXB_INDEX_BLOCK_BYTES(cap): uint64 count at byte 0 -- it may exceed cap --,
 * indices from byte 16) and ONE all-gather places the blocks in `blocks_all` (device,
 * n_ranks blocks, rank order = ascending row order).  *n_accepted: accepted rows of the
 * whole vector.  cap == 0: epsilon and count only (block pointers may be NULL).  The whole
 * vector holds fewer than 2^32 valid rows.  comm == NULL: one rank. */
#define VXB_INDEX_BLOCK_BYTES(cap) (16ull + ((((uint64_t)(cap)) * 8ull + 15ull) & ~15ull))
int vxb_sharded_select_epsilon(vxb_ctx* ctx, vxb_comm* comm, int precision,
                               const void* rho_local, const uint8_t* failed_local,
                               uint64_t n_local, uint64_t first_row, double accept_fraction,
                               double* epsilon, uint64_t* n_accepted, uint64_t cap,
                               void* block_local, void* blocks_all);
/* SPMD forms of configs 2 and 4 (every rank calls them; comm == NULL: one rank): rank r
 * works on partition(m_total or paths, n_ranks, 1)[r]; ONE ncclAllReduce(SUM) of the
 * 64-bit integer counters (exact in any order); every rank receives the totals of the
 * whole job -- counts / p-values, and the MLMC estimator formed from the exact sums. */
int vxb_sharded_ppp_pvalues(vxb_ctx* ctx, vxb_comm* comm, const vxb_model* model,
                            const double* lambda, const double* log_norm, uint32_t n_lambda,
                            uint64_t m_total, uint64_t seed, double ybar_obs, uint64_t* counts,
                            double* pvalues);
int vxb_sharded_mlmc_tauleap(vxb_ctx* ctx, vxb_comm* comm, const vxb_model* model,
                             const vxb_mlmc_cfg* cfg, vxb_mlmc_out* out);
/* Host-side concatenation of gathered blocks (a HOST copy of packed_all) in rank
 * order: at most cap_out rows are written (*n_written of them); *n_accepted is the
 * full count (a rank whose count exceeded layout->cap contributes only its first cap
 * rows -- check *overflowed).  overflowed and n_written may be NULL. */
int vxb_accept_unpack(const vxb_accept_layout* layout, int precision, uint32_t dim, int n_ranks,
                      const void* packed_all_host, uint64_t cap_out, uint64_t* n_accepted,
                      uint64_t* idx, void* params, void* rho, int* overflowed,
                      uint64_t* n_written);

/* One process, several GPUs.  device_ids == NULL or n_dev == 0: every visible
 * device.  With one device no communicator is created (NCCL is not loaded). */
int vxb_multi_init(vxb_multi** multi, const int* device_ids, int n_dev);
/* Diagnostics for boxes with fewer GPUs than ranks: n_ranks contexts on ONE device
 * joined by a LOOPBACK group instead of NCCL -- a collective is a host rendezvous of the
 * ranks' threads (stream drained, barrier, device-to-device copies, barrier); no kernel
 * ever waits for another rank.  Every vxb_multi_* driver then runs its multi-rank logic
 * (sharding, packed gathers, chunk-total reduction, append order) for real.  A rank that
 * fails releases the ranks waiting for it at the next collective (the call returns the
 * root cause, the group is reset and stays usable); VXB_LOOPBACK_FAIL_RANK=r injects one
 * such failure for the tests.  With NCCL, as in any NCCL program, a rank-local failure in
 * the middle of a call leaves its peers waiting: argument and shape errors are raised
 * identically on every rank before the first collective. */
int vxb_multi_init_loopback(vxb_multi** multi, int device, int n_ranks);
void vxb_multi_shutdown(vxb_multi* multi);
int vxb_multi_size(const vxb_multi* multi);
vxb_ctx* vxb_multi_ctx(vxb_multi* multi, int rank);
vxb_comm* vxb_multi_comm(vxb_multi* multi, int rank); /* NULL with one device */
/* abc::run_prior_predictive (abc.cpp:26-73) with the rows split over the devices
 * by partition(n, G, 1): device g fills rows [begin_g, end_g) of the caller's HOST
 * buffers (no collective; the keying -- VXB_KEY_WORKER included -- addresses rows
 * globally, so the result does not depend on G). */
int vxb_multi_abc_prior_predictive(vxb_multi* multi, const vxb_model* model, const vxb_keying* key,
                                   uint64_t n, const double* observed, void* params,
                                   void* summaries, void* rho, uint8_t* failed);
/* Fused fixed-epsilon rejection over all devices + the NCCL gather of the
 * accepted samples; host outputs as vxb_abc_reject (cap = total rows kept). */
int vxb_multi_abc_reject(vxb_multi* multi, const vxb_model* model, const vxb_keying* key,
                         uint64_t n_total, const double* observed, double epsilon, uint64_t cap,
                         uint64_t* n_accepted, uint64_t* idx, void* params, void* rho);
/* select_epsilon over HOST arrays with every device taking the rows of its partition
 * range (vxb_sharded_select_epsilon on one host thread per device); arguments and
 * results as vxb_select_epsilon. */
int vxb_multi_select_epsilon(vxb_multi* multi, int precision, const void* rho,
                             const uint8_t* failed, uint64_t n, double accept_fraction,
                             double* epsilon, uint64_t cap, uint64_t* n_accepted, uint64_t* idx);
/* Configs 2 and 4 over all devices: the SPMD forms (vxb_sharded_ppp_pvalues /
 * vxb_sharded_mlmc_tauleap) on one host thread per device -- disjoint dataset / path
 * ranges, one all-reduce of the exact integer counters. */
int vxb_multi_ppp_pvalues(vxb_multi* multi, const vxb_model* model, const double* lambda,
                          const double* log_norm, uint32_t n_lambda, uint64_t m_total,
                          uint64_t seed, double ybar_obs, uint64_t* counts, double* pvalues);
int vxb_multi_mlmc_tauleap(vxb_multi* multi, const vxb_model* model, const vxb_mlmc_cfg* cfg,
                           vxb_mlmc_out* out);
/* Config 3 over several GPUs.  SPMD form (every rank calls it; comm == NULL: one rank)
 * and the one-process form.  Same scheme and the same bits as vxb_abcsmc_run for any
 * number of ranks: proposals of a round and new particles of a generation sharded by
 * global index; per round ONE ncclAllGather of the packed accepted proposals, per
 * generation one ncclAllGather of the unnormalised weights and one ncclAllReduce(SUM)
 * of the chunk totals of the weight sum (exact: one non-zero contributor per entry);
 * rounds issued ahead of the host, state on the device (vxb_abcsmc_append_round). */
int vxb_sharded_abcsmc_run(vxb_ctx* ctx, vxb_comm* comm, const vxb_model* model,
                           const vxb_abcsmc_cfg* cfg, const double* observed,
                           vxb_abcsmc_out* out);
int vxb_multi_abcsmc_run(vxb_multi* multi, const vxb_model* model, const vxb_abcsmc_cfg* cfg,
                         const double* observed, vxb_abcsmc_out* out);
/* run_weak_info_test (weak_info.cpp:163-277) with the hyperparameter rows split over
 * the devices -- the reference's own task split over `workers` (weak_info.cpp:248-270);
 * sampler seeds are keyed by (row, dataset): the table does not depend on the device
 * count.  Arguments as vxb_weak_info_test. */
int vxb_multi_weak_info_test(vxb_multi* multi, const vxb_weakinfo_cfg* cfg, double* lambda,
                             double* gamma, uint8_t* weakly, uint64_t* completed,
                             double* evidence);

#ifdef __cplusplus
}
#endif
#endif /* VEXBAYES_CUDA_H */
