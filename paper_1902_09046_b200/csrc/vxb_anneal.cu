// vxb_anneal.cu -- likelihood-annealed SMC evidence estimates for the
// weak-informativity test (the paper's case study 1).
//
// Reference pieces replaced here:
//   bioassay model            weak_info.cpp:18-160 (log1p_exp, ll_lane, hooks)
//   sample_prior_predictive   weak_info.cpp:82-106
//   smc::run_smc              smc.cpp:352-488 with workers = 1, fixed scale:
//     find_temperature :221-253, reweight_and_update_evidence :255-266,
//     resample_multinomial :268-300, make_kernel :311-325, move_range :77-150,
//     steps_from_acceptance :302-309
//   run_weak_info_test        weak_info.cpp:163-277
//
// The test needs 2 (K+1) N independent SMC runs of N_p particles each (the paper:
// K = N = 400, N_p = 500 => 320 800 runs).  The reference spreads hyperparameters
// over threads and runs each sampler serially; here ONE CTA owns one run for its
// whole life: the ensemble (theta, log w, log L, log prior) lives in shared
// memory (six arrays of N_p doubles), the temperature bisection, evidence update, ESS, cumulative weights and
// covariance are block reductions / scans, and the tempered random-walk moves run
// one particle per thread with every variate addressed at the reference's stream
// position (smc.cpp:66-76), so proposals and accept decisions replay the
// reference's.  Nothing but the run descriptors and one evidence per run touches
// HBM.
//
// Arithmetic: the model and the MCMC moves use the reference's polynomial
// fastmath with separately rounded operations (bit-identical given equal inputs);
// the weight algebra calls exp/log where the reference calls libm and sums in a
// fixed tree order, so evidences agree with the CPU to rounding (~1e-13), not bit
// for bit.

#include <algorithm>
#include <cmath>
#include <limits>
#include <vector>

#include "vxb_internal.cuh"

namespace vxb {

constexpr int kAnnealBlock = 128;
constexpr int kMaxGroups = 16;
constexpr uint32_t kMaxIterations = 1000;  // SmcConfig defaults, smc.hpp:119-123
constexpr uint32_t kStepCap = 100;
constexpr double kBisectionTol = 1e-10;
constexpr double kJitter = 1e-10;
enum { kRolePilot = 0, kRoleMove = 1, kRoleTrial = 2, kRoleCoordinator = 3 };       // smc.cpp:21-24
enum { kRunOk = 0, kRunInvalidModel = 1, kRunDegenerate = 2, kRunNoConvergence = 3 };

__host__ __device__ inline uint64_t derive_seed_dev(uint64_t seed, const uint64_t* path, int n) {
    uint64_t h = splitmix64(seed);  // rng.cpp:29-35
    for (int i = 0; i < n; ++i) h = splitmix64(h ^ path[i]);
    return h;
}

struct Design {
    uint32_t groups;
    double dose[kMaxGroups];
    double size[kMaxGroups];
    double log_choose[kMaxGroups][8];  // log C(size_g, y), y <= 7 (host libm); larger sizes: table below
    const double* log_choose_big;      // groups x (max_size + 1), device, or nullptr
    uint32_t big_stride;
};

// -log p = log(1 + e^b): weak_info.cpp:20-24
// A: Exact (separate multiply and add, the reference's arithmetic bit for bit) or Fused
// (VXB_ARITH_FMA: the same polynomials and the same random numbers with the compiler
// free to contract a * b + c, about half the FP64 instructions; results agree with the
// exact mode to rounding as long as no accept decision sits within rounding of its
// threshold)
template <class A>
__device__ __forceinline__ double softplus(double b) {
    const double pos = b > 0.0 ? b : 0.0;
    const double mag = b > 0.0 ? b : -b;
    return A::add(pos, ln_pos<A>(A::add(1.0, exp2_clamped<A>(A::mul(-mag, kInvLn2)))));
}

struct RunModel {  // one dataset under one prior
    double hit[kMaxGroups], miss[kMaxGroups], choose[kMaxGroups];
    double l1, l2, log_norm;
};

// ll_lane: weak_info.cpp:26-40
// throughput-generator instance: table-based 2^z / log2 (vxb_rng.cuh), FMA
__device__ __forceinline__ double softplus_fast(double b, const double2* tbl) {
    const double pos = b > 0.0 ? b : 0.0;
    const double mag = b > 0.0 ? b : -b;
    return fma(kLn2, fast_log2_short(1.0 + fast_exp2_neg4(-mag * kInvLn2, tbl), tbl), pos);
}
template <class A = Exact, bool kFast = false>
__device__ __forceinline__ double log_lik(const Design& d, const RunModel& m, double b0, double b1,
                                          const double2* tbl = nullptr) {
    double total = 0.0;
    for (uint32_t g = 0; g < d.groups; ++g) {
        const double b = A::mad(b1, d.dose[g], b0);
        const double lse = kFast ? softplus_fast(b, tbl) : softplus<A>(b);
        total = A::add(total, m.choose[g]);
        if (m.hit[g] > 0.0) total = A::mad(-m.hit[g], lse, total);
        if (m.miss[g] > 0.0) total = A::mad(m.miss[g], A::sub(b, lse), total);
    }
    return total;
}
// log_prior hook: weak_info.cpp:144-148
template <class A = Exact>
__device__ __forceinline__ double log_prior(const RunModel& m, double b0, double b1) {
    const double a = A::div(b0, m.l1);
    const double b = A::div(b1, m.l2);
    return A::sub(m.log_norm, A::mul(0.5, A::mad(b, b, A::mul(a, a))));
}

// ------------------------------------------------------------ block collectives
// One __syncthreads per reduction: warp results go to one of two alternating
// slots (so the next reduction cannot overwrite values a slow warp is still
// reading), and every thread finishes the reduction itself in warp order -- the
// result is the same value in every thread, a pure function of the inputs.
constexpr int kAnnealWarps = kAnnealBlock / 32;
constexpr int kMaxEsjdScales = 16;
struct BlockScratch {
    double a[2][kAnnealWarps], b[2][kAnnealWarps];
    double scan[kAnnealWarps];  // warp totals of the cumulative-weight scan
    unsigned long long count;   // accepted proposals of a sweep
};
struct Reducer {
    BlockScratch& s;
    int phase = 0;
    __device__ __forceinline__ double max(double v) {
        for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
        if ((threadIdx.x & 31) == 0) s.a[phase][threadIdx.x >> 5] = v;
        __syncthreads();
        double m = s.a[phase][0];
#pragma unroll
        for (int w = 1; w < kAnnealWarps; ++w) m = fmax(m, s.a[phase][w]);
        phase ^= 1;
        return m;
    }
    // two sums at once (fixed order: strided partials, shuffle tree, warps left to right)
    __device__ __forceinline__ void sum2(double& x, double& y) {
        for (int o = 16; o > 0; o >>= 1) {
            x += __shfl_xor_sync(0xffffffffu, x, o);
            y += __shfl_xor_sync(0xffffffffu, y, o);
        }
        if ((threadIdx.x & 31) == 0) {
            s.a[phase][threadIdx.x >> 5] = x;
            s.b[phase][threadIdx.x >> 5] = y;
        }
        __syncthreads();
        double p = 0.0, q = 0.0;
#pragma unroll
        for (int w = 0; w < kAnnealWarps; ++w) {
            p += s.a[phase][w];
            q += s.b[phase][w];
        }
        x = p;
        y = q;
        phase ^= 1;
    }
};

struct Ensemble {  // views into dynamic shared memory, np entries each
    double *t0, *t1, *lw, *ll, *lp;  // current
    double* cum;                     // cumulative weights; staging row of the resampling gather
};

// Reweighted ESS at temperature increment dt >= 0 (smc.cpp:226-239) for an ensemble
// whose log weights are all equal to lw0 -- true whenever the sampler looks for a
// temperature, because it resamples every iteration.  x -> fl(lw0 + dt x) is
// monotone, so the reference's max_i (lw_i + dt ll_i) is fl(lw0 + dt max_i ll_i):
// the maximum of the log likelihoods is taken once per iteration, not once per
// bisection step.
template <bool kFast = false>
__device__ double ess_after(const Ensemble& e, uint32_t np, double dt, double lw0, double ll_max,
                            Reducer& red, const double2* tbl = nullptr) {
    const double top = fma(dt, ll_max, lw0);
    if (top == -INFINITY) return 0.0;
    double s1 = 0.0, s2 = 0.0;
    for (uint32_t i = threadIdx.x; i < np; i += kAnnealBlock) {
        const double x = fma(dt, e.ll[i], lw0) - top;  // <= 0
        const double w = kFast ? fast_exp2_neg4(x * kInvLn2, tbl) : exp(x);
        s1 += w;
        s2 = fma(w, w, s2);
    }
    red.sum2(s1, s2);
    return s1 * s1 / s2;
}
// logsumexp: numeric.cpp:11-18
__device__ double block_logsumexp(const double* x, uint32_t np, Reducer& red) {
    double top = -INFINITY;
    for (uint32_t i = threadIdx.x; i < np; i += kAnnealBlock) top = fmax(top, x[i]);
    top = red.max(top);
    if (!isfinite(top)) return top;
    double acc = 0.0, unused = 0.0;
    for (uint32_t i = threadIdx.x; i < np; i += kAnnealBlock) acc += exp(x[i] - top);
    red.sum2(acc, unused);
    return top + log(acc);
}

struct AnnealParams {
    Design design;
    uint64_t n_runs;
    uint32_t np;
    double c, scale, neg_log_np;
    const uint32_t* deaths;   // n_runs x groups
    const double* lambda;     // n_runs x 2
    const double* log_norm;   // n_runs: -log(2 pi l1 l2) (host libm, weak_info.cpp:135)
    const uint64_t* seeds;    // n_runs
    double* log_evidence;
    uint32_t* iterations;
    uint8_t* status;
    double* trace;            // optional: n_runs x trace_rows x 6 (temperature, ess, steps, p_acc, log evidence, scale)
    uint32_t trace_rows;
    double* ensemble;         // optional: n_runs x 5 x np (theta0, theta1, log w, log L, log prior)
    const double2* fast_table;  // throughput generator: log / trig / exp tables
    uint32_t n_scales;        // ESJD scale adaptation (kEsjd instance): the scale grid
    double scales[kMaxEsjdScales];
};

// One tempered random-walk sweep (move_range, smc.cpp:77-150): particle q, step r
// reads the Gaussian pair q*R + r and the uniform at 2 np R + q R + r of stream
// (seed, id).  Returns this thread's number of accepted proposals.
// The ESJD instance (kJumps) starts at stream position `base` (even), takes the
// proposal scale of particle q from a cyclic grid when one is given, and adds
// h^2 |z|^2 of every accepted proposal to jumps[q] (smc.cpp:138-144).
// kFast: the throughput generator -- proposal (q, r) of stream (iteration, role) takes
// its normal pair from Philox4x32 block (q R + r, noise domain | stream tag) and its
// acceptance uniform from block (q R + r, uniform domain | stream tag) of the run's key;
// table-based Box-Muller, log and softplus.  `key` is then the stream tag.
template <bool kJumps = false, class A = Exact, bool kFast = false>
__device__ uint32_t sweep(const Design& d, const RunModel& m, Ensemble& e, uint32_t np, uint64_t key,
                          uint32_t steps, double temperature, double h_all, double l00, double l10,
                          double l11, uint64_t base = 0, const double* scales = nullptr,
                          uint32_t n_scales = 0, double* jumps = nullptr, const FastKeys* fk = nullptr,
                          const double2* tbl = nullptr) {
    uint32_t accepted = 0;
    const uint64_t unif_base = base + static_cast<uint64_t>(np) * steps * 2;
    for (uint32_t q = threadIdx.x; q < np; q += kAnnealBlock) {
        double c0 = e.t0[q], c1 = e.t1[q], cll = e.ll[q], clp = e.lp[q];
        const double h = (kJumps && n_scales) ? scales[q % n_scales] : h_all;
        for (uint32_t r = 0; r < steps; ++r) {
            const uint64_t pair = (kJumps ? base / 2 : 0) + static_cast<uint64_t>(q) * steps + r;
            double z0, z1;
            if (kFast)
                fast_box_muller(philox4x32(*fk, static_cast<uint32_t>(pair), kDomNoise | static_cast<uint32_t>(key),
                                           0u, 0u), tbl, z0, z1);
            else
                box_muller<A>(philox2x64(key, pair), z0, z1);
            const double inc0 = A::mad(l00, z0, 0.0);
            const double inc1 = A::mad(l11, z1, A::mad(l10, z0, 0.0));
            const double p0 = A::mad(h, inc0, c0);
            const double p1 = A::mad(h, inc1, c1);
            const double lp_new = log_prior<A>(m, p0, p1);
            const double ll_new = log_lik<A, kFast>(d, m, p0, p1, tbl);
            const double log_alpha = A::sub(A::add(A::mul(temperature, A::sub(ll_new, cll)), lp_new), clp);
            double u, log_u;
            if (kFast) {
                const Words32 w = philox4x32(*fk, static_cast<uint32_t>(pair), kDomProposal | static_cast<uint32_t>(key),
                                             0u, 0u);
                u = fast_unit(w.a, w.b);
                log_u = u > 0.0 ? kLn2 * fast_log2_short(u, tbl) : -INFINITY;
            } else {
                const uint64_t upos = unif_base + static_cast<uint64_t>(q) * steps + r;
                const Words w = philox2x64(key, upos >> 1);
                u = to_unit((upos & 1) ? w.w1 : w.w0);
                log_u = u > 0.0 ? ln_pos<A>(u) : -INFINITY;
            }
            if (!isnan(log_alpha) && log_alpha > -INFINITY && log_u <= log_alpha) {
                ++accepted;
                c0 = p0;
                c1 = p1;
                cll = ll_new;
                clp = lp_new;
                if (kJumps) {
                    const double zz = __dadd_rn(__dadd_rn(0.0, __dmul_rn(z0, z0)), __dmul_rn(z1, z1));
                    jumps[q] = __dadd_rn(jumps[q], __dmul_rn(__dmul_rn(h, h), zz));
                }
            }
        }
        e.t0[q] = c0;
        e.t1[q] = c1;
        e.ll[q] = cll;
        e.lp[q] = clp;
    }
    return accepted;
}

// Type-7 median (numeric.cpp:20-36,53) of the `count` values x[offset + j * stride] by
// rank counting (no sort: the samples are a few hundred values in shared memory).
// Every thread returns the same value.
__device__ double block_median(const double* x, uint32_t count, uint32_t stride, uint32_t offset,
                               BlockScratch& s) {
    const double hpos = static_cast<double>(count - 1) * 0.5;
    const uint32_t lo = static_cast<uint32_t>(hpos);
    const uint32_t want_hi = (count > 1 && lo + 1 < count) ? lo + 1 : lo;
    __syncthreads();
    for (uint32_t j = threadIdx.x; j < count; j += kAnnealBlock) {
        const double v = x[offset + j * stride];
        uint32_t rank = 0;
        for (uint32_t k = 0; k < count; ++k) {
            const double o = x[offset + k * stride];
            rank += (o < v || (o == v && k < j)) ? 1 : 0;
        }
        if (rank == lo) s.a[0][0] = v;
        if (rank == want_hi) s.a[0][1] = v;
    }
    __syncthreads();
    const double v_lo = s.a[0][0], v_hi = s.a[0][1];
    __syncthreads();
    if (count == 1) return v_lo;
    if (lo + 1 >= count) return v_hi;  // (not reached at level 0.5; kept for the general rule)
    const double frac = hpos - static_cast<double>(lo);
    return __dadd_rn(v_lo, __dmul_rn(frac, __dsub_rn(v_hi, v_lo)));
}

// kEsjd: the ESJD scale adaptation of run_smc (esjd_core, smc.cpp:156-204) instead of
// the fixed-scale pilot + move sweeps.  A separate instance so that the fixed-scale
// kernel (the weak-informativity test's) keeps its register budget.
#ifndef VXB_ANNEAL_CTAS
#define VXB_ANNEAL_CTAS 6  // swept 4-8 at the paper size of the weak-informativity test: 0.40 / 0.37 / 0.353 / 0.366 / 0.367 s
#endif
// kMode: 0 the reference's arithmetic and streams; 1 the same streams with contracted
// multiply-adds (VXB_ARITH_FMA); 2 the throughput generator (VXB_RNG_FAST) with FMA.
template <bool kEsjd, int kMode>
__global__ void __launch_bounds__(kAnnealBlock, VXB_ANNEAL_CTAS) anneal_kernel(const __grid_constant__ AnnealParams p) {
    using A = typename std::conditional<kMode != 0, Fused, Exact>::type;
    constexpr bool kFast = kMode == 2;
    __shared__ double2 s_tab[kFast ? kFastTableSize : 1];
    __shared__ FastKeys s_fk;
    extern __shared__ double smem[];
    __shared__ BlockScratch scratch;
    Reducer red{scratch};
    __shared__ RunModel model;
    const uint64_t run = blockIdx.x;
    const uint32_t np = p.np;
    Ensemble e;
    e.t0 = smem;
    e.t1 = e.t0 + np;
    e.lw = e.t1 + np;
    e.ll = e.lw + np;
    e.lp = e.ll + np;
    e.cum = e.lp + np;
    const Design& d = p.design;

    if (threadIdx.x == 0) {
        model.l1 = p.lambda[2 * run];
        model.l2 = p.lambda[2 * run + 1];
        model.log_norm = p.log_norm[run];
        for (uint32_t g = 0; g < d.groups; ++g) {
            const uint32_t y = p.deaths[run * d.groups + g];
            model.hit[g] = static_cast<double>(y);
            model.miss[g] = d.size[g] - static_cast<double>(y);
            model.choose[g] = d.log_choose_big ? d.log_choose_big[g * d.big_stride + y] : d.log_choose[g][y];
        }
    }
    const uint64_t seed_hash = splitmix64(p.seeds[run]);
    if (kFast) {
        for (int i = threadIdx.x; i < kFastTableSize; i += kAnnealBlock) s_tab[i] = p.fast_table[i];
        if (threadIdx.x == 0) {  // the run's Philox4x32 key schedule (make_fast_keys)
            const uint64_t kk = splitmix64(seed_hash);
            uint32_t k0 = static_cast<uint32_t>(kk), k1 = static_cast<uint32_t>(kk >> 32);
            for (int r = 0; r < 10; ++r) {
                s_fk.rk[2 * r] = k0;
                s_fk.rk[2 * r + 1] = k1;
                k0 += 0x9E3779B9u;
                k1 += 0xBB67AE85u;
            }
        }
    }
    __syncthreads();
    // exact / FMA: the reference's stream key of (iteration, role); throughput generator:
    // the tag that separates the streams inside the counter's domain word
    const auto key_of = [&](uint32_t iteration, uint32_t role) -> uint64_t {
        if (kFast) return (role << 8) | (iteration << 12);
        return stream_key(seed_hash, static_cast<uint32_t>((iteration << 16) | role));  // smc.cpp:26-28
    };

    // ---- initial ensemble: prior draw i = Gaussian pair i of the pilot stream (smc.cpp:386-393)
    int bad = 0, finite_any = 0;
    {
        const uint64_t key = key_of(0, kRolePilot);
        for (uint32_t i = threadIdx.x; i < np; i += kAnnealBlock) {
            double z0, z1;
            if (kFast)
                fast_box_muller(philox4x32(s_fk, i, kDomPrior | static_cast<uint32_t>(key), 0u, 0u), s_tab, z0, z1);
            else
                box_muller<A>(philox2x64(key, i), z0, z1);
            const double b0 = A::mul(model.l1, z0), b1 = A::mul(model.l2, z1);
            const double ll = log_lik<A, kFast>(d, model, b0, b1, s_tab);
            e.t0[i] = b0;
            e.t1[i] = b1;
            e.lw[i] = p.neg_log_np;
            e.ll[i] = ll;
            e.lp[i] = log_prior<A>(model, b0, b1);
            bad |= (isnan(ll) || ll == INFINITY) ? 1 : 0;
            finite_any |= ll > -INFINITY ? 1 : 0;
        }
    }
    bad = __syncthreads_or(bad);
    finite_any = __syncthreads_or(finite_any);
    int status = (bad || !finite_any) ? kRunInvalidModel : kRunOk;

    double temperature = 0.0, log_evidence = 0.0;
    const double h = p.scale > 0.0 ? p.scale : 2.38 / sqrt(2.0);
    const double half = static_cast<double>(np) / 2.0;
    uint32_t n = 0;
    while (status == kRunOk && temperature < 1.0) {
        ++n;
        if (n > kMaxIterations) {
            status = kRunNoConvergence;
            break;
        }
        // ---- find_temperature (smc.cpp:221-253)
        double t_next = 1.0;
        {
            const double room = 1.0 - temperature;
            double ll_max = -INFINITY;
            for (uint32_t i = threadIdx.x; i < np; i += kAnnealBlock) ll_max = fmax(ll_max, e.ll[i]);
            ll_max = red.max(ll_max);
            if (!(ess_after<kFast>(e, np, room, p.neg_log_np, ll_max, red, s_tab) >= half)) {
                double lo = 0.0, hi = room;
                while (hi - lo > kBisectionTol) {
                    const double mid = 0.5 * (lo + hi);
                    if (ess_after<kFast>(e, np, mid, p.neg_log_np, ll_max, red, s_tab) >= half) lo = mid; else hi = mid;
                }
                t_next = temperature + 0.5 * (lo + hi);
            }
        }
        // ---- reweight_and_update_evidence (smc.cpp:255-266)
        {
            const double before = block_logsumexp(e.lw, np, red);
            const double dt = t_next - temperature;
            for (uint32_t i = threadIdx.x; i < np; i += kAnnealBlock) e.lw[i] = fma(dt, e.ll[i], e.lw[i]);
            __syncthreads();
            log_evidence += block_logsumexp(e.lw, np, red) - before;
            temperature = t_next;
        }
        // ---- ess (trace only) and cumulative weights (smc.cpp:208-219, 268-283)
        double top = -INFINITY;
        for (uint32_t i = threadIdx.x; i < np; i += kAnnealBlock) top = fmax(top, e.lw[i]);
        top = red.max(top);
        if (top == -INFINITY) {
            status = kRunDegenerate;
            break;
        }
        double ess_now = 0.0;
        {
            // contiguous chunk per thread, sequential inside, exclusive scan of the chunk totals
            const uint32_t chunk = (np + kAnnealBlock - 1) / kAnnealBlock;
            const uint32_t i0 = min(np, threadIdx.x * chunk), i1 = min(np, i0 + chunk);
            double run_sum = 0.0, sq = 0.0;
            for (uint32_t i = i0; i < i1; ++i) {
                const double w = exp(e.lw[i] - top);
                run_sum += w;
                sq = fma(w, w, sq);
                e.cum[i] = run_sum;
            }
            // inclusive scan over threads: warp shuffle, then warp totals
            double incl = run_sum;
            for (int o = 1; o < 32; o <<= 1) {
                const double up = __shfl_up_sync(0xffffffffu, incl, o);
                if ((threadIdx.x & 31) >= o) incl += up;
            }
            if ((threadIdx.x & 31) == 31) scratch.scan[threadIdx.x >> 5] = incl;
            __syncthreads();
            double offset = incl - run_sum;
            for (int w = 0; w < (threadIdx.x >> 5); ++w) offset += scratch.scan[w];
            __syncthreads();
            for (uint32_t i = i0; i < i1; ++i) e.cum[i] += offset;
            double s1 = run_sum;
            red.sum2(s1, sq);
            ess_now = s1 * s1 / sq;
        }
        __syncthreads();
        const double total = e.cum[np - 1];
        if (!(isfinite(total) && total > 0.0)) {
            status = kRunDegenerate;
            break;
        }
        // ---- resample_multinomial draws (smc.cpp:285-299): draw i = position i of the coordinator stream
        {
            // (the resampling uniforms stay on the reference stream in every mode)
            const uint64_t key = stream_key(seed_hash, static_cast<uint32_t>((n << 16) | kRoleCoordinator));
            // ancestor indices are parked in the log-weight array (reset right after)
            uint32_t* const anc = reinterpret_cast<uint32_t*>(e.lw);
            for (uint32_t i = threadIdx.x; i < np; i += kAnnealBlock) {
                const Words w = philox2x64(key, i >> 1);
                const double target = __dmul_rn(to_unit((i & 1) ? w.w1 : w.w0), total);
                uint32_t lo = 0, hi = np;  // std::upper_bound, clamped
                while (lo < hi) {
                    const uint32_t mid = lo + ((hi - lo) >> 1);
                    if (target < e.cum[mid]) hi = mid; else lo = mid + 1;
                }
                anc[i] = lo >= np ? np - 1 : lo;
            }
            __syncthreads();
            // gather the cached rows one array at a time through `cum` (free once the
            // ancestors are known): thread i reads X[anc[i]], all threads meet, thread i
            // writes X[i]
            double* const rows[4] = {e.t0, e.t1, e.ll, e.lp};
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                for (uint32_t i = threadIdx.x; i < np; i += kAnnealBlock) e.cum[i] = rows[r][anc[i]];
                __syncthreads();
                for (uint32_t i = threadIdx.x; i < np; i += kAnnealBlock) rows[r][i] = e.cum[i];
            }
            for (uint32_t i = threadIdx.x; i < np; i += kAnnealBlock) e.lw[i] = p.neg_log_np;
        }
        // ---- make_kernel: sample covariance + Cholesky + jitter (numeric.cpp:55-96, smc.cpp:311-325)
        double l00, l10, l11;
        {
            double m0 = 0.0, m1 = 0.0;
            for (uint32_t i = threadIdx.x; i < np; i += kAnnealBlock) {
                m0 += e.t0[i];
                m1 += e.t1[i];
            }
            red.sum2(m0, m1);
            m0 /= static_cast<double>(np);
            m1 /= static_cast<double>(np);
            double c00 = 0.0, c10 = 0.0, c11 = 0.0, unused = 0.0;
            for (uint32_t i = threadIdx.x; i < np; i += kAnnealBlock) {
                const double d0 = e.t0[i] - m0, d1 = e.t1[i] - m1;
                c00 = fma(d0, d0, c00);
                c10 = fma(d1, d0, c10);
                c11 = fma(d1, d1, c11);
            }
            red.sum2(c00, c10);
            red.sum2(c11, unused);
            const double norm = 1.0 / static_cast<double>(np - 1);
            c00 *= norm;
            c10 *= norm;
            c11 *= norm;
            bool ok = false;
            for (int attempt = 0; attempt < 2 && !ok; ++attempt) {
                const double a00 = c00 + (attempt ? kJitter : 0.0), a11 = c11 + (attempt ? kJitter : 0.0);
                if (a00 > 0.0) {
                    l00 = sqrt(a00);
                    l10 = c10 / l00;
                    const double rest = a11 - l10 * l10;
                    if (rest > 0.0) {
                        l11 = sqrt(rest);
                        ok = true;
                    }
                }
            }
            if (!ok) {
                status = kRunDegenerate;
                break;
            }
        }
        double p_acc, h_used = h;
        uint32_t steps;
        if (!kEsjd) {
            // ---- pilot sweep, step count, move sweep (smc.cpp:441-452)
            uint32_t acc = sweep<false, A, kFast>(d, model, e, np, key_of(n, kRolePilot), 1, temperature, h, l00, l10,
                                                  l11, 0, nullptr, 0, nullptr, &s_fk, s_tab);
            if (threadIdx.x == 0) scratch.count = 0;
            __syncthreads();
            atomicAdd(&scratch.count, static_cast<unsigned long long>(acc));
            __syncthreads();
            p_acc = static_cast<double>(scratch.count) / static_cast<double>(np);
            __syncthreads();
            {   // steps_from_acceptance: smc.cpp:302-309
                const double pc = fmin(fmax(p_acc, 0.01), 0.99);
                const double raw = ceil(log(p.c) / log(1.0 - pc));
                steps = !(raw >= 1.0) ? 1u : static_cast<uint32_t>(fmin(raw, static_cast<double>(kStepCap)));
            }
            sweep<false, A, kFast>(d, model, e, np, key_of(n, kRoleMove), steps, temperature, h, l00, l10, l11, 0,
                                   nullptr, 0, nullptr, &s_fk, s_tab);
            __syncthreads();
        } else {
            // ---- esjd_core (smc.cpp:156-204).  The jump distances live in the log-weight
            // array (every log weight is -log N after the resampling; restored below).
            double* const jumps = e.lw;
            for (uint32_t i = threadIdx.x; i < np; i += kAnnealBlock) jumps[i] = 0.0;
            __syncthreads();
            uint32_t acc = sweep<true>(d, model, e, np, key_of(n, kRoleTrial), 1, temperature, 0.0, l00, l10,
                                       l11, 0, p.scales, p.n_scales, jumps);
            if (threadIdx.x == 0) scratch.count = 0;
            __syncthreads();
            atomicAdd(&scratch.count, static_cast<unsigned long long>(acc));
            __syncthreads();
            p_acc = static_cast<double>(scratch.count) / static_cast<double>(np);
            const double trial_median = block_median(jumps, np, 1, 0, scratch);
            double best = -1.0;
            bool any_jump = false;
            h_used = 0.0;
            for (uint32_t sidx = 0; sidx < p.n_scales; ++sidx) {
                if (sidx >= np) continue;  // no particle carries this scale
                const uint32_t count = (np - sidx + p.n_scales - 1) / p.n_scales;
                const double med = block_median(jumps, count, p.n_scales, sidx, scratch);
                if (med > 0.0) any_jump = true;
                if (med > best) {
                    best = med;
                    h_used = p.scales[sidx];
                }
            }
            if (!any_jump) {
                int some = 0;
                for (uint32_t i = threadIdx.x; i < np; i += kAnnealBlock) some |= jumps[i] > 0.0 ? 1 : 0;
                any_jump = __syncthreads_or(some) != 0;
            }
            if (!any_jump) h_used = 2.38 / sqrt(2.0);
            steps = 0;
            uint64_t pos = 0;  // position of the move stream (continues from sweep to sweep)
            const uint64_t move_key = key_of(n, kRoleMove);
            while (steps < kStepCap) {
                int moved = 0;
                for (uint32_t i = threadIdx.x; i < np; i += kAnnealBlock) moved += jumps[i] > trial_median ? 1 : 0;
                if (threadIdx.x == 0) scratch.count = 0;
                __syncthreads();
                atomicAdd(&scratch.count, static_cast<unsigned long long>(moved));
                __syncthreads();
                const bool enough = 2 * scratch.count >= np;
                __syncthreads();
                if (enough) break;
                pos += pos & 1;  // align_even
                sweep<true>(d, model, e, np, move_key, 1, temperature, h_used, l00, l10, l11, pos, nullptr, 0,
                            jumps);
                __syncthreads();
                pos += 3ull * np;
                ++steps;
            }
            for (uint32_t i = threadIdx.x; i < np; i += kAnnealBlock) e.lw[i] = p.neg_log_np;
            __syncthreads();
        }
        if (p.trace && threadIdx.x == 0 && n <= p.trace_rows) {
            double* row = p.trace + (run * p.trace_rows + (n - 1)) * 6;
            row[0] = temperature;
            row[1] = ess_now;
            row[2] = static_cast<double>(steps);
            row[3] = p_acc;
            row[4] = log_evidence;
            row[5] = h_used;
        }
    }
    if (p.ensemble) {  // the final ensemble (SmcResult::ensemble)
        __syncthreads();
        double* out = p.ensemble + run * 5 * np;
        const double* rows[5] = {e.t0, e.t1, e.lw, e.ll, e.lp};
#pragma unroll
        for (int r = 0; r < 5; ++r)
            for (uint32_t i = threadIdx.x; i < np; i += kAnnealBlock) out[r * np + i] = rows[r][i];
    }
    if (threadIdx.x == 0) {
        p.log_evidence[run] = status == kRunOk ? log_evidence : __longlong_as_double(0x7FF8000000000000LL);
        p.iterations[run] = n;
        p.status[run] = static_cast<uint8_t>(status);
    }
}

// ------------------------------------------------- prior-predictive datasets
// sample_prior_predictive (weak_info.cpp:82-106) from RngStream(seed, 0): one draw
// per thread.
struct DrawParams {
    Design design;
    uint64_t n;
    const double* lambda;   // n x 2
    const uint64_t* seeds;  // n
    double* theta;          // n x 2 (optional)
    uint32_t* deaths;       // n x groups
};
__global__ void bioassay_draw_kernel(const __grid_constant__ DrawParams p) {
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= p.n) return;
    const Design& d = p.design;
    const uint64_t key = stream_key(splitmix64(p.seeds[i]), 0);
    double z0, z1;
    box_muller<Exact>(philox2x64(key, 0), z0, z1);
    const double b0 = __dmul_rn(p.lambda[2 * i], z0), b1 = __dmul_rn(p.lambda[2 * i + 1], z1);
    if (p.theta) {
        p.theta[2 * i] = b0;
        p.theta[2 * i + 1] = b1;
    }
    uint64_t pos = 2;
    for (uint32_t g = 0; g < d.groups; ++g) {
        const double b = __dadd_rn(b0, __dmul_rn(b1, d.dose[g]));
        const double prob = exp2_clamped<Exact>(__dmul_rn(-softplus<Exact>(b), kInvLn2));
        uint32_t k = 0;
        const uint32_t animals = static_cast<uint32_t>(d.size[g]);
        for (uint32_t j = 0; j < animals; ++j, ++pos) {
            const Words w = philox2x64(key, pos >> 1);
            k += to_unit((pos & 1) ? w.w1 : w.w0) < prob ? 1u : 0u;
        }
        p.deaths[i * d.groups + g] = k;
    }
}

__global__ void bioassay_ll_kernel(Design d, const double* beta, uint64_t lanes, const uint32_t* deaths,
                                   double* out) {
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= lanes) return;
    RunModel m;
    for (uint32_t g = 0; g < d.groups; ++g) {
        m.hit[g] = static_cast<double>(deaths[g]);
        m.miss[g] = d.size[g] - m.hit[g];
        m.choose[g] = d.log_choose_big ? d.log_choose_big[g * d.big_stride + deaths[g]] : d.log_choose[g][deaths[g]];
    }
    out[i] = log_lik(d, m, beta[2 * i], beta[2 * i + 1]);
}

// Run descriptors of the weak-informativity test, built on the device: row k,
// dataset i, which = 0 (base data) / 1 (data from prior k): seeds and priors as in
// weak_info.cpp:217-236.
struct PlanParams {
    uint64_t rows, first_row, datasets, seed;  // rows of this shard; k = first_row + local row
    int redraw_base;
    double base0, base1;
    const double* lambda_rows;  // rows x 2
    double* draw_lambda;        // draws x 2
    uint64_t* draw_seed;        // draws
    double* run_lambda;         // runs x 2
    uint64_t* run_seed;         // runs
};
// draws: [0, rows*datasets): hyper datasets (k, i); then base datasets: shared
// (datasets of them) or redrawn (rows*datasets).
__global__ void weakinfo_plan_kernel(PlanParams p) {
    const uint64_t t = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const uint64_t pairs = p.rows * p.datasets;
    if (t >= pairs) return;
    const uint64_t local = t / p.datasets, k = p.first_row + local, i = t % p.datasets;
    {
        const uint64_t path[3] = {3, k, i};
        p.draw_seed[t] = derive_seed_dev(p.seed, path, 3);
        p.draw_lambda[2 * t] = p.lambda_rows[2 * local];
        p.draw_lambda[2 * t + 1] = p.lambda_rows[2 * local + 1];
    }
    if (p.redraw_base) {
        const uint64_t path[3] = {5, k, i};
        p.draw_seed[pairs + t] = derive_seed_dev(p.seed, path, 3);
        p.draw_lambda[2 * (pairs + t)] = p.base0;
        p.draw_lambda[2 * (pairs + t) + 1] = p.base1;
    } else if (local == 0) {  // the shared base datasets: the same for every shard
        const uint64_t path[2] = {2, i};
        p.draw_seed[pairs + i] = derive_seed_dev(p.seed, path, 2);
        p.draw_lambda[2 * (pairs + i)] = p.base0;
        p.draw_lambda[2 * (pairs + i) + 1] = p.base1;
    }
    for (uint64_t which = 0; which < 2; ++which) {
        const uint64_t r = 2 * t + which;  // run index: (k, i, which)
        const uint64_t path[4] = {4, k, which, i};
        p.run_seed[r] = derive_seed_dev(p.seed, path, 4);
        p.run_lambda[2 * r] = p.lambda_rows[2 * local];
        p.run_lambda[2 * r + 1] = p.lambda_rows[2 * local + 1];
    }
}
// deaths of run (k, i, which) from the draws
__global__ void weakinfo_gather_kernel(uint64_t rows, uint64_t datasets, uint32_t groups, int redraw_base,
                                       const uint32_t* draw_deaths, uint32_t* run_deaths) {
    const uint64_t t = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const uint64_t pairs = rows * datasets;
    if (t >= pairs) return;
    const uint64_t i = t % datasets;
    const uint64_t base_draw = pairs + (redraw_base ? t : i);
    for (uint32_t g = 0; g < groups; ++g) {
        run_deaths[(2 * t) * groups + g] = draw_deaths[base_draw * groups + g];
        run_deaths[(2 * t + 1) * groups + g] = draw_deaths[t * groups + g];
    }
}

// ------------------------------------------------------------------ host side
static Design make_design(vxb_ctx* ctx, uint32_t groups, const double* dose, const uint32_t* group_size,
                          Scratch** big_holder) {
    require(groups >= 1 && groups <= static_cast<uint32_t>(kMaxGroups), "invalid-argument",
            "between 1 and 16 dose groups");
    require(dose && group_size, "invalid-argument", "null design");
    Design d{};
    d.groups = groups;
    uint32_t max_size = 0;
    for (uint32_t g = 0; g < groups; ++g) {
        d.dose[g] = dose[g];
        d.size[g] = static_cast<double>(group_size[g]);
        max_size = std::max(max_size, group_size[g]);
    }
    // log_binomial (numeric.cpp:98-102) on the host, as the reference computes it
    const auto log_choose = [](uint32_t n, uint32_t k) {
        return std::lgamma(static_cast<double>(n) + 1.0) - std::lgamma(static_cast<double>(k) + 1.0) -
               std::lgamma(static_cast<double>(n - k) + 1.0);
    };
    if (max_size <= 7) {
        for (uint32_t g = 0; g < groups; ++g)
            for (uint32_t y = 0; y <= group_size[g]; ++y) d.log_choose[g][y] = log_choose(group_size[g], y);
        d.log_choose_big = nullptr;
    } else {
        const uint32_t stride = max_size + 1;
        std::vector<double> table(static_cast<size_t>(groups) * stride, 0.0);
        for (uint32_t g = 0; g < groups; ++g)
            for (uint32_t y = 0; y <= group_size[g]; ++y) table[g * stride + y] = log_choose(group_size[g], y);
        *big_holder = new Scratch(ctx, table.size() * 8);
        VXB_CUDA(cudaMemcpyAsync((*big_holder)->as<void>(), table.data(), table.size() * 8,
                                 cudaMemcpyHostToDevice, ctx->stream));
        VXB_CUDA(cudaStreamSynchronize(ctx->stream));
        d.log_choose_big = (*big_holder)->as<double>();
        d.big_stride = stride;
    }
    return d;
}

static void check_sampler_args(uint64_t particles, uint64_t block_width, double c) {
    require(block_width == 1 || block_width == 2 || block_width == 4 || block_width == 8 ||
                block_width == 16,
            "invalid-shape", "unsupported block width");  // blocked.cpp:10-12
    require(particles >= 2 * block_width, "invalid-shape", "need at least two particle blocks");
    require(particles <= 2048, "invalid-shape", "at most 2048 particles per device run");
    require(c > 0.0 && c < 1.0, "invalid-argument", "tuning constant must lie in (0, 1)");
}

// all pointers device; log_norm computed here from lambda (host libm)
static void anneal_device(vxb_ctx* ctx, const Design& design, uint64_t n_runs, uint64_t particles, double c,
                          double scale, const uint32_t* deaths, const double* lambda, const double* lambda_host,
                          const uint64_t* seeds, double* log_evidence, uint32_t* iterations, uint8_t* status,
                          double* trace, uint32_t trace_rows, double* ensemble = nullptr,
                          const double* esjd_scales = nullptr, uint32_t n_scales = 0,
                          int arith = VXB_ARITH_EXACT, int rng = VXB_RNG_REF) {
    require(arith == VXB_ARITH_EXACT || arith == VXB_ARITH_FMA, "invalid-argument", "bad arithmetic mode");
    require(n_scales <= kMaxEsjdScales, "invalid-argument", "at most 16 ESJD scales");
    for (uint32_t k = 0; k < n_scales; ++k)
        require(esjd_scales[k] > 0.0, "invalid-scale", "ESJD scales must be positive");
    std::vector<double> norm(n_runs);
    for (uint64_t r = 0; r < n_runs; ++r) {
        require(lambda_host[2 * r] > 0.0 && lambda_host[2 * r + 1] > 0.0, "invalid-argument",
                "prior scales must be positive");
        norm[r] = -std::log(2.0 * 3.141592653589793238462643 * lambda_host[2 * r] * lambda_host[2 * r + 1]);
    }
    Scratch d_norm(ctx, n_runs * 8);
    VXB_CUDA(cudaMemcpyAsync(d_norm.as<void>(), norm.data(), n_runs * 8, cudaMemcpyHostToDevice, ctx->stream));
    AnnealParams p{};
    p.design = design;
    p.n_runs = n_runs;
    p.np = static_cast<uint32_t>(particles);
    p.c = c;
    p.scale = scale;
    p.neg_log_np = -std::log(static_cast<double>(particles));
    p.deaths = deaths;
    p.lambda = lambda;
    p.log_norm = d_norm.as<double>();
    p.seeds = seeds;
    p.log_evidence = log_evidence;
    p.iterations = iterations;
    p.status = status;
    p.trace = trace;
    p.trace_rows = trace_rows;
    p.ensemble = ensemble;
    p.n_scales = n_scales;
    for (uint32_t k = 0; k < n_scales; ++k) p.scales[k] = esjd_scales[k];
    const size_t smem = particles * 6 * sizeof(double);
    require(!(n_scales && arith == VXB_ARITH_FMA), "invalid-argument",
            "the ESJD instance runs in the reference's arithmetic");
    require(rng == VXB_RNG_REF || rng == VXB_RNG_FAST, "invalid-argument", "bad generator mode");
    require(!(n_scales && rng == VXB_RNG_FAST), "invalid-argument",
            "the ESJD instance runs on the reference's streams");
    p.fast_table = ctx->log_table;
    auto kernel = n_scales ? anneal_kernel<true, 0>
                  : rng == VXB_RNG_FAST ? anneal_kernel<false, 2>
                  : arith == VXB_ARITH_FMA ? anneal_kernel<false, 1> : anneal_kernel<false, 0>;
    VXB_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    {
        LaunchScope scope(ctx, VXB_K_RESAMPLE);
        // the grid is one CTA per run; launch in slices below the grid limit
        for (uint64_t first = 0; first < n_runs; first += 1u << 30) {
            AnnealParams q = p;
            const uint64_t count = std::min<uint64_t>(n_runs - first, 1u << 30);
            q.deaths += first * design.groups;
            q.lambda += 2 * first;
            q.log_norm += first;
            q.seeds += first;
            q.log_evidence += first;
            q.iterations += first;
            q.status += first;
            if (q.trace) q.trace += first * trace_rows * 6;
            if (q.ensemble) q.ensemble += first * 5 * particles;
            kernel<<<static_cast<unsigned>(count), kAnnealBlock, smem, ctx->stream>>>(q);
        }
        check_launch("anneal_kernel");
    }
    VXB_CUDA(cudaStreamSynchronize(ctx->stream));  // norm (host vector) must outlive the copy
}

}  // namespace vxb

using namespace vxb;

extern "C" int vxb_bioassay_log_likelihood(vxb_ctx* ctx, const double* beta, uint64_t lanes, uint32_t groups,
                                           const double* dose, const uint32_t* group_size,
                                           const uint32_t* deaths, double* out) {
    return guarded([&] {
        use(ctx);
        require(beta && deaths && out, "invalid-argument", "null argument");
        Scratch* big = nullptr;
        const Design d = make_design(ctx, groups, dose, group_size, &big);
        for (uint32_t g = 0; g < groups; ++g)
            require(deaths[g] <= group_size[g], "invalid-argument", "more deaths than animals in a group");
        Staged d_beta(ctx, beta, lanes * 16, true, false);
        Staged d_y(ctx, deaths, groups * 4, true, false);
        Staged d_out(ctx, out, lanes * 8, false, true);
        {
            LaunchScope scope(ctx, VXB_K_MISC);
            bioassay_ll_kernel<<<grid_for(lanes, 128), 128, 0, ctx->stream>>>(
                d, d_beta.as<double>(), lanes, d_y.as<uint32_t>(), d_out.as<double>());
            check_launch("bioassay_ll_kernel");
        }
        d_out.finish();
        VXB_CUDA(cudaStreamSynchronize(ctx->stream));
        delete big;
    });
}

extern "C" int vxb_bioassay_sample(vxb_ctx* ctx, uint64_t n, uint32_t groups, const double* dose,
                                   const uint32_t* group_size, const double* lambda, const uint64_t* seeds,
                                   double* theta, uint32_t* deaths) {
    return guarded([&] {
        use(ctx);
        require(lambda && seeds && deaths, "invalid-argument", "null argument");
        Scratch* big = nullptr;
        DrawParams p{};
        p.design = make_design(ctx, groups, dose, group_size, &big);
        p.n = n;
        Staged d_l(ctx, lambda, n * 16, true, false);
        Staged d_s(ctx, seeds, n * 8, true, false);
        Staged d_t(ctx, theta, n * 16, false, true);
        Staged d_y(ctx, deaths, n * groups * 4, false, true);
        p.lambda = d_l.as<double>();
        p.seeds = d_s.as<uint64_t>();
        p.theta = d_t.as<double>();
        p.deaths = d_y.as<uint32_t>();
        {
            LaunchScope scope(ctx, VXB_K_MISC);
            bioassay_draw_kernel<<<grid_for(n, 128), 128, 0, ctx->stream>>>(p);
            check_launch("bioassay_draw_kernel");
        }
        d_t.finish();
        d_y.finish();
        VXB_CUDA(cudaStreamSynchronize(ctx->stream));
        delete big;
    });
}

extern "C" int vxb_smc_bioassay(vxb_ctx* ctx, uint64_t n_runs, uint32_t groups, const double* dose,
                                const uint32_t* group_size, const uint32_t* deaths, const double* lambda,
                                const uint64_t* seeds, uint64_t particles, uint64_t block_width, double c,
                                double scale, double* log_evidence, uint32_t* iterations, uint8_t* status,
                                double* trace, uint32_t trace_rows) {
    return guarded([&] {
        use(ctx);
        require(deaths && lambda && seeds && log_evidence, "invalid-argument", "null argument");
        require(!is_device_pointer(lambda) && !is_device_pointer(deaths), "invalid-argument",
                "deaths, lambda and seeds are host arrays");
        check_sampler_args(particles, block_width, c);
        if (n_runs == 0) return;
        for (uint64_t r = 0; r < n_runs; ++r)
            for (uint32_t g = 0; g < groups; ++g)
                require(deaths[r * groups + g] <= group_size[g], "invalid-argument",
                        "more deaths than animals in a group");
        Scratch* big = nullptr;
        const Design d = make_design(ctx, groups, dose, group_size, &big);
        Staged d_y(ctx, deaths, n_runs * groups * 4, true, false);
        Staged d_l(ctx, lambda, n_runs * 16, true, false);
        Staged d_s(ctx, seeds, n_runs * 8, true, false);
        Staged d_ev(ctx, log_evidence, n_runs * 8, false, true);
        Scratch it_tmp(ctx, n_runs * 4), st_tmp(ctx, n_runs);
        Staged d_it(ctx, iterations, n_runs * 4, false, true);
        Staged d_st(ctx, status, n_runs, false, true);
        Staged d_tr(ctx, trace, n_runs * trace_rows * 48, false, true);
        if (trace) VXB_CUDA(cudaMemsetAsync(d_tr.ptr(), 0, n_runs * trace_rows * 48, ctx->stream));
        anneal_device(ctx, d, n_runs, particles, c, scale, d_y.as<uint32_t>(), d_l.as<double>(), lambda,
                      d_s.as<uint64_t>(), d_ev.as<double>(),
                      iterations ? d_it.as<uint32_t>() : it_tmp.as<uint32_t>(),
                      status ? d_st.as<uint8_t>() : st_tmp.as<uint8_t>(), trace ? d_tr.as<double>() : nullptr,
                      trace_rows);
        d_ev.finish();
        d_it.finish();
        d_st.finish();
        d_tr.finish();
        VXB_CUDA(cudaStreamSynchronize(ctx->stream));
        delete big;
    });
}

// One run with its final ensemble: smc::run_smc (smc.cpp:352-488) on
// make_bioassay_model(deaths, lambda) -> SmcResult.
extern "C" int vxb_smc_bioassay_ensemble(vxb_ctx* ctx, uint32_t groups, const double* dose,
                                         const uint32_t* group_size, const uint32_t* deaths,
                                         const double* lambda, uint64_t seed, uint64_t particles,
                                         uint64_t block_width, double c, double scale, double* log_evidence,
                                         uint32_t* iterations, double* ensemble, double* trace,
                                         uint32_t trace_rows, const double* esjd_scales,
                                         uint32_t n_scales) {
    return guarded([&] {
        use(ctx);
        require(deaths && lambda && log_evidence && ensemble, "invalid-argument", "null argument");
        check_sampler_args(particles, block_width, c);
        for (uint32_t g = 0; g < groups; ++g)
            require(deaths[g] <= group_size[g], "invalid-argument", "more deaths than animals in a group");
        Scratch* big = nullptr;
        const Design d = make_design(ctx, groups, dose, group_size, &big);
        Staged d_y(ctx, deaths, groups * 4, true, false);
        Staged d_l(ctx, lambda, 16, true, false);
        Staged d_s(ctx, &seed, 8, true, false);
        Scratch d_ev(ctx, 8), d_it(ctx, 4), d_st(ctx, 1);
        Staged d_en(ctx, ensemble, particles * 40, false, true);
        Staged d_tr(ctx, trace, static_cast<size_t>(trace_rows) * 48, false, true);
        if (trace) VXB_CUDA(cudaMemsetAsync(d_tr.ptr(), 0, static_cast<size_t>(trace_rows) * 48, ctx->stream));
        require(n_scales == 0 || esjd_scales, "invalid-argument", "null scale grid");
        anneal_device(ctx, d, 1, particles, c, scale, d_y.as<uint32_t>(), d_l.as<double>(), lambda,
                      d_s.as<uint64_t>(), d_ev.as<double>(), d_it.as<uint32_t>(), d_st.as<uint8_t>(),
                      trace ? d_tr.as<double>() : nullptr, trace_rows, d_en.as<double>(), esjd_scales, n_scales);
        uint32_t it = 0;
        uint8_t st = 0;
        VXB_CUDA(cudaMemcpyAsync(log_evidence, d_ev.as<void>(), 8, cudaMemcpyDeviceToHost, ctx->stream));
        VXB_CUDA(cudaMemcpyAsync(&it, d_it.as<void>(), 4, cudaMemcpyDeviceToHost, ctx->stream));
        VXB_CUDA(cudaMemcpyAsync(&st, d_st.as<void>(), 1, cudaMemcpyDeviceToHost, ctx->stream));
        d_en.finish();
        d_tr.finish();
        VXB_CUDA(cudaStreamSynchronize(ctx->stream));
        delete big;
        if (iterations) *iterations = it;
        // the reference raises here (smc.cpp:395-402, 208-211, 412-414)
        require(st != kRunInvalidModel, "invalid-model", "log-likelihood is not finite at initialization");
        require(st != kRunDegenerate, "degenerate-ensemble", "all weights are zero");
        require(st != kRunNoConvergence, "non-convergence",
                "temperature failed to reach 1 within the iteration cap");
    });
}

// hyperparameters: lambda_k ~ U([0.1,10] x [0.1,20]) from RngStream(derive_seed(seed,{1}), 0)
// (weak_info.cpp:174-182); next_uniform's clamp (rng.cpp:101-110) on the host
extern "C" int vxb_weak_info_lambdas(vxb_ctx* ctx, const vxb_weakinfo_cfg* cfg, double* lambda) {
    return guarded([&] {
        use(ctx);
        require(cfg && lambda, "invalid-argument", "null argument");
        lambda[0] = cfg->base[0];
        lambda[1] = cfg->base[1];
        if (cfg->hyper_count == 0) return;
        std::vector<uint64_t> words(2 * cfg->hyper_count);
        const uint64_t one = 1;
        require(vxb_rng_fill_u64(ctx, vxb_derive_seed(cfg->seed, &one, 1), 0, 0, words.size(),
                                 words.data()) == 0,
                "internal", vxb_last_error());
        for (uint64_t j = 0; j < words.size(); ++j) {
            const double a = 0.1, b = (j & 1) ? 20.0 : 10.0;
            const double u = static_cast<double>(words[j] >> 11) * 0x1.0p-53;
            const double top = std::nextafter(b, a);
            const double r = a + u * (b - a);
            lambda[2 + j] = r < a ? a : (r > top ? top : r);
        }
    });
}

// evidences of rows [first_row, first_row + n_rows): n_rows x N x 2 (base data, data
// drawn under the row's prior); NaN where the sampler failed
extern "C" int vxb_weak_info_evidence(vxb_ctx* ctx, const vxb_weakinfo_cfg* cfg, const double* lambda,
                                      uint64_t first_row, uint64_t n_rows, double* evidence) {
    return guarded([&] {
        use(ctx);
        require(cfg && lambda && evidence, "invalid-argument", "null argument");
        require(cfg->datasets >= 1, "invalid-argument", "need at least one dataset per prior");
        require(first_row + n_rows <= cfg->hyper_count + 1, "invalid-shape", "row range exceeds the table");
        check_sampler_args(cfg->particles, cfg->block_width, cfg->c);
        if (n_rows == 0) return;
        const uint64_t n = cfg->datasets, pairs = n_rows * n, runs = 2 * pairs;
        Scratch* big = nullptr;
        const Design design = make_design(ctx, cfg->groups, cfg->dose, cfg->group_size, &big);
        const uint32_t groups = cfg->groups;
        const uint64_t base_draws = cfg->redraw_base ? pairs : n, draws = pairs + base_draws;
        Scratch d_rows(ctx, n_rows * 16), d_dl(ctx, draws * 16), d_ds(ctx, draws * 8), d_rl(ctx, runs * 16),
            d_rs(ctx, runs * 8), d_dy(ctx, draws * groups * 4), d_ry(ctx, runs * groups * 4),
            d_it(ctx, runs * 4), d_st(ctx, runs);
        Staged d_ev(ctx, evidence, runs * 8, false, true);
        VXB_CUDA(cudaMemcpyAsync(d_rows.as<void>(), lambda + 2 * first_row, n_rows * 16,
                                 cudaMemcpyHostToDevice, ctx->stream));
        {
            LaunchScope scope(ctx, VXB_K_MISC);
            PlanParams pp{n_rows, first_row, n, cfg->seed, cfg->redraw_base, cfg->base[0], cfg->base[1],
                          d_rows.as<double>(), d_dl.as<double>(), d_ds.as<uint64_t>(), d_rl.as<double>(),
                          d_rs.as<uint64_t>()};
            weakinfo_plan_kernel<<<grid_for(pairs, 128), 128, 0, ctx->stream>>>(pp);
            DrawParams dp{};
            dp.design = design;
            dp.n = draws;
            dp.lambda = d_dl.as<double>();
            dp.seeds = d_ds.as<uint64_t>();
            dp.theta = nullptr;
            dp.deaths = d_dy.as<uint32_t>();
            bioassay_draw_kernel<<<grid_for(draws, 128), 128, 0, ctx->stream>>>(dp);
            weakinfo_gather_kernel<<<grid_for(pairs, 128), 128, 0, ctx->stream>>>(
                n_rows, n, groups, cfg->redraw_base, d_dy.as<uint32_t>(), d_ry.as<uint32_t>());
            check_launch("weak-info plan kernels");
        }
        std::vector<double> run_lambda(runs * 2);
        for (uint64_t t = 0; t < pairs; ++t)
            for (int which = 0; which < 2; ++which) {
                run_lambda[2 * (2 * t + which)] = lambda[2 * (first_row + t / n)];
                run_lambda[2 * (2 * t + which) + 1] = lambda[2 * (first_row + t / n) + 1];
            }
        anneal_device(ctx, design, runs, cfg->particles, cfg->c, cfg->scale, d_ry.as<uint32_t>(),
                      d_rl.as<double>(), run_lambda.data(), d_rs.as<uint64_t>(), d_ev.as<double>(),
                      d_it.as<uint32_t>(), d_st.as<uint8_t>(), nullptr, 0, nullptr, nullptr, 0, cfg->arith, cfg->rng);
        d_ev.finish();
        VXB_CUDA(cudaStreamSynchronize(ctx->stream));
        delete big;
    });
}

// p-values and cut-offs per row (weak_info.cpp:238-246, 108-125, 272-275); host only.
// evidence: (K+1) x N x 2, NaN = failed sampler run.
extern "C" int vxb_weak_info_cutoffs(const vxb_weakinfo_cfg* cfg, const double* evidence, double* gamma,
                                     uint8_t* weakly, uint64_t* completed) {
    return guarded([&] {
        require(cfg && evidence && gamma && weakly && completed, "invalid-argument", "null argument");
        require(cfg->alpha > 0.0 && cfg->alpha < 1.0, "invalid-argument", "alpha must lie in (0, 1)");
        const uint64_t rows = cfg->hyper_count + 1, n = cfg->datasets;
        for (uint64_t k = 0; k < rows; ++k) {
            std::vector<double> base_ev, hyper_ev;
            uint64_t both = 0;
            for (uint64_t i = 0; i < n; ++i) {
                const double eb = evidence[2 * (k * n + i)], eh = evidence[2 * (k * n + i) + 1];
                const bool ok_b = !std::isnan(eb), ok_h = !std::isnan(eh);
                if (ok_b) base_ev.push_back(eb);
                if (ok_h) hyper_ev.push_back(eh);
                both += (ok_b && ok_h) ? 1 : 0;
            }
            completed[k] = both;
            gamma[k] = std::numeric_limits<double>::quiet_NaN();
            if (base_ev.empty() || hyper_ev.empty()) continue;
            std::sort(hyper_ev.begin(), hyper_ev.end());
            std::vector<double> pv(base_ev.size());
            for (size_t i = 0; i < base_ev.size(); ++i)
                pv[i] = static_cast<double>(std::upper_bound(hyper_ev.begin(), hyper_ev.end(), base_ev[i]) -
                                            hyper_ev.begin()) /
                        static_cast<double>(hyper_ev.size());
            std::sort(pv.begin(), pv.end());
            const size_t m = pv.size();  // type-7 quantile, numeric.cpp:20-30
            if (m == 1) {
                gamma[k] = pv[0];
            } else {
                const double hq = static_cast<double>(m - 1) * cfg->alpha;
                const size_t lo = static_cast<size_t>(hq);
                gamma[k] = lo + 1 >= m ? pv[m - 1] : pv[lo] + (hq - static_cast<double>(lo)) * (pv[lo + 1] - pv[lo]);
            }
        }
        for (uint64_t k = 0; k < rows; ++k) weakly[k] = (k != 0 && gamma[k] > gamma[0]) ? 1 : 0;
    });
}

extern "C" int vxb_weak_info_test(vxb_ctx* ctx, const vxb_weakinfo_cfg* cfg, double* lambda, double* gamma,
                                  uint8_t* weakly, uint64_t* completed, double* evidence) {
    return guarded([&] {
        require(cfg && lambda && gamma && weakly && completed, "invalid-argument", "null argument");
        require(cfg->datasets >= 1, "invalid-argument", "need at least one dataset per prior");
        require(cfg->alpha > 0.0 && cfg->alpha < 1.0, "invalid-argument", "alpha must lie in (0, 1)");
        const uint64_t rows = cfg->hyper_count + 1;
        std::vector<double> own;
        if (!evidence) {
            own.resize(rows * cfg->datasets * 2);
            evidence = own.data();
        }
        const auto must = [](int rc) {  // pass a stage's "code: message" through unchanged
            if (rc == 0) return;
            const std::string text = vxb_last_error();
            const size_t cut = text.find(": ");
            if (cut == std::string::npos) throw Error{"internal", text};
            throw Error{text.substr(0, cut), text.substr(cut + 2)};
        };
        must(vxb_weak_info_lambdas(ctx, cfg, lambda));
        must(vxb_weak_info_evidence(ctx, cfg, lambda, 0, rows, evidence));
        must(vxb_weak_info_cutoffs(cfg, evidence, gamma, weakly, completed));
    });
}
