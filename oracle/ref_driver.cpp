// oracle/ref_driver.cpp -- TEST INFRASTRUCTURE, not product code.
//
// A thin extern "C" driver around the UNMODIFIED reference library.  It is
// compiled together with the reference's own translation units, in place
// under /root/reference/proj/core/src, by oracle/Makefile into
// oracle/_ref/libvxb_ref.so (git-ignored).  Nothing from the reference is
// copied into this repository; this file only *calls* the reference API:
//   RngStream / splitmix64 / derive_seed      (vexbayes/rng.hpp)
//   fastmath::*                                (vexbayes/fastmath.hpp)
//   quantile / sample_covariance / cholesky    (vexbayes/numeric.hpp)
//   partition                                  (vexbayes/blocked.hpp)
//   ModelHooks                                 (vexbayes/model.hpp)
//   abc::run_prior_predictive / select_epsilon (vexbayes/abc.hpp)
//   smc::ess / resample_multinomial            (vexbayes/smc.hpp)
//   weakinfo::estimate_pvalues / compute_cutoff(vexbayes/weak_info.hpp)
//   toggle::make_abc_model                     (vexbayes/toggle_switch.hpp)
//   smc::run_smc, weakinfo::make_bioassay_model / sample_prior_predictive /
//   run_weak_info_test / write_csv             (vexbayes/smc.hpp, weak_info.hpp)
//   tb::gillespie_simulate / tb_summaries / make_abc_model (vexbayes/tb_model.hpp)
//   abc::write_csv, bench::write_csv / amdahl_bound / tb_observed_summaries
//                                              (vexbayes/abc.hpp, bench.hpp)
//
// The workloads of BASELINE.json that the reference does not contain (the
// logistic SDE, the normal-mean p-value) are expressed here as ModelHooks /
// RngStream clients in the mould of toggle_switch.cpp:135-152, so that the
// reference's own sampler, RNG and numerics produce the expected values.
// Used (a) to pin oracle/vxb_oracle.cpp, (b) to generate tests/golden/*, and
// (c) as the CPU baseline of bench.py (`cpu_baseline.kind = "reference"`).

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <fstream>
#include <sstream>
#include <limits>
#include <string>
#include <thread>
#include <vector>

#include "vexbayes/abc.hpp"
#include "vexbayes/bench.hpp"
#include "vexbayes/blocked.hpp"
#include "vexbayes/errors.hpp"
#include "vexbayes/fastmath.hpp"
#include "vexbayes/model.hpp"
#include "vexbayes/numeric.hpp"
#include "vexbayes/rng.hpp"
#include "vexbayes/smc.hpp"
#include "vexbayes/tb_model.hpp"
#include "vexbayes/toggle_switch.hpp"
#include "vexbayes/weak_info.hpp"

#include "../include/vexbayes_cuda.h"  // vxb_model only (plain struct)

using namespace vexbayes;

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const Error& e) {
        g_err = e.what();
        return 1;
    } catch (const std::exception& e) {
        g_err = std::string("internal: ") + e.what();
        return 2;
    }
}

// Logistic-growth SDE as a ModelHooks client.  Real = double reproduces the
// fp64 configs; Real = float is the fp32 variant: the prior draw and the
// standard normals come from the same fp64 stream positions and are rounded
// to float once; all state arithmetic is float.
template <class Real>
ModelHooks make_logistic_model(const vxb_model& m, std::vector<Real>* f32_shadow = nullptr) {
    (void)f32_shadow;
    ModelHooks hooks;
    hooks.dim = 3;
    hooks.summary_dim = m.steps / m.obs_stride;
    const std::array<double, 3> lo{m.prior_lo[0], m.prior_lo[1], m.prior_lo[2]};
    const std::array<double, 3> hi{m.prior_hi[0], m.prior_hi[1], m.prior_hi[2]};
    hooks.sample_prior = [lo, hi](RngStream& stream, std::span<double> out) {
        std::array<double, 3> unit;
        stream.fill_uniform(unit, 0.0, 1.0);
        for (std::size_t k = 0; k < 3; ++k) {
            const double th = lo[k] + unit[k] * (hi[k] - lo[k]);
            out[k] = static_cast<double>(static_cast<Real>(th));
        }
    };
    const std::size_t steps = m.steps, stride = m.obs_stride;
    const Real dt = static_cast<Real>(m.dt), sqdt = static_cast<Real>(m.consts[0]);
    const Real x0 = static_cast<Real>(m.x0);
    hooks.simulate = [steps, stride, dt, sqdt, x0](std::span<const double> theta,
                                                   RngStream& stream, std::size_t block_width,
                                                   std::span<double> out) {
        require(is_supported_block_width(block_width), "invalid-shape", "unsupported block width");
        require(steps >= 1 && stride >= 1, "invalid-horizon", "need at least one step");
        stream.align_even();
        std::vector<double> z(steps + (steps & 1));
        stream.fill_gaussian(z, 0.0, 1.0);
        const Real r = static_cast<Real>(theta[0]);
        const Real k = static_cast<Real>(theta[1]);
        const Real sigma = static_cast<Real>(theta[2]);
        const Real a = r * dt;
        const Real c = sigma * sqdt;
        const Real inv_k = Real(1) / k;
        Real x = x0;
        std::size_t next = 0, since = 0;
        for (std::size_t j = 0; j < steps; ++j) {
            const Real zj = static_cast<Real>(z[j]);
            const Real drift = (a * x) * (Real(1) - x * inv_k);
            const Real diff = (c * x) * zj;
            x = (x + drift) + diff;
            if (++since == stride) {
                since = 0;
                if (next < out.size()) out[next++] = static_cast<double>(x);
            }
        }
        for (double v : out) require(std::isfinite(v), "invalid-state", "state left the reals");
    };
    return hooks;
}

ModelHooks logistic_for(const vxb_model& m) {
    return m.precision == VXB_F32 ? make_logistic_model<float>(m) : make_logistic_model<double>(m);
}

// abc::discrepancy in float for the fp32 variant (same order as abc.cpp:16-24).
double discrepancy_f32(std::span<const double> sim, std::span<const double> obs) {
    float ss = 0.0f;
    for (std::size_t i = 0; i < sim.size(); ++i) {
        const float d = static_cast<float>(sim[i]) - static_cast<float>(obs[i]);
        ss += d * d;
    }
    return static_cast<double>(std::sqrt(ss));
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// ---------------------------------------------------------------- substrate
std::uint64_t ref_splitmix64(std::uint64_t z) { return splitmix64(z); }

std::uint64_t ref_derive_seed(std::uint64_t seed, const std::uint64_t* path, std::size_t n) {
    // derive_seed takes an initializer_list; fold the same way it does by
    // chaining single-element calls is NOT equivalent, so dispatch on length.
    switch (n) {
        case 0: return derive_seed(seed, {});
        case 1: return derive_seed(seed, {path[0]});
        case 2: return derive_seed(seed, {path[0], path[1]});
        case 3: return derive_seed(seed, {path[0], path[1], path[2]});
        case 4: return derive_seed(seed, {path[0], path[1], path[2], path[3]});
        default: return 0;
    }
}

int ref_stream_u64(std::uint64_t seed, std::uint32_t id, std::uint64_t pos, std::uint64_t n,
                   std::uint64_t* out) {
    return guarded([&] {
        RngStream s(seed, id);
        s.set_counter(pos);
        for (std::uint64_t i = 0; i < n; ++i) out[i] = s.next_u64();
    });
}

int ref_fill_uniform(std::uint64_t seed, std::uint32_t id, std::uint64_t pos, std::uint64_t n,
                     double a, double b, double* out, std::uint64_t* end_pos) {
    return guarded([&] {
        RngStream s(seed, id);
        s.set_counter(pos);
        s.fill_uniform(std::span<double>(out, n), a, b);
        if (end_pos) *end_pos = s.counter_lo();
    });
}

// n may be odd: the tail is taken with next_gaussian (rng.cpp:112-123).
int ref_fill_gaussian(std::uint64_t seed, std::uint32_t id, std::uint64_t pos, std::uint64_t n,
                      double mu, double sigma, double* out) {
    return guarded([&] {
        RngStream s(seed, id);
        s.set_counter(pos);
        const std::uint64_t even = n & ~std::uint64_t(1);
        // fill_gaussian handles an odd starting position itself but needs an
        // even length; split accordingly.
        if (pos & 1) {
            for (std::uint64_t i = 0; i < n; ++i) out[i] = s.next_gaussian(mu, sigma);
        } else {
            s.fill_gaussian(std::span<double>(out, even), mu, sigma);
            if (n & 1) out[n - 1] = s.next_gaussian(mu, sigma);
        }
    });
}

int ref_fastmath(int fn, const double* x, const double* y, std::uint64_t n, double* out) {
    return guarded([&] {
        for (std::uint64_t i = 0; i < n; ++i) {
            switch (fn) {
                case 0: out[i] = fastmath::log2_pos(x[i]); break;
                case 1: out[i] = fastmath::ln_pos(x[i]); break;
                case 2: out[i] = fastmath::exp2_clamped(x[i]); break;
                case 3: out[i] = fastmath::sinpi(x[i]); break;
                case 4: out[i] = fastmath::cospi(x[i]); break;
                case 5: out[i] = fastmath::pow_pos(x[i], y[i]); break;
                default: raise("invalid-argument", "unknown fastmath function");
            }
        }
    });
}

int ref_quantile(const double* sample, std::uint64_t n, double level, double* out) {
    return guarded([&] { *out = quantile(std::span<const double>(sample, n), level); });
}

int ref_logsumexp(const double* x, std::uint64_t n, double* out) {
    return guarded([&] { *out = logsumexp(std::span<const double>(x, n)); });
}

int ref_sample_covariance(const double* data, std::uint64_t rows, std::uint64_t dim, double* cov) {
    return guarded([&] {
        const auto c = sample_covariance(std::span<const double>(data, rows * dim), rows, dim);
        std::copy(c.begin(), c.end(), cov);
    });
}

// returns 0 ok / 1 not positive definite (a is overwritten either way)
int ref_cholesky(double* a, std::uint64_t dim) {
    return cholesky(std::span<double>(a, dim * dim), dim) ? 0 : 1;
}

int ref_partition(std::uint64_t total, std::uint64_t workers, std::uint64_t width,
                  std::uint64_t* ranges) {
    return guarded([&] {
        const WorkPartition p = partition(total, workers, width);
        for (std::size_t w = 0; w < p.ranges.size(); ++w) {
            ranges[2 * w] = p.ranges[w].first;
            ranges[2 * w + 1] = p.ranges[w].second;
        }
    });
}

double ref_discrepancy(const double* sim, const double* obs, std::uint64_t n) {
    return abc::discrepancy(std::span<const double>(sim, n), std::span<const double>(obs, n));
}

// --------------------------------------------------------------- ABC (C0/C1)
// The real abc::run_prior_predictive on the logistic hooks: worker keying,
// deterministic for (seed, workers, block_width).  fp32: discrepancies are
// recomputed in float from the float-valued summaries.
int ref_logistic_abc(const vxb_model* m, std::uint64_t n, std::uint64_t workers,
                     std::uint64_t block_width, std::uint64_t seed, const double* observed,
                     double* params, double* summaries, double* rho, std::uint8_t* failed) {
    return guarded([&] {
        const ModelHooks hooks = logistic_for(*m);
        const std::size_t sd = hooks.summary_dim;
        std::vector<double> obs(observed, observed + sd);
        if (m->precision == VXB_F32)
            for (double& v : obs) v = static_cast<double>(static_cast<float>(v));
        const abc::PriorPredictiveSet set = abc::run_prior_predictive(
            hooks, n, workers, block_width, seed, std::span<const double>(obs));
        if (params) std::copy(set.params.begin(), set.params.end(), params);
        if (summaries) std::copy(set.summaries.begin(), set.summaries.end(), summaries);
        if (failed) std::copy(set.failed.begin(), set.failed.end(), failed);
        if (rho) {
            for (std::size_t r = 0; r < n; ++r) {
                rho[r] = set.discrepancies[r];
                if (m->precision == VXB_F32 && !set.failed[r])
                    rho[r] = discrepancy_f32(set.summary_row(r), obs);
            }
        }
    });
}

// Particle keying: row i of [first, first+count) owns RngStream(seed, i); the
// per-row sequence is exactly abc.cpp:51-60 (prior, align_even, simulate,
// discrepancy, failure flag).  Rows are spread over `threads` std::threads.
int ref_logistic_abc_particle(const vxb_model* m, std::uint64_t first, std::uint64_t count,
                              std::uint64_t seed, const double* observed, double* params,
                              double* summaries, double* rho, std::uint8_t* failed,
                              unsigned threads) {
    return guarded([&] {
        const ModelHooks hooks = logistic_for(*m);
        const std::size_t d = hooks.dim, sd = hooks.summary_dim;
        std::vector<double> obs(observed, observed + sd);
        if (m->precision == VXB_F32)
            for (double& v : obs) v = static_cast<double>(static_cast<float>(v));
        if (threads < 1) threads = 1;
        auto body = [&](unsigned t) {
            std::vector<double> theta(d), summary(sd);
            for (std::uint64_t r = t; r < count; r += threads) {
                RngStream stream(seed, static_cast<std::uint32_t>(first + r));
                hooks.sample_prior(stream, theta);
                stream.align_even();
                double dist = std::numeric_limits<double>::quiet_NaN();
                std::uint8_t bad = 0;
                try {
                    hooks.simulate(theta, stream, 1, summary);
                    dist = m->precision == VXB_F32 ? discrepancy_f32(summary, obs)
                                                   : abc::discrepancy(summary, obs);
                } catch (const Error&) {
                    bad = 1;
                    std::fill(summary.begin(), summary.end(), 0.0);
                }
                if (params) std::copy(theta.begin(), theta.end(), params + r * d);
                if (summaries) std::copy(summary.begin(), summary.end(), summaries + r * sd);
                if (rho) rho[r] = dist;
                if (failed) failed[r] = bad;
            }
        };
        if (threads == 1) {
            body(0);
        } else {
            std::vector<std::thread> pool;
            for (unsigned t = 0; t < threads; ++t) pool.emplace_back(body, t);
            for (auto& th : pool) th.join();
        }
    });
}

// One simulation at theta from RngStream(seed, id) positioned at pos
// (the way bench.cpp:69-77 builds observed summaries).
int ref_logistic_simulate(const vxb_model* m, const double* theta, std::uint64_t seed,
                          std::uint32_t id, std::uint64_t pos, double* summary) {
    return guarded([&] {
        const ModelHooks hooks = logistic_for(*m);
        RngStream stream(seed, id);
        stream.set_counter(pos);
        std::vector<double> th(theta, theta + 3);
        if (m->precision == VXB_F32)
            for (double& v : th) v = static_cast<double>(static_cast<float>(v));
        hooks.simulate(th, stream, 1, std::span<double>(summary, hooks.summary_dim));
    });
}

// The real abc::select_epsilon on caller-supplied discrepancies.
int ref_select_epsilon(const double* rho, const std::uint8_t* failed, std::uint64_t n, double q,
                       double* eps, std::uint64_t cap, std::uint64_t* n_acc, std::uint64_t* idx) {
    return guarded([&] {
        abc::PriorPredictiveSet set;
        set.rows = n;
        set.dim = 0;
        set.summary_dim = 0;
        set.discrepancies.assign(rho, rho + n);
        if (failed) {
            set.failed.assign(failed, failed + n);
        } else {
            set.failed.assign(n, 0);
        }
        const abc::EpsilonSelection sel = abc::select_epsilon(set, q);
        *eps = sel.epsilon;
        *n_acc = sel.accepted.size();
        if (idx)
            for (std::size_t i = 0; i < sel.accepted.size() && i < cap; ++i) idx[i] = sel.accepted[i];
    });
}

// Toggle-switch ABC exactly as bench.cpp:97-103 runs it (known-answer values
// of SURVEY.md section 8c).
int ref_toggle_abc(std::uint64_t steps, std::uint64_t cells, std::uint64_t n,
                   std::uint64_t workers, std::uint64_t block_width, std::uint64_t seed,
                   double* observed_out, double* params, double* summaries, double* rho,
                   std::uint8_t* failed) {
    return guarded([&] {
        const toggle::ToggleParams theta{325.0, 0.275, 0.2, 25.0, 25.0, 3.5, 3.5};
        RngStream stream(derive_seed(seed, {90}), 0);
        const auto obs = toggle::simulate(theta, steps, cells, stream, block_width);
        const auto q = toggle::summary_quantiles(obs);
        const std::vector<double> observed(q.begin(), q.end());
        if (observed_out) std::copy(observed.begin(), observed.end(), observed_out);
        const ModelHooks model = toggle::make_abc_model(steps, cells);
        const auto set = abc::run_prior_predictive(model, n, workers, block_width, seed, observed);
        if (params) std::copy(set.params.begin(), set.params.end(), params);
        if (summaries) std::copy(set.summaries.begin(), set.summaries.end(), summaries);
        if (rho) std::copy(set.discrepancies.begin(), set.discrepancies.end(), rho);
        if (failed) std::copy(set.failed.begin(), set.failed.end(), failed);
    });
}

// Raw toggle observations y[cells] for one theta (test_toggle.cpp:122-143).
int ref_toggle_simulate(const double* theta7, std::uint64_t steps, std::uint64_t cells,
                        std::uint64_t seed, std::uint32_t id, std::uint64_t pos,
                        std::uint64_t block_width, double* y, std::uint64_t* end_pos) {
    return guarded([&] {
        RngStream stream(seed, id);
        stream.set_counter(pos);
        const auto obs = toggle::simulate(
            toggle::ToggleParams::from_span(std::span<const double>(theta7, 7)), steps, cells,
            stream, block_width);
        std::copy(obs.y.begin(), obs.y.end(), y);
        if (end_pos) *end_pos = stream.counter_lo();
    });
}

// ------------------------------------------------------------ p-values (C2)
int ref_estimate_pvalues(const double* base, std::uint64_t nb, const double* k, std::uint64_t nk,
                         double* out) {
    return guarded([&] {
        const auto p = weakinfo::estimate_pvalues(std::span<const double>(base, nb),
                                                  std::span<const double>(k, nk));
        std::copy(p.begin(), p.end(), out);
    });
}

int ref_compute_cutoff(const double* p, std::uint64_t n, double alpha, double* out) {
    return guarded([&] { *out = weakinfo::compute_cutoff(std::span<const double>(p, n), alpha); });
}

// Normal-mean prior-predictive log marginal densities for one lambda, drawn in
// the order of weak_info.cpp:82-106 (align_even; Gaussian prior draw -- the
// second half of the pair is discarded; then the data).  Dataset j of
// hyperparameter k owns RngStream(derive_seed(seed,{k}), j).
int ref_normal_mean_logm(std::uint64_t seed, std::uint64_t k, double lambda, double log_norm,
                         std::uint64_t n_data, std::uint64_t first, std::uint64_t count,
                         double* ybar_out, double* logm_out) {
    return guarded([&] {
        const std::uint64_t sk = derive_seed(seed, {k});
        const double v = lambda * lambda + 1.0 / static_cast<double>(n_data);
        std::vector<double> z(n_data + (n_data & 1));
        for (std::uint64_t j = 0; j < count; ++j) {
            RngStream stream(sk, static_cast<std::uint32_t>(first + j));
            stream.align_even();
            std::array<double, 2> zp;
            stream.fill_gaussian(zp, 0.0, 1.0);
            const double theta = lambda * zp[0];
            stream.fill_gaussian(z, 0.0, 1.0);
            double sum = 0.0;
            for (std::uint64_t i = 0; i < n_data; ++i) sum += theta + z[i];
            const double ybar = sum / static_cast<double>(n_data);
            if (ybar_out) ybar_out[j] = ybar;
            if (logm_out) logm_out[j] = log_norm - ((0.5 * ybar) * ybar) / v;
        }
    });
}

// -------------------------------------------------------------- SMC pieces
int ref_ess(const double* lw, std::uint64_t n, double* out) {
    return guarded([&] { *out = smc::ess(std::span<const double>(lw, n)); });
}

// The real smc::resample_multinomial.  Ancestors are recovered by running it
// a second time (same stream) on an ensemble whose single coordinate is the
// particle index.
int ref_resample_multinomial(std::uint64_t n, std::uint32_t dim, const double* log_w,
                             const double* particles, std::uint64_t seed, std::uint32_t id,
                             double* particles_out, std::uint64_t* ancestors) {
    return guarded([&] {
        smc::ParticleEnsemble ens;
        ens.count = n;
        ens.dim = dim;
        ens.particles.assign(particles, particles + n * dim);
        ens.log_weights.assign(log_w, log_w + n);
        ens.log_liks.assign(n, 0.0);
        RngStream s(seed, id);
        smc::resample_multinomial(ens, s);
        if (particles_out) std::copy(ens.particles.begin(), ens.particles.end(), particles_out);
        if (ancestors) {
            smc::ParticleEnsemble tag;
            tag.count = n;
            tag.dim = 1;
            tag.particles.resize(n);
            for (std::uint64_t i = 0; i < n; ++i) tag.particles[i] = static_cast<double>(i);
            tag.log_weights.assign(log_w, log_w + n);
            tag.log_liks.assign(n, 0.0);
            RngStream s2(seed, id);
            smc::resample_multinomial(tag, s2);
            for (std::uint64_t i = 0; i < n; ++i)
                ancestors[i] = static_cast<std::uint64_t>(tag.particles[i]);
        }
    });
}

// ------------------------------------------------ reference-format outputs
// abc::write_csv (abc.cpp:99-124) of the set the reference's own
// run_prior_predictive produces for the logistic hooks.
int ref_logistic_abc_csv(const vxb_model* m, std::uint64_t n, std::uint64_t workers,
                         std::uint64_t block_width, std::uint64_t seed, const double* observed,
                         const char* path) {
    return guarded([&] {
        const ModelHooks hooks = logistic_for(*m);
        std::vector<double> obs(observed, observed + hooks.summary_dim);
        const abc::PriorPredictiveSet set = abc::run_prior_predictive(
            hooks, n, workers, block_width, seed, std::span<const double>(obs));
        abc::write_csv(set, std::string(path));
    });
}

// bench::write_csv (bench.cpp:215-230: records section + summary section) of
// caller-supplied records; experiment 0..3 = toggle-abc, weakinfo, bege, tb;
// mode 0 scalar, 1 blocked.
int ref_bench_csv(std::uint64_t n, const std::int32_t* experiment, const std::int32_t* mode,
                  const std::uint64_t* threads, const std::uint64_t* width,
                  const std::uint64_t* replicate, const double* runtime,
                  const std::uint8_t* failed, const char* path) {
    return guarded([&] {
        std::vector<bench::BenchmarkRecord> records;
        for (std::uint64_t i = 0; i < n; ++i)
            records.push_back({static_cast<bench::Experiment>(experiment[i]),
                               static_cast<bench::Mode>(mode[i]), threads[i], width[i],
                               replicate[i], runtime[i], failed[i] != 0});
        bench::write_csv(records, std::string(path));
    });
}

int ref_amdahl_bound(double serial, double parallel, double units, double* out) {
    return guarded([&] { *out = bench::amdahl_bound(serial, parallel, units); });
}

// ------------------------------------ likelihood-annealed SMC / weak-info test
//   The bioassay model (weak_info.cpp:18-160), the adaptive
// sampler smc::run_smc (smc.cpp:352-488) and run_weak_info_test
// (weak_info.cpp:163-277), called as they are.
static weakinfo::BioassayData make_data(const double* dose, const std::uint32_t* group_size,
                                        const std::uint32_t* deaths, std::uint32_t groups) {
    weakinfo::BioassayData d;
    d.dose.assign(dose, dose + groups);
    d.group_size.assign(group_size, group_size + groups);
    if (deaths) d.deaths.assign(deaths, deaths + groups);
    return d;
}

int ref_bioassay_ll(const double* beta, std::uint64_t lanes, const double* dose,
                    const std::uint32_t* group_size, const std::uint32_t* deaths,
                    std::uint32_t groups, double* out) {
    return guarded([&] {
        const auto data = make_data(dose, group_size, deaths, groups);
        weakinfo::bioassay_block_log_likelihood(std::span<const double>(beta, 2 * lanes), lanes,
                                                data, std::span<double>(out, lanes));
    });
}

int ref_bioassay_sample(double lambda1, double lambda2, const double* dose,
                        const std::uint32_t* group_size, std::uint32_t groups, std::uint64_t seed,
                        double* theta, std::uint32_t* deaths) {
    return guarded([&] {
        RngStream stream(seed, 0);
        const auto draw = weakinfo::sample_prior_predictive({lambda1, lambda2},
                                                            make_data(dose, group_size, nullptr, groups),
                                                            stream);
        theta[0] = draw.theta[0];
        theta[1] = draw.theta[1];
        std::copy(draw.data.deaths.begin(), draw.data.deaths.end(), deaths);
    });
}

// One evidence estimate (the evidence_of closure of weak_info.cpp:200-215);
// trace receives the sampler's per-iteration CSV (smc.hpp:125).
int ref_smc_bioassay(const double* dose, const std::uint32_t* group_size,
                     const std::uint32_t* deaths, std::uint32_t groups, double lambda1,
                     double lambda2, std::uint64_t particles, std::uint64_t block_width, double c,
                     double scale, std::uint64_t seed, double* log_evidence,
                     std::uint64_t* iterations, char* trace, std::uint64_t trace_cap) {
    return guarded([&] {
        smc::SmcConfig cfg;
        cfg.particles = particles;
        cfg.block_width = block_width;
        cfg.workers = 1;
        cfg.c = c;
        cfg.scale = scale;
        cfg.seed = seed;
        std::ostringstream text;
        text.precision(17);
        if (trace) cfg.trace = &text;
        const auto model = weakinfo::make_bioassay_model(make_data(dose, group_size, deaths, groups),
                                                         {lambda1, lambda2});
        const smc::SmcResult res = smc::run_smc(model, cfg);
        *log_evidence = res.log_evidence;
        *iterations = res.iterations;
        if (trace && trace_cap) {
            const std::string t = text.str();
            const std::size_t k = std::min<std::size_t>(t.size(), trace_cap - 1);
            std::memcpy(trace, t.data(), k);
            trace[k] = 0;
        }
    });
}

// One run returning the reference's SmcResult: ensemble as 5 x particles doubles
// (theta0, theta1, log weights, log likelihoods, log priors) and the trace CSV text.
int ref_smc_bioassay_ensemble(const double* dose, const std::uint32_t* group_size,
                              const std::uint32_t* deaths, std::uint32_t groups, double lambda1,
                              double lambda2, std::uint64_t particles, std::uint64_t block_width,
                              double c, double scale, std::uint64_t seed, double* log_evidence,
                              std::uint64_t* iterations, double* ensemble, char* trace,
                              std::uint64_t trace_cap, const double* esjd_scales,
                              std::uint64_t n_scales) {
    return guarded([&] {
        smc::SmcConfig cfg;
        cfg.particles = particles;
        cfg.block_width = block_width;
        cfg.workers = 1;
        cfg.c = c;
        cfg.scale = scale;
        cfg.seed = seed;
        if (n_scales) {
            cfg.esjd = true;
            cfg.esjd_scales.assign(esjd_scales, esjd_scales + n_scales);
        }
        std::ostringstream text;
        text.precision(17);
        if (trace) cfg.trace = &text;
        const auto model = weakinfo::make_bioassay_model(make_data(dose, group_size, deaths, groups),
                                                         {lambda1, lambda2});
        const smc::SmcResult res = smc::run_smc(model, cfg);
        *log_evidence = res.log_evidence;
        *iterations = res.iterations;
        const smc::ParticleEnsemble& e = res.ensemble;
        for (std::uint64_t i = 0; i < particles; ++i) {
            ensemble[i] = e.particles[2 * i];
            ensemble[particles + i] = e.particles[2 * i + 1];
            ensemble[2 * particles + i] = e.log_weights[i];
            ensemble[3 * particles + i] = e.log_liks[i];
            ensemble[4 * particles + i] = e.log_priors[i];
        }
        if (trace && trace_cap) {
            const std::string t = text.str();
            const std::size_t k = std::min<std::size_t>(t.size(), trace_cap - 1);
            std::memcpy(trace, t.data(), k);
            trace[k] = 0;
        }
    });
}

int ref_weak_info_test(std::uint64_t hyper_count, std::uint64_t datasets, std::uint64_t particles,
                       double alpha, double c, double scale, std::uint64_t workers,
                       std::uint64_t block_width, std::uint64_t seed, int redraw_base,
                       double* lambda /* (K+1) x 2 */, double* gamma, std::uint8_t* weakly,
                       std::uint64_t* completed, const char* csv_path) {
    return guarded([&] {
        weakinfo::WeakInfoConfig cfg;
        cfg.hyper_count = hyper_count;
        cfg.datasets = datasets;
        cfg.particles = particles;
        cfg.alpha = alpha;
        cfg.c = c;
        cfg.scale = scale;
        cfg.workers = workers;
        cfg.block_width = block_width;
        cfg.seed = seed;
        cfg.redraw_base = redraw_base != 0;
        const weakinfo::CutoffTable table = weakinfo::run_weak_info_test(cfg);
        for (std::size_t k = 0; k < table.rows.size(); ++k) {
            const auto& row = table.rows[k];
            lambda[2 * k] = row.lambda.lambda1;
            lambda[2 * k + 1] = row.lambda.lambda2;
            gamma[k] = row.gamma;
            weakly[k] = row.weakly_informative ? 1 : 0;
            completed[k] = row.completed;
        }
        if (csv_path) {
            std::ofstream out(csv_path);
            weakinfo::write_csv(table, out);
        }
    });
}

// ----------------------------------------------- TB Gillespie ABC
// tb::gillespie_simulate / tb_summaries / make_abc_model (tb_model.cpp:39-167) as
// they are.  ref_tb_simulate: one path at theta from RngStream(seed, id) at pos;
// out = (time, total, genotypes, G summary, H summary or NaN when extinct),
// pos_after = the stream position the path stopped at.
int ref_tb_simulate(const double* theta, std::uint64_t initial, double horizon, double target,
                    std::uint64_t seed, std::uint32_t id, std::uint64_t pos,
                    std::uint64_t block_width, double* out, std::uint64_t* pos_after,
                    double* counts_out, std::uint64_t counts_cap, std::uint64_t* n_counts) {
    return guarded([&] {
        RngStream stream(seed, id);
        stream.set_counter(pos);
        const tb::TbState st = tb::gillespie_simulate({theta[0], theta[1], theta[2]}, initial,
                                                      {horizon, target}, stream, block_width);
        out[0] = st.time;
        out[1] = st.total;
        out[2] = static_cast<double>(st.genotypes);
        out[3] = out[4] = std::numeric_limits<double>::quiet_NaN();
        if (st.total >= 1.0) {
            const tb::TbSummaries sm = tb::tb_summaries(st);
            out[3] = sm.genotypes;
            out[4] = sm.diversity;
        }
        if (pos_after) *pos_after = stream.counter_lo();
        if (n_counts) *n_counts = st.counts.size();
        for (std::size_t k = 0; counts_out && k < st.counts.size() && k < counts_cap; ++k)
            counts_out[k] = st.counts[k];
    });
}

// Rows [first, first+count) keyed per particle: row i owns RngStream(seed, i) and
// runs the row sequence of abc.cpp:51-60 on tb::make_abc_model.
int ref_tb_abc_particle(std::uint64_t initial, double horizon, double target, std::uint64_t first,
                        std::uint64_t count, std::uint64_t seed, const double* observed,
                        double* params, double* summaries, double* rho, std::uint8_t* failed,
                        unsigned threads) {
    return guarded([&] {
        const ModelHooks hooks = tb::make_abc_model(initial, {horizon, target});
        const std::vector<double> obs(observed, observed + 2);
        if (threads < 1) threads = 1;
        auto body = [&](unsigned t) {
            std::vector<double> theta(3), summary(2);
            for (std::uint64_t r = t; r < count; r += threads) {
                RngStream stream(seed, static_cast<std::uint32_t>(first + r));
                hooks.sample_prior(stream, theta);
                stream.align_even();
                double dist = std::numeric_limits<double>::quiet_NaN();
                std::uint8_t bad = 0;
                try {
                    hooks.simulate(theta, stream, 4, summary);
                    dist = abc::discrepancy(summary, obs);
                } catch (const Error&) {
                    bad = 1;
                    std::fill(summary.begin(), summary.end(), 0.0);
                }
                if (params) std::copy(theta.begin(), theta.end(), params + r * 3);
                if (summaries) std::copy(summary.begin(), summary.end(), summaries + r * 2);
                if (rho) rho[r] = dist;
                if (failed) failed[r] = bad;
            }
        };
        std::vector<std::thread> pool;
        for (unsigned t = 0; t < threads; ++t) pool.emplace_back(body, t);
        for (auto& th : pool) th.join();
    });
}

// bench::tb_observed_summaries (bench.cpp:79-92)
int ref_tb_observed(std::uint64_t initial, double horizon, double target, std::uint64_t seed,
                    std::uint64_t block_width, double* out) {
    return guarded([&] {
        const auto s = bench::tb_observed_summaries(initial, {horizon, target}, seed, block_width);
        out[0] = s[0];
        out[1] = s[1];
    });
}

}  // extern "C"
