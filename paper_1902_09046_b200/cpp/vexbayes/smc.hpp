// vexbayes/smc.hpp (B200 shim) -- the SMC building blocks on the hot path
// (smc.hpp:35-49): ParticleEnsemble, ess, resample_multinomial; plus the
// ABC-SMC driver of BASELINE config 3 (not in the reference).
#pragma once

#include <cmath>
#include <cstdint>
#include <span>
#include <vector>

#include "cuda_context.hpp"
#include "model.hpp"

namespace vexbayes::smc {

struct ParticleEnsemble {
    std::size_t count = 0;
    std::size_t dim = 0;
    std::vector<double> particles;    // count x dim
    std::vector<double> log_weights;  // count
    std::vector<double> log_liks;     // count
    std::vector<double> log_priors;   // count
    double temperature = 0.0;
    double log_evidence = 0.0;
    std::size_t iteration = 0;
    std::span<double> row(std::size_t i) { return {particles.data() + i * dim, dim}; }
    std::span<const double> row(std::size_t i) const { return {particles.data() + i * dim, dim}; }
};

// smc::ess (smc.cpp:208-219)
inline double ess(std::span<const double> log_weights) {
    double out = 0.0;
    cuda::check(vxb_ess(cuda::context(), log_weights.data(), log_weights.size(), &out));
    return out;
}

// smc::resample_multinomial (smc.cpp:268-300).  The reference takes the
// coordinator's RngStream; the device needs its identity: (seed, stream_id),
// positioned at 0.  Cached rows are permuted consistently; weights reset.
inline void resample_multinomial(ParticleEnsemble& ensemble, std::uint64_t seed,
                                 std::uint32_t stream_id) {
    const std::size_t np = ensemble.count, d = ensemble.dim;
    std::vector<double> moved(np * d);
    std::vector<std::uint64_t> anc(np);
    cuda::check(vxb_resample_multinomial(cuda::context(), np, static_cast<std::uint32_t>(d),
                                         ensemble.log_weights.data(), ensemble.particles.data(),
                                         seed, stream_id, moved.data(), anc.data()));
    ensemble.particles = std::move(moved);
    const bool has_priors = ensemble.log_priors.size() == np;
    std::vector<double> lls(np), lps(has_priors ? np : 0);
    for (std::size_t i = 0; i < np; ++i) {
        if (ensemble.log_liks.size() == np) lls[i] = ensemble.log_liks[anc[i]];
        if (has_priors) lps[i] = ensemble.log_priors[anc[i]];
    }
    if (ensemble.log_liks.size() == np) ensemble.log_liks = std::move(lls);
    if (has_priors) ensemble.log_priors = std::move(lps);
    ensemble.log_weights.assign(np, -std::log(static_cast<double>(np)));
}

struct AbcSmcConfig {
    std::size_t particles = 100000;
    std::size_t generations = 10;
    double quantile = 0.5;       // epsilon_g = this quantile of the previous distances
    double kernel_scale = 2.0;   // covariance multiplier of the Gaussian random walk
    double jitter = 1e-10;
    std::size_t round_size = 0;  // proposals per round (0: particles)
    std::size_t max_rounds = 0;  // 0: 1000
    std::uint64_t seed = 0;
};
struct AbcSmcResult {
    std::size_t dim = 0;
    std::vector<double> particles, weights, discrepancies;           // final population
    std::vector<double> epsilon, ess, accept_rate, mean, covariance;  // per generation
    std::vector<std::uint64_t> proposals;
};
inline AbcSmcResult run_abc_smc(const ModelHooks& model, const AbcSmcConfig& cfg,
                                std::span<const double> observed) {
    require(static_cast<bool>(model.device), "unsupported-model", "model has no device descriptor");
    require(observed.size() == model.summary_dim, "invalid-summary",
            "observed summary length differs from the model summary dimension");
    const std::size_t n = cfg.particles, g = cfg.generations, d = model.dim;
    AbcSmcResult r;
    r.dim = d;
    r.particles.resize(n * d);
    r.weights.resize(n);
    r.discrepancies.resize(n);
    r.epsilon.resize(g);
    r.ess.resize(g);
    r.accept_rate.resize(g);
    r.mean.resize(g * d);
    r.covariance.resize(g * d * d);
    r.proposals.resize(g);
    vxb_abcsmc_cfg c{n, static_cast<std::uint32_t>(g), 0, cfg.quantile, cfg.kernel_scale,
                     cfg.jitter, cfg.round_size, cfg.max_rounds, cfg.seed};
    vxb_abcsmc_out out{r.particles.data(), r.weights.data(), r.discrepancies.data(),
                       r.epsilon.data(), r.ess.data(), r.accept_rate.data(), r.proposals.data(),
                       r.mean.data(), r.covariance.data()};
    cuda::check(vxb_abcsmc_run(cuda::context(), model.device.get(), &c, observed.data(), &out));
    return r;
}

}  // namespace vexbayes::smc
