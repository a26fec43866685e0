// vexbayes/smc.hpp (B200 shim) -- the SMC building blocks on the hot path
// (smc.hpp:35-49): ParticleEnsemble, ess, resample_multinomial; run_smc
// (smc.hpp:112-138) for the model the paper runs it on; plus the ABC-SMC
// driver of BASELINE config 3 (not in the reference).
#pragma once

#include <cmath>
#include <cstdint>
#include <ostream>
#include <span>
#include <string_view>
#include <vector>

#include "bioassay.hpp"
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

// ---------------------------------------------------------------- run_smc
// SmcConfig / SmcResult: smc.hpp:112-131, same members and defaults.
struct SmcConfig {
    std::size_t particles = 2000;
    std::size_t block_width = 4;
    std::size_t workers = 1;  // accepted for source compatibility; the device replays the
                              // reference's workers = 1 stream layout whatever is asked
    double c = 0.01;
    double scale = 0.0;       // <= 0 selects 2.38/sqrt(d)
    bool esjd = false;
    std::vector<double> esjd_scales = {0.1, 0.2, 0.3, 0.4, 0.5, 0.6, 0.7, 0.8, 0.9, 1.0};
    double bisection_tol = 1e-10;
    double jitter = 1e-10;
    std::size_t max_iterations = 1000;
    std::size_t step_cap = 100;
    std::uint64_t seed = 0;
    std::ostream* trace = nullptr;  // per-iteration CSV: n,t_n,ess,log_evidence,R_n,p_acc,h
};
struct SmcResult {
    ParticleEnsemble ensemble;
    double log_evidence = 0.0;
    std::size_t iterations = 0;
};

// smc::run_smc (smc.cpp:352-488): the whole adaptive sampler is ONE kernel with
// the ensemble in shared memory (csrc/vxb_anneal.cu), so the model has to be one
// the kernel knows: the bioassay model of the case study (make_bioassay_model).
// Non-default tolerances/caps are fixed on the device and rejected here rather than
// silently ignored; the ESJD scale adaptation (config.esjd) runs on the device with a
// grid of up to 16 scales.
inline SmcResult run_smc(const ModelHooks& model, const SmcConfig& cfg) {
    require(model.family && std::string_view(model.family) == "bioassay" && model.binding,
            "unsupported-model", "run_smc on the device needs make_bioassay_model()");
    require(!cfg.esjd || (!cfg.esjd_scales.empty() && cfg.esjd_scales.size() <= 16), "invalid-argument",
            cfg.esjd_scales.empty() ? "scale grid must not be empty" : "at most 16 ESJD scales on the device");
    require(cfg.bisection_tol == 1e-10 && cfg.jitter == 1e-10 && cfg.max_iterations == 1000 &&
                cfg.step_cap == 100,
            "unsupported-config", "tolerance, jitter and caps are fixed at the reference defaults");
    require(cfg.workers >= 1, "invalid-argument", "need at least one worker");
    const auto& b = *static_cast<const weakinfo::BioassayBinding*>(model.binding.get());
    const std::size_t np = cfg.particles;
    const double lam[2] = {b.prior.lambda1, b.prior.lambda2};
    const std::uint32_t rows = 1000;
    std::vector<double> packed(5 * np), trace(cfg.trace ? rows * 6 : 0);
    SmcResult r;
    std::uint32_t it = 0;
    cuda::check(vxb_smc_bioassay_ensemble(
        cuda::context(), static_cast<std::uint32_t>(b.data.groups()), b.data.dose.data(),
        b.data.group_size.data(), b.data.deaths.data(), lam, cfg.seed, np, cfg.block_width, cfg.c,
        cfg.scale, &r.log_evidence, &it, packed.data(), cfg.trace ? trace.data() : nullptr,
        cfg.trace ? rows : 0, cfg.esjd ? cfg.esjd_scales.data() : nullptr,
        cfg.esjd ? static_cast<std::uint32_t>(cfg.esjd_scales.size()) : 0));
    r.iterations = it;
    ParticleEnsemble& e = r.ensemble;
    e.count = np;
    e.dim = 2;
    e.particles.resize(2 * np);
    for (std::size_t i = 0; i < np; ++i) {
        e.particles[2 * i] = packed[i];
        e.particles[2 * i + 1] = packed[np + i];
    }
    e.log_weights.assign(packed.begin() + 2 * np, packed.begin() + 3 * np);
    e.log_liks.assign(packed.begin() + 3 * np, packed.begin() + 4 * np);
    e.log_priors.assign(packed.begin() + 4 * np, packed.end());
    e.temperature = 1.0;
    e.log_evidence = r.log_evidence;
    e.iteration = it;
    if (cfg.trace) {
        *cfg.trace << "n,t_n,ess,log_evidence,R_n,p_acc,h\n";
        for (std::uint32_t n = 0; n < it; ++n) {
            const double* row = &trace[6 * n];
            *cfg.trace << (n + 1) << ',' << row[0] << ',' << row[1] << ',' << row[4] << ','
                       << static_cast<std::size_t>(row[2]) << ',' << row[3] << ',' << row[5] << '\n';
        }
    }
    return r;
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
    // every GPU in use (cuda::set_devices): proposals and new particles sharded by global
    // index, accepted proposals / weights gathered and the weight sum reduced over NCCL
    // inside the library; the same bits as one GPU (vxb_abcsmc_run) for any device count
    cuda::check(vxb_multi_abcsmc_run(cuda::multi(), model.device.get(), &c, observed.data(), &out));
    return r;
}

}  // namespace vexbayes::smc
