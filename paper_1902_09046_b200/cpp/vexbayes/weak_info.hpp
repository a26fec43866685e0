// vexbayes/weak_info.hpp (B200 shim) -- the weak-informativity test of the
// reference (weak_info.hpp:13-104) over the device sampler, and the
// prior-predictive p-value grid of BASELINE config 2.
//
// Same types and free functions as the reference header: Hyperparam,
// BioassayData, default_design, bioassay_log_likelihood /
// bioassay_block_log_likelihood, sample_prior_predictive, estimate_pvalues,
// compute_cutoff, WeakInfoConfig, CutoffRow/CutoffTable, run_weak_info_test,
// write_csv.  Every sampler run of the test (2 (K+1) N of them) is one CTA of one
// launch per GPU in use (vxb_multi_weak_info_test: rows split over the devices, the
// reference's own task split); `workers` is accepted and has no device meaning.
// Differences at the boundary: sample_prior_predictive takes the stream's
// identity (seed) instead of an RngStream&; log_evidence adds the single-run
// entry (the evidence_of closure of weak_info.cpp:200-215).
#pragma once

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <limits>
#include <ostream>
#include <span>
#include <vector>

#include "bioassay.hpp"
#include "cuda_context.hpp"

namespace vexbayes::weakinfo {

// estimate_pvalues (weak_info.cpp:108-120): p_i = #{ j : k_j <= base_i } / N,
// ties count.  Host-side (the inputs are small evidence vectors).
inline std::vector<double> estimate_pvalues(std::span<const double> evidences_base,
                                            std::span<const double> evidences_k) {
    require(!evidences_k.empty(), "invalid-argument", "need at least one comparison evidence");
    std::vector<double> sorted(evidences_k.begin(), evidences_k.end());
    std::sort(sorted.begin(), sorted.end());
    std::vector<double> p(evidences_base.size());
    for (std::size_t i = 0; i < p.size(); ++i)
        p[i] = static_cast<double>(std::upper_bound(sorted.begin(), sorted.end(), evidences_base[i]) -
                                   sorted.begin()) /
               static_cast<double>(sorted.size());
    return p;
}

// Hyperparam, BioassayData, default_design, make_bioassay_model: bioassay.hpp

inline void bioassay_block_log_likelihood(std::span<const double> params, std::size_t lanes,
                                          const BioassayData& data, std::span<double> out) {
    detail::check_design(data, true);
    cuda::check(vxb_bioassay_log_likelihood(cuda::context(), params.data(), lanes,
                                            static_cast<std::uint32_t>(data.groups()), data.dose.data(),
                                            data.group_size.data(), data.deaths.data(), out.data()));
}
inline double bioassay_log_likelihood(double beta0, double beta1, const BioassayData& data) {
    const double beta[2] = {beta0, beta1};
    double out = 0.0;
    bioassay_block_log_likelihood(beta, 1, data, {&out, 1});
    return out;
}

struct PriorPredictiveDraw {
    std::array<double, 2> theta;
    BioassayData data;
};
// draw from RngStream(seed, 0) (the reference passes the stream itself)
inline PriorPredictiveDraw sample_prior_predictive(const Hyperparam& lambda, const BioassayData& design,
                                                   std::uint64_t seed) {
    detail::check_design(design, false);
    require(lambda.lambda1 >= 0.0 && lambda.lambda2 >= 0.0, "invalid-argument",
            "prior scales must be nonnegative");
    PriorPredictiveDraw draw;
    draw.data = design;
    draw.data.deaths.assign(design.groups(), 0);
    const double lam[2] = {lambda.lambda1, lambda.lambda2};
    cuda::check(vxb_bioassay_sample(cuda::context(), 1, static_cast<std::uint32_t>(design.groups()),
                                    design.dose.data(), design.group_size.data(), lam, &seed,
                                    draw.theta.data(), draw.data.deaths.data()));
    return draw;
}

// log evidence of one dataset under one prior by the adaptive annealed sampler
// (smc::run_smc with the test's settings); NaN-free: sampler failures throw.
inline double log_evidence(const BioassayData& data, const Hyperparam& prior, std::size_t particles,
                           std::size_t block_width, double c, double scale, std::uint64_t seed,
                           std::size_t* iterations = nullptr) {
    detail::check_design(data, true);
    const double lam[2] = {prior.lambda1, prior.lambda2};
    double ev = 0.0;
    std::uint32_t it = 0;
    std::uint8_t status = 0;
    cuda::check(vxb_smc_bioassay(cuda::context(), 1, static_cast<std::uint32_t>(data.groups()),
                                 data.dose.data(), data.group_size.data(), data.deaths.data(), lam, &seed,
                                 particles, block_width, c, scale, &ev, &it, &status, nullptr, 0));
    static const char* const codes[] = {"", "invalid-model", "degenerate-ensemble", "non-convergence"};
    require(status == 0, codes[status < 4 ? status : 1], "the annealed sampler did not complete");
    if (iterations) *iterations = it;
    return ev;
}

// compute_cutoff (weak_info.cpp:122-125): type-7 alpha-quantile of the p-values
inline double compute_cutoff(std::span<const double> pvalues, double alpha) {
    require(alpha > 0.0 && alpha < 1.0, "invalid-argument", "alpha must lie in (0, 1)");
    require(!pvalues.empty(), "insufficient-data", "quantile of an empty sample");
    std::vector<double> sorted(pvalues.begin(), pvalues.end());
    std::sort(sorted.begin(), sorted.end());
    const std::size_t n = sorted.size();
    if (n == 1) return sorted[0];
    const double h = static_cast<double>(n - 1) * alpha;
    const auto lo = static_cast<std::size_t>(h);
    if (lo + 1 >= n) return sorted[n - 1];
    return sorted[lo] + (h - static_cast<double>(lo)) * (sorted[lo + 1] - sorted[lo]);
}

struct WeakInfoConfig {
    std::size_t hyper_count = 400;
    std::size_t datasets = 400;
    std::size_t particles = 500;
    double alpha = 0.05;
    double c = 0.01;
    double scale = 1.6828427124746189;
    std::size_t workers = 1;
    std::size_t block_width = 4;
    std::uint64_t seed = 0;
    bool redraw_base = false;
    Hyperparam base = kBasePrior;
    BioassayData design;
    // not in the reference: run the sampler with contracted multiply-adds
    // (VXB_ARITH_FMA -- same random numbers, evidences equal to rounding, ~10 % faster)
    bool fused_arithmetic = false;
    // not in the reference: the throughput generator (VXB_RNG_FAST -- other random numbers,
    // statistically equivalent estimates, ~1.75x faster); implies fused arithmetic
    bool throughput_generator = false;
};
struct CutoffRow {
    std::size_t index;
    Hyperparam lambda;
    double gamma;
    bool weakly_informative;
    std::size_t completed;
};
struct CutoffTable {
    double alpha = 0.0;
    std::vector<CutoffRow> rows;
};

inline CutoffTable run_weak_info_test(const WeakInfoConfig& config) {
    require(config.datasets >= 1, "invalid-argument", "need at least one dataset per prior");
    require(config.workers >= 1, "invalid-argument", "need at least one worker");
    const BioassayData design = config.design.dose.empty() ? default_design() : config.design;
    detail::check_design(design, false);
    require(design.groups() >= 1 && design.groups() <= 16, "invalid-argument",
            "between 1 and 16 dose groups");
    vxb_weakinfo_cfg cfg{};
    cfg.hyper_count = config.hyper_count;
    cfg.datasets = config.datasets;
    cfg.particles = config.particles;
    cfg.block_width = config.block_width;
    cfg.seed = config.seed;
    cfg.alpha = config.alpha;
    cfg.c = config.c;
    cfg.scale = config.scale;
    cfg.base[0] = config.base.lambda1;
    cfg.base[1] = config.base.lambda2;
    cfg.redraw_base = config.redraw_base ? 1 : 0;
    cfg.arith = config.fused_arithmetic ? VXB_ARITH_FMA : VXB_ARITH_EXACT;
    cfg.rng = config.throughput_generator ? VXB_RNG_FAST : VXB_RNG_REF;
    cfg.groups = static_cast<std::uint32_t>(design.groups());
    for (std::size_t g = 0; g < design.groups(); ++g) {
        cfg.dose[g] = design.dose[g];
        cfg.group_size[g] = design.group_size[g];
    }
    const std::size_t rows = config.hyper_count + 1;
    std::vector<double> lambda(2 * rows), gamma(rows);
    std::vector<std::uint8_t> weakly(rows);
    std::vector<std::uint64_t> completed(rows);
    cuda::check(vxb_multi_weak_info_test(cuda::multi(), &cfg, lambda.data(), gamma.data(), weakly.data(),
                                   completed.data(), nullptr));
    CutoffTable table;
    table.alpha = config.alpha;
    for (std::size_t k = 0; k < rows; ++k)
        table.rows.push_back({k, {lambda[2 * k], lambda[2 * k + 1]}, gamma[k], weakly[k] != 0, completed[k]});
    return table;
}

// CSV: k,lambda1,lambda2,gamma_alpha,weakly_informative (weak_info.cpp:279-293)
inline void write_csv(const CutoffTable& table, std::ostream& out) {
    out << "k,lambda1,lambda2,gamma_alpha,weakly_informative\n";
    char text[64];
    for (const CutoffRow& row : table.rows) {
        out << row.index;
        for (double v : {row.lambda.lambda1, row.lambda.lambda2, row.gamma}) {
            std::snprintf(text, sizeof(text), "%.17g", v);
            out << ',' << text;
        }
        out << ',' << (row.weakly_informative ? 1 : 0) << '\n';
    }
}

// Prior-predictive p-values of the normal-mean model over a lambda grid: the
// fused device form of {sample_prior_predictive, density, estimate_pvalues}.
struct PvalueGrid {
    std::vector<std::uint64_t> counts;
    std::vector<double> pvalues;
};
inline PvalueGrid prior_predictive_pvalues(std::span<const double> lambda, std::size_t n_data,
                                           std::uint64_t datasets, std::uint64_t seed,
                                           double ybar_observed, bool fast_generator = false) {
    vxb_model m{};
    m.model = VXB_MODEL_NORMAL_MEAN;
    m.precision = VXB_F64;
    m.rng = fast_generator ? VXB_RNG_FAST : VXB_RNG_REF;
    m.dim = m.summary_dim = 1;
    m.steps = m.obs_stride = static_cast<std::uint32_t>(n_data);
    std::vector<double> log_norm(lambda.size());
    const double pi = 3.141592653589793238462643383279502884;
    for (std::size_t k = 0; k < lambda.size(); ++k)
        log_norm[k] = -0.5 * std::log(2.0 * pi * (lambda[k] * lambda[k] + 1.0 / static_cast<double>(n_data)));
    PvalueGrid g;
    g.counts.resize(lambda.size());
    g.pvalues.resize(lambda.size());
    cuda::check(vxb_ppp_pvalues(cuda::context(), &m, lambda.data(), log_norm.data(),
                                static_cast<std::uint32_t>(lambda.size()), datasets, 0, datasets, seed,
                                ybar_observed, g.counts.data(), g.pvalues.data(), nullptr));
    return g;
}

}  // namespace vexbayes::weakinfo
