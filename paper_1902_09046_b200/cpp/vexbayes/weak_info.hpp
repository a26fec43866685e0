// vexbayes/weak_info.hpp (B200 shim) -- the p-value step of the weak-
// informativity test (weak_info.hpp:55-61) and the prior-predictive p-value
// grid of BASELINE config 2.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <span>
#include <vector>

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
