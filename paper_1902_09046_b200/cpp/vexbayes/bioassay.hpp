// vexbayes/bioassay.hpp (B200 shim) -- the bioassay dose-response model of the
// weak-informativity case study (weak_info.hpp:14-45): data, hyperparameters and
// the ModelHooks factory.  Shared by weak_info.hpp and smc.hpp.
#pragma once

#include <cstdint>
#include <memory>
#include <vector>

#include "errors.hpp"
#include "model.hpp"

namespace vexbayes::weakinfo {

struct Hyperparam {
    double lambda1;
    double lambda2;
};
inline constexpr Hyperparam kBasePrior{10.0, 2.5};

struct BioassayData {
    std::vector<double> dose;
    std::vector<unsigned> group_size;
    std::vector<unsigned> deaths;
    std::size_t groups() const { return dose.size(); }
};
inline BioassayData default_design() { return {{-0.86, -0.3, -0.05, -0.75}, {5, 5, 5, 5}, {}}; }

namespace detail {
inline void check_design(const BioassayData& data, bool with_deaths) {
    require(data.dose.size() == data.group_size.size(), "invalid-argument",
            "dose and group size lengths differ");
    if (!with_deaths) return;
    require(data.deaths.size() == data.dose.size(), "invalid-argument",
            "death count length differs from the design");
    for (std::size_t g = 0; g < data.groups(); ++g)
        require(data.deaths[g] <= data.group_size[g], "invalid-argument",
                "more deaths than animals in a group");
}
}  // namespace detail


// What the annealed-sampler kernel needs of the model: the dataset and the prior.
struct BioassayBinding {
    BioassayData data;
    Hyperparam prior;
};

// make_bioassay_model (weak_info.cpp:84-106): dim 2, prior N(0, diag(lambda^2)).
// The host closures of the reference are not populated (a kernel cannot call
// them); smc::run_smc recognises the model through `family` / `binding`.
inline ModelHooks make_bioassay_model(BioassayData data, const Hyperparam& prior) {
    detail::check_design(data, true);
    require(prior.lambda1 > 0.0 && prior.lambda2 > 0.0, "invalid-argument",
            "prior scales must be positive");
    ModelHooks m;
    m.dim = 2;
    m.summary_dim = 0;
    m.family = "bioassay";
    m.binding = std::make_shared<const BioassayBinding>(BioassayBinding{std::move(data), prior});
    return m;
}

}  // namespace vexbayes::weakinfo
