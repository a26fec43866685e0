// Exercises the C++ shim the way a user of the reference would call the
// reference API (abc.hpp / smc.hpp / weak_info.hpp), and dumps the results as
// hex doubles for tests/test_gpu_cpp_shim.py to compare with the oracle.
#include <cstdio>
#include <cstring>
#include <vector>

#include "vexbayes/abc.hpp"
#include "vexbayes/logistic.hpp"
#include "vexbayes/rng.hpp"
#include "vexbayes/smc.hpp"
#include "vexbayes/weak_info.hpp"

using namespace vexbayes;

static void dump(const char* name, const std::vector<double>& v) {
    std::printf("%s %zu", name, v.size());
    for (double x : v) {
        unsigned long long b;
        std::memcpy(&b, &x, 8);
        std::printf(" %016llx", b);
    }
    std::printf("\n");
}

int main() {
    try {
        const ModelHooks model = logistic::make_abc_model();
        const std::vector<double> theta{0.5, 100.0, 0.05};
        const auto observed = logistic::simulate_at(model, theta, derive_seed(1, {90}), 0, 0);
        dump("observed", observed);

        const abc::PriorPredictiveSet set = abc::run_prior_predictive(model, 500, 3, 4, 1337, observed);
        dump("params", set.params);
        dump("summaries", set.summaries);
        dump("rho", set.discrepancies);
        const abc::EpsilonSelection sel = abc::select_epsilon(set, 0.05);
        dump("epsilon", {sel.epsilon});
        std::printf("accepted %zu", sel.accepted.size());
        for (auto r : sel.accepted) std::printf(" %zu", r);
        std::printf("\n");
        std::printf("discrepancy %.17g\n", abc::discrepancy(std::vector<double>{0.0, 0.0}, std::vector<double>{3.0, 4.0}));

        const auto acc = abc::reject_fixed_epsilon(model, 20000, 0, 20000, 1337, observed, sel.epsilon, 20000);
        std::printf("reject %llu", static_cast<unsigned long long>(acc.total_accepted));
        for (auto r : acc.rows) std::printf(" %llu", static_cast<unsigned long long>(r));
        std::printf("\n");

        // error behaviour mirrors the reference
        int ok = 0;
        try { abc::run_prior_predictive(model, 0, 1, 1, 1, observed); } catch (const Error& e) { ok += e.code() == "invalid-shape"; }
        try { abc::run_prior_predictive(model, 8, 0, 1, 1, observed); } catch (const Error& e) { ok += e.code() == "invalid-shape"; }
        try { abc::run_prior_predictive(model, 8, 1, 3, 1, observed); } catch (const Error& e) { ok += e.code() == "invalid-shape"; }
        try { abc::run_prior_predictive(model, 8, 1, 1, 1, std::vector<double>(3)); } catch (const Error& e) { ok += e.code() == "invalid-summary"; }
        try { abc::select_epsilon(set, 0.0); } catch (const Error& e) { ok += e.code() == "invalid-argument"; }
        try { abc::run_prior_predictive(ModelHooks{}, 8, 1, 1, 1, {}); } catch (const Error& e) { ok += e.code() == "unsupported-model"; }
        std::printf("errors %d\n", ok);

        // SMC pieces
        smc::ParticleEnsemble ens;
        ens.count = 256;
        ens.dim = 2;
        const auto g = fill_gaussian(7, 1, 0, 768, 0.0, 1.0);
        ens.particles.assign(g.begin(), g.begin() + 512);
        ens.log_weights.assign(g.begin() + 512, g.end());
        ens.log_liks.assign(256, 0.0);
        std::printf("ess %.17g\n", smc::ess(ens.log_weights));
        smc::resample_multinomial(ens, 2718, 3);
        dump("resampled", ens.particles);

        const std::vector<double> lambda{0.1, 1.0, 10.0, 100.0};
        const auto pv = weakinfo::prior_predictive_pvalues(lambda, 100, 20000, 1337, 2.9);
        std::printf("counts");
        for (auto c : pv.counts) std::printf(" %llu", static_cast<unsigned long long>(c));
        std::printf("\n");
        const auto p2 = weakinfo::estimate_pvalues(std::vector<double>{2.0, 5.0}, std::vector<double>{1.0, 3.0, 4.0, 6.0});
        std::printf("pvalues %.17g %.17g\n", p2[0], p2[1]);
    } catch (const Error& e) {
        std::printf("FAILED %s\n", e.what());
        return 1;
    }
    return 0;
}
