// Exercises the C++ shim the way a user of the reference would call the
// reference API (abc.hpp / smc.hpp / weak_info.hpp), and dumps the results as
// hex doubles for tests/test_gpu_cpp_shim.py to compare with the oracle.
#include <cstdio>
#include <cstring>
#include <fstream>
#include <sstream>
#include <vector>

#include "vexbayes/abc.hpp"
#include "vexbayes/bench.hpp"
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

// Reference-format outputs (argv: golden bench csv, observed hex file, out dir):
// the set of the fixture's (n, P, V, seed) case written by abc::write_csv, the
// golden bench file parsed and written again, and a short run_benchmark sweep.
static int csv_mode(const char* bench_golden, const char* out_dir) {
    const std::string dir(out_dir);
    std::ifstream in(bench_golden);
    const auto records = bench::parse_csv(in);
    bench::write_csv(records, dir + "/bench_rewritten.csv");

    auto dm = std::make_shared<DeviceModel>(*logistic::make_abc_model().device);
    dm->steps = 400;
    dm->obs_stride = 100;
    dm->summary_dim = 4;
    dm->prior_hi[0] = 4000.0;
    ModelHooks bad;
    bad.dim = 3;
    bad.summary_dim = 4;
    bad.device = dm;
    auto good = std::make_shared<DeviceModel>(*dm);
    good->prior_hi[0] = 1.0;
    ModelHooks ok = bad;
    ok.device = good;
    const auto observed = logistic::simulate_at(ok, std::vector<double>{0.5, 100.0, 0.05}, 5, 0, 0);
    abc::write_csv(abc::run_prior_predictive(bad, 24, 3, 2, 21, observed), dir + "/set.csv");

    // the weak-informativity test through the reference's own interface
    weakinfo::WeakInfoConfig wcfg;
    wcfg.hyper_count = 3;
    wcfg.datasets = 12;
    wcfg.particles = 200;
    wcfg.seed = 1337;
    {
        std::ofstream wout(dir + "/weakinfo_table.csv");
        weakinfo::write_csv(weakinfo::run_weak_info_test(wcfg), wout);
    }
    auto design = weakinfo::default_design();
    const auto draw = weakinfo::sample_prior_predictive({10.0, 2.5}, design, 1234);
    std::size_t its = 0;
    const double ev = weakinfo::log_evidence(draw.data, {10.0, 2.5}, 500, 4, 0.01, 1.6828427124746189, 3702, &its);
    std::printf("evidence %.17g %zu %u%u%u%u\n", ev, its, draw.data.deaths[0], draw.data.deaths[1],
                draw.data.deaths[2], draw.data.deaths[3]);
    {   // smc::run_smc as the reference's weak_info.cpp calls it (weak_info.cpp:199-208)
        const auto d3 = weakinfo::sample_prior_predictive({4.0, 0.2}, design, 5);
        smc::SmcConfig sc;
        sc.particles = 64;
        sc.scale = 1.6828427124746189;
        sc.seed = 15;
        std::ostringstream tr;
        tr.precision(17);
        sc.trace = &tr;
        const smc::SmcResult res = smc::run_smc(weakinfo::make_bioassay_model(d3.data, {4.0, 0.2}), sc);
        std::printf("run_smc %.17g %zu %zu %zu %.17g\n", res.log_evidence, res.iterations,
                    res.ensemble.count, res.ensemble.dim, res.ensemble.temperature);
        dump("run_smc_particles", res.ensemble.particles);
        dump("run_smc_log_liks", res.ensemble.log_liks);
        std::ofstream(dir + "/smc_trace.csv") << tr.str();
        int refused = 0;
        {   // SmcConfig::esjd = true: the scale adaptation, default grid
            smc::SmcConfig se;
            se.particles = 333;
            se.seed = 15;
            se.esjd = true;
            std::ostringstream te;
            te.precision(17);
            se.trace = &te;
            const smc::SmcResult re = smc::run_smc(weakinfo::make_bioassay_model(d3.data, {4.0, 0.2}), se);
            std::printf("run_smc_esjd %.17g %zu\n", re.log_evidence, re.iterations);
            std::ofstream(dir + "/smc_trace_esjd.csv") << te.str();
            se.esjd_scales.assign(17, 0.1);
            try { smc::run_smc(weakinfo::make_bioassay_model(d3.data, {4.0, 0.2}), se); } catch (const Error& e) { refused += e.code() == "invalid-argument"; }
        }
        try { smc::run_smc(ModelHooks{}, sc); } catch (const Error& e) { refused += e.code() == "unsupported-model"; }
        sc.particles = 6;
        try { smc::run_smc(weakinfo::make_bioassay_model(d3.data, {4.0, 0.2}), sc); } catch (const Error& e) { refused += e.code() == "invalid-shape"; }
        std::printf("run_smc_refused %d\n", refused);
    }
    {
        bench::ExperimentSizes ws;
        bench::run_experiment_once(bench::Experiment::weakinfo, ws, 2, 4, 1337);
        bench::run_experiment_once(bench::Experiment::tb, ws, 2, 4, 1337);
        const auto tb_obs = bench::tb_observed_summaries(10, {10.0, 10000.0}, 1337, 4);
        const auto tb_set = abc::run_prior_predictive(tb::make_abc_model(10, {10.0, 10000.0}), 40, 2, 4, 1337, tb_obs);
        std::printf("tb %.17g %.17g %.17g %.17g %d\n", tb_obs[0], tb_obs[1], tb_set.summaries[0],
                    tb_set.discrepancies[1], static_cast<int>(tb_set.failed[0] + tb_set.failed[1]));
    }

    bench::BenchConfig cfg;
    cfg.threads = {1, 3};
    cfg.block_widths = {1, 4};
    cfg.replicates = 2;
    cfg.sizes.samples = 32;
    const auto sweep = bench::run_benchmark(cfg);
    bench::write_csv(sweep, dir + "/sweep.csv");
    int failures = 0;
    for (const auto& r : sweep) failures += r.failed ? 1 : 0;
    std::printf("sweep %zu %d\n", sweep.size(), failures);
    int codes = 0;
    try { bench::run_experiment_once(bench::Experiment::bege, cfg.sizes, 1, 1, 1); } catch (const Error& e) { codes += e.code() == "unsupported-model"; }
    try { bench::amdahl_bound(0.0, 0.0, 2.0); } catch (const Error& e) { codes += e.code() == "invalid-input"; }
    try { bench::experiment_from_string("toggle"); } catch (const Error& e) { codes += e.code() == "invalid-input"; }
    std::printf("bench_errors %d amdahl %.17g\n", codes, bench::amdahl_bound(1.0, 9.0, 4.0));
    return 0;
}

int main(int argc, char** argv) {
    try {
        if (argc == 4 && std::string(argv[1]) == "csv") return csv_mode(argv[2], argv[3]);
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
        {   // early rejection (opt-in): the same accepted set, bit for bit
            cuda::set_early_reject(true);
            const auto early = abc::reject_fixed_epsilon(model, 20000, 0, 20000, 1337, observed, sel.epsilon, 20000);
            cuda::set_early_reject(false);
            std::printf("early_reject_identical %d\n",
                        static_cast<int>(early.total_accepted == acc.total_accepted && early.rows == acc.rows &&
                                         early.params == acc.params && early.discrepancies == acc.discrepancies));
        }

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
