// vexbayes/abc.hpp (B200 shim) -- drop-in for the reference ABC sampler
// interface (abc.hpp:16-58): same names, argument meaning and error behaviour,
// executed by libvexbayes_cuda.so.
//
//   run_prior_predictive   -> vxb_multi_abc_prior_predictive with VXB_KEY_WORKER, so
//       the result is bit-identical to the reference for the same
//       (seed, workers, block_width)  (abc.cpp:26-73).  `workers` keeps its
//       meaning for the STREAM LAYOUT (worker w owns stream (seed, w)); the rows
//       themselves are split over the GPUs in use (cuda::set_devices, default:
//       every visible device) by partition(n, G, 1) -- a device where the
//       reference has a worker thread (abc.cpp:43-71);
//   select_epsilon         -> vxb_multi_select_epsilon     (abc.cpp:75-97): the rows are
//       split over the GPUs in use, the digit histograms of the radix select are
//       all-reduced -- same epsilon and indices for any device count;
//   discrepancy            -> host arithmetic, left-to-right (abc.cpp:16-24);
//   write_csv              -> same column layout, %.17g      (abc.cpp:99-124).
// Extension for jobs that do not fit the fixed-N container (config 1):
//   reject_fixed_epsilon   -> vxb_abc_reject (only accepted rows leave the GPU);
//   reject_fixed_epsilon (whole job) -> vxb_multi_abc_reject: rows sharded over the
//       GPUs in use, accepted samples gathered over NCCL inside the library.
#pragma once

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <fstream>
#include <ostream>
#include <span>
#include <string>
#include <vector>

#include "cuda_context.hpp"
#include "model.hpp"

namespace vexbayes::abc {

struct PriorPredictiveSet {
    std::size_t rows = 0;
    std::size_t dim = 0;
    std::size_t summary_dim = 0;
    std::vector<double> params;         // rows x dim
    std::vector<double> summaries;      // rows x summary_dim
    std::vector<double> discrepancies;  // rows (NaN where failed)
    std::vector<std::uint8_t> failed;   // rows

    std::span<const double> param_row(std::size_t r) const { return {params.data() + r * dim, dim}; }
    std::span<const double> summary_row(std::size_t r) const {
        return {summaries.data() + r * summary_dim, summary_dim};
    }
};

struct EpsilonSelection {
    double epsilon = 0.0;
    std::vector<std::size_t> accepted;  // ascending row indices with rho <= epsilon
};

inline double discrepancy(std::span<const double> sim, std::span<const double> obs) {
    require(sim.size() == obs.size(), "invalid-summary", "summary vector lengths differ");
    double ss = 0.0;
    for (std::size_t i = 0; i < sim.size(); ++i) {
        const double d = sim[i] - obs[i];
        ss += d * d;
    }
    return std::sqrt(ss);
}

inline const DeviceModel& device_model(const ModelHooks& model) {
    require(static_cast<bool>(model.device), "unsupported-model",
            "model has no device descriptor (the GPU build has no CPU fallback)");
    return *model.device;
}

inline PriorPredictiveSet run_prior_predictive(const ModelHooks& model, std::size_t n,
                                               std::size_t workers, std::size_t block_width,
                                               std::uint64_t seed,
                                               std::span<const double> observed) {
    require(n >= 1, "invalid-shape", "need at least one prior predictive sample");
    require(workers >= 1, "invalid-shape", "need at least one worker");
    require(observed.size() == model.summary_dim, "invalid-summary",
            "observed summary length differs from the model summary dimension");
    const DeviceModel& dm = device_model(model);
    require(dm.precision == VXB_F64, "invalid-argument", "the reference container is fp64");
    PriorPredictiveSet set;
    set.rows = n;
    set.dim = model.dim;
    set.summary_dim = model.summary_dim;
    set.params.resize(n * model.dim);
    set.summaries.resize(n * model.summary_dim);
    set.discrepancies.resize(n);
    set.failed.resize(n);
    vxb_keying key{VXB_KEY_WORKER, static_cast<std::uint32_t>(workers),
                   static_cast<std::uint32_t>(block_width), 0, seed};
    if (dm.model == VXB_MODEL_TOGGLE && dm.rng == VXB_RNG_FAST) {
        // throughput mode of the toggle model: rows keyed per particle
        key = vxb_keying{VXB_KEY_PARTICLE, 1, 1, 0, seed};
    }
    if (dm.model == VXB_MODEL_TB) {
        // a TB path consumes a data-dependent number of variates: rows are keyed per
        // particle (tb_model.hpp of this shim); block_width is validated as the
        // reference does (blocked.cpp:10-12)
        require(block_width == 1 || block_width == 2 || block_width == 4 || block_width == 8 ||
                    block_width == 16,
                "invalid-shape", "unsupported block width");
        key = vxb_keying{VXB_KEY_PARTICLE, 1, 1, 0, seed};
    }
    cuda::check(vxb_multi_abc_prior_predictive(cuda::multi(), &dm, &key, n, observed.data(),
                                               set.params.data(), set.summaries.data(),
                                               set.discrepancies.data(), set.failed.data()));
    return set;
}

inline EpsilonSelection select_epsilon(const PriorPredictiveSet& set, double accept_fraction) {
    require(accept_fraction > 0.0 && accept_fraction <= 1.0, "invalid-argument",
            "accept fraction must lie in (0, 1]");
    require(set.rows >= 1, "empty-set", "every prior predictive row failed");
    std::vector<std::uint64_t> idx(set.rows);
    std::uint64_t n_acc = 0;
    EpsilonSelection sel;
    cuda::check(vxb_multi_select_epsilon(cuda::multi(), VXB_F64, set.discrepancies.data(),
                                         set.failed.data(), set.rows, accept_fraction, &sel.epsilon,
                                         idx.size(), &n_acc, idx.data()));
    sel.accepted.assign(idx.begin(), idx.begin() + static_cast<std::ptrdiff_t>(n_acc));
    return sel;
}

// Fixed-epsilon rejection over rows [first, first+count) of an n_total-row job
// keyed per particle (shard-independent).  Accepted rows only.
struct AcceptedSet {
    std::uint64_t total_accepted = 0;       // may exceed the kept rows when capped
    std::vector<std::uint64_t> rows;        // ascending global row numbers
    std::vector<double> params;             // kept x dim
    std::vector<double> discrepancies;      // kept
};
inline AcceptedSet reject_fixed_epsilon(const ModelHooks& model, std::uint64_t n_total,
                                        std::uint64_t first, std::uint64_t count,
                                        std::uint64_t seed, std::span<const double> observed,
                                        double epsilon, std::uint64_t cap) {
    require(observed.size() == model.summary_dim, "invalid-summary",
            "observed summary length differs from the model summary dimension");
    const DeviceModel& dm = device_model(model);
    require(dm.precision == VXB_F64, "invalid-argument", "this container is fp64");
    AcceptedSet out;
    out.rows.resize(cap);
    out.params.resize(cap * model.dim);
    out.discrepancies.resize(cap);
    vxb_keying key{VXB_KEY_PARTICLE, 1, 1, 0, seed};
    cuda::check(vxb_abc_reject(cuda::context(), &dm, &key, n_total, first, count, observed.data(),
                               epsilon, cap, &out.total_accepted, out.rows.data(),
                               out.params.data(), out.discrepancies.data()));
    const std::uint64_t kept = out.total_accepted < cap ? out.total_accepted : cap;
    out.rows.resize(kept);
    out.params.resize(kept * model.dim);
    out.discrepancies.resize(kept);
    return out;
}

// The whole n_total-row job over every GPU in use (config 1): device g simulates
// partition(n_total, G, 1)[g]; the accepted samples are gathered over NCCL inside
// the library; identical to the one-GPU result for any G.  `cap` = rows kept.
inline AcceptedSet reject_fixed_epsilon(const ModelHooks& model, std::uint64_t n_total,
                                        std::uint64_t seed, std::span<const double> observed,
                                        double epsilon, std::uint64_t cap) {
    require(observed.size() == model.summary_dim, "invalid-summary",
            "observed summary length differs from the model summary dimension");
    const DeviceModel& dm = device_model(model);
    require(dm.precision == VXB_F64, "invalid-argument", "this container is fp64");
    AcceptedSet out;
    out.rows.resize(cap);
    out.params.resize(cap * model.dim);
    out.discrepancies.resize(cap);
    vxb_keying key{VXB_KEY_PARTICLE, 1, 1, 0, seed};
    cuda::check(vxb_multi_abc_reject(cuda::multi(), &dm, &key, n_total, observed.data(), epsilon,
                                     cap, &out.total_accepted, out.rows.data(), out.params.data(),
                                     out.discrepancies.data()));
    const std::uint64_t kept = out.total_accepted < cap ? out.total_accepted : cap;
    out.rows.resize(kept);
    out.params.resize(kept * model.dim);
    out.discrepancies.resize(kept);
    return out;
}

inline void write_csv(const PriorPredictiveSet& set, std::ostream& out) {
    out << "row";
    for (std::size_t k = 1; k <= set.dim; ++k) out << ",theta_" << k;
    for (std::size_t k = 1; k <= set.summary_dim; ++k) out << ",s_" << k;
    out << ",rho,failed\n";
    char buf[64];
    for (std::size_t r = 0; r < set.rows; ++r) {
        out << r;
        auto put = [&](double v) {
            std::snprintf(buf, sizeof(buf), "%.17g", v);
            out << ',' << buf;
        };
        for (double v : set.param_row(r)) put(v);
        for (double v : set.summary_row(r)) put(v);
        put(set.discrepancies[r]);
        out << ',' << static_cast<int>(set.failed[r]) << '\n';
    }
}
inline void write_csv(const PriorPredictiveSet& set, const std::string& path) {
    std::ofstream out(path);
    require(out.good(), "io-error", "cannot open " + path + " for writing");
    write_csv(set, out);
    require(out.good(), "io-error", "write to " + path + " failed");
}

}  // namespace vexbayes::abc
