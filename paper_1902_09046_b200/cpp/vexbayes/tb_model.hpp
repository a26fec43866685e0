// vexbayes/tb_model.hpp (B200 shim) -- the reference's TB transmission model
// (tb_model.hpp:12-76) as a device-backed ModelHooks factory: theta = (alpha,
// delta, tau) with the prior of tb::sample_prior, exact Gillespie simulation (one
// warp per path), summaries (G, H).  abc::run_prior_predictive on these hooks uses
// particle keying (row i owns RngStream(seed, i)) -- a path consumes a
// data-dependent number of variates, so the per-worker sequential keying of the
// CPU sampler cannot be addressed in parallel; `workers` and `block_width` are
// accepted and do not change the result.
#pragma once

#include <limits>
#include <memory>
#include <vector>

#include "cuda_context.hpp"
#include "model.hpp"

namespace vexbayes::tb {

struct TbParams {
    double alpha;
    double delta;
    double tau;
};
struct StopRule {
    double time_horizon = 50.0;
    double case_target = 10000.0;
};
struct TbSummaries {
    double genotypes;  // G
    double diversity;  // H = 1 - sum (X_i/N)^2
};
inline constexpr double kNoHorizon = std::numeric_limits<double>::infinity();

inline ModelHooks make_abc_model(std::size_t initial_cases, StopRule stop) {
    auto dm = std::make_shared<DeviceModel>();
    *dm = DeviceModel{};
    dm->model = VXB_MODEL_TB;
    dm->precision = VXB_F64;
    dm->rng = VXB_RNG_REF;
    dm->arith = VXB_ARITH_EXACT;
    dm->dim = 3;
    dm->summary_dim = 2;
    dm->consts[0] = static_cast<double>(initial_cases);
    dm->consts[1] = stop.time_horizon;
    dm->consts[2] = stop.case_target;
    dm->consts[3] = 1.0;
    dm->prior_hi[0] = 2.0;
    dm->prior_hi[2] = 1.0;
    ModelHooks hooks;
    hooks.dim = 3;
    hooks.summary_dim = 2;
    hooks.device = dm;
    return hooks;
}

// One path at theta from RngStream(seed, stream_id) at pos, reduced to (G, H);
// extinct-population when the path dies out (tb_summaries, tb_model.cpp:129-131).
// attempts > 1 retries from where the stream stands (bench.cpp:83-90).
inline TbSummaries simulate_summaries(const TbParams& theta, std::size_t initial_cases, StopRule stop,
                                      std::uint64_t seed, std::uint32_t stream_id, std::uint64_t pos,
                                      unsigned attempts = 1) {
    ModelHooks model = make_abc_model(initial_cases, stop);
    auto dm = std::make_shared<DeviceModel>(*model.device);
    dm->consts[3] = static_cast<double>(attempts);
    const double th[3] = {theta.alpha, theta.delta, theta.tau};
    double out[2] = {0.0, 0.0};
    cuda::check(vxb_simulate_at(cuda::context(), dm.get(), th, seed, stream_id, pos, out));
    return {out[0], out[1]};
}

}  // namespace vexbayes::tb
