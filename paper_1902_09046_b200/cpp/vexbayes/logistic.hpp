// vexbayes/logistic.hpp -- the stochastic logistic-growth model of BASELINE
// configs 0/1/3 as a ModelHooks factory in the mould of the reference's
// toggle::make_abc_model (toggle_switch.cpp:135-152).  Only the device
// descriptor is filled: the simulator runs on the GPU.
#pragma once

#include <array>
#include <cmath>
#include <memory>

#include "model.hpp"

namespace vexbayes::logistic {

inline constexpr std::size_t kLogisticDim = 3;  // theta = (r, K, sigma)

struct LogisticConfig {
    std::size_t steps = 2000;       // Euler-Maruyama steps
    std::size_t obs_stride = 100;   // state recorded every obs_stride steps
    double dt = 0.01;
    double x0 = 10.0;
    std::array<double, 3> prior_lo{0.0, 50.0, 0.0};
    std::array<double, 3> prior_hi{1.0, 150.0, 0.2};
};

inline ModelHooks make_abc_model(const LogisticConfig& cfg = {}) {
    auto dm = std::make_shared<DeviceModel>();
    *dm = DeviceModel{};
    dm->model = VXB_MODEL_LOGISTIC_SDE;
    dm->precision = VXB_F64;
    dm->rng = VXB_RNG_REF;
    dm->arith = VXB_ARITH_EXACT;
    dm->dim = kLogisticDim;
    dm->steps = static_cast<std::uint32_t>(cfg.steps);
    dm->obs_stride = static_cast<std::uint32_t>(cfg.obs_stride);
    dm->summary_dim = cfg.obs_stride ? static_cast<std::uint32_t>(cfg.steps / cfg.obs_stride) : 0;
    dm->dt = cfg.dt;
    dm->x0 = cfg.x0;
    for (int k = 0; k < 3; ++k) {
        dm->prior_lo[k] = cfg.prior_lo[k];
        dm->prior_hi[k] = cfg.prior_hi[k];
    }
    dm->consts[0] = std::sqrt(cfg.dt);
    ModelHooks hooks;
    hooks.dim = kLogisticDim;
    hooks.summary_dim = dm->summary_dim;
    hooks.device = dm;
    return hooks;
}

// One simulation at theta from stream (seed, stream_id) at position pos, the way
// the reference builds synthetic observed summaries (bench.cpp:69-77).
inline std::vector<double> simulate_at(const ModelHooks& model, std::span<const double> theta,
                                       std::uint64_t seed, std::uint32_t stream_id,
                                       std::uint64_t pos);

}  // namespace vexbayes::logistic

#include "cuda_context.hpp"
#include "errors.hpp"

namespace vexbayes::logistic {
inline std::vector<double> simulate_at(const ModelHooks& model, std::span<const double> theta,
                                       std::uint64_t seed, std::uint32_t stream_id,
                                       std::uint64_t pos) {
    require(static_cast<bool>(model.device), "unsupported-model", "model has no device descriptor");
    require(theta.size() == kLogisticDim, "invalid-argument", "logistic parameter vector needs 3 entries");
    std::vector<double> out(model.summary_dim);
    cuda::check(vxb_simulate_at(cuda::context(), model.device.get(), theta.data(), seed, stream_id,
                                pos, out.data()));
    return out;
}
}  // namespace vexbayes::logistic
