// vexbayes/toggle_switch.hpp (B200 shim) -- the reference's toggle-switch model
// (toggle_switch.hpp:16-82) as a device-backed ModelHooks factory.  Same
// parameter order theta = (mu, sigma, gamma, alpha_u, alpha_v, beta_u, beta_v),
// prior box (toggle_switch.cpp:17-22), canonical per-cell variate layout and 19
// quantile summaries; abc::run_prior_predictive on these hooks is bit-identical
// to the reference for the same (seed, workers, block_width).
#pragma once

#include <array>
#include <memory>
#include <span>
#include <vector>

#include "cuda_context.hpp"
#include "model.hpp"

namespace vexbayes::toggle {

inline constexpr std::size_t kToggleDim = 7;
inline constexpr std::size_t kToggleSummaryDim = 19;

struct ToggleParams {
    double mu, sigma, gamma, alpha_u, alpha_v, beta_u, beta_v;
    std::array<double, 7> as_array() const { return {mu, sigma, gamma, alpha_u, alpha_v, beta_u, beta_v}; }
};

inline constexpr std::size_t cell_stride(std::size_t steps) { return 2 * steps; }

// throughput = true selects the statistically validated fast mode (packed Philox4x32
// normals, table-based powers, FMA arithmetic, particle keying) instead of the
// bit-exact replay of the reference.
inline ModelHooks make_abc_model(std::size_t steps, std::size_t cells, bool throughput = false) {
    auto dm = std::make_shared<DeviceModel>();
    *dm = DeviceModel{};
    dm->model = VXB_MODEL_TOGGLE;
    dm->precision = VXB_F64;
    dm->rng = throughput ? VXB_RNG_FAST : VXB_RNG_REF;
    dm->arith = throughput ? VXB_ARITH_FMA : VXB_ARITH_EXACT;
    dm->dim = kToggleDim;
    dm->summary_dim = kToggleSummaryDim;
    dm->steps = dm->obs_stride = static_cast<std::uint32_t>(steps);
    dm->x0 = 10.0;
    const double lo[7] = {250.0, 0.05, 0.05, 0.0, 0.0, 0.0, 0.0};
    const double hi[7] = {400.0, 0.5, 0.35, 50.0, 50.0, 7.0, 7.0};
    for (int k = 0; k < 7; ++k) {
        dm->prior_lo[k] = lo[k];
        dm->prior_hi[k] = hi[k];
    }
    dm->consts[1] = static_cast<double>(cells);
    ModelHooks hooks;
    hooks.dim = kToggleDim;
    hooks.summary_dim = kToggleSummaryDim;
    hooks.device = dm;
    return hooks;
}

// The 19 summary quantiles of one simulation at theta from stream
// (seed, stream_id) at position pos (bench.cpp:69-77 builds observed data so).
inline std::vector<double> simulate_summaries(const ModelHooks& model, const ToggleParams& theta,
                                              std::uint64_t seed, std::uint32_t stream_id,
                                              std::uint64_t pos) {
    require(static_cast<bool>(model.device), "unsupported-model", "model has no device descriptor");
    const auto th = theta.as_array();
    std::vector<double> out(kToggleSummaryDim);
    cuda::check(vxb_simulate_at(cuda::context(), model.device.get(), th.data(), seed, stream_id, pos,
                                out.data()));
    return out;
}

}  // namespace vexbayes::toggle
