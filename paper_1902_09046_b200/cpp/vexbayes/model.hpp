// vexbayes/model.hpp (B200 shim) -- the model contract.
//
// The reference's ModelHooks (model.hpp:19-36) is a bag of std::function
// closures called once per row on the host.  A device cannot call them, so the
// GPU drivers identify a model by a POD descriptor instead; the hook members
// are kept so that existing aggregate-by-name initialisation still compiles,
// and one optional member is added: `device`.  Drivers in this shim require
// it and refuse (Error "unsupported-model") otherwise -- there is no CPU path.
#pragma once

#include <cstddef>
#include <functional>
#include <memory>
#include <span>

#include "../../../include/vexbayes_cuda.h"

namespace vexbayes {

class RngStream;  // host-side stream type of the reference; unused by the GPU drivers

using DeviceModel = vxb_model;

struct ModelHooks {
    std::size_t dim = 0;
    std::size_t summary_dim = 0;
    std::function<void(RngStream&, std::span<double>)> sample_prior;
    std::function<void(std::span<const double>, RngStream&, std::size_t, std::span<double>)> simulate;
    std::function<double(std::span<const double>)> log_prior;
    std::function<double(std::span<const double>)> log_likelihood;
    std::function<void(std::span<const double>, std::size_t, std::span<double>)> block_log_likelihood;
    // GPU descriptor of the same model (what the kernels read).
    std::shared_ptr<const DeviceModel> device;
    // Models whose device form needs more than the POD descriptor (a dataset):
    // a family tag and the family's own binding (bioassay.hpp).
    const char* family = nullptr;
    std::shared_ptr<const void> binding;
};

}  // namespace vexbayes
