// vexbayes/rng.hpp (B200 shim) -- seed derivation and device stream fills.
// Mirrors the free functions of the reference's rng.hpp:10-16,80-83; the
// per-draw RngStream object stays a host-side concept of the reference and is
// not needed by the batched drivers (streams are addressed by counter position
// on the device).
#pragma once

#include <cstdint>
#include <initializer_list>
#include <vector>

#include "cuda_context.hpp"

namespace vexbayes {

inline std::uint64_t splitmix64(std::uint64_t z) { return vxb_splitmix64(z); }

inline std::uint64_t derive_seed(std::uint64_t seed, std::initializer_list<std::uint64_t> path) {
    return vxb_derive_seed(seed, path.begin(), path.size());
}

// n uniforms / Gaussians of stream (seed, stream_id) starting at counter
// position pos, generated on the GPU, bit-identical to RngStream's fills.
inline std::vector<double> fill_uniform(std::uint64_t seed, std::uint32_t stream_id,
                                        std::uint64_t pos, std::size_t n, double a, double b) {
    std::vector<double> out(n);
    cuda::check(vxb_rng_fill_uniform(cuda::context(), seed, stream_id, pos, n, a, b, out.data()));
    return out;
}
inline std::vector<double> fill_gaussian(std::uint64_t seed, std::uint32_t stream_id,
                                         std::uint64_t pos, std::size_t n, double mu,
                                         double sigma) {
    std::vector<double> out(n);
    cuda::check(vxb_rng_fill_gaussian(cuda::context(), seed, stream_id, pos, n, mu, sigma, out.data()));
    return out;
}

}  // namespace vexbayes
