// vxb_ppp.cu -- prior-predictive p-values over a hyperparameter grid (config 2).
//
// Model: y_i ~ N(theta, 1), i < n, theta ~ N(0, lambda^2).  For every lambda_k
// the kernel draws M prior-predictive datasets, reduces each to its sample mean
// and counts how many have a prior-predictive density no larger than the
// observed one -- the counting rule of weakinfo::estimate_pvalues
// (weak_info.cpp:108-120: p = #{value <= observed}/N, ties count), with the
// per-dataset sort replaced by a fused compare + ballot + integer atomic.
//
// Draw order follows weakinfo::sample_prior_predictive (weak_info.cpp:82-106):
// align_even; one Gaussian pair for the prior draw (theta = lambda * z_0, the
// second half of the pair is unused); then the data y_i = theta + z_i from the
// following pairs.  Dataset (k, j) owns RngStream(derive_seed(seed,{k}), j).
// One dataset per thread; nothing but the 64 counters leaves the device.

#include <cmath>

#include "vxb_common.cuh"
#include "vxb_logistic.cuh"

#ifndef VXB_PPP_MINB
#define VXB_PPP_MINB 1
#endif

namespace vxb {

constexpr int kPppBlock = 256;
constexpr int kMaxLambda = 256;

struct PppParams {
    uint64_t first, count;
    uint32_t n_data, n_lambda;
    FastKeys fast;
    const double2* log_table;
    const uint64_t* seed_hash;  // n_lambda: splitmix64(derive_seed(seed,{k}))
    const double* lambda;       // n_lambda
    const double* log_norm;     // n_lambda
    const double* v;            // n_lambda: lambda^2 + 1/n
    const double* logm_obs;     // n_lambda
    unsigned long long* counts; // n_lambda
    double* ybar_out;           // optional: n_lambda x count
};

template <int kRng>
__global__ void __launch_bounds__(kPppBlock, VXB_PPP_MINB) ppp_kernel(const __grid_constant__ PppParams p) {
    __shared__ double2 s_log[kRng == VXB_RNG_FAST ? kFastTableSize : 1];
    __shared__ unsigned int s_count;
    if (kRng == VXB_RNG_FAST)
        for (int i = threadIdx.x; i < kFastTableSize; i += kPppBlock) s_log[i] = p.log_table[i];
    if (threadIdx.x == 0) s_count = 0;
    __syncthreads();
    const uint32_t k = blockIdx.y;
    const uint64_t r = static_cast<uint64_t>(blockIdx.x) * kPppBlock + threadIdx.x;
    bool hit = false;
    if (r < p.count) {
        const uint64_t j = p.first + r;
        const double lambda = p.lambda[k];
        const double dn = static_cast<double>(p.n_data);
        const uint32_t pairs = (p.n_data + 1) >> 1;
        double ybar;
        if (kRng == VXB_RNG_REF) {
            const uint64_t key = stream_key(p.seed_hash[k], j);
            double ze, zo;
            box_muller<Exact>(philox2x64(key, 0), ze, zo);
            const double theta = __dmul_rn(lambda, ze);
            double sum = 0.0;
            uint32_t i = 0;
            for (uint32_t q = 1; q <= pairs; ++q) {
                box_muller<Exact>(philox2x64(key, q), ze, zo);
                sum = __dadd_rn(sum, __dadd_rn(theta, ze));
                if (++i < p.n_data) {
                    sum = __dadd_rn(sum, __dadd_rn(theta, zo));
                    ++i;
                }
            }
            ybar = __ddiv_rn(sum, dn);
        } else {
            // throughput generator: batches of eight normals from three Philox blocks,
            // drawn one batch ahead (FastNoise64); normal 0 is the prior draw, normals
            // 1..n the data
            const uint32_t jl = static_cast<uint32_t>(j), jh = static_cast<uint32_t>(j >> 32);
            FastNoise64 noise(p.fast, s_log, jl, jh, 0u, kDomNoise | (k << 8));
            double z[8];
            noise.next(z);
            const double theta = lambda * z[0];
            double s0 = 0.0, s1 = 0.0;
            uint32_t left = p.n_data;
#pragma unroll
            for (int q = 1; q < 8; ++q) {
                if (left) {
                    (q & 1 ? s1 : s0) += z[q];
                    --left;
                }
            }
            while (left >= 8) {
                noise.next(z);
                s0 += (z[0] + z[2]) + (z[4] + z[6]);
                s1 += (z[1] + z[3]) + (z[5] + z[7]);
                left -= 8;
            }
            if (left) {
                noise.next(z);
#pragma unroll
                for (int q = 0; q < 8; ++q)
                    if (static_cast<uint32_t>(q) < left) (q & 1 ? s1 : s0) += z[q];
            }
            ybar = theta + (s0 + s1) / dn;
        }
        if (p.ybar_out) p.ybar_out[static_cast<uint64_t>(k) * p.count + r] = ybar;
        // logm = log_norm - ((0.5 ybar) ybar) / v
        const double logm =
            __dsub_rn(p.log_norm[k], __ddiv_rn(__dmul_rn(__dmul_rn(0.5, ybar), ybar), p.v[k]));
        hit = logm <= p.logm_obs[k];
    }
    const unsigned ballot = __ballot_sync(0xffffffffu, hit);
    if ((threadIdx.x & 31) == 0 && ballot) atomicAdd(&s_count, __popc(ballot));
    __syncthreads();
    if (threadIdx.x == 0 && s_count) atomicAdd(&p.counts[k], static_cast<unsigned long long>(s_count));
}

}  // namespace vxb

using namespace vxb;

extern "C" int vxb_ppp_pvalues(vxb_ctx* ctx, const vxb_model* model, const double* lambda,
                               const double* log_norm, uint32_t n_lambda, uint64_t m_total,
                               uint64_t first, uint64_t count, uint64_t seed, double ybar_obs,
                               uint64_t* counts, double* pvalues, double* ybar_out) {
    return guarded([&] {
        use(ctx);
        require(model && lambda && log_norm && counts, "invalid-argument", "null argument");
        require(model->model == VXB_MODEL_NORMAL_MEAN, "invalid-argument",
                "not the normal-mean model");
        require(model->steps >= 1, "insufficient-data",
                "need at least one observation per dataset");
        require(n_lambda >= 1 && n_lambda <= kMaxLambda && m_total >= 1 &&
                    first + count <= m_total,
                "invalid-shape", "bad lambda grid or dataset range");
        require(model->rng == VXB_RNG_REF || model->rng == VXB_RNG_FAST, "invalid-argument",
                "bad rng mode");
        const double dn = static_cast<double>(model->steps);
        std::vector<uint64_t> h_seed(n_lambda);
        std::vector<double> h_v(n_lambda), h_obs(n_lambda);
        for (uint32_t k = 0; k < n_lambda; ++k) {
            require(lambda[k] >= 0.0, "invalid-argument", "prior scales must be nonnegative");
            const uint64_t kk = k;
            h_seed[k] = splitmix64(vxb_derive_seed(seed, &kk, 1));
            h_v[k] = lambda[k] * lambda[k] + 1.0 / dn;
            h_obs[k] = log_norm[k] - ((0.5 * ybar_obs) * ybar_obs) / h_v[k];
        }
        PppParams p{};
        p.first = first;
        p.count = count;
        p.n_data = model->steps;
        p.n_lambda = n_lambda;
        p.fast = make_fast_keys(splitmix64(seed));
        p.log_table = ctx->log_table;
        Staged d_seed(ctx, h_seed.data(), n_lambda * 8, true, false);
        Staged d_lambda(ctx, lambda, n_lambda * 8, true, false);
        Staged d_ln(ctx, log_norm, n_lambda * 8, true, false);
        Staged d_v(ctx, h_v.data(), n_lambda * 8, true, false);
        Staged d_obs(ctx, h_obs.data(), n_lambda * 8, true, false);
        Scratch d_counts(ctx, n_lambda * 8);
        Staged d_ybar(ctx, ybar_out, static_cast<size_t>(n_lambda) * count * 8, false, true);
        VXB_CUDA(cudaMemsetAsync(d_counts.as<void>(), 0, n_lambda * 8, ctx->stream));
        p.seed_hash = d_seed.as<uint64_t>();
        p.lambda = d_lambda.as<double>();
        p.log_norm = d_ln.as<double>();
        p.v = d_v.as<double>();
        p.logm_obs = d_obs.as<double>();
        p.counts = d_counts.as<unsigned long long>();
        p.ybar_out = d_ybar.as<double>();
        if (count) {
            LaunchScope scope(ctx, VXB_K_PPP);
            const dim3 grid(grid_for(count, kPppBlock), n_lambda);
            if (model->rng == VXB_RNG_FAST)
                ppp_kernel<VXB_RNG_FAST><<<grid, kPppBlock, 0, ctx->stream>>>(p);
            else
                ppp_kernel<VXB_RNG_REF><<<grid, kPppBlock, 0, ctx->stream>>>(p);
            check_launch("ppp_kernel");
        }
        std::vector<unsigned long long> h_counts(n_lambda);
        VXB_CUDA(cudaMemcpyAsync(h_counts.data(), p.counts, n_lambda * 8, cudaMemcpyDeviceToHost,
                                 ctx->stream));
        d_ybar.finish();
        VXB_CUDA(cudaStreamSynchronize(ctx->stream));
        const bool counts_on_device = is_device_pointer(counts);
        for (uint32_t k = 0; k < n_lambda; ++k)
            if (pvalues && !is_device_pointer(pvalues))
                pvalues[k] = static_cast<double>(h_counts[k]) / static_cast<double>(m_total);
        if (counts_on_device)
            VXB_CUDA(cudaMemcpy(counts, h_counts.data(), n_lambda * 8, cudaMemcpyHostToDevice));
        else
            for (uint32_t k = 0; k < n_lambda; ++k) counts[k] = h_counts[k];
    });
}
