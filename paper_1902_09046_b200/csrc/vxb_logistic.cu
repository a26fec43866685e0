// vxb_logistic.cu -- ABC rejection on the logistic SDE (configs 0/1): the fused
// simulate -> summary -> distance kernel and the C-ABI entry points built on it
// (drop-ins for abc::run_prior_predictive, abc.cpp:26-73).
//
// Launch shape: one particle per thread, state in registers, 256-thread CTAs.
// The kernel is FP64-pipe bound (fp32: FP32/MUFU bound); HBM traffic is the
// per-row outputs only (<= 8 B/row on the fused fixed-epsilon path).

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <limits>

#include "vxb_internal.cuh"

namespace vxb {

struct AbcParams {
    uint64_t first, count;
    Keying key;
    LogisticModel model;
    double observed[VXB_MAX_SUMMARY];
    const double* theta_in;  // kKeyFixed: simulate at this theta, no prior draw
    const double2* log_table;  // fast fp64 generator: log + trig tables, kFastTableSize entries
    void* params;
    void* summaries;
    void* rho;
    uint8_t* failed;
    const void* noise;
    // early rejection: partial squared distance beyond which a row is lost; +inf: off
    double ss_bound = std::numeric_limits<double>::infinity();
    // Early rejection in SEGMENTS (vxb_abc_reject): this launch simulates observations
    // [obs_begin, obs_end) of its rows; rows that are still alive at the end of a segment
    // that is not the last are appended to the out-queue (row offset, state, partial sum)
    // and the next launch takes them from there, densely packed again -- a warp whose rows
    // died one by one would otherwise run on for its last survivor.
    uint32_t obs_begin = 0, obs_end = 0xFFFFFFFFu;
    const uint32_t* in_rows = nullptr;  // null: rows 0 .. count-1 from the initial state
    const void* in_x = nullptr;
    const void* in_ss = nullptr;
    const unsigned long long* in_count = nullptr;
    uint32_t* out_rows = nullptr;  // null: last segment
    void* out_x = nullptr;
    void* out_ss = nullptr;
    unsigned long long* out_count = nullptr;
};

#ifndef VXB_SIM_BLOCK
#define VXB_SIM_BLOCK 256
#endif
#ifndef VXB_SIM_MIN_BLOCKS
#define VXB_SIM_MIN_BLOCKS 1
#endif
constexpr int kBlock = VXB_SIM_BLOCK;

// kSeg: the segment form of early rejection (queues in / out, a range of observations, a
// strided loop over the items); false compiles to the plain one-row-per-thread kernel.
template <class Real, int kRng, bool kFma, bool kSeg>
// (block, CTAs per SM) swept on a B200: fp64 is best with the registers it asks for
// (2.73e8 sims/s at (256, 1) against 2.49-2.56e8 at 3-4 CTAs per SM); the fp32
// throughput instance gains 1.6 % from four CTAs per SM.
#ifndef VXB_SEG_MIN_BLOCKS
#define VXB_SEG_MIN_BLOCKS 2  // the segment form asks for 140 registers in fp64: capped at 128 (two CTAs per SM) 116.5 against 132.8 ms
#endif
__global__ void __launch_bounds__(kBlock, (sizeof(Real) == 4 && kRng == VXB_RNG_FAST) ? 4 : kSeg ? VXB_SEG_MIN_BLOCKS : VXB_SIM_MIN_BLOCKS)
logistic_abc_kernel(const __grid_constant__ AbcParams p) {
    // fast fp64 generator: stage the 2 KB log table in shared memory
    __shared__ double2 s_log[(kRng == VXB_RNG_FAST && sizeof(Real) == 8) ? kFastTableSize : 1];
    if (kRng == VXB_RNG_FAST && sizeof(Real) == 8) {
        for (int i = threadIdx.x; i < kFastTableSize; i += kBlock) s_log[i] = p.log_table[i];
        __syncthreads();
    }
    // one item per thread; a launch over a queue runs a fixed grid with a stride
    const bool queued = kSeg && p.in_rows != nullptr;
    const uint64_t n_items = queued ? *p.in_count : p.count;
    auto run_item = [&](const uint64_t item) {
        const uint64_t r = queued ? p.in_rows[item] : item;
        const uint64_t row = p.first + r;
        uint64_t key, base;
        locate_row(p.key, row, key, base);

        double theta[3];
        uint64_t noise_pos;
        if (p.theta_in) {
            theta[0] = p.theta_in[0];
            theta[1] = p.theta_in[1];
            theta[2] = p.theta_in[2];
            noise_pos = base + (base & 1);
        } else {
            if (kRng == VXB_RNG_FAST)
                draw_prior_fast(p.model, p.key.fast, row, theta);
            else
                draw_prior_ref(p.model, key, base, theta);
            noise_pos = base + 4;  // three uniforms, aligned to the pair boundary
        }
        if (sizeof(Real) == 4) {
            theta[0] = static_cast<double>(static_cast<float>(theta[0]));
            theta[1] = static_cast<double>(static_cast<float>(theta[1]));
            theta[2] = static_cast<double>(static_cast<float>(theta[2]));
        }
        if (p.params) {
            Real* out = static_cast<Real*>(p.params) + r * 3;
            out[0] = static_cast<Real>(theta[0]);
            out[1] = static_cast<Real>(theta[1]);
            out[2] = static_cast<Real>(theta[2]);
        }

        Real* summary = p.summaries ? static_cast<Real*>(p.summaries) + r * p.model.n_obs : nullptr;
        auto emit = [summary](uint32_t k, Real v) {
            if (summary) summary[k] = v;
        };
        using A = typename std::conditional<
            kFma, typename std::conditional<kRng == VXB_RNG_FAST && sizeof(Real) == 8, FusedCompact, Fused>::type,
            Exact>::type;
        bool bad;
        const Real ss_bound = static_cast<Real>(p.ss_bound);  // +inf stays +inf
        Real x = queued ? static_cast<const Real*>(p.in_x)[item] : static_cast<Real>(p.model.x0);
        Real ss = queued ? static_cast<const Real*>(p.in_ss)[item] : Real(0);
        const uint32_t obs_begin = kSeg ? p.obs_begin : 0u, obs_end = kSeg ? p.obs_end : 0xFFFFFFFFu;
        const uint32_t step0 = obs_begin * p.model.obs_stride;  // the noise source starts at the batch that holds it
        if (kRng == VXB_RNG_REF) {
            RefNoise<Real> noise(key, (noise_pos >> 1) + (step0 >> 1));
            logistic_segment<Real, A>(p.model, theta, p.observed, noise, emit, bad, ss_bound, obs_begin, obs_end, x, ss);
        } else if (kRng == VXB_RNG_FAST) {
            const uint32_t rl = static_cast<uint32_t>(row), rh = static_cast<uint32_t>(row >> 32);
            if constexpr (sizeof(Real) == 4) {
                FastNoise32 noise(p.key.fast, rl, rh, 3u * (step0 / FastNoise32::kBatch));
                logistic_segment<Real, A>(p.model, theta, p.observed, noise, emit, bad, ss_bound, obs_begin, obs_end, x, ss);
            } else {
                FastNoise64 noise(p.key.fast, s_log, rl, rh, 3u * (step0 / FastNoise64::kBatch));
                logistic_segment<Real, A>(p.model, theta, p.observed, noise, emit, bad, ss_bound, obs_begin, obs_end, x, ss);
            }
        } else {
            ExternalNoise<Real> noise{static_cast<const Real*>(p.noise) + r * p.model.steps, step0,
                                      p.model.steps};
            logistic_segment<Real, A>(p.model, theta, p.observed, noise, emit, bad, ss_bound, obs_begin, obs_end, x, ss);
        }
        if (kSeg && p.out_rows && ss <= ss_bound) {
            // alive at the end of a segment that is not the last: hand the row on (one
            // atomic per warp; the order inside the queue is irrelevant, rho is addressed by row)
            const unsigned alive = __activemask();
            const unsigned lane = threadIdx.x & 31u;
            const int leader = __ffs(alive) - 1;
            unsigned long long slot = 0;
            if (lane == static_cast<unsigned>(leader)) slot = atomicAdd(p.out_count, static_cast<unsigned long long>(__popc(alive)));
            slot = __shfl_sync(alive, slot, leader) + __popc(alive & ((1u << lane) - 1u));
            p.out_rows[slot] = static_cast<uint32_t>(r);
            static_cast<Real*>(p.out_x)[slot] = x;
            static_cast<Real*>(p.out_ss)[slot] = ss;
            return;
        }
        Real rho = Exact::sqrt(ss);
        if (bad) {  // abc.cpp:57-60: flag the row, zero its summary, rho stays NaN
            rho = static_cast<Real>(__longlong_as_double(0x7FF8000000000000LL));
            if (summary)
                for (uint32_t k = 0; k < p.model.n_obs; ++k) summary[k] = Real(0);
        }
        if (p.rho) static_cast<Real*>(p.rho)[r] = rho;
        if (p.failed) p.failed[r] = bad ? 1 : 0;
    };
    const uint64_t first_item = static_cast<uint64_t>(blockIdx.x) * kBlock + threadIdx.x;
    if constexpr (kSeg) {
        const uint64_t stride_items = static_cast<uint64_t>(gridDim.x) * kBlock;
        for (uint64_t item = first_item; item < n_items; item += stride_items) run_item(item);
    } else {
        if (first_item < n_items) run_item(first_item);
    }
}

// The standard normals the step loop of the throughput generator consumes for
// rows [first, first+rows): row r, step j -> out[r * per_row + j].  Validation
// aid (vxb_rng_fill_gaussian_fast); same noise sources as the kernels above.
template <class Real>
__global__ void __launch_bounds__(256) fast_normals_kernel(FastKeys fk, const double2* table,
                                                           uint64_t first, uint64_t rows,
                                                           uint32_t per_row, Real* out) {
    // One thread per batch (eight fp64 / sixteen fp32 normals from three Philox blocks,
    // the unit the step loop consumes); the threads of a CTA take consecutive batches
    // of one row, so a warp writes one contiguous 2 KB piece of the row.
    __shared__ double2 s_tab[sizeof(Real) == 8 ? kFastTableSize : 1];
    if (sizeof(Real) == 8) {
        for (int i = threadIdx.x; i < kFastTableSize; i += 256) s_tab[i] = table[i];
        __syncthreads();
    }
    constexpr uint32_t kB = sizeof(Real) == 8 ? 8 : 16;
    const uint32_t q = blockIdx.y * 256 + threadIdx.x;  // batch inside the row
    if (q * kB >= per_row) return;
    for (uint64_t r = blockIdx.x; r < rows; r += gridDim.x) {
        const uint64_t row = first + r;
        const uint32_t rl = static_cast<uint32_t>(row), rh = static_cast<uint32_t>(row >> 32);
        const Words32 u = philox4x32(fk, 3 * q, kDomNoise, rl, rh);
        const Words32 v = philox4x32(fk, 3 * q + 1, kDomNoise, rl, rh);
        const Words32 w = philox4x32(fk, 3 * q + 2, kDomNoise, rl, rh);
        Real z[kB];
        if constexpr (sizeof(Real) == 8)
            fast_box_muller_x4(u, v, w, s_tab, z);
        else
            box_muller_f32_x8(u, v, w, z);
        Real* dst = out + r * per_row + static_cast<uint64_t>(q) * kB;
        if (q * kB + kB <= per_row && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
            using V = typename std::conditional<sizeof(Real) == 8, double2, float4>::type;
            constexpr int kPer = 16 / sizeof(Real);
#pragma unroll
            for (int e = 0; e < static_cast<int>(kB) / kPer; ++e) {
                V pack;
                if constexpr (sizeof(Real) == 8) {
                    pack.x = z[2 * e];
                    pack.y = z[2 * e + 1];
                } else {
                    pack.x = z[4 * e];
                    pack.y = z[4 * e + 1];
                    pack.z = z[4 * e + 2];
                    pack.w = z[4 * e + 3];
                }
                reinterpret_cast<V*>(dst)[e] = pack;
            }
        } else {
            for (uint32_t k = 0; k < kB && q * kB + k < per_row; ++k) dst[k] = z[k];
        }
    }
}

// Re-derives the prior draw of accepted rows and gathers their rho (fused
// fixed-epsilon path: rejected rows never leave the device).
template <class Real, int kRng>
__global__ void gather_accepted_kernel(Keying key, LogisticModel model, uint64_t first,
                                       const uint64_t* __restrict__ idx, uint64_t n_acc,
                                       const Real* __restrict__ rho_all, Real* params_out,
                                       Real* rho_out,
                                       const unsigned long long* __restrict__ n_acc_dev) {
    const uint64_t a = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    // asynchronous form: the accepted count lives on the device, n_acc is the cap
    const uint64_t lim = n_acc_dev ? min(n_acc, static_cast<uint64_t>(*n_acc_dev)) : n_acc;
    if (a >= lim) return;
    const uint64_t row = idx[a];
    uint64_t k, base;
    locate_row(key, row, k, base);
    double theta[3];
    if (kRng == VXB_RNG_FAST)
        draw_prior_fast(model, key.fast, row, theta);
    else
        draw_prior_ref(model, k, base, theta);
    if (params_out) {
        params_out[a * 3 + 0] = static_cast<Real>(theta[0]);
        params_out[a * 3 + 1] = static_cast<Real>(theta[1]);
        params_out[a * 3 + 2] = static_cast<Real>(theta[2]);
    }
    if (rho_out) rho_out[a] = rho_all[row - first];
}

LogisticModel make_logistic(const vxb_model& m) {
    require(m.model == VXB_MODEL_LOGISTIC_SDE, "invalid-argument", "not a logistic model");
    require(m.dim == 3, "invalid-shape", "logistic model has three parameters");
    require(m.steps >= 1 && m.obs_stride >= 1, "invalid-horizon", "need at least one step");
    require(m.summary_dim >= 1 && m.summary_dim == m.steps / m.obs_stride, "invalid-summary",
            "summary_dim must equal steps / obs_stride");
    require(m.summary_dim <= VXB_MAX_SUMMARY, "invalid-summary", "summary dimension too large");
    require(m.precision == VXB_F64 || m.precision == VXB_F32, "invalid-argument", "bad precision");
    require(m.rng >= VXB_RNG_REF && m.rng <= VXB_RNG_EXTERNAL, "invalid-argument", "bad rng mode");
    LogisticModel d;
    d.steps = m.steps;
    d.obs_stride = m.obs_stride;
    d.n_obs = m.summary_dim;
    d.dt = m.dt;
    d.sqdt = m.consts[0];
    d.x0 = m.x0;
    for (int k = 0; k < 3; ++k) {
        require(m.prior_lo[k] <= m.prior_hi[k], "invalid-range",
                "uniform lower bound exceeds upper bound");
        d.lo[k] = m.prior_lo[k];
        d.hi[k] = m.prior_hi[k];
    }
    return d;
}

Keying make_keying(const vxb_keying& k, const vxb_model& m, uint64_t n_total) {
    Keying d{};
    d.seed_hash = splitmix64(k.seed);
    d.fast = make_fast_keys(d.seed_hash);
    if (k.mode == VXB_KEY_PARTICLE) {
        d.mode = kKeyParticle;
    } else if (k.mode == VXB_KEY_WORKER) {
        require(k.workers >= 1, "invalid-shape", "need at least one worker");
        const uint32_t v = k.block_width;
        require(v == 1 || v == 2 || v == 4 || v == 8 || v == 16, "invalid-shape",
                "block width must be one of 1, 2, 4, 8, 16");  // blocked.cpp:10-12
        require(m.rng != VXB_RNG_FAST, "invalid-argument",
                "worker keying is defined for the reference generator only");
        d.mode = kKeyWorker;
        const uint64_t blocks = (n_total + v - 1) / v;
        d.base_blocks = blocks / k.workers;
        d.extra_blocks = blocks % k.workers;
        d.width = v;
        d.row_stride = 4 + m.steps + (m.steps & 1);
    } else {
        raise("invalid-argument", "unknown keying mode");
    }
    return d;
}

template <class Real, int kRng>
void launch_abc2(vxb_ctx* ctx, const AbcParams& p, bool fma) {
    unsigned grid = grid_for(p.count, kBlock);
    const bool seg = p.in_rows || p.out_rows || p.obs_begin != 0 || p.obs_end < p.model.n_obs;
    if (seg) {
        if constexpr (kRng != VXB_RNG_EXTERNAL) {
            auto kernel = fma ? logistic_abc_kernel<Real, kRng, true, true> : logistic_abc_kernel<Real, kRng, false, true>;
            if (p.in_rows) {
                // over a queue whose length only the device knows: a grid of resident CTAs, strided
                int per_sm = 0;
                VXB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, kBlock, 0));
                grid = std::min<unsigned>(grid, static_cast<unsigned>(ctx->prop.multiProcessorCount * std::max(per_sm, 1) * 4));
            }
            LaunchScope scope(ctx, VXB_K_SIMULATE);
            kernel<<<grid, kBlock, 0, ctx->stream>>>(p);
            check_launch("logistic_abc_kernel (segment)");
        } else {
            raise("internal", "segments are driven by vxb_abc_reject only");
        }
        return;
    }
    LaunchScope scope(ctx, VXB_K_SIMULATE);
    if (fma)
        logistic_abc_kernel<Real, kRng, true, false><<<grid, kBlock, 0, ctx->stream>>>(p);
    else
        logistic_abc_kernel<Real, kRng, false, false><<<grid, kBlock, 0, ctx->stream>>>(p);
    check_launch("logistic_abc_kernel");
}
template <class Real>
void launch_abc1(vxb_ctx* ctx, const AbcParams& p, int rng, bool fma) {
    if (rng == VXB_RNG_REF)
        launch_abc2<Real, VXB_RNG_REF>(ctx, p, fma);
    else if (rng == VXB_RNG_FAST)
        launch_abc2<Real, VXB_RNG_FAST>(ctx, p, fma);
    else
        launch_abc2<Real, VXB_RNG_EXTERNAL>(ctx, p, fma);
}
void launch_abc(vxb_ctx* ctx, const vxb_model& m, AbcParams p) {
    if (p.count == 0) return;
    p.log_table = ctx->log_table;
    const bool fma = m.arith == VXB_ARITH_FMA || m.rng == VXB_RNG_FAST;
    if (m.precision == VXB_F32)
        launch_abc1<float>(ctx, p, m.rng, fma);
    else
        launch_abc1<double>(ctx, p, m.rng, fma);
}

}  // namespace vxb

using namespace vxb;

extern "C" int vxb_abc_prior_predictive(vxb_ctx* ctx, const vxb_model* model,
                                        const vxb_keying* key, uint64_t n_total, uint64_t first,
                                        uint64_t count, const double* observed, void* params,
                                        void* summaries, void* rho, uint8_t* failed,
                                        const void* external_noise) {
    return guarded([&] {
        use(ctx);
        require(model && key && observed, "invalid-argument", "null argument");
        require(n_total >= 1, "invalid-shape", "need at least one prior predictive sample");
        require(first + count <= n_total, "invalid-shape", "row range exceeds the job");
        if (model->model == VXB_MODEL_TB) {  // exact Gillespie TB model: vxb_tb.cu
            require(key->mode == VXB_KEY_PARTICLE, "invalid-argument",
                    "the TB model consumes a data-dependent number of variates per row: "
                    "particle keying only");
            Staged t_params(ctx, params, count * 3 * 8, false, true);
            Staged t_summ(ctx, summaries, count * 2 * 8, false, true);
            Staged t_rho(ctx, rho, count * 8, false, true);
            Staged t_failed(ctx, failed, count, false, true);
            tb_launch(ctx, *model, key->seed, first, count, observed, t_params.as<double>(),
                      t_summ.as<double>(), t_rho.as<double>(), t_failed.as<uint8_t>());
            t_params.finish();
            t_summ.finish();
            t_rho.finish();
            t_failed.finish();
            if (t_params.staged() || t_summ.staged() || t_rho.staged() || t_failed.staged())
                VXB_CUDA(cudaStreamSynchronize(ctx->stream));
            return;
        }
        if (model->model == VXB_MODEL_TOGGLE) {  // the reference's own SDE: vxb_toggle.cu
            const Keying tk = make_keying(*key, *model, n_total);
            Staged t_params(ctx, params, count * 7 * 8, false, true);
            Staged t_summ(ctx, summaries, count * 19 * 8, false, true);
            Staged t_rho(ctx, rho, count * 8, false, true);
            Staged t_failed(ctx, failed, count, false, true);
            toggle_launch(ctx, *model, tk, first, count,
                          key->mode == VXB_KEY_WORKER ? key->block_width : 1, observed, nullptr,
                          t_params.as<double>(), t_summ.as<double>(), t_rho.as<double>(),
                          t_failed.as<uint8_t>());
            t_params.finish();
            t_summ.finish();
            t_rho.finish();
            t_failed.finish();
            if (t_params.staged() || t_summ.staged() || t_rho.staged() || t_failed.staged())
                VXB_CUDA(cudaStreamSynchronize(ctx->stream));
            return;
        }
        AbcParams p{};
        p.model = make_logistic(*model);
        p.key = make_keying(*key, *model, n_total);
        p.first = first;
        p.count = count;
        for (uint32_t k = 0; k < p.model.n_obs; ++k)
            p.observed[k] = model->precision == VXB_F32
                                ? static_cast<double>(static_cast<float>(observed[k]))
                                : observed[k];
        require(model->rng != VXB_RNG_EXTERNAL || external_noise, "invalid-argument",
                "external rng mode needs a noise buffer");
        const size_t real = model->precision == VXB_F32 ? 4 : 8;
        Staged d_params(ctx, params, count * 3 * real, false, true);
        Staged d_summ(ctx, summaries, count * p.model.n_obs * real, false, true);
        Staged d_rho(ctx, rho, count * real, false, true);
        Staged d_failed(ctx, failed, count, false, true);
        Staged d_noise(ctx, model->rng == VXB_RNG_EXTERNAL ? external_noise : nullptr,
                       count * p.model.steps * real, true, false);
        p.params = d_params.ptr();
        p.summaries = d_summ.ptr();
        p.rho = d_rho.ptr();
        p.failed = d_failed.as<uint8_t>();
        p.noise = d_noise.ptr();
        launch_abc(ctx, *model, p);
        d_params.finish();
        d_summ.finish();
        d_rho.finish();
        d_failed.finish();
        if (d_params.staged() || d_summ.staged() || d_rho.staged() || d_failed.staged())
            VXB_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

extern "C" int vxb_simulate_at(vxb_ctx* ctx, const vxb_model* model, const double* theta,
                               uint64_t seed, uint32_t stream_id, uint64_t pos, void* summary) {
    return guarded([&] {
        use(ctx);
        require(model && theta && summary, "invalid-argument", "null argument");
        require(model->rng == VXB_RNG_REF, "invalid-argument",
                "simulate_at is defined for the reference generator");
        if (model->model == VXB_MODEL_TB) {
            // consts[3] > 1: retry from where the stream stands while the population dies
            // out, the way bench.cpp:79-92 builds observed summaries
            const uint32_t attempts = model->consts[3] >= 1.0 ? static_cast<uint32_t>(model->consts[3]) : 1;
            if (!is_device_pointer(theta))
                require(theta[0] >= 0 && theta[1] >= 0 && theta[2] >= 0, "invalid-argument",
                        "rates must be nonnegative");  // tb_model.cpp:43-44
            Staged t_theta(ctx, theta, 3 * sizeof(double), true, false);
            Staged t_summ(ctx, summary, 2 * sizeof(double), false, true);
            Scratch t_failed(ctx, 1);
            tb_simulate_fixed(ctx, *model, t_theta.as<double>(), stream_key(splitmix64(seed), stream_id),
                              pos, attempts, t_summ.as<double>(), t_failed.as<uint8_t>(), nullptr);
            uint8_t bad = 0;
            VXB_CUDA(cudaMemcpyAsync(&bad, t_failed.as<uint8_t>(), 1, cudaMemcpyDeviceToHost, ctx->stream));
            t_summ.finish();
            VXB_CUDA(cudaStreamSynchronize(ctx->stream));
            require(!bad, attempts > 1 ? "empty-set" : "extinct-population",
                    attempts > 1 ? "synthetic tb population kept going extinct"
                                 : "summaries need a surviving population");
            return;
        }
        if (model->model == VXB_MODEL_TOGGLE) {
            require(model->steps >= 2, "invalid-horizon",
                    "toggle simulation needs at least two time points");
            require(model->consts[1] >= 19.0, "insufficient-data",
                    "need at least 19 observations for the quantile summary");
            Keying tk{};
            tk.mode = kKeyFixed;
            tk.fixed_key = stream_key(splitmix64(seed), stream_id);
            tk.fixed_pos = pos;
            Staged t_theta(ctx, theta, 7 * sizeof(double), true, false);
            Staged t_summ(ctx, summary, 19 * sizeof(double), false, true);
            toggle_launch(ctx, *model, tk, 0, 1, 1, nullptr, t_theta.as<double>(), nullptr,
                          t_summ.as<double>(), nullptr, nullptr);
            t_summ.finish();
            VXB_CUDA(cudaStreamSynchronize(ctx->stream));
            return;
        }
        AbcParams p{};
        p.model = make_logistic(*model);
        p.key.mode = kKeyFixed;
        p.key.fixed_key = stream_key(splitmix64(seed), stream_id);
        p.key.fixed_pos = pos;
        p.first = 0;
        p.count = 1;
        const size_t real = model->precision == VXB_F32 ? 4 : 8;
        Staged d_theta(ctx, theta, 3 * sizeof(double), true, false);
        Staged d_summ(ctx, summary, p.model.n_obs * real, false, true);
        Scratch d_failed(ctx, 1);
        p.theta_in = d_theta.as<double>();
        p.summaries = d_summ.ptr();
        p.failed = d_failed.as<uint8_t>();
        launch_abc(ctx, *model, p);
        uint8_t bad = 0;
        VXB_CUDA(cudaMemcpyAsync(&bad, p.failed, 1, cudaMemcpyDeviceToHost, ctx->stream));
        d_summ.finish();
        VXB_CUDA(cudaStreamSynchronize(ctx->stream));
        require(!bad, "invalid-state", "state left the reals");
    });
}

// Partial squared distance beyond which a row cannot be accepted any more.  The sum of
// squares only grows (every term is added as RN(d^2 + ss) >= ss) and rho = RN(sqrt(ss)) is
// accepted iff rho <= epsilon (compared in double): ss > eps^2 (1 + m) gives
// sqrt(ss) > eps (1 + m/2 - m^2/8), which survives the rounding of the square root with
// m = 2^-50 in fp64 (one ulp is <= 2^-52 relative) and m = 2^-21 in fp32 (<= 2^-23).
// Rounded UP to the working precision; a negative or non-finite epsilon switches it off.
static double early_reject_bound(double epsilon, bool f32) {
    if (!(epsilon >= 0.0) || !std::isfinite(epsilon)) return std::numeric_limits<double>::infinity();
    const double b = epsilon * epsilon * (1.0 + (f32 ? 0x1p-21 : 0x1p-50));
    if (!std::isfinite(b)) return std::numeric_limits<double>::infinity();
    if (f32) {
        float bf = static_cast<float>(b);
        if (static_cast<double>(bf) < b) bf = std::nextafter(bf, std::numeric_limits<float>::infinity());
        return static_cast<double>(bf);
    }
    return std::nextafter(b, std::numeric_limits<double>::infinity());
}

// Early rejection in up to six launches (see AbcParams): observations [0, b1) for every
// row, [b1, b2) for the rows alive at b1, ... -- the survivors are re-packed between the
// launches, so warps stay full although most rows die early (BASELINE config 1: 34 % alive
// after 4 of 20 observations, 15 % after 6, 5 % after 8, 0.6 % after 12, 0.1 % at the end;
// scripts/survivors_probe.py).  Nothing returns to the host: queue lengths stay on the
// device.  false: not applicable (plain launch).
static bool early_reject_segments(vxb_ctx* ctx, const vxb_model& model, AbcParams p) {
    if (!std::isfinite(p.ss_bound) || p.count < (1u << 16) || p.count >= (1ull << 32)) return false;
    const uint32_t n_obs = p.model.n_obs;
    // a segment may begin inside a noise batch (logistic_segment skips the normals of the
    // previous segment), so every observation is a possible boundary.
    // Boundaries: VXB_EARLY_BOUNDS="b1,b2,..." (experiments) or 15 / 20 / 30 / 40 / 60 % of
    // the observations (BASELINE config 1 at 1e8 rows, fp64 throughput instance: 104 ms with
    // 4,6,8,12 against 117 ms with 4,8 and 351 ms without early rejection; the exact
    // instance 315 ms with 3,4,6,8,12 against 340 ms; scripts/early_reject_sweep.sh)
    uint32_t bounds[8] = {0};
    int n_seg = 1;
    if (const char* env = getenv("VXB_EARLY_BOUNDS")) {
        for (const char* c = env; *c && n_seg < 6;) {
            const uint32_t v = static_cast<uint32_t>(strtoul(c, const_cast<char**>(&c), 10));
            if (v > bounds[n_seg - 1] && v < n_obs) bounds[n_seg++] = v;
            while (*c == ',') ++c;
        }
    } else {
        for (const uint32_t twentieth : {3u, 4u, 6u, 8u, 12u}) {
            const uint32_t v = (n_obs * twentieth + 19) / 20;
            if (v > bounds[n_seg - 1] && v < n_obs) bounds[n_seg++] = v;
        }
    }
    if (n_seg < 2) return false;
    bounds[n_seg] = n_obs;
    const size_t real = model.precision == VXB_F32 ? 4 : 8;
    // two queues of `count` entries each (x, ss, then the u32 row offsets), used alternately;
    // in front of them one length counter per segment (64 bytes)
    const size_t per_queue = (p.count * (4 + 2 * real) + 64 + 15) & ~size_t(15);
    char* base = static_cast<char*>(arena_get(ctx, 3, 64 + 2 * per_queue));
    VXB_CUDA(cudaMemsetAsync(base, 0, 64, ctx->stream));
    auto* counts = reinterpret_cast<unsigned long long*>(base);
    struct Queue {
        uint32_t* rows;
        void *x, *ss;
    } q[2];
    for (int k = 0; k < 2; ++k) {
        char* b = base + 64 + k * per_queue;
        q[k].x = b;
        q[k].ss = b + p.count * real;
        q[k].rows = reinterpret_cast<uint32_t*>(b + 2 * p.count * real);
    }
    for (int seg = 0; seg < n_seg; ++seg) {
        AbcParams s = p;
        s.obs_begin = bounds[seg];
        s.obs_end = seg == n_seg - 1 ? 0xFFFFFFFFu : bounds[seg + 1];
        if (seg > 0) {  // queues alternate; every segment has its own counter
            s.in_rows = q[(seg - 1) & 1].rows;
            s.in_x = q[(seg - 1) & 1].x;
            s.in_ss = q[(seg - 1) & 1].ss;
            s.in_count = counts + (seg - 1);
        }
        if (seg < n_seg - 1) {
            s.out_rows = q[seg & 1].rows;
            s.out_x = q[seg & 1].x;
            s.out_ss = q[seg & 1].ss;
            s.out_count = counts + seg;
        }
        launch_abc(ctx, model, s);
    }
    return true;
}

extern "C" int vxb_set_option(vxb_ctx* ctx, int option, int64_t value) {
    return guarded([&] {
        use(ctx);
        require(option == VXB_OPT_EARLY_REJECT, "invalid-argument", "unknown option");
        ctx->early_reject = value != 0;
    });
}

extern "C" int vxb_abc_reject(vxb_ctx* ctx, const vxb_model* model, const vxb_keying* key,
                              uint64_t n_total, uint64_t first, uint64_t count,
                              const double* observed, double epsilon, uint64_t cap,
                              uint64_t* n_accepted, uint64_t* idx, void* params, void* rho) {
    return guarded([&] {
        use(ctx);
        require(model && key && observed && n_accepted, "invalid-argument", "null argument");
        require(n_total >= 1, "invalid-shape", "need at least one prior predictive sample");
        require(first + count <= n_total, "invalid-shape", "row range exceeds the job");
        require(model->rng != VXB_RNG_EXTERNAL, "invalid-argument",
                "the fused path generates its own noise");
        AbcParams p{};
        p.model = make_logistic(*model);
        p.key = make_keying(*key, *model, n_total);
        p.first = first;
        p.count = count;
        const bool f32 = model->precision == VXB_F32;
        for (uint32_t k = 0; k < p.model.n_obs; ++k)
            p.observed[k] = f32 ? static_cast<double>(static_cast<float>(observed[k])) : observed[k];
        const size_t real = f32 ? 4 : 8;
        p.rho = arena_get(ctx, 0, count * real);
        p.failed = static_cast<uint8_t*>(arena_get(ctx, 1, count));
        if (ctx->early_reject) p.ss_bound = early_reject_bound(epsilon, f32);
        if (!early_reject_segments(ctx, *model, p)) launch_abc(ctx, *model, p);

        Staged d_idx(ctx, idx, cap * sizeof(uint64_t), false, true);
        Scratch d_idx_tmp(ctx, d_idx.ptr() ? 0 : cap * sizeof(uint64_t));
        uint64_t* idx_dev = d_idx.ptr() ? d_idx.as<uint64_t>() : d_idx_tmp.as<uint64_t>();
        // n_accepted in device memory => fully asynchronous call: the count stays on
        // the device, nothing is copied to the host and the stream is not synchronised
        const bool async = is_device_pointer(n_accepted);
        require(!async || ((!idx || is_device_pointer(idx)) && (!params || is_device_pointer(params)) &&
                           (!rho || is_device_pointer(rho))),
                "invalid-argument", "a device-resident count needs device-resident outputs");
        uint64_t n_acc = 0;
        compact_accepted_device(ctx, model->precision, p.rho, p.failed, count, epsilon, first, cap,
                                async ? n_accepted : &n_acc, idx_dev);
        const unsigned long long* n_acc_dev =
            async ? reinterpret_cast<const unsigned long long*>(n_accepted) : nullptr;
        if (!async) *n_accepted = n_acc;
        const uint64_t kept = async ? cap : (n_acc < cap ? n_acc : cap);
        Staged d_params(ctx, params, cap * 3 * real, false, true);
        Staged d_rho(ctx, rho, cap * real, false, true);
        if (kept && (params || rho)) {
            LaunchScope scope(ctx, VXB_K_COMPACT);
            const unsigned grid = grid_for(kept, 128);
            if (f32) {
                if (model->rng == VXB_RNG_FAST)
                    gather_accepted_kernel<float, VXB_RNG_FAST><<<grid, 128, 0, ctx->stream>>>(
                        p.key, p.model, first, idx_dev, kept, static_cast<const float*>(p.rho),
                        d_params.as<float>(), d_rho.as<float>(), n_acc_dev);
                else
                    gather_accepted_kernel<float, VXB_RNG_REF><<<grid, 128, 0, ctx->stream>>>(
                        p.key, p.model, first, idx_dev, kept, static_cast<const float*>(p.rho),
                        d_params.as<float>(), d_rho.as<float>(), n_acc_dev);
            } else {
                if (model->rng == VXB_RNG_FAST)
                    gather_accepted_kernel<double, VXB_RNG_FAST><<<grid, 128, 0, ctx->stream>>>(
                        p.key, p.model, first, idx_dev, kept, static_cast<const double*>(p.rho),
                        d_params.as<double>(), d_rho.as<double>(), n_acc_dev);
                else
                    gather_accepted_kernel<double, VXB_RNG_REF><<<grid, 128, 0, ctx->stream>>>(
                        p.key, p.model, first, idx_dev, kept, static_cast<const double*>(p.rho),
                        d_params.as<double>(), d_rho.as<double>(), n_acc_dev);
            }
            check_launch("gather_accepted_kernel");
        }
        if (async) return;
        d_idx.finish(kept * sizeof(uint64_t));
        d_params.finish(kept * 3 * real);
        d_rho.finish(kept * real);
        VXB_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

// Device-side statistics of the throughput generator over rows x per_row normals,
// nothing but counters leaves the GPU (1e10+ samples in milliseconds): tail counts
// |z| > t_k, power sums, the largest |z|, and for fp32 the error of the MUFU
// evaluation against a double-precision evaluation of the SAME uniforms.
struct FastStats {
    unsigned long long tail[8];
    unsigned long long n;
    double sum[4];      // z, z^2, z^3, z^4
    double max_abs;
    double err_max;     // fp32: max |z32 - z64|
    double err_max_tail;  // ... over |z64| > 4
    double err_sq;      // sum (z32 - z64)^2
};
template <class Real>
__global__ void __launch_bounds__(256) fast_stats_kernel(FastKeys fk, const double2* table,
                                                         uint64_t first, uint64_t rows,
                                                         uint32_t per_row, const double* thr,
                                                         uint32_t n_thr, FastStats* out) {
    __shared__ double2 s_tab[sizeof(Real) == 8 ? kFastTableSize : 1];
    if (sizeof(Real) == 8) {
        for (int i = threadIdx.x; i < kFastTableSize; i += 256) s_tab[i] = table[i];
        __syncthreads();
    }
    constexpr uint32_t kB = sizeof(Real) == 8 ? 8 : 16;
    const uint32_t q = blockIdx.y * 256 + threadIdx.x;
    const bool live = q * kB < per_row;
    double t[8];
    for (uint32_t k = 0; k < 8; ++k) t[k] = k < n_thr ? thr[k] : 1e300;
    unsigned long long tail[8] = {0, 0, 0, 0, 0, 0, 0, 0}, n = 0;
    double s1 = 0, s2 = 0, s3 = 0, s4 = 0, mx = 0, emax = 0, etail = 0, esq = 0;
    if (live)
        for (uint64_t r = blockIdx.x; r < rows; r += gridDim.x) {
            const uint64_t row = first + r;
            const uint32_t rl = static_cast<uint32_t>(row), rh = static_cast<uint32_t>(row >> 32);
            const Words32 u = philox4x32(fk, 3 * q, kDomNoise, rl, rh);
            const Words32 v = philox4x32(fk, 3 * q + 1, kDomNoise, rl, rh);
            const Words32 w = philox4x32(fk, 3 * q + 2, kDomNoise, rl, rh);
            Real z[kB];
            double ze[kB];
            if constexpr (sizeof(Real) == 8) {
                fast_box_muller_x4(u, v, w, s_tab, z);
            } else {
                box_muller_f32_x8(u, v, w, z);
                uint32_t m1[8], m2[8];
                f32_batch_fields(u, v, w, m1, m2);
                for (int k = 0; k < 8; ++k) {  // the same uniforms, evaluated in fp64
                    const float u1 = f32_u1(m1[k]);
                    const double rad = sqrt(-2.0 * log(static_cast<double>(u1)));
                    const double ang = static_cast<double>(__uint_as_float(0x3F800000u | m2[k])) *
                                           6.283185307179586476925 - 9.424777960769379715;
                    ze[2 * k] = rad * cos(ang);
                    ze[2 * k + 1] = rad * sin(ang);
                }
            }
            const uint32_t valid = min(kB, per_row - q * kB);
            for (uint32_t e = 0; e < valid; ++e) {
                const double x = static_cast<double>(z[e]), a = fabs(x);
                ++n;
                s1 += x;
                s2 += x * x;
                s3 += x * x * x;
                s4 += x * x * x * x;
                mx = fmax(mx, a);
                for (uint32_t k = 0; k < 8; ++k) tail[k] += a > t[k];
                if constexpr (sizeof(Real) == 4) {
                    const double d = fabs(x - ze[e]);
                    emax = fmax(emax, d);
                    if (fabs(ze[e]) > 4.0) etail = fmax(etail, d);
                    esq += d * d;
                }
            }
        }
    // warp reduction, then one atomic per warp and field
    for (int o = 16; o; o >>= 1) {
        for (int k = 0; k < 8; ++k) tail[k] += __shfl_down_sync(0xffffffffu, tail[k], o);
        n += __shfl_down_sync(0xffffffffu, n, o);
        s1 += __shfl_down_sync(0xffffffffu, s1, o);
        s2 += __shfl_down_sync(0xffffffffu, s2, o);
        s3 += __shfl_down_sync(0xffffffffu, s3, o);
        s4 += __shfl_down_sync(0xffffffffu, s4, o);
        esq += __shfl_down_sync(0xffffffffu, esq, o);
        mx = fmax(mx, __shfl_down_sync(0xffffffffu, mx, o));
        emax = fmax(emax, __shfl_down_sync(0xffffffffu, emax, o));
        etail = fmax(etail, __shfl_down_sync(0xffffffffu, etail, o));
    }
    if ((threadIdx.x & 31) == 0) {
        for (int k = 0; k < 8; ++k)
            if (tail[k]) atomicAdd(&out->tail[k], tail[k]);
        atomicAdd(&out->n, n);
        atomicAdd(&out->sum[0], s1);
        atomicAdd(&out->sum[1], s2);
        atomicAdd(&out->sum[2], s3);
        atomicAdd(&out->sum[3], s4);
        atomicAdd(&out->err_sq, esq);
        // non-negative doubles order like their bit patterns
        atomicMax(reinterpret_cast<unsigned long long*>(&out->max_abs), __double_as_longlong(mx));
        atomicMax(reinterpret_cast<unsigned long long*>(&out->err_max), __double_as_longlong(emax));
        atomicMax(reinterpret_cast<unsigned long long*>(&out->err_max_tail), __double_as_longlong(etail));
    }
}

extern "C" int vxb_rng_fast_stats(vxb_ctx* ctx, int precision, uint64_t seed, uint64_t first_row,
                                  uint64_t rows, uint32_t per_row, const double* thresholds,
                                  uint32_t n_thresholds, uint64_t* tail_counts, double* moments) {
    return guarded([&] {
        use(ctx);
        require(precision == VXB_F64 || precision == VXB_F32, "invalid-argument", "unknown precision");
        require(n_thresholds <= 8 && (n_thresholds == 0 || (thresholds && tail_counts)) && moments,
                "invalid-argument", "at most 8 thresholds; null argument");
        require(rows >= 1 && per_row >= 1, "invalid-shape", "empty sample");
        Scratch d_thr(ctx, 8 * sizeof(double)), d_out(ctx, sizeof(FastStats));
        double h_thr[8] = {0};
        for (uint32_t k = 0; k < n_thresholds; ++k) h_thr[k] = thresholds[k];
        VXB_CUDA(cudaMemcpyAsync(d_thr.as<void>(), h_thr, sizeof(h_thr), cudaMemcpyHostToDevice, ctx->stream));
        VXB_CUDA(cudaMemsetAsync(d_out.as<void>(), 0, sizeof(FastStats), ctx->stream));
        const FastKeys fk = make_fast_keys(splitmix64(seed));
        {
            LaunchScope scope(ctx, VXB_K_RNGFILL);
            const uint32_t per_batch = precision == VXB_F32 ? 16 : 8;
            const uint32_t chunks = ((per_row + per_batch - 1) / per_batch + 255) / 256;
            require(chunks <= 65535, "invalid-shape", "too many values per row");
            const dim3 grid(static_cast<unsigned>(std::min<uint64_t>(rows, 148u * 64u)), chunks);
            if (precision == VXB_F32)
                fast_stats_kernel<float><<<grid, 256, 0, ctx->stream>>>(
                    fk, ctx->log_table, first_row, rows, per_row, d_thr.as<double>(), n_thresholds,
                    d_out.as<FastStats>());
            else
                fast_stats_kernel<double><<<grid, 256, 0, ctx->stream>>>(
                    fk, ctx->log_table, first_row, rows, per_row, d_thr.as<double>(), n_thresholds,
                    d_out.as<FastStats>());
            check_launch("fast_stats_kernel");
        }
        FastStats h;
        VXB_CUDA(cudaMemcpyAsync(&h, d_out.as<void>(), sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
        VXB_CUDA(cudaStreamSynchronize(ctx->stream));
        for (uint32_t k = 0; k < n_thresholds; ++k) tail_counts[k] = h.tail[k];
        moments[0] = static_cast<double>(h.n);
        for (int k = 0; k < 4; ++k) moments[1 + k] = h.sum[k];
        moments[5] = h.max_abs;
        moments[6] = h.err_max;
        moments[7] = h.err_max_tail;
        moments[8] = h.err_sq;
    });
}

extern "C" int vxb_rng_fill_gaussian_fast(vxb_ctx* ctx, int precision, uint64_t seed,
                                          uint64_t first_row, uint64_t rows, uint32_t per_row,
                                          void* out) {
    return guarded([&] {
        use(ctx);
        require(precision == VXB_F64 || precision == VXB_F32, "invalid-argument",
                "unknown precision");
        if (rows == 0 || per_row == 0) return;
        require(out != nullptr, "invalid-argument", "null output");
        const size_t elem = precision == VXB_F32 ? 4 : 8;
        Staged d_out(ctx, out, rows * per_row * elem, false, true);
        const FastKeys fk = make_fast_keys(splitmix64(seed));
        {
            LaunchScope scope(ctx, VXB_K_RNGFILL);
            const uint32_t per_batch = precision == VXB_F32 ? 16 : 8;
            const uint32_t chunks = ((per_row + per_batch - 1) / per_batch + 255) / 256;
            require(chunks <= 65535, "invalid-shape", "too many values per row");
            const dim3 grid(static_cast<unsigned>(std::min<uint64_t>(rows, 1u << 30)), chunks);
            if (precision == VXB_F32)
                fast_normals_kernel<float><<<grid, 256, 0, ctx->stream>>>(fk, ctx->log_table, first_row, rows,
                                                                         per_row, d_out.as<float>());
            else
                fast_normals_kernel<double><<<grid, 256, 0, ctx->stream>>>(fk, ctx->log_table, first_row, rows,
                                                                          per_row, d_out.as<double>());
            check_launch("fast_normals_kernel");
        }
        d_out.finish();
        if (d_out.staged()) VXB_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}
