// vxb_toggle.cu -- the reference's toggle-switch SDE on the GPU:
// toggle::simulate_block / simulate / summary_quantiles (toggle_switch.cpp:31-133)
// fused with the prior draw and the discrepancy of run_prior_predictive
// (abc.cpp:45-61).
//
// One CTA per prior-predictive sample: the C cells of a sample are spread over
// the threads (each cell is an independent 2-state Euler-Maruyama path of T-1
// steps with two pow_pos per step), their noisy observations land in shared
// memory, a bitonic sort orders them in place, and 19 threads read the type-7
// quantiles (numeric.cpp:20-30).  Variates are addressed by the reference's
// canonical layout (toggle_switch.hpp:52-57): cell c owns stream positions
// [b0 + c*2T, b0 + (c+1)*2T); ONE Philox block yields the (u, v) increments of a
// step (positions 2(j-1) and 2(j-1)+1 are the cos and sin halves of the same
// Box-Muller pair).  Nothing but theta, the 19 summaries and rho leaves the SM.

#include <cmath>

#include "vxb_internal.cuh"

namespace vxb {

constexpr int kTgBlock = 256;

struct ToggleParams {
    uint64_t first, count;
    Keying key;
    uint32_t steps, cells, sort_n;  // sort_n: power of two >= cells
    uint32_t invalid;               // steps < 2 or cells < 19: every row is flagged
    uint64_t padded_cells;          // worker keying: cells rounded up to V
    double lo[7], hi[7];
    double observed[19];
    const double* theta_in;  // kKeyFixed
    const double2* fast_table;
    double* params;
    double* summaries;
    double* rho;
    uint8_t* failed;
};

template <class A>
__device__ __forceinline__ double toggle_cell(const double* th, uint32_t steps, uint64_t key,
                                              uint64_t pair0) {
    const double mu = th[0], sigma = th[1], gamma = th[2];
    const double alpha_u = th[3], alpha_v = th[4], beta_u = th[5], beta_v = th[6];
    double u = 10.0, v = 10.0;
    uint64_t pair = pair0;
#ifdef VXB_TOGGLE_NO_FLOOR_SHORTCUT
    const bool shortcut = false;
#else
    const bool shortcut = beta_u >= 0.0 && beta_v >= 0.0;  // beta * (+0) = +0 (uniform over the sample)
#endif
    for (uint32_t j = 1; j < steps; ++j, ++pair) {
        double zu, zv;
        box_muller<A>(philox2x64(key, pair), zu, zv);
        // previous-step powers (toggle_switch.cpp:50-51); the state never drops below 1.
        // A species that sits ON the floor has the power 1 exactly (log2_pos(1) = +0,
        // exp2_clamped(beta * 0) = 1 for beta >= 0), and in a settled switch one of the two
        // species of a cell is on the floor 95 % of the time -- which one differs from cell
        // to cell.  So every lane evaluates ONE power, of whichever species is off the floor,
        // and the second evaluation runs only when some cell of the warp has both off it
        // (about half of the warp-steps).  Same bits as two evaluations per step.
        double p_u, p_v;
        if (shortcut) {
            const bool vf = v == 1.0, uf = u == 1.0;
            const double p1 = exp2_clamped<A>(A::mul(vf ? beta_v : beta_u, log2_pos<A, false>(vf ? u : v)));
            p_u = vf ? 1.0 : p1;
            p_v = vf ? p1 : 1.0;  // v off the floor: 1 if u is on it, else the second evaluation
            if (__any_sync(__activemask(), !vf && !uf)) {
                const double p2 = exp2_clamped<A>(A::mul(beta_v, log2_pos<A, false>(u)));
                if (!vf) p_v = p2;
            }
        } else {
            p_u = exp2_clamped<A>(A::mul(beta_u, log2_pos<A, false>(v)));
            p_v = exp2_clamped<A>(A::mul(beta_v, log2_pos<A, false>(u)));
        }
        double ut = A::mul(u, 0.97);
        ut = A::add(ut, A::sub(A::div(alpha_u, A::add(1.0, p_u)), 1.0));
        double vt = A::mul(v, 0.97);
        vt = A::add(vt, A::sub(A::div(alpha_v, A::add(1.0, p_v)), 1.0));
        ut = A::add(ut, A::mul(0.5, zu));
        vt = A::add(vt, A::mul(0.5, zv));
        u = ut >= 1.0 ? ut : 1.0;
        v = vt >= 1.0 ? vt : 1.0;
    }
    double eta, unused;
    box_muller<A>(philox2x64(key, pair), eta, unused);  // position 2(T-1): cos half
    const double pw = exp2_clamped<A>(A::mul(gamma, log2_pos<A, false>(u)));
    const double obs = A::add(A::add(u, mu), A::div(A::mul(A::mul(sigma, mu), eta), pw));
    return obs >= 1.0 ? obs : 1.0;
}

// Throughput mode of one cell (VXB_RNG_FAST): the same model with the packed
// Philox4x32 generator (eight normals = four steps per batch, drawn one batch
// ahead), table-based log2 / 2^z, a Newton reciprocal and FMA arithmetic.
// Statistically validated against the exact mode (tests/test_gpu_workloads.py).
__device__ __forceinline__ double toggle_cell_fast(const double* th, uint32_t steps, const FastKeys& fk,
                                                   const double2* tbl, uint32_t row_word,
                                                   uint32_t cell_word) {
    const double mu = th[0], sigma = th[1], gamma = th[2];
    const double alpha_u = th[3], alpha_v = th[4], beta_u = th[5], beta_v = th[6];
    double u = 10.0, v = 10.0;
    FastNoise64 noise(fk, tbl, row_word, cell_word, 0u);
    const auto step = [&](double zu, double zv) {
        // (the short forms: relative error of a power ~1e-13, the model's noise is 0.5 per step)
        // (the floor shortcut of the exact instance does not pay here: 309 against 286 ms at the
        // paper's size -- the short power forms are cheaper than the selects and the vote)
        const double p_u = fast_exp2_short(beta_u * fast_log2_short(v, tbl), tbl);
        const double p_v = fast_exp2_short(beta_v * fast_log2_short(u, tbl), tbl);
        const double ut = fma(0.5, zu, fma(u, 0.97, fma(alpha_u, fast_rcp(1.0 + p_u), -1.0)));
        const double vt = fma(0.5, zv, fma(v, 0.97, fma(alpha_v, fast_rcp(1.0 + p_v), -1.0)));
        u = fmax(ut, 1.0);
        v = fmax(vt, 1.0);
    };
    uint32_t left = steps - 1;
    double z[8];
    while (left >= 4) {
        noise.next(z);
        step(z[0], z[1]);
        step(z[2], z[3]);
        step(z[4], z[5]);
        step(z[6], z[7]);
        left -= 4;
    }
    noise.next(z);  // the ragged tail (< 4 steps) and the observation noise
#pragma unroll
    for (uint32_t q = 0; q < 3; ++q)
        if (q < left) step(z[2 * q], z[2 * q + 1]);
    const double eta = z[6];
    const double pw = fast_exp2(gamma * fast_log2(u, tbl), tbl);
    return fmax(u + mu + sigma * mu * eta * fast_rcp(pw), 1.0);
}

// CTAs per SM the register budget is sized for (64 KB of sort buffer per CTA at the
// paper's 8000 cells allow three): measured at the paper size, exact 1.74 / 1.16 / 1.06 s
// and throughput 0.33 / 0.30 / 0.31 s for 1 / 2 / 3.
template <bool kFast>
__global__ void __launch_bounds__(kTgBlock, kFast ? 2 : 3) toggle_abc_kernel(const __grid_constant__ ToggleParams p) {
    extern __shared__ double s_y[];
    __shared__ double s_q[19];
    __shared__ double2 s_tab[kFast ? kFastTableSize : 1];
    if (kFast) {
        for (int i = threadIdx.x; i < kFastTableSize; i += kTgBlock) s_tab[i] = p.fast_table[i];
        __syncthreads();
    }
    for (uint64_t r = blockIdx.x; r < p.count; r += gridDim.x) {
        const uint64_t row = p.first + r;
        uint64_t key, base;
        locate_row(p.key, row, key, base);
        double th[7];
        uint64_t b0;
        if (p.theta_in) {
#pragma unroll
            for (int k = 0; k < 7; ++k) th[k] = p.theta_in[k];
            b0 = base + (base & 1);
        } else if (kFast) {
            // throughput generator: seven uniforms from four Philox4x32 blocks of the row
            const uint32_t rl = static_cast<uint32_t>(row), rh = static_cast<uint32_t>(row >> 32);
            double un[8];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const Words32 w = philox4x32(p.key.fast, static_cast<uint32_t>(q), kDomPrior, rl, rh);
                un[2 * q] = fast_unit(w.a, w.b);
                un[2 * q + 1] = fast_unit(w.c, w.d);
            }
#pragma unroll
            for (int k = 0; k < 7; ++k) th[k] = p.lo[k] + un[k] * (p.hi[k] - p.lo[k]);
            b0 = 0;
        } else {
            // sample_prior (toggle_switch.cpp:25-29): 7 uniforms at base..base+6
#pragma unroll
            for (int b = 0; b < 4; ++b) {
                const Words w = philox2x64(key, (base >> 1) + b);
                th[2 * b] = __dadd_rn(p.lo[2 * b], __dmul_rn(to_unit(w.w0), __dsub_rn(p.hi[2 * b], p.lo[2 * b])));
                if (b < 3)
                    th[2 * b + 1] = __dadd_rn(p.lo[2 * b + 1],
                                              __dmul_rn(to_unit(w.w1), __dsub_rn(p.hi[2 * b + 1], p.lo[2 * b + 1])));
            }
            b0 = base + 8;
        }
        if (!p.invalid) {
            for (uint32_t c = threadIdx.x; c < p.sort_n; c += kTgBlock) {
                double y = INFINITY;  // padding sorts to the end
                if (c < p.cells) {
                    if (kFast)
                        y = toggle_cell_fast(th, p.steps, p.key.fast, s_tab, static_cast<uint32_t>(row),
                                             c | (static_cast<uint32_t>(row >> 32) << 14));
                    else
                        y = toggle_cell<Exact>(th, p.steps, key,
                                               (b0 >> 1) + static_cast<uint64_t>(c) * p.steps);
                }
                s_y[c] = y;
            }
            __syncthreads();
            // bitonic sort, ascending
            for (uint32_t k = 2; k <= p.sort_n; k <<= 1) {
                for (uint32_t j = k >> 1; j > 0; j >>= 1) {
                    for (uint32_t i = threadIdx.x; i < p.sort_n; i += kTgBlock) {
                        const uint32_t l = i ^ j;
                        if (l > i) {
                            const double a = s_y[i], b = s_y[l];
                            const bool up = (i & k) == 0;
                            if ((a > b) == up) {
                                s_y[i] = b;
                                s_y[l] = a;
                            }
                        }
                    }
                    __syncthreads();
                }
            }
            if (threadIdx.x < 19) {  // summary_quantiles (toggle_switch.cpp:123-133)
                const double level = __dmul_rn(0.05, static_cast<double>(threadIdx.x + 1));
                const uint32_t n = p.cells;
                const double h = __dmul_rn(static_cast<double>(n - 1), level);
                const uint32_t lo = static_cast<uint32_t>(h);
                double q;
                if (lo + 1 >= n) {
                    q = s_y[n - 1];
                } else {
                    const double frac = __dsub_rn(h, static_cast<double>(lo));
                    q = __dadd_rn(s_y[lo], __dmul_rn(frac, __dsub_rn(s_y[lo + 1], s_y[lo])));
                }
                s_q[threadIdx.x] = q;
            }
            __syncthreads();
        }
        if (threadIdx.x == 0) {
            double rho = __longlong_as_double(0x7FF8000000000000LL);
            if (!p.invalid) {
                double ss = 0.0;  // discrepancy (abc.cpp:16-24)
                for (int k = 0; k < 19; ++k) {
                    const double d = __dsub_rn(s_q[k], p.observed[k]);
                    ss = __dadd_rn(ss, __dmul_rn(d, d));
                }
                rho = __dsqrt_rn(ss);
            }
            if (p.rho) p.rho[r] = rho;
            if (p.failed) p.failed[r] = p.invalid ? 1 : 0;
            if (p.params)
                for (int k = 0; k < 7; ++k) p.params[r * 7 + k] = th[k];
        }
        if (p.summaries && threadIdx.x < 19)
            p.summaries[r * 19 + threadIdx.x] = p.invalid ? 0.0 : s_q[threadIdx.x];
        __syncthreads();
    }
}

static uint32_t next_pow2(uint32_t v) {
    uint32_t p = 1;
    while (p < v) p <<= 1;
    return p;
}

// Shared by vxb_abc_prior_predictive and vxb_simulate_at (dispatch in vxb_logistic.cu).
void toggle_launch(vxb_ctx* ctx, const vxb_model& m, const Keying& key, uint64_t first,
                   uint64_t count, uint64_t block_width, const double* observed_host,
                   const double* theta_dev, double* params, double* summaries, double* rho,
                   uint8_t* failed) {
    require(m.model == VXB_MODEL_TOGGLE, "invalid-argument", "not the toggle-switch model");
    require(m.dim == 7 && m.summary_dim == 19, "invalid-shape",
            "toggle model has 7 parameters and 19 summaries");
    require(m.precision == VXB_F64 && (m.rng == VXB_RNG_REF || m.rng == VXB_RNG_FAST),
            "invalid-argument", "the toggle model runs in fp64 (reference or throughput generator)");
    const bool fast = m.rng == VXB_RNG_FAST;
    require(!fast || (!theta_dev && key.mode == kKeyParticle), "invalid-argument",
            "the throughput generator keys rows per particle");
    const uint32_t cells = static_cast<uint32_t>(m.consts[1]);
    require(cells >= 1, "invalid-shape", "toggle simulation needs at least one cell");
    ToggleParams p{};
    p.first = first;
    p.count = count;
    p.key = key;
    p.steps = m.steps;
    p.cells = cells;
    p.sort_n = next_pow2(cells);
    p.invalid = (m.steps < 2 || cells < 19) ? 1u : 0u;
    p.padded_cells = (cells + block_width - 1) / block_width * block_width;
    if (p.key.mode == kKeyWorker) p.key.row_stride = 8 + p.padded_cells * 2 * m.steps;
    for (int k = 0; k < 7; ++k) {
        require(m.prior_lo[k] <= m.prior_hi[k], "invalid-range",
                "uniform lower bound exceeds upper bound");
        p.lo[k] = m.prior_lo[k];
        p.hi[k] = m.prior_hi[k];
    }
    for (int k = 0; k < 19; ++k) p.observed[k] = observed_host ? observed_host[k] : 0.0;
    p.theta_in = theta_dev;
    p.fast_table = ctx->log_table;
    p.params = params;
    p.summaries = summaries;
    p.rho = rho;
    p.failed = failed;
    if (count == 0) return;
    const size_t smem = static_cast<size_t>(p.sort_n) * sizeof(double);
    require(smem <= 200 * 1024, "invalid-shape", "too many cells for the in-CTA sort (max 16384)");
    const unsigned grid = static_cast<unsigned>(std::min<uint64_t>(count, 1u << 20));
    LaunchScope scope(ctx, VXB_K_SIMULATE);
    if (fast) {
        VXB_CUDA(cudaFuncSetAttribute(toggle_abc_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(smem)));
        toggle_abc_kernel<true><<<grid, kTgBlock, smem, ctx->stream>>>(p);
    } else {
        VXB_CUDA(cudaFuncSetAttribute(toggle_abc_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(smem)));
        toggle_abc_kernel<false><<<grid, kTgBlock, smem, ctx->stream>>>(p);
    }
    check_launch("toggle_abc_kernel");
}

}  // namespace vxb
