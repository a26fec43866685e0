// vxb_smc.cu -- SMC building blocks and the ABC-SMC driver (kernel 5, config 3).
//
// Reference pieces replaced here (all single-threaded on the coordinator in the
// reference):
//   smc::ess                    smc.cpp:208-219
//   logsumexp                   numeric.cpp:11-18
//   smc::resample_multinomial   smc.cpp:268-300  (inverse-CDF, draw i = stream position i)
//   make_kernel / cholesky      smc.cpp:311-325, numeric.cpp:81-96
//   proposal theta + L z        smc.cpp:115-119
// The ABC-SMC generation loop itself is not in the reference; it is
// defined by oracle/vxb_oracle.cpp (vxo_abcsmc_run) and reproduced here
// bit-for-bit: every reduction uses the canonical two-level order (chunks of
// 256 summed left to right, then the chunk totals left to right), which one
// thread per chunk reproduces exactly on the device, independent of launch
// shape and GPU count.

#include <algorithm>
#include <cmath>
#include <limits>
#include <vector>

#include "vxb_internal.cuh"
#include "vxb_libmexp.cuh"

#ifndef VXB_PROP_MINB
#define VXB_PROP_MINB 1
#endif

namespace vxb {

constexpr int kChunk = 256;  // canonical reduction chunk (oracle: kChunk)

// ------------------------------------------------------------- reductions
// Deterministic max / (sum e, sum e^2) with a fixed grid: per-thread strided
// partials, block tree in shared memory, per-block results finished by one
// thread in block order.
constexpr int kRedBlock = 256;
constexpr int kRedGrid = 296;

__global__ void __launch_bounds__(kRedBlock) max_partial_kernel(const double* __restrict__ x, uint64_t n,
                                                             double* __restrict__ part) {
    __shared__ double sh[kRedBlock];
    double m = -INFINITY;
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * kRedBlock + threadIdx.x; i < n;
         i += static_cast<uint64_t>(kRedGrid) * kRedBlock)
        m = fmax(m, x[i]);  // NaN-ignoring like std::max(m, v) with m first
    sh[threadIdx.x] = m;
    __syncthreads();
    for (int s = kRedBlock / 2; s > 0; s >>= 1) {
        if (threadIdx.x < s) sh[threadIdx.x] = fmax(sh[threadIdx.x], sh[threadIdx.x + s]);
        __syncthreads();
    }
    if (threadIdx.x == 0) part[blockIdx.x] = sh[0];
}
__global__ void max_final_kernel(const double* part, double* out) {
    double m = -INFINITY;
    for (int b = 0; b < kRedGrid; ++b) m = fmax(m, part[b]);
    *out = m;
}
// Strictly sequential sums in the reference's order (smc.cpp:208-219, 276-283,
// numeric.cpp:11-18): s1 = sum_i exp(x_i - max), s2 = sum_i exp(x_i - max)^2, added
// left to right, every exp the host libm's (vxb_libmexp.cuh) -- so ess, logsumexp and
// the cumulative weights of resample_multinomial are bit-identical to the CPU.  A
// floating-point running sum cannot be re-associated without changing its roundings,
// so the chain itself is one thread; what is parallel is everything around it: warps
// 1..3 evaluate the exponentials of the NEXT tile into shared memory (and, for the
// cumulative form, all threads store the finished tile) while thread 0 walks the
// current one.  The chain costs one dependent DADD per element.
constexpr int kSeqTile = 2048;
constexpr int kSeqThreads = 128;
template <bool kCum>
__global__ void __launch_bounds__(kSeqThreads)
seq_expsum_kernel(const double* __restrict__ x, const double* __restrict__ mx, uint64_t n,
                  double* __restrict__ cum, double* __restrict__ sums /* 2 */, int exp_variant) {
    __shared__ double buf[2][kSeqTile];
    const double m = *mx;
    const uint32_t tid = threadIdx.x;
    const uint64_t tiles = (n + kSeqTile - 1) / kSeqTile;
    for (uint64_t k = tid; k < min(static_cast<uint64_t>(kSeqTile), n); k += kSeqThreads)
        buf[0][k] = libm_exp(__dsub_rn(x[k], m), exp_variant);
    __syncthreads();
    double s1 = 0.0, s2 = 0.0;
    for (uint64_t t = 0; t < tiles; ++t) {
        const uint64_t t0 = t * kSeqTile;
        const uint32_t len = static_cast<uint32_t>(min(static_cast<uint64_t>(kSeqTile), n - t0));
        double* cur = buf[t & 1];
        if (tid == 0) {
            // the chain: one dependent DADD per element.  Blocks of 32 with the NEXT
            // block's loads issued before this block's adds, so that the shared-memory
            // latency (~30 cycles) hides behind the 32 adds instead of preceding every 8
            constexpr uint32_t kW = 32;
            double v[kW], nx[kW];
            uint32_t k0 = 0;
            if (len >= kW) {
#pragma unroll
                for (uint32_t q = 0; q < kW; ++q) v[q] = cur[q];
                for (; k0 + 2 * kW <= len; k0 += kW) {
#pragma unroll
                    for (uint32_t q = 0; q < kW; ++q) nx[q] = cur[k0 + kW + q];
#pragma unroll
                    for (uint32_t q = 0; q < kW; ++q) {
                        s1 = __dadd_rn(s1, v[q]);
                        if (kCum) cur[k0 + q] = s1; else s2 = __dadd_rn(s2, __dmul_rn(v[q], v[q]));
                    }
#pragma unroll
                    for (uint32_t q = 0; q < kW; ++q) v[q] = nx[q];
                }
#pragma unroll
                for (uint32_t q = 0; q < kW; ++q) {  // the last full block
                    s1 = __dadd_rn(s1, v[q]);
                    if (kCum) cur[k0 + q] = s1; else s2 = __dadd_rn(s2, __dmul_rn(v[q], v[q]));
                }
                k0 += kW;
            }
            for (uint32_t k = k0; k < len; ++k) {  // ragged tail of the last tile
                const double e = cur[k];
                s1 = __dadd_rn(s1, e);
                if (kCum) cur[k] = s1; else s2 = __dadd_rn(s2, __dmul_rn(e, e));
            }
        } else if (tid >= 32 && t + 1 < tiles) {
            const uint64_t n0 = t0 + kSeqTile;
            const uint32_t nlen = static_cast<uint32_t>(min(static_cast<uint64_t>(kSeqTile), n - n0));
            double* nxt = buf[(t + 1) & 1];
            for (uint32_t k = tid - 32; k < nlen; k += kSeqThreads - 32)
                nxt[k] = libm_exp(__dsub_rn(x[n0 + k], m), exp_variant);
        }
        __syncthreads();
        if (kCum) {
            for (uint32_t k = tid; k < len; k += kSeqThreads) cum[t0 + k] = cur[k];
            __syncthreads();  // the tile after next is written into this buffer
        }
    }
    if (tid == 0) {
        sums[0] = s1;
        sums[1] = s2;
    }
}

// max, then the sequential sums above.  cum_dev != nullptr: also the inclusive
// cumulative sums (resample_multinomial's `cum`); s2 is then not computed.
void max_and_expsums(vxb_ctx* ctx, const double* x_dev, uint64_t n, double* mx, double* s1,
                     double* s2, double* cum_dev = nullptr) {
    Scratch part(ctx, sizeof(double) * kRedGrid);
    Scratch res(ctx, sizeof(double) * 3);
    {
        LaunchScope scope(ctx, VXB_K_RESAMPLE);
        max_partial_kernel<<<kRedGrid, kRedBlock, 0, ctx->stream>>>(x_dev, n, part.as<double>());
        max_final_kernel<<<1, 1, 0, ctx->stream>>>(part.as<double>(), res.as<double>());
        check_launch("max kernels");
    }
    double h[3] = {0, 0, 0};
    VXB_CUDA(cudaMemcpyAsync(h, res.as<double>(), 8, cudaMemcpyDeviceToHost, ctx->stream));
    VXB_CUDA(cudaStreamSynchronize(ctx->stream));
    *mx = h[0];
    if (!(h[0] > -INFINITY) || !std::isfinite(h[0])) {
        *s1 = *s2 = 0.0;
        return;
    }
    {
        LaunchScope scope(ctx, VXB_K_RESAMPLE);
        if (cum_dev)
            seq_expsum_kernel<true><<<1, kSeqThreads, 0, ctx->stream>>>(x_dev, res.as<double>(), n,
                                                                        cum_dev, res.as<double>() + 1,
                                                                        ctx->exp_variant);
        else
            seq_expsum_kernel<false><<<1, kSeqThreads, 0, ctx->stream>>>(x_dev, res.as<double>(), n, nullptr,
                                                                         res.as<double>() + 1,
                                                                         ctx->exp_variant);
        check_launch("seq_expsum_kernel");
    }
    VXB_CUDA(cudaMemcpyAsync(h, res.as<double>(), 24, cudaMemcpyDeviceToHost, ctx->stream));
    VXB_CUDA(cudaStreamSynchronize(ctx->stream));
    *s1 = h[1];
    *s2 = h[2];
}

// --------------------------------------------- resample_multinomial pieces
__device__ __forceinline__ uint64_t upper_bound_dev(const double* __restrict__ cum, uint64_t n,
                                                    double target) {
    uint64_t lo = 0, hi = n;  // std::upper_bound (smc.cpp:287), clamped (smc.cpp:289)
    while (lo < hi) {
        const uint64_t mid = lo + ((hi - lo) >> 1);
        if (target < cum[mid]) hi = mid; else lo = mid + 1;
    }
    return lo >= n ? n - 1 : lo;
}
__global__ void resample_draw_kernel(const double* __restrict__ cum, uint64_t n, uint32_t dim,
                                     uint64_t key, const double* __restrict__ in,
                                     double* __restrict__ out, uint64_t* __restrict__ anc) {
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const Words w = philox2x64(key, i >> 1);  // draw i = stream position i (smc.cpp:285)
    const double u = to_unit((i & 1) ? w.w1 : w.w0);
    const double target = __dmul_rn(u, cum[n - 1]);
    const uint64_t a = upper_bound_dev(cum, n, target);
    if (anc) anc[i] = a;
    if (out)
        for (uint32_t k = 0; k < dim; ++k) out[i * dim + k] = in[a * dim + k];
}

// ---------------------------------------------------- canonical reductions
// One WARP per chunk of kChunk consecutive rows.  The rows are read once, coalesced,
// into shared memory; then lane q accumulates column q over the chunk's rows in row
// order -- the same operations in the same order as one thread per chunk would do,
// but with coalesced loads and the columns side by side.
// mode 0: w*theta_a (a<dim) and w*w  -> cols = dim+1
// mode 1: (w*(theta_a-mean_a))*(theta_b-mean_b), b<=a, row-major lower triangle
// mode 2: plain sum of v (cols = 1)
constexpr int kCanonWarps = 4;  // chunks per CTA
static size_t canon_smem(uint32_t dim) { return static_cast<size_t>(kCanonWarps) * kChunk * (dim + 1) * sizeof(double); }
__global__ void __launch_bounds__(kCanonWarps * 32)
canon_partial_kernel(int mode, const double* __restrict__ theta, const double* __restrict__ w,
                     const double* __restrict__ mean, uint64_t n, uint32_t dim, uint32_t cols,
                     double* __restrict__ part /* nchunks x cols */) {
    extern __shared__ double canon_sm[];
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint64_t c = static_cast<uint64_t>(blockIdx.x) * kCanonWarps + warp;
    const uint64_t i0 = c * kChunk;
    if (i0 >= n) return;
    const uint32_t rows = static_cast<uint32_t>(min(static_cast<uint64_t>(kChunk), n - i0));
    double* sw = canon_sm + static_cast<size_t>(warp) * kChunk * (dim + 1);
    double* st = sw + kChunk;
    for (uint32_t r = lane; r < rows; r += 32) sw[r] = w[i0 + r];
    if (mode != 2)
        for (uint32_t e = lane; e < rows * dim; e += 32) st[e] = theta[i0 * dim + e];
    __syncwarp();
    for (uint32_t q = lane; q < cols; q += 32) {
        double acc = 0.0;
        if (mode == 0) {
            if (q < dim)
                for (uint32_t r = 0; r < rows; ++r) acc = __dadd_rn(acc, __dmul_rn(sw[r], st[r * dim + q]));
            else
                for (uint32_t r = 0; r < rows; ++r) acc = __dadd_rn(acc, __dmul_rn(sw[r], sw[r]));
        } else if (mode == 1) {
            uint32_t a = 0;
            while ((a + 1) * (a + 2) / 2 <= q) ++a;  // q = a (a + 1) / 2 + b
            const uint32_t b = q - a * (a + 1) / 2;
            const double ma = mean[a], mb = mean[b];
            for (uint32_t r = 0; r < rows; ++r) {
                const double wa = __dmul_rn(sw[r], __dsub_rn(st[r * dim + a], ma));
                acc = __dadd_rn(acc, __dmul_rn(wa, __dsub_rn(st[r * dim + b], mb)));
            }
        } else {
            for (uint32_t r = 0; r < rows; ++r) acc = __dadd_rn(acc, sw[r]);
        }
        part[c * cols + q] = acc;
    }
}
__global__ void canon_final_kernel(const double* __restrict__ part, uint64_t nchunks, uint32_t cols,
                                   double* __restrict__ out) {
    const uint32_t q = threadIdx.x;
    if (q >= cols) return;
    double total = 0.0;
    for (uint64_t c = 0; c < nchunks; ++c) total = __dadd_rn(total, part[c * cols + q]);
    out[q] = total;
}
// canonical inclusive scan: cum[i] = offset(chunk) + local prefix.  One warp per
// chunk: coalesced load into shared memory, the running sum by one lane in row order,
// coalesced store.
__global__ void __launch_bounds__(kCanonWarps * 32)
cumsum_local_kernel(const double* __restrict__ w, uint64_t n, double* __restrict__ cum,
                    double* __restrict__ totals) {
    __shared__ double sm[kCanonWarps * kChunk];
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint64_t c = static_cast<uint64_t>(blockIdx.x) * kCanonWarps + warp;
    const uint64_t i0 = c * kChunk;
    if (i0 >= n) return;
    const uint32_t rows = static_cast<uint32_t>(min(static_cast<uint64_t>(kChunk), n - i0));
    double* sw = sm + warp * kChunk;
    for (uint32_t r = lane; r < rows; r += 32) sw[r] = w[i0 + r];
    __syncwarp();
    if (lane == 0) {
        double run = 0.0;
        for (uint32_t r = 0; r < rows; ++r) {
            run = __dadd_rn(run, sw[r]);
            sw[r] = run;
        }
        totals[c] = run;
    }
    __syncwarp();
    for (uint32_t r = lane; r < rows; r += 32) cum[i0 + r] = sw[r];
}
__global__ void cumsum_offsets_kernel(double* totals, uint64_t nchunks) {
    double offset = 0.0;  // totals[c] <- exclusive offset of chunk c
    for (uint64_t c = 0; c < nchunks; ++c) {
        const double t = totals[c];
        totals[c] = offset;
        offset = __dadd_rn(offset, t);
    }
}
__global__ void cumsum_apply_kernel(double* __restrict__ cum, const double* __restrict__ offsets,
                                    uint64_t n) {
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) cum[i] = __dadd_rn(offsets[i / kChunk], cum[i]);
}
__global__ void scale_kernel(double* __restrict__ v, uint64_t n, const double* __restrict__ total) {
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) v[i] = __ddiv_rn(v[i], *total);
}
__global__ void fill_kernel(double* __restrict__ v, uint64_t n, double value) {
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) v[i] = value;
}

static uint64_t n_chunks(uint64_t n) { return (n + kChunk - 1) / kChunk; }

void canon_reduce(vxb_ctx* ctx, int mode, const double* theta, const double* w, const double* mean,
                  uint64_t n, uint32_t dim, uint32_t cols, double* out_dev) {
    const uint64_t nc = n_chunks(n);
    Scratch part(ctx, nc * cols * sizeof(double));
    LaunchScope scope(ctx, VXB_K_RESAMPLE);
    if (canon_smem(dim) > 48 * 1024)
        VXB_CUDA(cudaFuncSetAttribute(canon_partial_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(canon_smem(dim))));
    canon_partial_kernel<<<grid_for(nc, kCanonWarps), kCanonWarps * 32, canon_smem(dim), ctx->stream>>>(
        mode, theta, w, mean, n, dim, cols, part.as<double>());
    canon_final_kernel<<<1, 64, 0, ctx->stream>>>(part.as<double>(), nc, cols, out_dev);
    check_launch("canon_reduce");
}

// Weighted mean / covariance with the oracle's operation order
// (vxo_weighted_moments_impl).  Results on the host; returns sum w^2.
double weighted_moments_device(vxb_ctx* ctx, const double* theta, const double* w, uint64_t n,
                               uint32_t dim, double* mean, double* cov) {
    require(dim >= 1 && dim <= 8, "invalid-shape", "dimension out of range");
    Scratch d_first(ctx, (dim + 1) * sizeof(double));
    canon_reduce(ctx, 0, theta, w, nullptr, n, dim, dim + 1, d_first.as<double>());
    const uint32_t tri = dim * (dim + 1) / 2;
    Scratch d_second(ctx, tri * sizeof(double));
    canon_reduce(ctx, 1, theta, w, d_first.as<double>(), n, dim, tri, d_second.as<double>());
    double h1[9], h2[36];
    VXB_CUDA(cudaMemcpyAsync(h1, d_first.as<double>(), (dim + 1) * 8, cudaMemcpyDeviceToHost, ctx->stream));
    VXB_CUDA(cudaMemcpyAsync(h2, d_second.as<double>(), tri * 8, cudaMemcpyDeviceToHost, ctx->stream));
    VXB_CUDA(cudaStreamSynchronize(ctx->stream));
    for (uint32_t a = 0; a < dim; ++a) mean[a] = h1[a];
    const double s2 = h1[dim];
    const double denom = 1.0 - s2;
    uint32_t q = 0;
    for (uint32_t a = 0; a < dim; ++a)
        for (uint32_t b = 0; b <= a; ++b, ++q) {
            cov[a * dim + b] = h2[q] / denom;
            cov[b * dim + a] = cov[a * dim + b];
        }
    return s2;
}

void canon_cumsum_device(vxb_ctx* ctx, const double* w, uint64_t n, double* cum) {
    const uint64_t nc = n_chunks(n);
    Scratch totals(ctx, nc * sizeof(double));
    LaunchScope scope(ctx, VXB_K_RESAMPLE);
    cumsum_local_kernel<<<grid_for(nc, kCanonWarps), kCanonWarps * 32, 0, ctx->stream>>>(w, n, cum, totals.as<double>());
    cumsum_offsets_kernel<<<1, 1, 0, ctx->stream>>>(totals.as<double>(), nc);
    cumsum_apply_kernel<<<grid_for(n, 256), 256, 0, ctx->stream>>>(cum, totals.as<double>(), n);
    check_launch("canon_cumsum");
}

// cholesky (numeric.cpp:81-96) and the jitter rule of make_kernel (smc.cpp:311-325)
static bool cholesky_host(double* a, uint32_t dim) {
    for (uint32_t j = 0; j < dim; ++j) {
        double d = a[j * dim + j];
        for (uint32_t k = 0; k < j; ++k) d -= a[j * dim + k] * a[j * dim + k];
        if (!(d > 0.0)) return false;
        const double ljj = std::sqrt(d);
        a[j * dim + j] = ljj;
        for (uint32_t i = j + 1; i < dim; ++i) {
            double s = a[i * dim + j];
            for (uint32_t k = 0; k < j; ++k) s -= a[i * dim + k] * a[j * dim + k];
            a[i * dim + j] = s / ljj;
        }
        for (uint32_t i = 0; i < j; ++i) a[i * dim + j] = 0.0;
    }
    return true;
}
static void make_kernel_host(const double* cov, uint32_t dim, double scale, double jitter,
                             double* chol) {
    double c[64];
    for (uint32_t i = 0; i < dim * dim; ++i) c[i] = scale * cov[i];
    std::copy(c, c + dim * dim, chol);
    if (!cholesky_host(chol, dim)) {
        for (uint32_t k = 0; k < dim; ++k) c[k * dim + k] += jitter;
        std::copy(c, c + dim * dim, chol);
        require(cholesky_host(chol, dim), "degenerate-ensemble",
                "covariance is rank deficient beyond jitter");
    }
}

// ------------------------------------------------------- ABC-SMC propagation
struct ProposeParams {
    uint64_t first, count, n_prev;
    uint64_t seed_hash;  // splitmix64(derive_seed(seed,{gen}))
    LogisticModel model;
    double observed[VXB_MAX_SUMMARY];
    double chol[9];
    double epsilon;
    const double* theta_prev;
    const double* cum_prev;
    double* theta_out;
    double* rho_out;
    uint8_t* flag_out;
    // optional gate (multi-GPU rounds issued ahead of the host's knowledge): the round
    // is skipped when the population is already full, state[0] >= gate_target
    const unsigned long long* gate;
    uint64_t gate_target;
};

// One proposal per thread (layout: vxo_abcsmc_propose): position 0 ancestor
// uniform, positions 2..4 the Gaussian increments, position 6+j the normal of
// simulation step j+1.
__global__ void __launch_bounds__(256, VXB_PROP_MINB) abcsmc_propose_kernel(const __grid_constant__ ProposeParams p) {
    const uint64_t r = static_cast<uint64_t>(blockIdx.x) * 256 + threadIdx.x;
    if (r >= p.count) return;
    if (p.gate && *p.gate >= p.gate_target) return;
    const uint64_t key = stream_key(p.seed_hash, p.first + r);
    const Words w0 = philox2x64(key, 0);
    const double target = __dmul_rn(to_unit(w0.w0), p.cum_prev[p.n_prev - 1]);
    const uint64_t a = upper_bound_dev(p.cum_prev, p.n_prev, target);
    double z[4];
    box_muller<Exact>(philox2x64(key, 1), z[0], z[1]);
    box_muller<Exact>(philox2x64(key, 2), z[2], z[3]);
    double th[3];
    bool inside = true;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        double inc = 0.0;
#pragma unroll
        for (int q = 0; q <= k; ++q) inc = __dadd_rn(inc, __dmul_rn(p.chol[k * 3 + q], z[q]));
        th[k] = __dadd_rn(p.theta_prev[a * 3 + k], inc);
        inside = inside && th[k] >= p.model.lo[k] && th[k] < p.model.hi[k];
    }
    double rho = __longlong_as_double(0x7FF8000000000000LL);
    uint8_t flag = 2;
    if (inside) {
        RefNoise<double> noise(key, 3);
        bool bad;
        auto emit = [](uint32_t, double) {};
        rho = logistic_path<double, Exact>(p.model, th, p.observed, noise, emit, bad);
        if (bad) {
            rho = __longlong_as_double(0x7FF8000000000000LL);
            flag = 3;
        } else {
            flag = rho <= p.epsilon ? 1 : 0;
        }
    }
    p.theta_out[r * 3 + 0] = th[0];
    p.theta_out[r * 3 + 1] = th[1];
    p.theta_out[r * 3 + 2] = th[2];
    p.rho_out[r] = rho;
    p.flag_out[r] = flag;
}

// Importance-weight denominator: one new particle per thread, previous
// population streamed through shared memory in index order, so the sum over j
// is the oracle's sequential sum (vxo_abcsmc_weights).
// 64-thread CTAs: at N = 1e5 new particles that is 1563 CTAs = 10.6 per SM, so the
// last wave costs 4% instead of the 12% of 128-thread CTAs (5.3 per SM).
constexpr int kWeightsBlock = 64;
template <int D>
__global__ void __launch_bounds__(kWeightsBlock)
abcsmc_weights_kernel(uint64_t count, const double* __restrict__ theta_new, uint64_t n_prev,
                      const double* __restrict__ theta_prev, const double* __restrict__ w_prev,
                      const double* __restrict__ chol, double* __restrict__ w_out) {
    constexpr int kTile = 128;
    __shared__ double s_theta[kTile * D];
    __shared__ double s_w[kTile];
    __shared__ double s_chol[D * D], s_invd[D];
    if (threadIdx.x < D * D) s_chol[threadIdx.x] = chol[threadIdx.x];
    if (threadIdx.x < D) s_invd[threadIdx.x] = __ddiv_rn(1.0, chol[threadIdx.x * D + threadIdx.x]);
    const uint64_t r = static_cast<uint64_t>(blockIdx.x) * kWeightsBlock + threadIdx.x;
    double ti[D];
#pragma unroll
    for (int k = 0; k < D; ++k) ti[k] = r < count ? theta_new[r * D + k] : 0.0;
    double sum = 0.0;
    for (uint64_t j0 = 0; j0 < n_prev; j0 += kTile) {
        const uint64_t len = min(static_cast<uint64_t>(kTile), n_prev - j0);
        __syncthreads();
        for (uint64_t t = threadIdx.x; t < len * D; t += kWeightsBlock) s_theta[t] = theta_prev[j0 * D + t];
        for (uint64_t t = threadIdx.x; t < len; t += kWeightsBlock) s_w[t] = w_prev[j0 + t];
        __syncthreads();
        // one term w_j exp(-q_ij / 2); terms are independent, only the running sum is
        // ordered: four terms are evaluated side by side (their Horner chains
        // interleave) and then added in index order
        const auto term = [&](uint64_t j) {
            double y[D];
            double q = 0.0;
#pragma unroll
            for (int k = 0; k < D; ++k) {
                double v = __dsub_rn(ti[k], s_theta[j * D + k]);
#pragma unroll
                for (int c = 0; c < k; ++c) v = __dsub_rn(v, __dmul_rn(s_chol[k * D + c], y[c]));
                y[k] = __dmul_rn(v, s_invd[k]);
                q = __dadd_rn(q, __dmul_rn(y[k], y[k]));
            }
            return __dmul_rn(s_w[j], exp2_clamped<Exact>(__dmul_rn(__dmul_rn(-0.5, q), kInvLn2)));
        };
        uint64_t j = 0;
        for (; j + 4 <= len; j += 4) {
            const double t0 = term(j), t1 = term(j + 1), t2 = term(j + 2), t3 = term(j + 3);
            sum = __dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(sum, t0), t1), t2), t3);
        }
        for (; j < len; ++j) sum = __dadd_rn(sum, term(j));
    }
    if (r < count) w_out[r] = __ddiv_rn(1.0, sum);
}

__global__ void gather_rows_kernel(const uint64_t* __restrict__ idx, uint64_t n_take, uint32_t dim,
                                   const double* __restrict__ src_theta,
                                   const double* __restrict__ src_rho, double* __restrict__ dst_theta,
                                   double* __restrict__ dst_rho) {
    const uint64_t t = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= n_take) return;
    const uint64_t s = idx[t];
    for (uint32_t k = 0; k < dim; ++k) dst_theta[t * dim + k] = src_theta[s * dim + k];
    dst_rho[t] = src_rho[s];
}

// ------------------------------------------- throughput mode (VXB_RNG_FAST)
// Same generation scheme with the throughput generator (Philox4x32, table-based
// normals, FMA arithmetic).  Statistically validated against the exact mode.
struct ProposeFastParams {
    ProposeParams base;
    FastKeys fast;
    uint32_t gen;
    const double2* fast_table;
};

__global__ void __launch_bounds__(256)
abcsmc_propose_fast_kernel(const __grid_constant__ ProposeFastParams pp) {
    __shared__ double2 s_tab[kFastTableSize];
    for (int i = threadIdx.x; i < kFastTableSize; i += 256) s_tab[i] = pp.fast_table[i];
    __syncthreads();
    const ProposeParams& p = pp.base;
    const uint64_t r = static_cast<uint64_t>(blockIdx.x) * 256 + threadIdx.x;
    if (r >= p.count) return;
    if (p.gate && *p.gate >= p.gate_target) return;
    const uint64_t row = p.first + r;
    const uint32_t rl = static_cast<uint32_t>(row), rh = static_cast<uint32_t>(row >> 32);
    const uint32_t dom = kDomProposal | (pp.gen << 8);
    const Words32 w0 = philox4x32(pp.fast, 0u, dom, rl, rh);
    const double target = fast_unit(w0.a, w0.b) * p.cum_prev[p.n_prev - 1];
    const uint64_t a = upper_bound_dev(p.cum_prev, p.n_prev, target);
    double z[4];
    fast_box_muller(philox4x32(pp.fast, 1u, dom, rl, rh), s_tab, z[0], z[1]);
    fast_box_muller(philox4x32(pp.fast, 2u, dom, rl, rh), s_tab, z[2], z[3]);
    double th[3];
    bool inside = true;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        double inc = 0.0;
#pragma unroll
        for (int q = 0; q <= k; ++q) inc = fma(p.chol[k * 3 + q], z[q], inc);
        th[k] = p.theta_prev[a * 3 + k] + inc;
        inside = inside && th[k] >= p.model.lo[k] && th[k] < p.model.hi[k];
    }
    double rho = __longlong_as_double(0x7FF8000000000000LL);
    uint8_t flag = 2;
    if (inside) {
        // noise domain of this generation: keeps it apart from the proposal draws
        // (domain kDomProposal) of the same row
        FastNoise64 noise(pp.fast, s_tab, rl, rh, 0u, kDomNoise | (pp.gen << 8));
        bool bad;
        auto emit = [](uint32_t, double) {};
        rho = logistic_path<double, FusedCompact>(p.model, th, p.observed, noise, emit, bad);
        if (bad) {
            rho = __longlong_as_double(0x7FF8000000000000LL);
            flag = 3;
        } else {
            flag = rho <= p.epsilon ? 1 : 0;
        }
    }
    p.theta_out[r * 3 + 0] = th[0];
    p.theta_out[r * 3 + 1] = th[1];
    p.theta_out[r * 3 + 2] = th[2];
    p.rho_out[r] = rho;
    p.flag_out[r] = flag;
}

// Whitening pre-pass for the throughput weights kernel: y = s L^-1 theta with
// s^2 = log2(e)/2, so that  w_j exp(-q_ij/2) = w_j 2^(2 y_i.y_j - |y_i|^2 - |y_j|^2).
// mode 0 (previous population): out = (2 y, -|y|^2 + log2 w) -- the weight rides in the
// exponent, so a kernel term is one 2^z and one add; mode 1 (new): out = (y, -|y|^2).
template <int D>
__global__ void whiten_kernel(int mode, uint64_t n, const double* __restrict__ theta,
                              const double* __restrict__ chol, const double* __restrict__ w,
                              double* __restrict__ out) {
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double s = 0.84932180028801907;  // sqrt(log2(e) / 2)
    double y[D], a = 0.0;
#pragma unroll
    for (int k = 0; k < D; ++k) {
        double v = theta[i * D + k];
#pragma unroll
        for (int c = 0; c < k; ++c) v = fma(-chol[k * D + c], y[c], v);
        y[k] = v / chol[k * D + k];
    }
#pragma unroll
    for (int k = 0; k < D; ++k) {
        y[k] *= s;
        a = fma(y[k], y[k], a);
        out[i * (D + 1) + k] = mode == 0 ? 2.0 * y[k] : y[k];
    }
    // (a weight that underflowed to 0 would put -inf into every exponent it meets)
    out[i * (D + 1) + D] = mode == 0 ? fmax(log2(w[i]), -1.0e4) - a : -a;
}

template <int D>
__global__ void __launch_bounds__(kWeightsBlock)
abcsmc_weights_fast_kernel(uint64_t count, const double* __restrict__ y_new, uint64_t n_prev,
                           const double* __restrict__ y_prev, const double2* __restrict__ fast_table,
                           double* __restrict__ w_out) {
    static_assert(D == 3, "rows of the whitened population are read as two 16-byte halves");
    constexpr int kTile = 128;
    __shared__ double2 s_y[kTile * 2];  // (2 y0, 2 y1), (2 y2, log2 w - |y|^2) per previous particle
    __shared__ double2 s_tab[kFastTableSize];
    for (int i = threadIdx.x; i < kFastTableSize; i += kWeightsBlock) s_tab[i] = fast_table[i];
    const uint64_t r = static_cast<uint64_t>(blockIdx.x) * kWeightsBlock + threadIdx.x;
    double yi[D + 1];
#pragma unroll
    for (int k = 0; k <= D; ++k) yi[k] = r < count ? y_new[r * (D + 1) + k] : 0.0;
    const double2* prev = reinterpret_cast<const double2*>(y_prev);
    double sum = 0.0;
    for (uint64_t j0 = 0; j0 < n_prev; j0 += kTile) {
        const uint64_t len = min(static_cast<uint64_t>(kTile), n_prev - j0);
        __syncthreads();
        for (uint64_t t = threadIdx.x; t < len * 2; t += kWeightsBlock) s_y[t] = prev[j0 * 2 + t];
        __syncthreads();
        const auto term = [&](uint64_t j) {  // w_j 2^(-|y_i - y_j|^2)
            const double2 lo = s_y[2 * j], hi = s_y[2 * j + 1];
            double z = fma(yi[0], lo.x, hi.y);
            z = fma(yi[1], lo.y, z);
            z = fma(yi[2], hi.x, z);
            return fast_exp2_neg4_finite(z + yi[D], s_tab);  // z <= 0 up to rounding, finite
        };
        uint64_t j = 0;
        for (; j + 4 <= len; j += 4) {  // four independent terms side by side, added in index order
            const double e0 = term(j), e1 = term(j + 1), e2 = term(j + 2), e3 = term(j + 3);
            sum = (((sum + e0) + e1) + e2) + e3;
        }
        for (; j < len; ++j) sum += term(j);
    }
    if (r < count) w_out[r] = 1.0 / sum;
}

// ---- rounds without host round trips (multi-GPU ABC-SMC, dist.sharded_abcsmc)
// state (device, 4 x uint64): [0] rows of the new population filled so far, [1]
// accepted proposals counted while filling, [2] rounds used, [3] reserved.
// pack: the accepted rows of this rank's slice of a round -> its packed block
// (vxb_accept_layout: count | idx | theta | rho); a round issued after the population
// filled up packs nothing.  append: the gathered blocks of all ranks, in rank order
// (= ascending proposal index), onto the population -- the first n accepted by
// proposal index, exactly as the one-GPU loop takes them.
__global__ void pack_rows_kernel(const uint64_t* __restrict__ idx, unsigned long long* count,
                                 uint64_t cap, uint32_t dim, const double* __restrict__ theta,
                                 const double* __restrict__ rho, double* __restrict__ dst_theta,
                                 double* __restrict__ dst_rho, const unsigned long long* gate,
                                 uint64_t gate_target) {
    const uint64_t t = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (gate && *gate >= gate_target) {
        if (t == 0) *count = 0;
        return;
    }
    const uint64_t n_take = min(static_cast<uint64_t>(*count), cap);
    if (t >= n_take) return;
    const uint64_t s = idx[t];
    for (uint32_t k = 0; k < dim; ++k) dst_theta[t * dim + k] = theta[s * dim + k];
    dst_rho[t] = rho[s];
}
__global__ void append_rows_kernel(const char* __restrict__ blocks, uint32_t n_blocks,
                                   vxb_accept_layout lay, uint32_t dim, double* __restrict__ pop_theta,
                                   double* __restrict__ pop_rho, uint64_t n,
                                   const unsigned long long* __restrict__ state) {
    const uint64_t base = state[0];
    if (base >= n) return;
    const uint32_t r = blockIdx.y;
    const uint64_t row = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    uint64_t before = 0, mine = 0;
    for (uint32_t q = 0; q <= r; ++q) {
        const uint64_t c = min(*reinterpret_cast<const unsigned long long*>(blocks + q * lay.stride + lay.off_count),
                               static_cast<unsigned long long>(lay.cap));
        if (q < r) before += c; else mine = c;
    }
    if (row >= mine) return;
    const uint64_t dest = base + before + row;
    if (dest >= n) return;
    const char* b = blocks + r * lay.stride;
    const double* th = reinterpret_cast<const double*>(b + lay.off_params);
    const double* rh = reinterpret_cast<const double*>(b + lay.off_rho);
    for (uint32_t k = 0; k < dim; ++k) pop_theta[dest * dim + k] = th[row * dim + k];
    pop_rho[dest] = rh[row];
}
__global__ void append_state_kernel(const char* __restrict__ blocks, uint32_t n_blocks,
                                    vxb_accept_layout lay, uint64_t n, unsigned long long* state) {
    if (state[0] >= n) return;
    unsigned long long total = 0;
    for (uint32_t q = 0; q < n_blocks; ++q)
        total += min(*reinterpret_cast<const unsigned long long*>(blocks + q * lay.stride + lay.off_count),
                     static_cast<unsigned long long>(lay.cap));
    state[1] += total;
    state[2] += 1;
    state[0] = min(static_cast<unsigned long long>(n), state[0] + total);
}
// total of the chunk totals, left to right (the canonical order), then w /= total
__global__ void chunk_total_kernel(const double* __restrict__ totals, uint64_t nchunks,
                                   double* __restrict__ out) {
    double t = 0.0;
    for (uint64_t c = 0; c < nchunks; ++c) t = __dadd_rn(t, totals[c]);
    *out = t;
}

void propose_device(vxb_ctx* ctx, const vxb_model& model, uint64_t seed, uint32_t gen,
                    uint64_t first, uint64_t count, uint64_t n_prev, const double* theta_prev,
                    const double* cum_prev, const double* chol_host, const double* observed_host,
                    double epsilon, double* theta_out, double* rho_out, uint8_t* flag_out,
                    const uint64_t* gate = nullptr, uint64_t gate_target = 0) {
    require(gen >= 1, "invalid-argument", "generation 0 is the prior predictive set");
    require(n_prev >= 1, "insufficient-data", "empty previous population");
    require(model.precision == VXB_F64 && (model.rng == VXB_RNG_REF || model.rng == VXB_RNG_FAST),
            "invalid-argument", "ABC-SMC propagation runs in fp64 (reference or throughput generator)");
    ProposeParams p{};
    p.model = make_logistic(model);
    p.first = first;
    p.count = count;
    p.n_prev = n_prev;
    const uint64_t g = gen;
    p.seed_hash = splitmix64(vxb_derive_seed(seed, &g, 1));
    for (uint32_t k = 0; k < p.model.n_obs; ++k) p.observed[k] = observed_host[k];
    for (int k = 0; k < 9; ++k) p.chol[k] = chol_host[k];
    p.epsilon = epsilon;
    p.theta_prev = theta_prev;
    p.cum_prev = cum_prev;
    p.theta_out = theta_out;
    p.rho_out = rho_out;
    p.flag_out = flag_out;
    p.gate = reinterpret_cast<const unsigned long long*>(gate);
    p.gate_target = gate_target;
    if (count == 0) return;
    LaunchScope scope(ctx, VXB_K_PROPOSE);
    if (model.rng == VXB_RNG_FAST) {
        ProposeFastParams pf{};
        pf.base = p;
        pf.fast = make_fast_keys(splitmix64(seed));
        pf.gen = gen;
        pf.fast_table = ctx->log_table;
        abcsmc_propose_fast_kernel<<<grid_for(count, 256), 256, 0, ctx->stream>>>(pf);
    } else {
        abcsmc_propose_kernel<<<grid_for(count, 256), 256, 0, ctx->stream>>>(p);
    }
    check_launch("abcsmc_propose_kernel");
}

// Throughput form of the importance weights: whiten both populations once, then
// one fused multiply-add per coordinate and a table-based exp2 per pair.
void weights_fast_device(vxb_ctx* ctx, uint32_t dim, uint64_t count, const double* theta_new,
                         uint64_t n_prev, const double* theta_prev, const double* w_prev,
                         const double* chol_dev, double* w_out) {
    require(dim == 3, "invalid-shape", "the throughput weights kernel is built for dim = 3");
    if (count == 0) return;
    Scratch y_prev(ctx, n_prev * 4 * sizeof(double)), y_new(ctx, count * 4 * sizeof(double));
    LaunchScope scope(ctx, VXB_K_WEIGHTS);
    whiten_kernel<3><<<grid_for(n_prev, 256), 256, 0, ctx->stream>>>(0, n_prev, theta_prev, chol_dev, w_prev,
                                                                    y_prev.as<double>());
    whiten_kernel<3><<<grid_for(count, 256), 256, 0, ctx->stream>>>(1, count, theta_new, chol_dev, nullptr,
                                                                   y_new.as<double>());
    abcsmc_weights_fast_kernel<3><<<grid_for(count, kWeightsBlock), kWeightsBlock, 0, ctx->stream>>>(
        count, y_new.as<double>(), n_prev, y_prev.as<double>(), ctx->log_table, w_out);
    check_launch("abcsmc_weights_fast_kernel");
}

void weights_device(vxb_ctx* ctx, uint32_t dim, uint64_t count, const double* theta_new,
                    uint64_t n_prev, const double* theta_prev, const double* w_prev,
                    const double* chol_dev, double* w_out) {
    if (count == 0) return;
    LaunchScope scope(ctx, VXB_K_WEIGHTS);
    const unsigned grid = grid_for(count, kWeightsBlock);
    switch (dim) {
        case 1: abcsmc_weights_kernel<1><<<grid, kWeightsBlock, 0, ctx->stream>>>(count, theta_new, n_prev, theta_prev, w_prev, chol_dev, w_out); break;
        case 2: abcsmc_weights_kernel<2><<<grid, kWeightsBlock, 0, ctx->stream>>>(count, theta_new, n_prev, theta_prev, w_prev, chol_dev, w_out); break;
        case 3: abcsmc_weights_kernel<3><<<grid, kWeightsBlock, 0, ctx->stream>>>(count, theta_new, n_prev, theta_prev, w_prev, chol_dev, w_out); break;
        case 4: abcsmc_weights_kernel<4><<<grid, kWeightsBlock, 0, ctx->stream>>>(count, theta_new, n_prev, theta_prev, w_prev, chol_dev, w_out); break;
        default: raise("invalid-shape", "dimension out of range (1..4)");
    }
    check_launch("abcsmc_weights_kernel");
}

}  // namespace vxb

using namespace vxb;

extern "C" int vxb_ess(vxb_ctx* ctx, const double* log_w, uint64_t n, double* ess) {
    return guarded([&] {
        use(ctx);
        require(log_w && ess && n >= 1, "invalid-argument", "null or empty argument");
        Staged d(ctx, log_w, n * 8, true, false);
        double mx, s1, s2;
        max_and_expsums(ctx, d.as<double>(), n, &mx, &s1, &s2);
        require(mx > -INFINITY, "degenerate-ensemble", "all weights are zero");
        *ess = s1 * s1 / s2;
    });
}

extern "C" int vxb_logsumexp(vxb_ctx* ctx, const double* x, uint64_t n, double* out) {
    return guarded([&] {
        use(ctx);
        require(out != nullptr, "invalid-argument", "null output");
        if (n == 0) {
            *out = -INFINITY;
            return;
        }
        Staged d(ctx, x, n * 8, true, false);
        double mx, s1, s2;
        max_and_expsums(ctx, d.as<double>(), n, &mx, &s1, &s2);
        *out = std::isfinite(mx) ? mx + std::log(s1) : mx;
    });
}

extern "C" int vxb_resample_multinomial(vxb_ctx* ctx, uint64_t n, uint32_t dim, const double* log_w,
                                        const double* particles_in, uint64_t seed,
                                        uint32_t stream_id, double* particles_out,
                                        uint64_t* ancestors) {
    return guarded([&] {
        use(ctx);
        require(log_w && n >= 1, "invalid-argument", "null or empty argument");
        require(!particles_out || particles_in, "invalid-argument", "missing input particles");
        Staged d_lw(ctx, log_w, n * 8, true, false);
        Staged d_in(ctx, particles_in, n * dim * 8, true, false);
        Staged d_out(ctx, particles_out, n * dim * 8, false, true);
        Staged d_anc(ctx, ancestors, n * 8, false, true);
        double mx, s1, s2;
        Scratch d_cum(ctx, n * 8);
        max_and_expsums(ctx, d_lw.as<double>(), n, &mx, &s1, &s2, d_cum.as<double>());
        require(mx > -INFINITY, "degenerate-ensemble", "all weights are zero");
        require(std::isfinite(s1) && s1 > 0.0, "degenerate-ensemble", "weight sum is not finite");
        {
            LaunchScope scope(ctx, VXB_K_RESAMPLE);
            resample_draw_kernel<<<grid_for(n, 256), 256, 0, ctx->stream>>>(
                d_cum.as<double>(), n, dim, stream_key(splitmix64(seed), stream_id), d_in.as<double>(),
                d_out.as<double>(), d_anc.as<uint64_t>());
            check_launch("resample kernels");
        }
        d_out.finish();
        d_anc.finish();
        VXB_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

extern "C" int vxb_abcsmc_propose(vxb_ctx* ctx, const vxb_model* model, uint64_t seed, uint32_t gen,
                                  uint64_t first, uint64_t count, uint64_t n_prev,
                                  const double* theta_prev, const double* cum_prev,
                                  const double* chol, const double* observed, double epsilon,
                                  double* theta_out, double* rho_out, uint8_t* flag_out,
                                  const uint64_t* state, uint64_t n_target) {
    return guarded([&] {
        use(ctx);
        if (count == 0) return;  // an empty shard (more ranks than proposals in the round)
        require(model && theta_prev && cum_prev && chol && observed && theta_out && rho_out &&
                    flag_out,
                "invalid-argument", "null argument");
        require(!state || is_device_pointer(state), "invalid-argument",
                "the round state lives in device memory");
        require(!is_device_pointer(chol) && !is_device_pointer(observed), "invalid-argument",
                "chol and observed are host arrays");
        Staged d_tp(ctx, theta_prev, n_prev * 3 * 8, true, false);
        Staged d_cp(ctx, cum_prev, n_prev * 8, true, false);
        Staged d_th(ctx, theta_out, count * 3 * 8, false, true);
        Staged d_rho(ctx, rho_out, count * 8, false, true);
        Staged d_flag(ctx, flag_out, count, false, true);
        propose_device(ctx, *model, seed, gen, first, count, n_prev, d_tp.as<double>(),
                       d_cp.as<double>(), chol, observed, epsilon, d_th.as<double>(),
                       d_rho.as<double>(), d_flag.as<uint8_t>(), state, n_target);
        d_th.finish();
        d_rho.finish();
        d_flag.finish();
        // all-device buffers: stay asynchronous (rounds are queued back to back)
        if (d_tp.staged() || d_cp.staged() || d_th.staged() || d_rho.staged() || d_flag.staged())
            VXB_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

// The accepted rows (finite rho <= epsilon, !failed) of `count` evaluated rows, packed
// into one block (vxb_accept_layout of (VXB_F64, dim, cap)): count | local row numbers |
// theta | rho.  Device buffers only; asynchronous.
extern "C" int vxb_abcsmc_pack_round(vxb_ctx* ctx, uint32_t dim, const double* theta,
                                     const double* rho, const uint8_t* failed, uint64_t count,
                                     double epsilon, const vxb_accept_layout* layout, void* block,
                                     const uint64_t* state, uint64_t n_target) {
    return guarded([&] {
        use(ctx);
        require(layout && block && is_device_pointer(block), "invalid-argument",
                "block is a device buffer");
        require(!state || is_device_pointer(state), "invalid-argument",
                "the round state lives in device memory");
        char* base = static_cast<char*>(block);
        auto* cnt = reinterpret_cast<unsigned long long*>(base + layout->off_count);
        if (count == 0) {
            VXB_CUDA(cudaMemsetAsync(cnt, 0, 8, ctx->stream));
            return;
        }
        require(theta && rho && is_device_pointer(theta) && is_device_pointer(rho) &&
                    (!failed || is_device_pointer(failed)),
                "invalid-argument", "theta, rho and failed are device buffers");
        require(count <= layout->cap, "invalid-shape", "the block is smaller than the slice");
        auto* idx = reinterpret_cast<uint64_t*>(base + layout->off_idx);
        compact_accepted_device(ctx, VXB_F64, rho, failed, count, epsilon, 0, layout->cap,
                                reinterpret_cast<uint64_t*>(cnt), idx);
        LaunchScope scope(ctx, VXB_K_COMPACT);
        pack_rows_kernel<<<grid_for(count, 256), 256, 0, ctx->stream>>>(
            idx, cnt, layout->cap, dim, theta, rho, reinterpret_cast<double*>(base + layout->off_params),
            reinterpret_cast<double*>(base + layout->off_rho),
            reinterpret_cast<const unsigned long long*>(state), n_target);
        check_launch("pack_rows_kernel");
    });
}

// Appends the gathered blocks of a round (n_blocks of them, rank order) to the new
// population (pop_theta: n x dim, pop_rho: n) behind the rows already filled, up to n
// rows, and advances the state.  A round that arrives after the population filled up
// changes nothing.  Device buffers only; asynchronous.
extern "C" int vxb_abcsmc_append_round(vxb_ctx* ctx, uint32_t dim, const void* blocks,
                                       uint32_t n_blocks, const vxb_accept_layout* layout,
                                       double* pop_theta, double* pop_rho, uint64_t n,
                                       uint64_t* state) {
    return guarded([&] {
        use(ctx);
        require(blocks && layout && pop_theta && pop_rho && state && n_blocks >= 1,
                "invalid-argument", "null argument");
        require(is_device_pointer(blocks) && is_device_pointer(pop_theta) &&
                    is_device_pointer(pop_rho) && is_device_pointer(state),
                "invalid-argument", "device buffers only");
        LaunchScope scope(ctx, VXB_K_COMPACT);
        const dim3 grid(grid_for(layout->cap, 256), n_blocks);
        append_rows_kernel<<<grid, 256, 0, ctx->stream>>>(
            static_cast<const char*>(blocks), n_blocks, *layout, dim, pop_theta, pop_rho, n,
            reinterpret_cast<const unsigned long long*>(state));
        append_state_kernel<<<1, 1, 0, ctx->stream>>>(static_cast<const char*>(blocks), n_blocks, *layout,
                                                     n, reinterpret_cast<unsigned long long*>(state));
        check_launch("append kernels");
    });
}

// w[i] <- w[i] / (sum of the chunk totals, added left to right): the weight
// normalisation with the divisor formed on the device in the canonical order.
// total_out (optional, device): the divisor.  Device buffers only; asynchronous.
extern "C" int vxb_normalise_by_chunk_totals(vxb_ctx* ctx, double* w, uint64_t n,
                                             const double* chunk_totals, uint64_t n_chunks_in,
                                             double* total_out) {
    return guarded([&] {
        use(ctx);
        require(w && chunk_totals && n >= 1 && n_chunks_in >= 1, "invalid-argument", "null argument");
        require(is_device_pointer(w) && is_device_pointer(chunk_totals) &&
                    (!total_out || is_device_pointer(total_out)),
                "invalid-argument", "device buffers only");
        Scratch d_total(ctx, total_out ? 0 : 8);
        double* t = total_out ? total_out : d_total.as<double>();
        LaunchScope scope(ctx, VXB_K_MISC);
        chunk_total_kernel<<<1, 1, 0, ctx->stream>>>(chunk_totals, n_chunks_in, t);
        scale_kernel<<<grid_for(n, 256), 256, 0, ctx->stream>>>(w, n, t);
        check_launch("normalise kernels");
    });
}

extern "C" int vxb_abcsmc_weights(vxb_ctx* ctx, int rng, uint32_t dim, uint64_t count,
                                  const double* theta_new, uint64_t n_prev,
                                  const double* theta_prev, const double* w_prev,
                                  const double* chol, double* w_out) {
    return guarded([&] {
        use(ctx);
        require(rng == VXB_RNG_REF || rng == VXB_RNG_FAST, "invalid-argument", "bad rng mode");
        require(dim >= 1 && dim <= 4, "invalid-shape", "dimension out of range (1..4)");
        if (count == 0) return;  // an empty shard (more ranks than chunks) is not an error
        require(theta_new && theta_prev && w_prev && chol && w_out, "invalid-argument",
                "null argument");
        Staged d_tn(ctx, theta_new, count * dim * 8, true, false);
        Staged d_tp(ctx, theta_prev, n_prev * dim * 8, true, false);
        Staged d_wp(ctx, w_prev, n_prev * 8, true, false);
        Staged d_ch(ctx, chol, dim * dim * 8, true, false);
        Staged d_out(ctx, w_out, count * 8, false, true);
        if (rng == VXB_RNG_FAST)  // the form vxb_abcsmc_run uses for a VXB_RNG_FAST model
            weights_fast_device(ctx, dim, count, d_tn.as<double>(), n_prev, d_tp.as<double>(),
                                d_wp.as<double>(), d_ch.as<double>(), d_out.as<double>());
        else
            weights_device(ctx, dim, count, d_tn.as<double>(), n_prev, d_tp.as<double>(),
                           d_wp.as<double>(), d_ch.as<double>(), d_out.as<double>());
        d_out.finish();
        // device-resident output: stay asynchronous (the multi-GPU host queues the
        // collectives behind it on the same stream)
        if (d_out.staged() || d_tn.staged() || d_tp.staged() || d_wp.staged() || d_ch.staged())
            VXB_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

// ---- population statistics in the canonical order, for the multi-GPU host
extern "C" int vxb_weighted_moments(vxb_ctx* ctx, const double* theta, const double* w, uint64_t n,
                                    uint32_t dim, double* mean, double* cov, double* sum_w2) {
    return guarded([&] {
        use(ctx);
        require(theta && w && mean && cov, "invalid-argument", "null argument");
        require(n >= 2, "insufficient-data", "covariance needs at least two rows");
        require(!is_device_pointer(mean) && !is_device_pointer(cov), "invalid-argument",
                "mean and cov are host arrays");
        Staged d_th(ctx, theta, n * dim * 8, true, false);
        Staged d_w(ctx, w, n * 8, true, false);
        const double s2 = weighted_moments_device(ctx, d_th.as<double>(), d_w.as<double>(), n, dim,
                                                  mean, cov);
        if (sum_w2) *sum_w2 = s2;
    });
}

extern "C" int vxb_canon_cumsum(vxb_ctx* ctx, const double* w, uint64_t n, double* cum) {
    return guarded([&] {
        use(ctx);
        require(w && cum && n >= 1, "invalid-argument", "null argument");
        Staged d_w(ctx, w, n * 8, true, false);
        Staged d_c(ctx, cum, n * 8, false, true);
        canon_cumsum_device(ctx, d_w.as<double>(), n, d_c.as<double>());
        d_c.finish();
        if (d_c.staged()) VXB_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

extern "C" int vxb_canon_chunk_sums(vxb_ctx* ctx, const double* v, uint64_t n, double* chunk_sums) {
    return guarded([&] {
        use(ctx);
        require(v && chunk_sums && n >= 1, "invalid-argument", "null argument");
        const uint64_t nc = n_chunks(n);
        Staged d_v(ctx, v, n * 8, true, false);
        Staged d_s(ctx, chunk_sums, nc * 8, false, true);
        {
            LaunchScope scope(ctx, VXB_K_RESAMPLE);
            canon_partial_kernel<<<grid_for(nc, kCanonWarps), kCanonWarps * 32, canon_smem(1), ctx->stream>>>(
                2, nullptr, d_v.as<double>(), nullptr, n, 1, 1, d_s.as<double>());
            check_launch("canon_partial_kernel");
        }
        d_s.finish();
        if (d_s.staged()) VXB_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

extern "C" int vxb_quantile(vxb_ctx* ctx, const double* values, uint64_t n, double level,
                            double* out) {
    return guarded([&] {
        use(ctx);
        require(values && out, "invalid-argument", "null argument");
        require(n >= 1, "insufficient-data", "quantile of an empty sample");
        Staged d_v(ctx, values, n * 8, true, false);
        *out = quantile_device(ctx, d_v.as<double>(), n, level);
    });
}

extern "C" int vxb_divide(vxb_ctx* ctx, double* v, uint64_t n, double divisor) {
    return guarded([&] {
        use(ctx);
        require(v && n >= 1, "invalid-argument", "null argument");
        Staged d_v(ctx, v, n * 8, true, true);
        Scratch d_div(ctx, 8);
        VXB_CUDA(cudaMemcpyAsync(d_div.as<void>(), &divisor, 8, cudaMemcpyHostToDevice, ctx->stream));
        {
            LaunchScope scope(ctx, VXB_K_MISC);
            scale_kernel<<<grid_for(n, 256), 256, 0, ctx->stream>>>(d_v.as<double>(), n,
                                                                  d_div.as<double>());
            check_launch("scale_kernel");
        }
        d_v.finish();
        // `divisor` is a stack variable of the caller: the copy must have left it
        VXB_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

extern "C" int vxb_make_kernel(const double* cov, uint32_t dim, double scale, double jitter,
                               double* chol) {
    return guarded([&] {
        require(cov && chol, "invalid-argument", "null argument");
        require(dim >= 1 && dim <= 8, "invalid-shape", "dimension out of range");
        make_kernel_host(cov, dim, scale, jitter, chol);
    });
}

// Full run, device resident; follows vxo_abcsmc_run step for step.
extern "C" int vxb_abcsmc_run(vxb_ctx* ctx, const vxb_model* model, const vxb_abcsmc_cfg* cfg,
                              const double* observed, vxb_abcsmc_out* out) {
    return guarded([&] {
        use(ctx);
        require(model && cfg && observed && out, "invalid-argument", "null argument");
        const LogisticModel lm = make_logistic(*model);
        (void)lm;
        require(model->precision == VXB_F64 &&
                    (model->rng == VXB_RNG_REF || model->rng == VXB_RNG_FAST),
                "invalid-argument", "ABC-SMC runs in fp64 (reference or throughput generator)");
        const bool fast = model->rng == VXB_RNG_FAST;
        const uint64_t n = cfg->particles;
        const uint32_t d = 3;
        require(n >= 2, "insufficient-data", "need at least two particles");
        require(cfg->generations >= 1, "invalid-argument", "need at least one generation");
        require(cfg->quantile > 0.0 && cfg->quantile <= 1.0, "invalid-argument",
                "quantile must lie in (0, 1]");
        const uint64_t round = cfg->round_size ? cfg->round_size : n;
        const uint64_t max_rounds = cfg->max_rounds ? cfg->max_rounds : 1000;
        const uint64_t zero = 0;

        Scratch theta(ctx, n * d * 8), w(ctx, n * 8), rho(ctx, n * 8), cum(ctx, n * 8);
        Scratch th_new(ctx, n * d * 8), rho_new(ctx, n * 8), w_new(ctx, n * 8);
        Scratch p_theta(ctx, round * d * 8), p_rho(ctx, round * 8), p_flag(ctx, round);
        Scratch p_idx(ctx, round * 8), d_chol(ctx, 9 * 8), d_total(ctx, 8);
        double* cur_theta = theta.as<double>();
        double* cur_w = w.as<double>();
        double* cur_rho = rho.as<double>();
        double* nxt_theta = th_new.as<double>();
        double* nxt_w = w_new.as<double>();
        double* nxt_rho = rho_new.as<double>();

        for (uint32_t g = 0; g < cfg->generations; ++g) {
            double eps = std::numeric_limits<double>::infinity();
            double chol[9] = {0};
            if (g >= 1) {
                eps = quantile_device(ctx, cur_rho, n, cfg->quantile);
                double mean[3], cov[9];
                weighted_moments_device(ctx, cur_theta, cur_w, n, d, mean, cov);
                make_kernel_host(cov, d, cfg->kernel_scale, cfg->jitter, chol);
                canon_cumsum_device(ctx, cur_w, n, cum.as<double>());
                VXB_CUDA(cudaMemcpyAsync(d_chol.as<void>(), chol, sizeof(chol), cudaMemcpyHostToDevice,
                                         ctx->stream));
            }
            uint64_t got = 0, evaluated = 0, accepted_total = 0;
            for (uint64_t t = 0; t < max_rounds && got < n; ++t) {
                if (g == 0) {
                    vxb_keying key{VXB_KEY_PARTICLE, 1, 1, 0, vxb_derive_seed(cfg->seed, &zero, 1)};
                    const int rc = vxb_abc_prior_predictive(
                        ctx, model, &key, (t + 1) * round, t * round, round, observed,
                        p_theta.as<double>(), nullptr, p_rho.as<double>(), p_flag.as<uint8_t>(),
                        nullptr);
                    require(rc == 0, "internal", vxb_last_error());
                } else {
                    propose_device(ctx, *model, cfg->seed, g, t * round, round, n, cur_theta,
                                   cum.as<double>(), chol, observed, eps, p_theta.as<double>(),
                                   p_rho.as<double>(), p_flag.as<uint8_t>());
                }
                evaluated += round;
                // accepted <=> finite rho <= eps (rejected / outside / failed rows carry
                // rho > eps or NaN); generation 0: failed flag excludes the row
                uint64_t acc = 0;
                compact_accepted_device(ctx, VXB_F64, p_rho.as<double>(),
                                        g == 0 ? p_flag.as<uint8_t>() : nullptr, round, eps, 0, round,
                                        &acc, p_idx.as<uint64_t>());
                accepted_total += acc;
                const uint64_t take = std::min(acc, n - got);
                if (take) {
                    LaunchScope scope(ctx, VXB_K_COMPACT);
                    gather_rows_kernel<<<grid_for(take, 256), 256, 0, ctx->stream>>>(
                        p_idx.as<uint64_t>(), take, d, p_theta.as<double>(), p_rho.as<double>(),
                        nxt_theta + got * d, nxt_rho + got);
                    check_launch("gather_rows_kernel");
                }
                got += take;
            }
            require(got == n, "empty-set", "generation did not fill within max_rounds");
            if (g == 0) {
                LaunchScope scope(ctx, VXB_K_MISC);
                fill_kernel<<<grid_for(n, 256), 256, 0, ctx->stream>>>(nxt_w, n, 1.0 / static_cast<double>(n));
                check_launch("fill_kernel");
            } else {
                if (fast)
                    weights_fast_device(ctx, d, n, nxt_theta, n, cur_theta, cur_w, d_chol.as<double>(), nxt_w);
                else
                    weights_device(ctx, d, n, nxt_theta, n, cur_theta, cur_w, d_chol.as<double>(), nxt_w);
                canon_reduce(ctx, 2, nullptr, nxt_w, nullptr, n, d, 1, d_total.as<double>());
                double total = 0.0;
                VXB_CUDA(cudaMemcpyAsync(&total, d_total.as<void>(), 8, cudaMemcpyDeviceToHost, ctx->stream));
                VXB_CUDA(cudaStreamSynchronize(ctx->stream));
                require(std::isfinite(total) && total > 0.0, "degenerate-ensemble",
                        "weight sum is not finite");
                LaunchScope scope(ctx, VXB_K_MISC);
                scale_kernel<<<grid_for(n, 256), 256, 0, ctx->stream>>>(nxt_w, n, d_total.as<double>());
                check_launch("scale_kernel");
            }
            std::swap(cur_theta, nxt_theta);
            std::swap(cur_w, nxt_w);
            std::swap(cur_rho, nxt_rho);
            double mean[3], cov[9];
            const double s2 = weighted_moments_device(ctx, cur_theta, cur_w, n, d, mean, cov);
            if (out->epsilon) out->epsilon[g] = eps;
            if (out->ess) out->ess[g] = 1.0 / s2;
            if (out->accept_rate)
                out->accept_rate[g] = static_cast<double>(accepted_total) / static_cast<double>(evaluated);
            if (out->proposals) out->proposals[g] = evaluated;
            if (out->mean) std::copy(mean, mean + d, out->mean + g * d);
            if (out->cov) std::copy(cov, cov + d * d, out->cov + g * d * d);
        }
        if (out->theta) VXB_CUDA(cudaMemcpyAsync(out->theta, cur_theta, n * d * 8, cudaMemcpyDefault, ctx->stream));
        if (out->weight) VXB_CUDA(cudaMemcpyAsync(out->weight, cur_w, n * 8, cudaMemcpyDefault, ctx->stream));
        if (out->rho) VXB_CUDA(cudaMemcpyAsync(out->rho, cur_rho, n * 8, cudaMemcpyDefault, ctx->stream));
        VXB_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

// ---------------------------------------------------------------------------
// ABC-SMC over several GPUs, SPMD: every rank calls this with its context and
// communicator (comm == NULL: one rank).  The scheme and every number are those of
// vxb_abcsmc_run -- the result is bit-identical for any number of ranks -- with the
// proposals of a round and the new particles of a generation sharded by global index
// (partition(., ranks, 1)):
//   * per round ONE all-gather of each rank's packed block of accepted proposals
//     (vxb_accept_layout), appended in rank order = ascending proposal index;
//   * per generation one all-gather of the unnormalised weights (shards aligned to the
//     256-row canonical chunks, padded to the largest) and one all-reduce(SUM) of the
//     chunk totals (one non-zero contributor per entry: exact); the divisor is formed
//     on the device, chunk totals left to right.
// Rounds are issued ahead of the host's knowledge (device-resident state, gated
// kernels); the host reads the 4-word state once per batch of rounds.  The previous
// population is replicated; its statistics are recomputed on every rank.
// The Python mirror of this loop is dist.sharded_abcsmc (gloo-testable).
extern "C" int vxb_sharded_abcsmc_run(vxb_ctx* ctx, vxb_comm* comm, const vxb_model* model,
                                      const vxb_abcsmc_cfg* cfg, const double* observed,
                                      vxb_abcsmc_out* out) {
    return guarded([&] {
        use(ctx);
        require(model && cfg && observed && out, "invalid-argument", "null argument");
        require(model->precision == VXB_F64 &&
                    (model->rng == VXB_RNG_REF || model->rng == VXB_RNG_FAST),
                "invalid-argument", "ABC-SMC runs in fp64 (reference or throughput generator)");
        const bool fast = model->rng == VXB_RNG_FAST;
        const uint64_t n = cfg->particles;
        const uint32_t d = 3;
        require(n >= 2, "insufficient-data", "need at least two particles");
        require(cfg->generations >= 1, "invalid-argument", "need at least one generation");
        require(cfg->quantile > 0.0 && cfg->quantile <= 1.0, "invalid-argument",
                "quantile must lie in (0, 1]");
        const uint64_t round = cfg->round_size ? cfg->round_size : n;
        const uint64_t max_rounds = cfg->max_rounds ? cfg->max_rounds : 1000;
        const uint64_t world = comm_size(comm), rank = comm_rank(comm);
        // a communicator of ONE rank still runs every collective (that is how the NCCL path
        // is executed on a one-GPU box); without a communicator nothing is exchanged
        const bool exchange = comm != nullptr;
        const uint64_t zero = 0;
        const uint64_t seed0 = vxb_derive_seed(cfg->seed, &zero, 1);

        // this rank's slice of a round and of the weights
        uint64_t rb, re, cap_b, cap_e;
        shard_of(round, world, rank, &rb, &re);
        shard_of(round, world, 0, &cap_b, &cap_e);
        const uint64_t slice = re - rb, cap = std::max<uint64_t>(1, cap_e - cap_b);
        const uint64_t nc = n_chunks(n);
        uint64_t cb, ce, c0b, c0e;
        shard_of(nc, world, rank, &cb, &ce);
        shard_of(nc, world, 0, &c0b, &c0e);
        const uint64_t w_begin = std::min(n, cb * kChunk), w_end = std::min(n, ce * kChunk);
        const uint64_t w_pad = std::max<uint64_t>(1, (c0e - c0b) * kChunk);

        vxb_accept_layout lay;
        require(vxb_accept_layout_of(VXB_F64, d, cap, &lay) == 0, "internal", vxb_last_error());
        Scratch theta_a(ctx, n * d * 8), theta_b(ctx, n * d * 8), rho_a(ctx, n * 8), rho_b(ctx, n * 8);
        Scratch w_a(ctx, n * 8), w_b(ctx, n * 8), cum(ctx, n * 8);
        Scratch p_theta(ctx, cap * d * 8), p_rho(ctx, cap * 8), p_flag(ctx, cap);
        Scratch block(ctx, lay.stride), blocks(ctx, exchange ? world * lay.stride : 0);
        Scratch state(ctx, 4 * 8), d_chol(ctx, 9 * 8), totals(ctx, nc * 8);
        Scratch w_send(ctx, exchange ? w_pad * 8 : 0), w_recv(ctx, exchange ? world * w_pad * 8 : 0);
        VXB_CUDA(cudaMemsetAsync(block.as<void>(), 0, lay.stride, ctx->stream));
        double* th[2] = {theta_a.as<double>(), theta_b.as<double>()};
        double* rh[2] = {rho_a.as<double>(), rho_b.as<double>()};
        double* ww[2] = {w_a.as<double>(), w_b.as<double>()};
        const void* gathered = exchange ? blocks.as<void>() : block.as<void>();
        auto* st = state.as<uint64_t>();

        double rate = 1.0;
        for (uint32_t g = 0; g < cfg->generations; ++g) {
            const double* cur_theta = th[(g + 1) & 1];
            const double* cur_w = ww[(g + 1) & 1];
            const double* cur_rho = rh[(g + 1) & 1];
            double* nxt_theta = th[g & 1];
            double* nxt_w = ww[g & 1];
            double* nxt_rho = rh[g & 1];
            double eps = std::numeric_limits<double>::infinity();
            double chol[9] = {0};
            if (g >= 1) {
                eps = quantile_device(ctx, cur_rho, n, cfg->quantile);
                double mean[3], cov[9];
                weighted_moments_device(ctx, cur_theta, cur_w, n, d, mean, cov);
                make_kernel_host(cov, d, cfg->kernel_scale, cfg->jitter, chol);
                canon_cumsum_device(ctx, cur_w, n, cum.as<double>());
                VXB_CUDA(cudaMemcpyAsync(d_chol.as<void>(), chol, sizeof(chol), cudaMemcpyHostToDevice,
                                         ctx->stream));
            }
            VXB_CUDA(cudaMemsetAsync(st, 0, 4 * 8, ctx->stream));
            uint64_t issued = 0, h_state[4] = {0, 0, 0, 0};
            while (h_state[0] < n && issued < max_rounds) {
                // generation 0 accepts every non-failed row: no slack; later: what the
                // estimated acceptance rate asks for, half as much again, plus one
                const double need = static_cast<double>(n - h_state[0]) / (static_cast<double>(round) * rate);
                uint64_t ahead = static_cast<uint64_t>(std::ceil(g == 0 ? need : 1.5 * need)) + (g == 0 ? 0 : 1);
                ahead = std::max<uint64_t>(1, std::min(ahead, max_rounds - issued));
                for (uint64_t t = issued; t < issued + ahead; ++t) {
                    const uint64_t first = t * round + rb;
                    if (g == 0) {
                        if (slice) {
                            vxb_keying key{VXB_KEY_PARTICLE, 1, 1, 0, seed0};
                            require(vxb_abc_prior_predictive(ctx, model, &key, (t + 1) * round, first, slice,
                                                             observed, p_theta.as<double>(), nullptr,
                                                             p_rho.as<double>(), p_flag.as<uint8_t>(),
                                                             nullptr) == 0,
                                    "internal", vxb_last_error());
                        }
                    } else {
                        propose_device(ctx, *model, cfg->seed, g, first, slice, n, cur_theta,
                                       cum.as<double>(), chol, observed, eps, p_theta.as<double>(),
                                       p_rho.as<double>(), p_flag.as<uint8_t>(), st, n);
                    }
                    require(vxb_abcsmc_pack_round(ctx, d, p_theta.as<double>(), p_rho.as<double>(),
                                                  g == 0 ? p_flag.as<uint8_t>() : nullptr, slice, eps, &lay,
                                                  block.as<void>(), st, n) == 0,
                            "internal", vxb_last_error());
                    if (exchange) comm_allgather(comm, block.as<void>(), blocks.as<void>(), lay.stride);
                    require(vxb_abcsmc_append_round(ctx, d, gathered, static_cast<uint32_t>(world), &lay,
                                                    nxt_theta, nxt_rho, n, st) == 0,
                            "internal", vxb_last_error());
                }
                issued += ahead;
                VXB_CUDA(cudaMemcpyAsync(h_state, st, sizeof(h_state), cudaMemcpyDeviceToHost, ctx->stream));
                VXB_CUDA(cudaStreamSynchronize(ctx->stream));  // one read per batch of rounds
                if (h_state[2])
                    rate = std::max(static_cast<double>(h_state[1]) /
                                        (static_cast<double>(h_state[2]) * static_cast<double>(round)),
                                    1e-9);
            }
            require(h_state[0] == n, "empty-set", "generation did not fill within max_rounds");
            const uint64_t evaluated = h_state[2] * round, accepted_total = h_state[1];
            rate *= 0.8;  // the acceptance rate falls from one generation to the next
            if (g == 0) {
                LaunchScope scope(ctx, VXB_K_MISC);
                fill_kernel<<<grid_for(n, 256), 256, 0, ctx->stream>>>(nxt_w, n, 1.0 / static_cast<double>(n));
                check_launch("fill_kernel");
            } else {
                const uint64_t mine = w_end - w_begin;
                double* w_local = exchange ? w_send.as<double>() : nxt_w;
                if (exchange) VXB_CUDA(cudaMemsetAsync(w_local, 0, w_pad * 8, ctx->stream));
                if (mine) {
                    if (fast)
                        weights_fast_device(ctx, d, mine, nxt_theta + w_begin * d, n, cur_theta, cur_w,
                                            d_chol.as<double>(), w_local);
                    else
                        weights_device(ctx, d, mine, nxt_theta + w_begin * d, n, cur_theta, cur_w,
                                       d_chol.as<double>(), w_local);
                }
                VXB_CUDA(cudaMemsetAsync(totals.as<void>(), 0, nc * 8, ctx->stream));
                if (mine) {
                    LaunchScope scope(ctx, VXB_K_RESAMPLE);
                    const uint64_t my_chunks = n_chunks(mine);
                    canon_partial_kernel<<<grid_for(my_chunks, kCanonWarps), kCanonWarps * 32, canon_smem(1),
                                           ctx->stream>>>(2, nullptr, w_local, nullptr, mine, 1, 1,
                                                          totals.as<double>() + cb);
                    check_launch("canon_partial_kernel");
                }
                if (exchange) {
                    comm_allgather(comm, w_send.as<void>(), w_recv.as<void>(), w_pad * 8);
                    for (uint64_t r = 0; r < world; ++r) {  // rank order = index order
                        uint64_t b2, e2;
                        shard_of(nc, world, r, &b2, &e2);
                        const uint64_t lo = std::min(n, b2 * kChunk), hi = std::min(n, e2 * kChunk);
                        if (hi > lo)
                            VXB_CUDA(cudaMemcpyAsync(nxt_w + lo, w_recv.as<double>() + r * w_pad, (hi - lo) * 8,
                                                     cudaMemcpyDeviceToDevice, ctx->stream));
                    }
                    comm_allreduce_sum_f64(comm, totals.as<double>(), nc);
                }
                require(vxb_normalise_by_chunk_totals(ctx, nxt_w, n, totals.as<double>(), nc, nullptr) == 0,
                        "internal", vxb_last_error());
            }
            double mean[3], cov[9];
            const double s2 = weighted_moments_device(ctx, nxt_theta, nxt_w, n, d, mean, cov);
            require(std::isfinite(s2) && s2 > 0.0, "degenerate-ensemble", "weight sum is not finite");
            if (out->epsilon) out->epsilon[g] = eps;
            if (out->ess) out->ess[g] = 1.0 / s2;
            if (out->accept_rate)
                out->accept_rate[g] = static_cast<double>(accepted_total) / static_cast<double>(evaluated);
            if (out->proposals) out->proposals[g] = evaluated;
            if (out->mean) std::copy(mean, mean + d, out->mean + g * d);
            if (out->cov) std::copy(cov, cov + d * d, out->cov + g * d * d);
        }
        const uint32_t last = (cfg->generations - 1) & 1;
        if (out->theta) VXB_CUDA(cudaMemcpyAsync(out->theta, th[last], n * d * 8, cudaMemcpyDefault, ctx->stream));
        if (out->weight) VXB_CUDA(cudaMemcpyAsync(out->weight, ww[last], n * 8, cudaMemcpyDefault, ctx->stream));
        if (out->rho) VXB_CUDA(cudaMemcpyAsync(out->rho, rh[last], n * 8, cudaMemcpyDefault, ctx->stream));
        VXB_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}
