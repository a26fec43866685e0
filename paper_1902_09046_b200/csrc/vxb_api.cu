// vxb_api.cu -- context lifecycle, error reporting, profiler, and the
// substrate entry points of the C ABI (RNG fills, fastmath evaluation,
// partition).  See include/vexbayes_cuda.h for the contract of each function.

#include <algorithm>
#include <cmath>
#include <cstring>

#include "vxb_common.cuh"
#include "vxb_rng.cuh"
#include "vxb_libmexp.cuh"

namespace vxb {

static thread_local std::string g_last_error;
void set_last_error(const std::string& text) { g_last_error = text; }

// Table of the fast fp64 logarithm (see fast_radius in vxb_rng.cuh).
void build_fast_log_table(double* table) {
    auto from_hi = [](uint32_t hi) {
        const uint64_t bits = static_cast<uint64_t>(hi) << 32;
        double v;
        std::memcpy(&v, &bits, 8);
        return v;
    };
    const uint32_t one_entry = (0x3FF00000u - 0x3FE6A09Eu) >> 13;
    for (uint32_t i = 0; i < kLogTableSize; ++i) {
        const double lo = from_hi(0x3FE6A09Eu + (i << 13));
        const double hi = from_hi(0x3FE6A09Eu + ((i + 1) << 13));
        double c = 1.0 / (0.5 * (lo + hi));
        double t = 2.0 * std::log(c);
        if (i == one_entry) {  // exact around u = 1
            c = 1.0;
            t = 1e-300;  // keeps -2 ln u > 0 when u == 1 exactly (no NaN from rsqrt(0))
        }
        table[2 * i] = c;
        table[2 * i + 1] = t;
    }
    const double two_pi = 6.283185307179586476925286766559;
    for (uint32_t i = 0; i < kTrigTableSize; ++i) {
        const double a = two_pi * (static_cast<double>(i) + 0.5) / kTrigTableSize;
        table[2 * (kLogTableSize + i)] = std::cos(a);
        table[2 * (kLogTableSize + i) + 1] = std::sin(a);
    }
    for (uint32_t j = 0; j < kExpTableSize; ++j)  // 2^(j/64) for fast_exp2_neg
        table[2 * (kLogTableSize + kTrigTableSize) + j] = std::exp2(static_cast<double>(j) / 64.0);
}

// ------------------------------------------------------------ fill kernels
// Thread t produces the pair block t of the requested range and writes the
// one or two positions of it that fall inside [pos, pos+n): one Philox call
// per two outputs, as in RngStream::current_pair_block (rng.cpp:80-90).
__global__ void fill_u64_kernel(uint64_t key, uint64_t pos, uint64_t n, uint64_t* out) {
    const uint64_t first_pair = pos >> 1;
    const uint64_t n_pairs = ((pos + n + 1) >> 1) - first_pair;
    const uint64_t t = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= n_pairs) return;
    const uint64_t pair = first_pair + t;
    const Words w = philox2x64(key, pair);
    const uint64_t p0 = pair << 1;
    if (p0 >= pos && p0 < pos + n) out[p0 - pos] = w.w0;
    if (p0 + 1 >= pos && p0 + 1 < pos + n) out[p0 + 1 - pos] = w.w1;
}

// fill_uniform (rng.cpp:125-140): a + u*(b-a) clamped to [a, nextafter(b,a)].
__global__ void fill_uniform_kernel(uint64_t key, uint64_t pos, uint64_t n, double a, double width,
                                    double top, double* out) {
    const uint64_t first_pair = pos >> 1;
    const uint64_t n_pairs = ((pos + n + 1) >> 1) - first_pair;
    const uint64_t t = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= n_pairs) return;
    const uint64_t pair = first_pair + t;
    const Words w = philox2x64(key, pair);
    const uint64_t p0 = pair << 1;
    const uint64_t words[2] = {w.w0, w.w1};
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const uint64_t p = p0 + h;
        if (p >= pos && p < pos + n) {
            double r = __dadd_rn(a, __dmul_rn(to_unit(words[h]), width));
            r = r < a ? a : (r > top ? top : r);
            out[p - pos] = width == 0.0 ? a : r;  // degenerate range is exact (rng.cpp:127-133)
        }
    }
}

// fill_gaussian (rng.cpp:142-164): mu + sigma * z.
__global__ void fill_gaussian_kernel(uint64_t key, uint64_t pos, uint64_t n, double mu,
                                     double sigma, double* out) {
    const uint64_t first_pair = pos >> 1;
    const uint64_t n_pairs = ((pos + n + 1) >> 1) - first_pair;
    const uint64_t t = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= n_pairs) return;
    const uint64_t pair = first_pair + t;
    const Words w = philox2x64(key, pair);
    // same operations as box_muller<Exact>, with the caller's mu and sigma
    const double u1 = to_unit(w.w0);
    const double ang = to_unit_x2(w.w1);
    const double r = __dsqrt_rn(__dmul_rn(-2.0, ln_pos<Exact, false>(__dsub_rn(1.0, u1))));
    double sn, cs;
    sincospi<Exact>(ang, sn, cs);
    const double z[2] = {__dmul_rn(r, cs), __dmul_rn(r, sn)};
    const uint64_t p0 = pair << 1;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const uint64_t p = p0 + h;
        if (p >= pos && p < pos + n) out[p - pos] = __dadd_rn(mu, __dmul_rn(sigma, z[h]));
    }
}

__global__ void fastmath_kernel(int fn, const double* x, const double* y, uint64_t n, double* out,
                                const double2* fast_table, int exp_variant) {
    // functions 6-8: the throughput-mode log2 / 2^z / reciprocal on the shared tables
    __shared__ double2 s_tab[kFastTableSize];
    if (fn >= 6 && fn <= 8) {
        for (int k = threadIdx.x; k < kFastTableSize; k += blockDim.x) s_tab[k] = fast_table[k];
        __syncthreads();
    }
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double a = x[i];
    double r;
    switch (fn) {
        case 0: r = log2_pos<Exact>(a); break;
        case 1: r = ln_pos<Exact>(a); break;
        case 2: r = exp2_clamped<Exact>(a); break;
        case 3: r = sinpi<Exact>(a); break;
        case 4: r = cospi<Exact>(a); break;
        case 5: r = pow_pos<Exact>(a, y[i]); break;
        case 6: r = fast_log2(a, s_tab); break;
        case 7: r = fast_exp2(a, s_tab); break;
        case 8: r = fast_rcp(a); break;
        case 9: r = libm_exp(a, exp_variant); break;  // the variant of this host
        case 10: r = libm_exp_t<true>(a); break;     // FMA build
        default: r = libm_exp_t<false>(a); break;    // plain build
    }
    out[i] = r;
}

}  // namespace vxb

using namespace vxb;

extern "C" int vxb_abi_version(void) { return VXB_ABI_VERSION; }
extern "C" int vxb_fast_generator_rounds(void) { return VXB_FAST_ROUNDS; }

extern "C" const char* vxb_last_error(void) { return g_last_error.c_str(); }

extern "C" int vxb_init(vxb_ctx** out, int device) {
    return guarded([&] {
        require(out != nullptr, "invalid-argument", "null context pointer");
        int count = 0;
        cudaError_t e = cudaGetDeviceCount(&count);
        if (e != cudaSuccess || count == 0)
            raise("device-error", "no CUDA device available (there is no CPU fallback)");
        if (device < 0) VXB_CUDA(cudaGetDevice(&device));
        require(device < count, "invalid-argument", "device index out of range");
        VXB_CUDA(cudaSetDevice(device));
        auto* ctx = new vxb_ctx();
        ctx->device = device;
        VXB_CUDA(cudaGetDeviceProperties(&ctx->prop, device));
        VXB_CUDA(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
        // keep stream-ordered scratch cached between calls -- in a pool of our own
        cudaMemPoolProps props{};
        props.allocType = cudaMemAllocationTypePinned;
        props.handleTypes = cudaMemHandleTypeNone;
        props.location.type = cudaMemLocationTypeDevice;
        props.location.id = device;
        VXB_CUDA(cudaMemPoolCreate(&ctx->pool, &props));
        uint64_t threshold = ~0ull;
        VXB_CUDA(cudaMemPoolSetAttribute(ctx->pool, cudaMemPoolAttrReleaseThreshold, &threshold));
        ctx->exp_variant = host_exp_variant();
        const char* guard = getenv("VXB_GUARD");
        ctx->guard = guard && *guard && *guard != '0';
        double table[2 * kFastTableSize];
        build_fast_log_table(table);
        VXB_CUDA(cudaMalloc(&ctx->log_table, sizeof(table)));
        VXB_CUDA(cudaMemcpy(ctx->log_table, table, sizeof(table), cudaMemcpyHostToDevice));
        *out = ctx;
    });
}

extern "C" void vxb_shutdown(vxb_ctx* ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    for (auto& t : ctx->pending) {
        cudaEventDestroy(std::get<1>(t));
        cudaEventDestroy(std::get<2>(t));
    }
    for (cudaEvent_t e : ctx->event_pool) cudaEventDestroy(e);
    cudaFree(ctx->log_table);
    for (int k = 0; k < 4; ++k) {
        if (!ctx->arena[k]) continue;
        if (ctx->guard)
            guard_release(ctx, ctx->arena[k], ctx->arena_bytes[k], false, "arena");
        else
            cudaFree(ctx->arena[k]);
    }
    if (ctx->guard)
        std::fprintf(stderr, "vxb guard: %llu violation(s) in this context\n", ctx->guard_violations);
    cudaStreamDestroy(ctx->stream);
    if (ctx->pool) cudaMemPoolDestroy(ctx->pool);
    delete ctx;
}

// guard mode (VXB_GUARD=1): the number of canary violations seen so far in this
// context; with selftest != 0 first provokes one (a kernel writes one byte past a
// 100-byte scratch buffer) and reports through *detected whether the guard saw it.
__global__ void guard_poke_kernel(unsigned char* p, size_t offset) { p[offset] = 0x3C; }
extern "C" int vxb_guard_report(vxb_ctx* ctx, int selftest, unsigned long long* violations,
                                int* detected) {
    return guarded([&] {
        use(ctx);
        require(violations != nullptr, "invalid-argument", "null output");
        if (selftest) {
            require(ctx->guard && detected, "invalid-argument",
                    "the self-test needs guard mode (VXB_GUARD=1 at vxb_init)");
            const unsigned long long before = ctx->guard_violations;
            {
                Scratch buf(ctx, 100);
                guard_poke_kernel<<<1, 1, 0, ctx->stream>>>(buf.as<unsigned char>(), 100);
                check_launch("guard_poke_kernel");
            }
            *detected = ctx->guard_violations == before + 1;
            ctx->guard_violations = before;  // the provoked one does not count
        }
        *violations = ctx->guard_violations;
    });
}

extern "C" int vxb_host_exp_variant(vxb_ctx* ctx, int* variant) {
    return guarded([&] {
        require(variant != nullptr, "invalid-argument", "null argument");
        *variant = ctx ? ctx->exp_variant : host_exp_variant();  // no context: probe this process
    });
}

extern "C" int vxb_device_info(vxb_ctx* ctx, vxb_device_props* out) {
    return guarded([&] {
        use(ctx);
        require(out != nullptr, "invalid-argument", "null output");
        std::memset(out, 0, sizeof(*out));
        out->device = ctx->device;
        out->sm_count = ctx->prop.multiProcessorCount;
        out->cc_major = ctx->prop.major;
        out->cc_minor = ctx->prop.minor;
        int khz = 0;
        cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, ctx->device);
        out->clock_khz = khz;
        out->global_mem = ctx->prop.totalGlobalMem;
        std::strncpy(out->name, ctx->prop.name, sizeof(out->name) - 1);
    });
}

extern "C" void* vxb_stream(vxb_ctx* ctx) { return ctx ? ctx->stream : nullptr; }

extern "C" int vxb_synchronize(vxb_ctx* ctx) {
    return guarded([&] {
        use(ctx);
        VXB_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

extern "C" int vxb_profile_enable(vxb_ctx* ctx, int on) {
    return guarded([&] {
        use(ctx);
        ctx->profiling = on != 0;
    });
}

static void drain_events(vxb_ctx* ctx) {
    VXB_CUDA(cudaStreamSynchronize(ctx->stream));
    for (auto& t : ctx->pending) {
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, std::get<1>(t), std::get<2>(t)) == cudaSuccess)
            ctx->profile.total_ms[std::get<0>(t)] += ms;
        ctx->event_pool.push_back(std::get<1>(t));
        ctx->event_pool.push_back(std::get<2>(t));
    }
    ctx->pending.clear();
}

extern "C" int vxb_profile_reset(vxb_ctx* ctx) {
    return guarded([&] {
        use(ctx);
        drain_events(ctx);
        std::memset(&ctx->profile, 0, sizeof(ctx->profile));
    });
}

extern "C" int vxb_profile_read(vxb_ctx* ctx, vxb_profile* out) {
    return guarded([&] {
        use(ctx);
        require(out != nullptr, "invalid-argument", "null output");
        drain_events(ctx);
        *out = ctx->profile;
    });
}

extern "C" int vxb_device_alloc(vxb_ctx* ctx, size_t bytes, void** out) {
    return guarded([&] {
        use(ctx);
        require(out != nullptr, "invalid-argument", "null output");
        VXB_CUDA(cudaMalloc(out, bytes ? bytes : 1));
    });
}

extern "C" int vxb_device_free(vxb_ctx* ctx, void* p) {
    return guarded([&] {
        use(ctx);
        VXB_CUDA(cudaStreamSynchronize(ctx->stream));
        VXB_CUDA(cudaFree(p));
    });
}

extern "C" int vxb_copy(vxb_ctx* ctx, void* dst, const void* src, size_t bytes) {
    return guarded([&] {
        use(ctx);
        VXB_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, ctx->stream));
        VXB_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

extern "C" uint64_t vxb_splitmix64(uint64_t z) { return splitmix64(z); }

extern "C" uint64_t vxb_derive_seed(uint64_t seed, const uint64_t* path, size_t n_path) {
    uint64_t h = splitmix64(seed);  // rng.cpp:29-35
    for (size_t i = 0; i < n_path; ++i) h = splitmix64(h ^ path[i]);
    return h;
}

extern "C" int vxb_rng_fill_u64(vxb_ctx* ctx, uint64_t seed, uint32_t stream_id, uint64_t pos,
                                uint64_t n, uint64_t* out) {
    return guarded([&] {
        use(ctx);
        if (n == 0) return;
        require(out != nullptr, "invalid-argument", "null output");
        Staged d_out(ctx, out, n * 8, false, true);
        const uint64_t n_pairs = ((pos + n + 1) >> 1) - (pos >> 1);
        {
            LaunchScope scope(ctx, VXB_K_RNGFILL);
            fill_u64_kernel<<<grid_for(n_pairs, 256), 256, 0, ctx->stream>>>(
                stream_key(splitmix64(seed), stream_id), pos, n, d_out.as<uint64_t>());
            check_launch("fill_u64_kernel");
        }
        d_out.finish();
        if (d_out.staged()) VXB_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

extern "C" int vxb_rng_fill_uniform(vxb_ctx* ctx, uint64_t seed, uint32_t stream_id, uint64_t pos,
                                    uint64_t n, double a, double b, double* out) {
    return guarded([&] {
        use(ctx);
        require(a <= b, "invalid-range", "uniform lower bound exceeds upper bound");
        if (n == 0) return;
        require(out != nullptr, "invalid-argument", "null output");
        Staged d_out(ctx, out, n * 8, false, true);
        const uint64_t n_pairs = ((pos + n + 1) >> 1) - (pos >> 1);
        const double top = a < b ? std::nextafter(b, a) : a;
        {
            LaunchScope scope(ctx, VXB_K_RNGFILL);
            fill_uniform_kernel<<<grid_for(n_pairs, 256), 256, 0, ctx->stream>>>(
                stream_key(splitmix64(seed), stream_id), pos, n, a, b - a, top,
                d_out.as<double>());
            check_launch("fill_uniform_kernel");
        }
        d_out.finish();
        if (d_out.staged()) VXB_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

extern "C" int vxb_rng_fill_gaussian(vxb_ctx* ctx, uint64_t seed, uint32_t stream_id, uint64_t pos,
                                     uint64_t n, double mu, double sigma, double* out) {
    return guarded([&] {
        use(ctx);
        require(sigma >= 0.0, "invalid-scale", "gaussian sigma must be nonnegative");
        if (n == 0) return;
        require(out != nullptr, "invalid-argument", "null output");
        Staged d_out(ctx, out, n * 8, false, true);
        const uint64_t n_pairs = ((pos + n + 1) >> 1) - (pos >> 1);
        {
            LaunchScope scope(ctx, VXB_K_RNGFILL);
            fill_gaussian_kernel<<<grid_for(n_pairs, 256), 256, 0, ctx->stream>>>(
                stream_key(splitmix64(seed), stream_id), pos, n, mu, sigma, d_out.as<double>());
            check_launch("fill_gaussian_kernel");
        }
        d_out.finish();
        if (d_out.staged()) VXB_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

extern "C" int vxb_fastmath_eval(vxb_ctx* ctx, int fn, const double* x, const double* y,
                                 uint64_t n, double* out) {
    return guarded([&] {
        use(ctx);
        require(fn >= 0 && fn <= 11, "invalid-argument", "unknown fastmath function");
        if (n == 0) return;
        require(x && out && (fn != 5 || y), "invalid-argument", "null argument");
        Staged d_x(ctx, x, n * 8, true, false);
        Staged d_y(ctx, fn == 5 ? y : nullptr, n * 8, true, false);
        Staged d_out(ctx, out, n * 8, false, true);
        {
            LaunchScope scope(ctx, VXB_K_MISC);
            fastmath_kernel<<<grid_for(n, 256), 256, 0, ctx->stream>>>(
                fn, d_x.as<double>(), d_y.as<double>(), n, d_out.as<double>(), ctx->log_table,
                ctx->exp_variant);
            check_launch("fastmath_kernel");
        }
        d_out.finish();
        if (d_out.staged()) VXB_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

// partition (blocked.cpp:34-63)
extern "C" int vxb_partition(uint64_t total, uint64_t workers, uint64_t block_width,
                             uint64_t* ranges) {
    return guarded([&] {
        require(total >= 1, "invalid-shape", "partition needs at least one item");
        require(workers >= 1, "invalid-shape", "partition needs at least one worker");
        require(block_width >= 1, "invalid-shape", "partition needs a positive block width");
        require(ranges != nullptr, "invalid-argument", "null output");
        const uint64_t blocks = (total + block_width - 1) / block_width;
        const uint64_t base = blocks / workers, extra = blocks % workers;
        uint64_t begin_block = 0;
        for (uint64_t w = 0; w < workers; ++w) {
            const uint64_t nb = base + (w < extra ? 1 : 0);
            const uint64_t begin = begin_block * block_width;
            const uint64_t end = std::min(total, (begin_block + nb) * block_width);
            ranges[2 * w] = begin > total ? total : begin;
            ranges[2 * w + 1] = begin > total ? total : end;
            begin_block += nb;
        }
    });
}

// ------------------------------------------------------------ FMA peak probe
namespace vxb {
template <class Real>
__global__ void __launch_bounds__(256) fma_peak_kernel(uint32_t iters, Real seed, Real* sink) {
    Real a[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = seed + Real(k + threadIdx.x) * Real(1e-3);
    const Real m = Real(0.999), c = Real(1e-3);
    for (uint32_t i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) a[k] = a[k] * m + c;  // contracted to one FMA
    }
    Real s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += a[k];
    if (s == Real(-1)) sink[0] = s;  // never true: keeps the chains alive
}
}  // namespace vxb

extern "C" int vxb_fma_peak(vxb_ctx* ctx, int precision, uint32_t iters, double* tflops,
                            double* ms_out) {
    return guarded([&] {
        use(ctx);
        require(tflops != nullptr && iters >= 1, "invalid-argument", "bad probe arguments");
        Scratch sink(ctx, 16);
        const unsigned blocks = static_cast<unsigned>(ctx->prop.multiProcessorCount) * 8;
        cudaEvent_t a, b;
        VXB_CUDA(cudaEventCreate(&a));
        VXB_CUDA(cudaEventCreate(&b));
        float best = 1e30f;
        for (int rep = 0; rep < 4; ++rep) {  // first repetition is the warm-up
            VXB_CUDA(cudaEventRecord(a, ctx->stream));
            if (precision == VXB_F32)
                fma_peak_kernel<float><<<blocks, 256, 0, ctx->stream>>>(iters, 1.0f, sink.as<float>());
            else
                fma_peak_kernel<double><<<blocks, 256, 0, ctx->stream>>>(iters, 1.0, sink.as<double>());
            VXB_CUDA(cudaEventRecord(b, ctx->stream));
            VXB_CUDA(cudaEventSynchronize(b));
            float ms = 0.f;
            VXB_CUDA(cudaEventElapsedTime(&ms, a, b));
            if (rep > 0 && ms < best) best = ms;
        }
        cudaEventDestroy(a);
        cudaEventDestroy(b);
        check_launch("fma_peak_kernel");
        const double flops = 2.0 * 8.0 * static_cast<double>(iters) * 256.0 * blocks;
        *tflops = flops / (best * 1e-3) / 1e12;
        if (ms_out) *ms_out = best;
    });
}
