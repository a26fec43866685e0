// vxb_common.cuh -- host-side plumbing shared by the C-ABI translation units:
// the context, the error convention (errors.hpp:11-28 "code: message" carried
// across the ABI as a thread-local string), host/device buffer staging and the
// per-launch event profiler.
#pragma once

#include <cstdint>
#include <cstdio>
#include <string>
#include <tuple>
#include <vector>

#include <cuda_runtime.h>

#include "../../include/vexbayes_cuda.h"

namespace vxb {

struct Error {
    std::string code, message;
};
[[noreturn]] inline void raise(const char* code, const std::string& message) {
    throw Error{code, message};
}
inline void require(bool ok, const char* code, const char* message) {
    if (!ok) raise(code, message);
}
void set_last_error(const std::string& text);

inline void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess)
        raise("device-error", std::string(what) + ": " + cudaGetErrorString(e));
}
#define VXB_CUDA(call) ::vxb::cuda_check((call), #call)

// Runs `f`, maps vxb::Error to the ABI convention (0 ok / 1 library error).
template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const Error& e) {
        set_last_error(e.code + ": " + e.message);
        return 1;
    } catch (const std::exception& e) {
        set_last_error(std::string("internal: ") + e.what());
        return 2;
    }
}

}  // namespace vxb

struct vxb_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    // private stream-ordered pool for Staged / Scratch: the release threshold is set
    // on THIS pool only, and vxb_shutdown destroys it -- the device's default pool
    // (shared with torch or any other cudaMallocAsync user in the process) is untouched
    cudaMemPool_t pool = nullptr;
    cudaDeviceProp prop{};
    double2* log_table = nullptr;  // fast fp64 generator table (vxb_rng.cuh)
    bool profiling = false;
    vxb_profile profile{};
    std::vector<std::tuple<int, cudaEvent_t, cudaEvent_t>> pending;
    std::vector<cudaEvent_t> event_pool;
    // grow-only device arenas for the large per-call temporaries (kept across
    // calls so that the steady state performs no allocation at all)
    void* arena[4] = {nullptr, nullptr, nullptr, nullptr};
    size_t arena_bytes[4] = {0, 0, 0, 0};
    // guard mode (environment VXB_GUARD=1 at vxb_init; diagnostics, slow): every
    // library-owned device allocation is bracketed by canary zones that are verified
    // when it is released -- the library's own out-of-bounds-write check, for pools
    // where compute-sanitizer is not available
    bool guard = false;
    unsigned long long guard_violations = 0;
    // which build of the host libm's exp the device reproduces (csrc/vxb_libmexp.cuh):
    // 0 FMA build, 1 plain build, -1 neither matched the live std::exp (FMA build used)
    int exp_variant = 0;
    // vxb_set_option(VXB_OPT_EARLY_REJECT): vxb_abc_reject stops rows that can no longer be accepted
    bool early_reject = false;
};

namespace vxb {

inline void use(vxb_ctx* ctx) {
    require(ctx != nullptr, "invalid-argument", "null context");
    VXB_CUDA(cudaSetDevice(ctx->device));
}

inline bool is_device_pointer(const void* p) {
    if (!p) return false;
    cudaPointerAttributes attr{};
    if (cudaPointerGetAttributes(&attr, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return attr.type == cudaMemoryTypeDevice || attr.type == cudaMemoryTypeManaged;
}

// ---- guard mode: canaries around library-owned device allocations
constexpr size_t kGuardBytes = 256;
constexpr int kGuardPattern = 0xA5;
inline void* guard_alloc(vxb_ctx* ctx, size_t bytes, bool pooled) {
    char* raw = nullptr;
    const size_t total = bytes + 2 * kGuardBytes;
    if (pooled)
        VXB_CUDA(cudaMallocFromPoolAsync(reinterpret_cast<void**>(&raw), total, ctx->pool, ctx->stream));
    else
        VXB_CUDA(cudaMalloc(reinterpret_cast<void**>(&raw), total));
    VXB_CUDA(cudaMemsetAsync(raw, kGuardPattern, kGuardBytes, ctx->stream));
    VXB_CUDA(cudaMemsetAsync(raw + kGuardBytes + bytes, kGuardPattern, kGuardBytes, ctx->stream));
    return raw + kGuardBytes;
}
// verifies both canaries (synchronises) and releases the allocation
inline void guard_release(vxb_ctx* ctx, void* p, size_t bytes, bool pooled, const char* what) {
    char* raw = static_cast<char*>(p) - kGuardBytes;
    unsigned char h[2 * kGuardBytes];
    cudaMemcpyAsync(h, raw, kGuardBytes, cudaMemcpyDeviceToHost, ctx->stream);
    cudaMemcpyAsync(h + kGuardBytes, raw + kGuardBytes + bytes, kGuardBytes, cudaMemcpyDeviceToHost,
                    ctx->stream);
    cudaStreamSynchronize(ctx->stream);
    size_t before = 0, after = 0;
    for (size_t i = 0; i < kGuardBytes; ++i) {
        before += h[i] != kGuardPattern;
        after += h[kGuardBytes + i] != kGuardPattern;
    }
    if (before || after) {
        ++ctx->guard_violations;
        std::fprintf(stderr, "vxb guard: out-of-bounds write on a %zu-byte %s buffer (%zu bytes before, %zu after)\n",
                     bytes, what, before, after);
    }
    if (pooled)
        cudaFreeAsync(raw, ctx->stream);
    else
        cudaFree(raw);
}

// A device view of a caller buffer.  Device pointers pass through; host
// pointers are staged through stream-ordered scratch (input: copied in on
// construction; output: copied back by finish()).
class Staged {
public:
    Staged() = default;
    Staged(vxb_ctx* ctx, const void* user, size_t bytes, bool is_input, bool is_output)
        : ctx_(ctx), user_(const_cast<void*>(user)), bytes_(bytes), out_(is_output) {
        if (!user || bytes == 0) return;
        if (is_device_pointer(user)) {
            dev_ = user_;
            return;
        }
        owned_ = true;
        if (ctx->guard)
            dev_ = guard_alloc(ctx, bytes, true);
        else
            VXB_CUDA(cudaMallocFromPoolAsync(&dev_, bytes, ctx->pool, ctx->stream));
        if (is_input)
            VXB_CUDA(cudaMemcpyAsync(dev_, user, bytes, cudaMemcpyHostToDevice, ctx->stream));
    }
    Staged(const Staged&) = delete;
    Staged& operator=(const Staged&) = delete;
    ~Staged() {
        if (!owned_ || !dev_) return;
        if (ctx_->guard)
            guard_release(ctx_, dev_, bytes_, true, "staged");
        else
            cudaFreeAsync(dev_, ctx_->stream);
    }
    // queue the device->host copy of an output (no-op for device buffers)
    void finish(size_t bytes = ~size_t(0)) {
        if (owned_ && out_ && dev_) {
            const size_t n = bytes < bytes_ ? bytes : bytes_;
            if (n) VXB_CUDA(cudaMemcpyAsync(user_, dev_, n, cudaMemcpyDeviceToHost, ctx_->stream));
        }
    }
    template <class T>
    T* as() const {
        return static_cast<T*>(dev_);
    }
    void* ptr() const { return dev_; }
    bool staged() const { return owned_; }

private:
    vxb_ctx* ctx_ = nullptr;
    void* user_ = nullptr;
    void* dev_ = nullptr;
    size_t bytes_ = 0;
    bool owned_ = false, out_ = false;
};

// Persistent scratch slot `slot` of at least `bytes` (grow-only; the contents do
// not survive a growth).  Stream-ordered use only.
inline void* arena_get(vxb_ctx* ctx, int slot, size_t bytes) {
    if (ctx->guard) {  // guard mode: a fresh bracketed allocation per request
        if (ctx->arena[slot]) guard_release(ctx, ctx->arena[slot], ctx->arena_bytes[slot], false, "arena");
        ctx->arena[slot] = guard_alloc(ctx, bytes, false);
        ctx->arena_bytes[slot] = bytes;
        return ctx->arena[slot];
    }
    if (ctx->arena_bytes[slot] < bytes) {
        VXB_CUDA(cudaStreamSynchronize(ctx->stream));
        if (ctx->arena[slot]) VXB_CUDA(cudaFree(ctx->arena[slot]));
        ctx->arena[slot] = nullptr;
        ctx->arena_bytes[slot] = 0;
        VXB_CUDA(cudaMalloc(&ctx->arena[slot], bytes));
        ctx->arena_bytes[slot] = bytes;
    }
    return ctx->arena[slot];
}

// Stream-ordered scratch with RAII.
class Scratch {
public:
    Scratch(vxb_ctx* ctx, size_t bytes) : ctx_(ctx), bytes_(bytes) {
        if (!bytes) return;
        if (ctx->guard)
            p_ = guard_alloc(ctx, bytes, true);
        else
            VXB_CUDA(cudaMallocFromPoolAsync(&p_, bytes, ctx->pool, ctx->stream));
    }
    Scratch(const Scratch&) = delete;
    Scratch& operator=(const Scratch&) = delete;
    ~Scratch() {
        if (!p_) return;
        if (ctx_->guard)
            guard_release(ctx_, p_, bytes_, true, "scratch");
        else
            cudaFreeAsync(p_, ctx_->stream);
    }
    template <class T>
    T* as() const {
        return static_cast<T*>(p_);
    }

private:
    vxb_ctx* ctx_;
    void* p_ = nullptr;
    size_t bytes_ = 0;
};

// Counts a launch of family `kind`; with profiling on, brackets it by events.
class LaunchScope {
public:
    LaunchScope(vxb_ctx* ctx, int kind) : ctx_(ctx), kind_(kind) {
        ctx->profile.launches[kind]++;
        if (ctx->profiling) {
            a_ = take();
            b_ = take();
            cudaEventRecord(a_, ctx->stream);
        }
    }
    ~LaunchScope() {
        if (ctx_->profiling) {
            cudaEventRecord(b_, ctx_->stream);
            ctx_->pending.emplace_back(kind_, a_, b_);
        }
    }

private:
    cudaEvent_t take() {
        if (!ctx_->event_pool.empty()) {
            cudaEvent_t e = ctx_->event_pool.back();
            ctx_->event_pool.pop_back();
            return e;
        }
        cudaEvent_t e;
        cudaEventCreate(&e);
        return e;
    }
    vxb_ctx* ctx_;
    int kind_;
    cudaEvent_t a_ = nullptr, b_ = nullptr;
};

inline void check_launch(const char* what) { cuda_check(cudaGetLastError(), what); }

inline unsigned grid_for(uint64_t n, unsigned block) {
    return static_cast<unsigned>((n + block - 1) / block);
}

}  // namespace vxb
