// vexbayes/cuda_context.hpp -- process-wide access to the C-ABI context.
//
// The reference has no global state (drivers spawn and join their own threads,
// abc.cpp:64-71).  The GPU build needs one vxb_ctx per host thread that calls
// into the library (the single-owner rule of rng.hpp:30-31 carried over), so
// the shim keeps a thread_local context, created on first use on the device
// selected by set_device().  There is no CPU fallback: without the CUDA
// library or a GPU the first call throws vexbayes::Error("device-error").
#pragma once

#include <memory>

#include "../../../include/vexbayes_cuda.h"
#include "errors.hpp"

namespace vexbayes::cuda {

inline int& selected_device() {
    static thread_local int device = -1;  // -1: current CUDA device
    return device;
}
inline void set_device(int device) { selected_device() = device; }

inline void check(int rc) {
    if (rc != 0) rethrow(vxb_last_error());
}

inline vxb_ctx* context() {
    struct Holder {
        vxb_ctx* ctx = nullptr;
        ~Holder() { vxb_shutdown(ctx); }
    };
    static thread_local Holder holder;
    if (!holder.ctx) check(vxb_init(&holder.ctx, selected_device()));
    return holder.ctx;
}

}  // namespace vexbayes::cuda
