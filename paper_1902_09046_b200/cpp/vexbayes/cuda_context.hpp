// vexbayes/cuda_context.hpp -- process-wide access to the C-ABI contexts.
//
// The reference has no global state (drivers spawn and join their own threads,
// abc.cpp:64-71).  The GPU build needs one vxb_ctx per device and host thread
// that calls into the library (the single-owner rule of rng.hpp:30-31 carried
// over), so the shim keeps a thread_local vxb_multi: one context per selected
// device (every visible GPU unless set_devices() / set_device() narrows it),
// created on first use, with the library's NCCL communicators when there is more
// than one.  The batch drivers (abc::run_prior_predictive, reject_fixed_epsilon)
// split their rows over those devices with partition(n, G, 1)
// (blocked.cpp:34-63) the way the reference splits them over `workers` threads;
// everything else runs on the first device, context().  There is no CPU
// fallback: without the CUDA library or a GPU the first call throws
// vexbayes::Error("device-error").
#pragma once

#include <memory>
#include <vector>

#include "../../../include/vexbayes_cuda.h"
#include "errors.hpp"

namespace vexbayes::cuda {

inline void check(int rc) {
    if (rc != 0) rethrow(vxb_last_error());
}

namespace detail {
struct Holder {
    vxb_multi* multi = nullptr;
    std::vector<int> devices;  // empty: every visible device
    ~Holder() { vxb_multi_shutdown(multi); }
    void reset(std::vector<int> ids) {
        vxb_multi_shutdown(multi);
        multi = nullptr;
        devices = std::move(ids);
    }
};
inline Holder& holder() {
    static thread_local Holder h;
    return h;
}
}  // namespace detail

// Number of CUDA devices the process can see (0 without a GPU).
inline int device_count() {
    int n = 0;
    check(vxb_device_count(&n));
    return n;
}
// Devices the batch drivers shard over; takes effect on the next call.
inline void set_devices(std::vector<int> ids) { detail::holder().reset(std::move(ids)); }
inline void set_device(int device) {
    if (device < 0)
        set_devices({});
    else
        set_devices({device});
}

inline vxb_multi* multi() {
    auto& h = detail::holder();
    if (!h.multi)
        check(vxb_multi_init(&h.multi, h.devices.empty() ? nullptr : h.devices.data(),
                             static_cast<int>(h.devices.size())));
    return h.multi;
}
// Number of devices in use (>= 1 once a context exists).
inline int devices_in_use() { return vxb_multi_size(multi()); }
// The first device's context: single-GPU entry points run here.
inline vxb_ctx* context() { return vxb_multi_ctx(multi(), 0); }
// Early rejection in abc::reject_fixed_epsilon (VXB_OPT_EARLY_REJECT, off by default): rows
// stop once their partial distance is beyond epsilon; the accepted set is unchanged, bit
// for bit.  Applies to the devices in use now (set it again after set_devices).
inline void set_early_reject(bool on) {
    for (int r = 0; r < devices_in_use(); ++r)
        check(vxb_set_option(vxb_multi_ctx(multi(), r), VXB_OPT_EARLY_REJECT, on ? 1 : 0));
}

}  // namespace vexbayes::cuda
