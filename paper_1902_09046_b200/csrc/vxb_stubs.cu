// vxb_stubs.cu -- entry points declared in include/vexbayes_cuda.h whose device
// implementation has not landed yet.  They fail loudly (never fall back).
#include "vxb_common.cuh"
using namespace vxb;
#define VXB_STUB(name, ...)                                                        \
    extern "C" int name(__VA_ARGS__) {                                             \
        return guarded([&] { raise("not-implemented", #name " is not built yet"); }); \
    }
VXB_STUB(vxb_ess, vxb_ctx*, const double*, uint64_t, double*)
VXB_STUB(vxb_logsumexp, vxb_ctx*, const double*, uint64_t, double*)
VXB_STUB(vxb_resample_multinomial, vxb_ctx*, uint64_t, uint32_t, const double*, const double*, uint64_t, uint32_t, double*, uint64_t*)
VXB_STUB(vxb_abcsmc_run, vxb_ctx*, const vxb_model*, const vxb_abcsmc_cfg*, const double*, vxb_abcsmc_out*)
VXB_STUB(vxb_abcsmc_propose, vxb_ctx*, const vxb_model*, uint64_t, uint32_t, uint64_t, uint64_t, uint64_t, const double*, const double*, const double*, const double*, double, double*, double*, uint8_t*)
VXB_STUB(vxb_abcsmc_weights, vxb_ctx*, uint32_t, uint64_t, const double*, uint64_t, const double*, const double*, const double*, double*)
VXB_STUB(vxb_mlmc_level, vxb_ctx*, const vxb_model*, const vxb_mlmc_cfg*, uint32_t, uint64_t, uint64_t, int64_t*, int32_t*)
VXB_STUB(vxb_mlmc_tauleap, vxb_ctx*, const vxb_model*, const vxb_mlmc_cfg*, vxb_mlmc_out*)
