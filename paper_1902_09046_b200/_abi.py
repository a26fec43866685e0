"""ctypes mirror of include/vexbayes_cuda.h (struct layouts and enums only).

No computation lives here; the module exists so that Python callers (tests,
bench.py, the torch.distributed host layer) can build the POD descriptors the
C ABI takes.  Field order and types must match the header exactly.
"""
import ctypes as C

VXB_OPT_EARLY_REJECT = 1
VXB_ABI_VERSION = 2

VXB_MODEL_LOGISTIC_SDE, VXB_MODEL_NORMAL_MEAN, VXB_MODEL_MM_TAULEAP, VXB_MODEL_TOGGLE = 1, 2, 3, 4
VXB_MODEL_TB = 5
VXB_F64, VXB_F32 = 0, 1
VXB_RNG_REF, VXB_RNG_FAST, VXB_RNG_EXTERNAL = 0, 1, 2
VXB_ARITH_EXACT, VXB_ARITH_FMA = 0, 1
VXB_KEY_PARTICLE, VXB_KEY_WORKER = 0, 1

VXB_K_NAMES = ("simulate", "select", "compact", "ppp", "resample", "weights", "propose",
               "tauleap", "rngfill", "misc")
VXB_K_COUNT = len(VXB_K_NAMES)


class vxb_model(C.Structure):
    _fields_ = [
        ("model", C.c_int32), ("precision", C.c_int32), ("rng", C.c_int32), ("arith", C.c_int32),
        ("dim", C.c_uint32), ("summary_dim", C.c_uint32), ("steps", C.c_uint32),
        ("obs_stride", C.c_uint32),
        ("dt", C.c_double), ("x0", C.c_double),
        ("prior_lo", C.c_double * 8), ("prior_hi", C.c_double * 8), ("consts", C.c_double * 16),
    ]


class vxb_keying(C.Structure):
    _fields_ = [("mode", C.c_int32), ("workers", C.c_uint32), ("block_width", C.c_uint32),
                ("reserved", C.c_uint32), ("seed", C.c_uint64)]


class vxb_device_props(C.Structure):
    _fields_ = [("device", C.c_int32), ("sm_count", C.c_int32), ("cc_major", C.c_int32),
                ("cc_minor", C.c_int32), ("clock_khz", C.c_int32), ("reserved", C.c_int32),
                ("global_mem", C.c_uint64), ("name", C.c_char * 128)]


class vxb_profile(C.Structure):
    _fields_ = [("launches", C.c_uint64 * VXB_K_COUNT), ("total_ms", C.c_double * VXB_K_COUNT)]


class vxb_abcsmc_cfg(C.Structure):
    _fields_ = [("particles", C.c_uint64), ("generations", C.c_uint32), ("reserved", C.c_uint32),
                ("quantile", C.c_double), ("kernel_scale", C.c_double), ("jitter", C.c_double),
                ("round_size", C.c_uint64), ("max_rounds", C.c_uint64), ("seed", C.c_uint64)]


class vxb_abcsmc_out(C.Structure):
    _fields_ = [("theta", C.c_void_p), ("weight", C.c_void_p), ("rho", C.c_void_p),
                ("epsilon", C.c_void_p), ("ess", C.c_void_p), ("accept_rate", C.c_void_p),
                ("proposals", C.c_void_p), ("mean", C.c_void_p), ("cov", C.c_void_p)]


class vxb_weakinfo_cfg(C.Structure):
    _fields_ = [("hyper_count", C.c_uint64), ("datasets", C.c_uint64), ("particles", C.c_uint64),
                ("block_width", C.c_uint64), ("seed", C.c_uint64), ("alpha", C.c_double),
                ("c", C.c_double), ("scale", C.c_double), ("base", C.c_double * 2),
                ("redraw_base", C.c_int32), ("groups", C.c_uint32),
                ("group_size", C.c_uint32 * 16), ("dose", C.c_double * 16),
                ("arith", C.c_int32), ("rng", C.c_int32)]


class vxb_mlmc_cfg(C.Structure):
    _fields_ = [("levels", C.c_uint32), ("refine", C.c_uint32), ("tau0", C.c_double),
                ("t_end", C.c_double), ("paths", C.c_uint64), ("seed", C.c_uint64)]


class vxb_mlmc_out(C.Structure):
    _fields_ = [("level_mean", C.c_void_p), ("level_var", C.c_void_p), ("level_cost", C.c_void_p),
                ("estimate", C.c_double), ("std_error", C.c_double)]


VXB_COMM_ID_BYTES = 128
VXB_DT_U8, VXB_DT_I64, VXB_DT_U64, VXB_DT_F64, VXB_DT_U32 = 0, 1, 2, 3, 4
VXB_OP_SUM, VXB_OP_MAX = 0, 1


class vxb_accept_layout(C.Structure):
    _fields_ = [("cap", C.c_uint64), ("off_count", C.c_uint64), ("off_idx", C.c_uint64),
                ("off_params", C.c_uint64), ("off_rho", C.c_uint64), ("stride", C.c_uint64)]


# Every symbol include/vexbayes_cuda.h declares (tests check the .so exports all).
EXPORTED_SYMBOLS = (
    "vxb_abi_version", "vxb_init", "vxb_shutdown", "vxb_last_error", "vxb_device_info",
    "vxb_stream", "vxb_synchronize", "vxb_profile_enable", "vxb_profile_reset",
    "vxb_profile_read", "vxb_fma_peak", "vxb_device_alloc", "vxb_device_free", "vxb_copy",
    "vxb_splitmix64", "vxb_derive_seed", "vxb_rng_fill_u64", "vxb_rng_fill_uniform",
    "vxb_rng_fill_gaussian", "vxb_rng_fill_gaussian_fast", "vxb_fastmath_eval", "vxb_partition",
    "vxb_abc_prior_predictive", "vxb_select_epsilon", "vxb_order_statistics",
    "vxb_compact_accepted", "vxb_abc_reject", "vxb_simulate_at", "vxb_ppp_pvalues",
    "vxb_ess", "vxb_logsumexp", "vxb_resample_multinomial", "vxb_abcsmc_run",
    "vxb_abcsmc_propose", "vxb_abcsmc_weights", "vxb_weighted_moments", "vxb_canon_cumsum",
    "vxb_canon_chunk_sums", "vxb_quantile", "vxb_divide", "vxb_make_kernel", "vxb_bioassay_log_likelihood", "vxb_bioassay_sample", "vxb_smc_bioassay", "vxb_smc_bioassay_ensemble",
    "vxb_weak_info_test", "vxb_weak_info_lambdas", "vxb_weak_info_evidence",
    "vxb_weak_info_cutoffs", "vxb_mlmc_level", "vxb_mlmc_tauleap",
    "vxb_device_count", "vxb_comm_version", "vxb_comm_unique_id", "vxb_comm_init_rank",
    "vxb_comm_destroy", "vxb_comm_rank", "vxb_comm_size", "vxb_comm_allgather",
    "vxb_comm_allreduce", "vxb_accept_layout_of", "vxb_sharded_abc_reject", "vxb_accept_unpack",
    "vxb_multi_init", "vxb_multi_shutdown", "vxb_multi_size", "vxb_multi_ctx", "vxb_multi_comm",
    "vxb_multi_abc_prior_predictive", "vxb_multi_abc_reject", "vxb_multi_ppp_pvalues",
    "vxb_multi_mlmc_tauleap", "vxb_abcsmc_pack_round", "vxb_abcsmc_append_round",
    "vxb_normalise_by_chunk_totals", "vxb_guard_report", "vxb_rng_fast_stats",
    "vxb_sharded_abcsmc_run", "vxb_multi_abcsmc_run", "vxb_fast_generator_rounds", "vxb_multi_init_loopback", "vxb_multi_weak_info_test", "vxb_host_exp_variant",
    "vxb_sharded_ppp_pvalues", "vxb_sharded_mlmc_tauleap", "vxb_sharded_select_epsilon", "vxb_multi_select_epsilon", "vxb_set_option",
)
