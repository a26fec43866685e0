"""ctypes binding of libvexbayes_cuda.so -- the Python face of the C ABI.

Thin by design: every method forwards to one ``vxb_*`` entry point of
include/vexbayes_cuda.h, passing numpy arrays (host buffers), torch CUDA
tensors or raw device pointers straight through.  There is no CPU fallback: if
the shared object or a CUDA device is missing, loading / ``Context()`` raises.
"""
import ctypes as C
import os

import numpy as np

from . import _abi as A

HERE = os.path.dirname(os.path.abspath(__file__))
# VXB_LIBRARY selects another build of the same ABI (the Philox4x32-7 opt-in of
# paper_1902_09046_b200/build.py --rounds7); the default is the product library.
LIB_PATH = os.environ.get("VXB_LIBRARY") or os.path.join(HERE, "libvexbayes_cuda.so")

u64, u32, f64, i32 = C.c_uint64, C.c_uint32, C.c_double, C.c_int32
P = C.c_void_p
_lib = None


class VxbError(RuntimeError):
    """Mirror of vexbayes::Error (errors.hpp:11-28): ``code`` + message."""

    def __init__(self, text):
        super().__init__(text)
        self.code = text.split(":", 1)[0]


def load():
    """Load the CUDA library (built in-tree by paper_1902_09046_b200.build)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise FileNotFoundError(
                f"{LIB_PATH} is missing: run `python -m paper_1902_09046_b200.build` "
                "(there is no CPU fallback)")
        _lib = C.CDLL(LIB_PATH)
        _lib.vxb_last_error.restype = C.c_char_p
        _lib.vxb_stream.restype = P
        _lib.vxb_stream.argtypes = [P]
        _lib.vxb_splitmix64.restype = u64
        _lib.vxb_splitmix64.argtypes = [u64]
        _lib.vxb_derive_seed.restype = u64
        _lib.vxb_derive_seed.argtypes = [u64, P, C.c_size_t]
        _lib.vxb_multi_ctx.restype = P
        _lib.vxb_multi_ctx.argtypes = [P, C.c_int]
        _lib.vxb_multi_comm.restype = P
        _lib.vxb_multi_comm.argtypes = [P, C.c_int]
        _lib.vxb_multi_size.argtypes = [P]
        _lib.vxb_multi_shutdown.argtypes = [P]
        _lib.vxb_multi_shutdown.restype = None
        _lib.vxb_comm_destroy.argtypes = [P]
        _lib.vxb_comm_destroy.restype = None
        _lib.vxb_comm_rank.argtypes = [P]
        _lib.vxb_comm_size.argtypes = [P]
    return _lib


def _ptr(a):
    """numpy array / torch tensor / int address / None -> c_void_p."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        assert a.flags["C_CONTIGUOUS"], "buffers must be contiguous"
        return C.c_void_p(a.ctypes.data)
    if hasattr(a, "data_ptr"):  # torch tensor (host or device)
        assert a.is_contiguous()
        return C.c_void_p(a.data_ptr())
    return C.c_void_p(int(a))


def splitmix64(z):
    return int(load().vxb_splitmix64(z))


def derive_seed(seed, path):
    a = np.asarray(path, dtype=np.uint64)
    return int(load().vxb_derive_seed(seed, _ptr(a), len(a)))


def make_kernel(cov, scale, jitter=1e-10):
    """chol(scale * cov) with the jitter rule of smc.cpp:311-325 (host side)."""
    cov = np.ascontiguousarray(cov, dtype=np.float64)
    chol = np.zeros_like(cov)
    rc = load().vxb_make_kernel(_ptr(cov), u32(cov.shape[0]), f64(scale), f64(jitter), _ptr(chol))
    if rc:
        raise VxbError(load().vxb_last_error().decode())
    return chol


def weak_info_cutoffs(cfg, evidence):
    """p-values, cut-offs and flags from the full evidence table (host side)."""
    ev = np.ascontiguousarray(evidence, dtype=np.float64)
    k = cfg.hyper_count + 1
    gamma, weakly, completed = np.zeros(k), np.zeros(k, dtype=np.uint8), np.zeros(k, dtype=np.uint64)
    rc = load().vxb_weak_info_cutoffs(C.byref(cfg), _ptr(ev), _ptr(gamma), _ptr(weakly), _ptr(completed))
    if rc:
        raise VxbError(load().vxb_last_error().decode())
    return gamma, weakly, completed


def partition(total, workers, block_width):
    r = np.zeros((workers, 2), dtype=np.uint64)
    rc = load().vxb_partition(u64(total), u64(workers), u64(block_width), _ptr(r))
    if rc:
        raise VxbError(load().vxb_last_error().decode())
    return r


def _raise_last():
    raise VxbError(load().vxb_last_error().decode())


def host_exp_variant():
    """Probe of the calling process' std::exp (no GPU needed): 0 FMA build of the
    library's algorithm, 1 plain build, -1 neither."""
    v = C.c_int()
    if load().vxb_host_exp_variant(None, C.byref(v)):
        _raise_last()
    return v.value


def device_count():
    n = C.c_int()
    if load().vxb_device_count(C.byref(n)):
        _raise_last()
    return n.value


def accept_layout(precision, dim, cap):
    """Layout of one rank's packed accepted set (vxb_accept_layout_of)."""
    lay = A.vxb_accept_layout()
    if load().vxb_accept_layout_of(i32(precision), u32(dim), u64(cap), C.byref(lay)):
        _raise_last()
    return lay


def accept_unpack(layout, precision, dim, n_ranks, packed_all_host, cap_out=None):
    """Concatenate gathered blocks (a host uint8 array) in rank order.
    Returns (n_accepted, idx, params, rho, overflowed)."""
    buf = np.ascontiguousarray(packed_all_host, dtype=np.uint8)
    assert buf.size >= n_ranks * layout.stride
    cap_out = n_ranks * layout.cap if cap_out is None else cap_out
    dt = np.float32 if precision == A.VXB_F32 else np.float64
    idx = np.zeros(cap_out, dtype=np.uint64)
    params, rho = np.zeros((cap_out, dim), dtype=dt), np.zeros(cap_out, dtype=dt)
    n_acc, over, written = u64(), C.c_int(), u64()
    if load().vxb_accept_unpack(C.byref(layout), i32(precision), u32(dim), C.c_int(n_ranks),
                                _ptr(buf), u64(cap_out), C.byref(n_acc), _ptr(idx), _ptr(params),
                                _ptr(rho), C.byref(over), C.byref(written)):
        _raise_last()
    k = written.value
    return n_acc.value, idx[:k], params[:k], rho[:k], bool(over.value)


def comm_unique_id():
    """128-byte NCCL unique id (rank 0 creates it and ships it to the other ranks)."""
    buf = np.zeros(A.VXB_COMM_ID_BYTES, dtype=np.uint8)
    if load().vxb_comm_unique_id(_ptr(buf)):
        _raise_last()
    return buf


def comm_version():
    v = C.c_int()
    if load().vxb_comm_version(C.byref(v)):
        _raise_last()
    return v.value


class Comm:
    """The library's own NCCL communicator of one rank (vxb_comm); collectives are
    queued on the context's stream."""

    def __init__(self, ctx, unique_id, rank, n_ranks, handle=None):
        self.ctx, self.lib = ctx, load()
        self.owned = handle is None
        self.handle = P(handle) if handle is not None else P()
        if self.owned:
            uid = np.ascontiguousarray(unique_id, dtype=np.uint8)
            ctx._check(self.lib.vxb_comm_init_rank(ctx.handle, _ptr(uid), C.c_int(rank),
                                                   C.c_int(n_ranks), C.byref(self.handle)))

    @property
    def rank(self):
        return int(self.lib.vxb_comm_rank(self.handle))

    @property
    def size(self):
        return int(self.lib.vxb_comm_size(self.handle))

    def allgather(self, send, recv, nbytes):
        self.ctx._check(self.lib.vxb_comm_allgather(self.handle, _ptr(send), _ptr(recv),
                                                    C.c_size_t(nbytes)))

    def allreduce(self, buf, count, dtype=A.VXB_DT_F64, op=A.VXB_OP_SUM):
        self.ctx._check(self.lib.vxb_comm_allreduce(self.handle, _ptr(buf), C.c_size_t(count),
                                                    i32(dtype), i32(op)))

    def close(self):
        if self.owned and self.handle:
            self.lib.vxb_comm_destroy(self.handle)
        self.handle = P()


class Multi:
    """One process, several GPUs (vxb_multi): a context (and an NCCL communicator)
    per device; the calls fork one host thread per device and join."""

    def __init__(self, device_ids=None, loopback_ranks=None, device=0):
        """loopback_ranks=n (diagnostics): n contexts on ONE device joined by the
        library's loopback group instead of NCCL (vxb_multi_init_loopback)."""
        self.lib = load()
        self.handle = P()
        if loopback_ranks is not None:
            if self.lib.vxb_multi_init_loopback(C.byref(self.handle), C.c_int(device),
                                                C.c_int(loopback_ranks)):
                _raise_last()
            return
        ids = None if device_ids is None else np.ascontiguousarray(device_ids, dtype=np.int32)
        if self.lib.vxb_multi_init(C.byref(self.handle), _ptr(ids), C.c_int(0 if ids is None else ids.size)):
            _raise_last()

    def _check(self, rc):
        if rc:
            _raise_last()

    @property
    def size(self):
        return int(self.lib.vxb_multi_size(self.handle))

    def close(self):
        if self.handle:
            self.lib.vxb_multi_shutdown(self.handle)
            self.handle = P()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_early_reject(self, on=True):
        """VXB_OPT_EARLY_REJECT on every device of the group (see Context.set_early_reject)."""
        for r in range(self.size):
            self._check(self.lib.vxb_set_option(P(self.lib.vxb_multi_ctx(self.handle, r)),
                                                i32(A.VXB_OPT_EARLY_REJECT), C.c_int64(1 if on else 0)))

    def abc_prior_predictive(self, model, key, n, observed, want_summaries=True):
        dt = np.float32 if model.precision == A.VXB_F32 else np.float64
        obs = np.ascontiguousarray(observed, dtype=np.float64)
        params = np.zeros((n, model.dim), dtype=dt)
        summ = np.zeros((n, model.summary_dim), dtype=dt) if want_summaries else None
        rho, failed = np.zeros(n, dtype=dt), np.zeros(n, dtype=np.uint8)
        self._check(self.lib.vxb_multi_abc_prior_predictive(
            self.handle, C.byref(model), C.byref(key), u64(n), _ptr(obs), _ptr(params), _ptr(summ),
            _ptr(rho), _ptr(failed)))
        return params, summ, rho, failed

    def abc_reject(self, model, key, n_total, observed, eps, cap):
        dt = np.float32 if model.precision == A.VXB_F32 else np.float64
        obs = np.ascontiguousarray(observed, dtype=np.float64)
        idx = np.zeros(cap, dtype=np.uint64)
        params, rho = np.zeros((cap, model.dim), dtype=dt), np.zeros(cap, dtype=dt)
        nacc = u64()
        self._check(self.lib.vxb_multi_abc_reject(self.handle, C.byref(model), C.byref(key),
                                                  u64(n_total), _ptr(obs), f64(eps), u64(cap),
                                                  C.byref(nacc), _ptr(idx), _ptr(params), _ptr(rho)))
        k = min(nacc.value, cap)
        return nacc.value, idx[:k], params[:k], rho[:k]

    def select_epsilon(self, rho, failed, q, cap=None):
        """select_epsilon (abc.cpp:74-106) over host arrays, the rows split over the devices."""
        rho = np.ascontiguousarray(rho)
        failed = None if failed is None else np.ascontiguousarray(failed, dtype=np.uint8)
        precision = A.VXB_F32 if rho.dtype == np.float32 else A.VXB_F64
        cap = rho.size if cap is None else cap
        idx = np.zeros(cap, dtype=np.uint64)
        eps, nacc = f64(), u64()
        self._check(self.lib.vxb_multi_select_epsilon(self.handle, i32(precision), _ptr(rho), _ptr(failed),
                                                      u64(rho.size), f64(q), C.byref(eps), u64(cap),
                                                      C.byref(nacc), _ptr(idx)))
        return eps.value, idx[:min(nacc.value, cap)], nacc.value

    def ppp_pvalues(self, model, lam, log_norm, m_total, seed, ybar_obs):
        lam = np.ascontiguousarray(lam, dtype=np.float64)
        ln = np.ascontiguousarray(log_norm, dtype=np.float64)
        counts, pv = np.zeros(lam.size, dtype=np.uint64), np.zeros(lam.size)
        self._check(self.lib.vxb_multi_ppp_pvalues(self.handle, C.byref(model), _ptr(lam), _ptr(ln),
                                                   u32(lam.size), u64(m_total), u64(seed),
                                                   f64(ybar_obs), _ptr(counts), _ptr(pv)))
        return counts, pv

    def abcsmc_run(self, model, cfg, observed):
        n, g, d = cfg.particles, cfg.generations, model.dim
        obs = np.ascontiguousarray(observed, dtype=np.float64)
        res = dict(theta=np.zeros((n, d)), weight=np.zeros(n), rho=np.zeros(n),
                   epsilon=np.zeros(g), ess=np.zeros(g), accept_rate=np.zeros(g),
                   proposals=np.zeros(g, dtype=np.uint64), mean=np.zeros((g, d)),
                   cov=np.zeros((g, d, d)))
        out = A.vxb_abcsmc_out(*[res[k].ctypes.data for k in
                                 ("theta", "weight", "rho", "epsilon", "ess", "accept_rate",
                                  "proposals", "mean", "cov")])
        self._check(self.lib.vxb_multi_abcsmc_run(self.handle, C.byref(model), C.byref(cfg), _ptr(obs),
                                                  C.byref(out)))
        return res

    def weak_info_test(self, cfg, want_evidence=False):
        k = cfg.hyper_count + 1
        lam, gamma = np.zeros((k, 2)), np.zeros(k)
        weakly, completed = np.zeros(k, dtype=np.uint8), np.zeros(k, dtype=np.uint64)
        ev = np.zeros((k, cfg.datasets, 2)) if want_evidence else None
        self._check(self.lib.vxb_multi_weak_info_test(self.handle, C.byref(cfg), _ptr(lam), _ptr(gamma),
                                                      _ptr(weakly), _ptr(completed), _ptr(ev)))
        return dict(lambda_=lam, gamma=gamma, weakly=weakly, completed=completed, evidence=ev)

    def mlmc_tauleap(self, model, cfg):
        L = cfg.levels
        res = dict(level_mean=np.zeros(L), level_var=np.zeros(L), level_cost=np.zeros(L))
        out = A.vxb_mlmc_out(res["level_mean"].ctypes.data, res["level_var"].ctypes.data,
                             res["level_cost"].ctypes.data, 0.0, 0.0)
        self._check(self.lib.vxb_multi_mlmc_tauleap(self.handle, C.byref(model), C.byref(cfg),
                                                    C.byref(out)))
        res["estimate"], res["std_error"] = out.estimate, out.std_error
        return res


class Context:
    """One GPU, one stream (vxb_ctx)."""

    def __init__(self, device=-1):
        self.lib = load()
        self.handle = P()
        self._check(self.lib.vxb_init(C.byref(self.handle), i32(device)))

    def _check(self, rc):
        if rc != 0:
            raise VxbError(self.lib.vxb_last_error().decode())

    def close(self):
        if self.handle:
            self.lib.vxb_shutdown(self.handle)
            self.handle = P()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- plumbing
    def device_info(self):
        out = A.vxb_device_props()
        self._check(self.lib.vxb_device_info(self.handle, C.byref(out)))
        return dict(device=out.device, sm_count=out.sm_count, cc=(out.cc_major, out.cc_minor),
                    clock_khz=out.clock_khz, global_mem=out.global_mem, name=out.name.decode())

    def stream(self):
        return self.lib.vxb_stream(self.handle)

    def synchronize(self):
        self._check(self.lib.vxb_synchronize(self.handle))

    def profile_enable(self, on=True):
        self._check(self.lib.vxb_profile_enable(self.handle, i32(1 if on else 0)))

    def profile_reset(self):
        self._check(self.lib.vxb_profile_reset(self.handle))

    def profile_read(self):
        out = A.vxb_profile()
        self._check(self.lib.vxb_profile_read(self.handle, C.byref(out)))
        return {name: dict(launches=int(out.launches[i]), total_ms=float(out.total_ms[i]))
                for i, name in enumerate(A.VXB_K_NAMES)}

    def fma_peak(self, precision=A.VXB_F64, iters=200000):
        """Measured FMA-chain throughput (TFLOP/s) -- the roofline denominator."""
        tf, ms = f64(), f64()
        self._check(self.lib.vxb_fma_peak(self.handle, i32(precision), u32(iters), C.byref(tf),
                                          C.byref(ms)))
        return tf.value, ms.value

    def host_exp_variant(self):
        """Which build of the host libm's exp the device reproduces: 0 FMA, 1 plain, -1 none."""
        v = C.c_int()
        self._check(self.lib.vxb_host_exp_variant(self.handle, C.byref(v)))
        return v.value

    def set_early_reject(self, on=True):
        """vxb_abc_reject stops rows whose partial distance already exceeds epsilon (same
        accepted set, bit for bit); off by default."""
        self._check(self.lib.vxb_set_option(self.handle, i32(A.VXB_OPT_EARLY_REJECT), C.c_int64(1 if on else 0)))

    def guard_report(self, selftest=False):
        """Guard mode (VXB_GUARD=1): (violations so far, self-test detected or None)."""
        v, d = C.c_ulonglong(), C.c_int(-1)
        self._check(self.lib.vxb_guard_report(self.handle, i32(1 if selftest else 0), C.byref(v),
                                              C.byref(d)))
        return v.value, (bool(d.value) if selftest else None)

    def device_alloc(self, nbytes):
        out = P()
        self._check(self.lib.vxb_device_alloc(self.handle, C.c_size_t(nbytes), C.byref(out)))
        return out.value

    def device_free(self, p):
        self._check(self.lib.vxb_device_free(self.handle, P(p)))

    def copy(self, dst, src, nbytes):
        self._check(self.lib.vxb_copy(self.handle, _ptr(dst), _ptr(src), C.c_size_t(nbytes)))

    # ---- substrate
    def rng_fill_u64(self, seed, stream_id, pos, n):
        out = np.zeros(n, dtype=np.uint64)
        self._check(self.lib.vxb_rng_fill_u64(self.handle, u64(seed), u32(stream_id), u64(pos),
                                              u64(n), _ptr(out)))
        return out

    def rng_fill_uniform(self, seed, stream_id, pos, n, a=0.0, b=1.0):
        out = np.zeros(n)
        self._check(self.lib.vxb_rng_fill_uniform(self.handle, u64(seed), u32(stream_id), u64(pos),
                                                  u64(n), f64(a), f64(b), _ptr(out)))
        return out

    def rng_fill_gaussian(self, seed, stream_id, pos, n, mu=0.0, sigma=1.0):
        out = np.zeros(n)
        self._check(self.lib.vxb_rng_fill_gaussian(self.handle, u64(seed), u32(stream_id),
                                                   u64(pos), u64(n), f64(mu), f64(sigma),
                                                   _ptr(out)))
        return out

    def rng_fill_gaussian_fast(self, precision, seed, first_row, rows, per_row):
        """Normals of the throughput generator as the step loop consumes them."""
        out = np.zeros((rows, per_row), dtype=np.float32 if precision == A.VXB_F32 else np.float64)
        self._check(self.lib.vxb_rng_fill_gaussian_fast(self.handle, i32(precision), u64(seed),
                                                        u64(first_row), u64(rows), u32(per_row),
                                                        _ptr(out)))
        return out

    def rng_fast_stats(self, precision, seed, first_row, rows, per_row, thresholds=()):
        """Device-side tail counts / moments / fp32 MUFU error of the throughput generator."""
        thr = np.ascontiguousarray(thresholds, dtype=np.float64)
        tails = np.zeros(max(thr.size, 1), dtype=np.uint64)
        mom = np.zeros(9)
        self._check(self.lib.vxb_rng_fast_stats(self.handle, i32(precision), u64(seed), u64(first_row),
                                                u64(rows), u32(per_row), _ptr(thr), u32(thr.size),
                                                _ptr(tails), _ptr(mom)))
        n = mom[0]
        return dict(n=int(n), tails=tails[:thr.size], mean=mom[1] / n, var=mom[2] / n - (mom[1] / n) ** 2,
                    skew=mom[3] / n, kurt=mom[4] / n, max_abs=mom[5], err_max=mom[6],
                    err_max_tail=mom[7], err_rms=float(np.sqrt(mom[8] / n)))

    def fastmath(self, fn, x, y=None):
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.ascontiguousarray(y, dtype=np.float64) if y is not None else None
        out = np.zeros_like(x)
        self._check(self.lib.vxb_fastmath_eval(self.handle, i32(fn), _ptr(x), _ptr(y), u64(x.size),
                                               _ptr(out)))
        return out

    # ---- ABC
    def abc_prior_predictive(self, model, key, n_total, first, count, observed, params=None,
                             summaries=None, rho=None, failed=None, noise=None):
        """Raw form: every buffer is caller-supplied (numpy / torch / address)."""
        obs = np.ascontiguousarray(observed, dtype=np.float64)
        self._check(self.lib.vxb_abc_prior_predictive(
            self.handle, C.byref(model), C.byref(key), u64(n_total), u64(first), u64(count),
            _ptr(obs), _ptr(params), _ptr(summaries), _ptr(rho), _ptr(failed), _ptr(noise)))

    def abc_prior_predictive_host(self, model, key, n_total, first, count, observed, noise=None,
                                  want_summaries=True):
        """Convenience form returning numpy arrays (params, summaries, rho, failed)."""
        dt = np.float32 if model.precision == A.VXB_F32 else np.float64
        params = np.zeros((count, model.dim), dtype=dt)
        summ = np.zeros((count, model.summary_dim), dtype=dt) if want_summaries else None
        rho = np.zeros(count, dtype=dt)
        failed = np.zeros(count, dtype=np.uint8)
        if noise is not None:
            noise = np.ascontiguousarray(noise, dtype=dt)
        self.abc_prior_predictive(model, key, n_total, first, count, observed, params, summ, rho,
                                  failed, noise)
        return params, summ, rho, failed

    def simulate_at(self, model, theta, seed, stream_id, pos):
        dt = np.float32 if model.precision == A.VXB_F32 else np.float64
        th = np.ascontiguousarray(theta, dtype=np.float64)
        out = np.zeros(model.summary_dim, dtype=dt)
        self._check(self.lib.vxb_simulate_at(self.handle, C.byref(model), _ptr(th), u64(seed),
                                             u32(stream_id), u64(pos), _ptr(out)))
        return out

    def select_epsilon(self, rho, failed, q, cap=None, precision=None, n=None, idx=None):
        if isinstance(rho, np.ndarray):
            n = rho.size
            precision = A.VXB_F32 if rho.dtype == np.float32 else A.VXB_F64
        cap = n if cap is None else cap
        if idx is None:
            idx = np.zeros(cap, dtype=np.uint64)
        eps, nacc = f64(), u64()
        self._check(self.lib.vxb_select_epsilon(self.handle, i32(precision), _ptr(rho),
                                                _ptr(failed), u64(n), f64(q), C.byref(eps),
                                                u64(cap), C.byref(nacc), _ptr(idx)))
        k = min(nacc.value, cap)
        return eps.value, (idx[:k] if isinstance(idx, np.ndarray) else idx), nacc.value

    def order_statistics(self, rho, failed, ranks, precision=None, n=None):
        if isinstance(rho, np.ndarray):
            n = rho.size
            precision = A.VXB_F32 if rho.dtype == np.float32 else A.VXB_F64
        ranks = np.ascontiguousarray(ranks, dtype=np.uint64)
        vals = np.zeros(ranks.size)
        nv = u64()
        self._check(self.lib.vxb_order_statistics(self.handle, i32(precision), _ptr(rho),
                                                  _ptr(failed), u64(n), _ptr(ranks),
                                                  u32(ranks.size), _ptr(vals), C.byref(nv)))
        return vals, nv.value

    def compact_accepted(self, rho, failed, eps, index_base=0, cap=None, precision=None, n=None,
                         idx=None):
        if isinstance(rho, np.ndarray):
            n = rho.size
            precision = A.VXB_F32 if rho.dtype == np.float32 else A.VXB_F64
        cap = n if cap is None else cap
        if idx is None:
            idx = np.zeros(cap, dtype=np.uint64)
        nacc = u64()
        self._check(self.lib.vxb_compact_accepted(self.handle, i32(precision), _ptr(rho),
                                                  _ptr(failed), u64(n), f64(eps), u64(index_base),
                                                  u64(cap), C.byref(nacc), _ptr(idx)))
        k = min(nacc.value, cap)
        return (idx[:k] if isinstance(idx, np.ndarray) else idx), nacc.value

    def abc_reject(self, model, key, n_total, first, count, observed, eps, cap, idx=None,
                   params=None, rho=None, n_accepted=None):
        """Fused fixed-epsilon rejection; host numpy outputs unless buffers are given.
        With ``n_accepted`` a device int64 tensor (and device outputs) the call is
        fully asynchronous: nothing returns to the host."""
        obs = np.ascontiguousarray(observed, dtype=np.float64)
        dt = np.float32 if model.precision == A.VXB_F32 else np.float64
        own = idx is None
        if own:  # every valid row is overwritten: no need to zero cap rows per call
            idx = np.empty(cap, dtype=np.uint64)
            params = np.empty((cap, model.dim), dtype=dt)
            rho = np.empty(cap, dtype=dt)
        if n_accepted is not None:
            # asynchronous form: the count is written to device memory, no host sync
            self._check(self.lib.vxb_abc_reject(self.handle, C.byref(model), C.byref(key),
                                                u64(n_total), u64(first), u64(count), _ptr(obs),
                                                f64(eps), u64(cap), _ptr(n_accepted), _ptr(idx),
                                                _ptr(params), _ptr(rho)))
            return n_accepted, idx, params, rho
        nacc = u64()
        self._check(self.lib.vxb_abc_reject(self.handle, C.byref(model), C.byref(key),
                                            u64(n_total), u64(first), u64(count), _ptr(obs),
                                            f64(eps), u64(cap), C.byref(nacc), _ptr(idx),
                                            _ptr(params), _ptr(rho)))
        k = min(nacc.value, cap)
        if own:
            return nacc.value, idx[:k], params[:k], rho[:k]
        return nacc.value, idx, params, rho

    def sharded_abc_reject(self, comm, model, key, n_total, observed, eps, layout, packed_local,
                           packed_all=None):
        """SPMD config 1: this rank's shard into `packed_local`, one NCCL all-gather into
        `packed_all` (device uint8 buffers; comm None = one rank).  Asynchronous."""
        obs = np.ascontiguousarray(observed, dtype=np.float64)
        self._check(self.lib.vxb_sharded_abc_reject(
            self.handle, comm.handle if comm is not None else None, C.byref(model), C.byref(key),
            u64(n_total), _ptr(obs), f64(eps), C.byref(layout), _ptr(packed_local), _ptr(packed_all)))

    def sharded_select_epsilon(self, comm, rho_local, failed_local, first_row, q, cap=0,
                               block_local=None, blocks_all=None, precision=None, n_local=None):
        """SPMD config 0 selection over a sharded distance vector (histogram all-reduce):
        (epsilon, accepted rows of the whole vector).  Buffers: numpy or device tensors."""
        if isinstance(rho_local, np.ndarray):
            n_local = rho_local.size
            precision = A.VXB_F32 if rho_local.dtype == np.float32 else A.VXB_F64
        eps, nacc = f64(), u64()
        self._check(self.lib.vxb_sharded_select_epsilon(
            self.handle, comm.handle if comm is not None else None, i32(precision), _ptr(rho_local),
            _ptr(failed_local), u64(n_local), u64(first_row), f64(q), C.byref(eps), C.byref(nacc), u64(cap),
            _ptr(block_local), _ptr(blocks_all)))
        return eps.value, nacc.value

    # ---- p-values
    def ppp_pvalues(self, model, lam, log_norm, m_total, first, count, seed, ybar_obs,
                    want_ybar=False):
        lam = np.ascontiguousarray(lam, dtype=np.float64)
        ln = np.ascontiguousarray(log_norm, dtype=np.float64)
        counts = np.zeros(lam.size, dtype=np.uint64)
        pv = np.zeros(lam.size)
        yb = np.zeros((lam.size, count)) if want_ybar else None
        self._check(self.lib.vxb_ppp_pvalues(self.handle, C.byref(model), _ptr(lam), _ptr(ln),
                                             u32(lam.size), u64(m_total), u64(first), u64(count),
                                             u64(seed), f64(ybar_obs), _ptr(counts), _ptr(pv),
                                             _ptr(yb)))
        return counts, pv, yb

    # ---- SMC pieces
    def ess(self, log_w):
        lw = np.ascontiguousarray(log_w, dtype=np.float64)
        out = f64()
        self._check(self.lib.vxb_ess(self.handle, _ptr(lw), u64(lw.size), C.byref(out)))
        return out.value

    def logsumexp(self, x):
        x = np.ascontiguousarray(x, dtype=np.float64)
        out = f64()
        self._check(self.lib.vxb_logsumexp(self.handle, _ptr(x), u64(x.size), C.byref(out)))
        return out.value

    def resample_multinomial(self, log_w, particles, seed, stream_id):
        lw = np.ascontiguousarray(log_w, dtype=np.float64)
        p = np.ascontiguousarray(particles, dtype=np.float64)
        n, d = p.shape
        out = np.zeros_like(p)
        anc = np.zeros(n, dtype=np.uint64)
        self._check(self.lib.vxb_resample_multinomial(self.handle, u64(n), u32(d), _ptr(lw),
                                                      _ptr(p), u64(seed), u32(stream_id),
                                                      _ptr(out), _ptr(anc)))
        return out, anc

    def abcsmc_propose(self, model, seed, gen, first, count, theta_prev, cum_prev, chol, observed,
                       eps):
        tp = np.ascontiguousarray(theta_prev, dtype=np.float64)
        cp = np.ascontiguousarray(cum_prev, dtype=np.float64)
        ch = np.ascontiguousarray(chol, dtype=np.float64)
        obs = np.ascontiguousarray(observed, dtype=np.float64)
        th = np.zeros((count, model.dim))
        rho = np.zeros(count)
        flag = np.zeros(count, dtype=np.uint8)
        self._check(self.lib.vxb_abcsmc_propose(self.handle, C.byref(model), u64(seed), u32(gen),
                                                u64(first), u64(count), u64(tp.shape[0]), _ptr(tp),
                                                _ptr(cp), _ptr(ch), _ptr(obs), f64(eps), _ptr(th),
                                                _ptr(rho), _ptr(flag), None, u64(0)))
        return th, rho, flag

    def abcsmc_weights(self, theta_new, theta_prev, w_prev, chol, rng=A.VXB_RNG_REF):
        tn = np.ascontiguousarray(theta_new, dtype=np.float64)
        tp = np.ascontiguousarray(theta_prev, dtype=np.float64)
        wp = np.ascontiguousarray(w_prev, dtype=np.float64)
        ch = np.ascontiguousarray(chol, dtype=np.float64)
        out = np.zeros(tn.shape[0])
        self._check(self.lib.vxb_abcsmc_weights(self.handle, i32(rng), u32(tn.shape[1]), u64(tn.shape[0]),
                                                _ptr(tn), u64(tp.shape[0]), _ptr(tp), _ptr(wp),
                                                _ptr(ch), _ptr(out)))
        return out

    def abcsmc_run(self, model, cfg, observed):
        n, g, d = cfg.particles, cfg.generations, model.dim
        obs = np.ascontiguousarray(observed, dtype=np.float64)
        res = dict(theta=np.zeros((n, d)), weight=np.zeros(n), rho=np.zeros(n),
                   epsilon=np.zeros(g), ess=np.zeros(g), accept_rate=np.zeros(g),
                   proposals=np.zeros(g, dtype=np.uint64), mean=np.zeros((g, d)),
                   cov=np.zeros((g, d, d)))
        out = A.vxb_abcsmc_out(*[res[k].ctypes.data for k in
                                 ("theta", "weight", "rho", "epsilon", "ess", "accept_rate",
                                  "proposals", "mean", "cov")])
        self._check(self.lib.vxb_abcsmc_run(self.handle, C.byref(model), C.byref(cfg), _ptr(obs),
                                            C.byref(out)))
        return res

    def sharded_abcsmc_run(self, comm, model, cfg, observed):
        """The native SPMD ABC-SMC driver (every rank calls it; comm None = one rank):
        same dictionary and the same bits as abcsmc_run."""
        n, g, d = cfg.particles, cfg.generations, model.dim
        obs = np.ascontiguousarray(observed, dtype=np.float64)
        res = dict(theta=np.zeros((n, d)), weight=np.zeros(n), rho=np.zeros(n),
                   epsilon=np.zeros(g), ess=np.zeros(g), accept_rate=np.zeros(g),
                   proposals=np.zeros(g, dtype=np.uint64), mean=np.zeros((g, d)),
                   cov=np.zeros((g, d, d)))
        out = A.vxb_abcsmc_out(*[res[k].ctypes.data for k in
                                 ("theta", "weight", "rho", "epsilon", "ess", "accept_rate",
                                  "proposals", "mean", "cov")])
        self._check(self.lib.vxb_sharded_abcsmc_run(
            self.handle, comm.handle if comm is not None else None, C.byref(model), C.byref(cfg),
            _ptr(obs), C.byref(out)))
        return res

    def sharded_ppp_pvalues(self, comm, model, lam, log_norm, m_total, seed, ybar_obs):
        """SPMD config 2 (every rank calls it; comm None = one rank): counts / p-values of the whole job."""
        lam = np.ascontiguousarray(lam, dtype=np.float64)
        ln = np.ascontiguousarray(log_norm, dtype=np.float64)
        counts, pv = np.zeros(lam.size, dtype=np.uint64), np.zeros(lam.size)
        self._check(self.lib.vxb_sharded_ppp_pvalues(
            self.handle, comm.handle if comm is not None else None, C.byref(model), _ptr(lam), _ptr(ln),
            u32(lam.size), u64(m_total), u64(seed), f64(ybar_obs), _ptr(counts), _ptr(pv)))
        return counts, pv

    def sharded_mlmc_tauleap(self, comm, model, cfg):
        """SPMD config 4 (every rank calls it; comm None = one rank): same dictionary as mlmc_tauleap."""
        L = cfg.levels
        res = dict(level_mean=np.zeros(L), level_var=np.zeros(L), level_cost=np.zeros(L))
        out = A.vxb_mlmc_out(res["level_mean"].ctypes.data, res["level_var"].ctypes.data,
                             res["level_cost"].ctypes.data, 0.0, 0.0)
        self._check(self.lib.vxb_sharded_mlmc_tauleap(
            self.handle, comm.handle if comm is not None else None, C.byref(model), C.byref(cfg), C.byref(out)))
        res["estimate"], res["std_error"] = out.estimate, out.std_error
        return res

    # ---- population statistics (canonical order) for the multi-GPU host
    def weighted_moments(self, theta, w, n=None, dim=None):
        """theta (n x dim), w (n): numpy arrays or device tensors."""
        if n is None:
            n, dim = int(theta.shape[0]), int(theta.shape[1])
        mean, cov, s2 = np.zeros(dim), np.zeros((dim, dim)), f64()
        self._check(self.lib.vxb_weighted_moments(self.handle, _ptr(theta), _ptr(w), u64(n),
                                                  u32(dim), _ptr(mean), _ptr(cov), C.byref(s2)))
        return mean, cov, s2.value

    def canon_cumsum(self, w, out=None):
        n = int(w.shape[0])
        if out is None:
            out = np.zeros(n)
        self._check(self.lib.vxb_canon_cumsum(self.handle, _ptr(w), u64(n), _ptr(out)))
        return out

    def canon_chunk_sums(self, v, out=None):
        n = int(v.shape[0])
        if out is None:
            out = np.zeros((n + 255) // 256)
        self._check(self.lib.vxb_canon_chunk_sums(self.handle, _ptr(v), u64(n), _ptr(out)))
        return out

    def divide(self, v, divisor):
        """In place: v[i] <- v[i] / divisor (IEEE division on the device)."""
        self._check(self.lib.vxb_divide(self.handle, _ptr(v), u64(int(v.shape[0])), f64(divisor)))
        return v

    def quantile(self, values, level):
        out = f64()
        self._check(self.lib.vxb_quantile(self.handle, _ptr(values), u64(int(values.shape[0])),
                                          f64(level), C.byref(out)))
        return out.value

    # ---- likelihood-annealed SMC / weak-informativity test
    @staticmethod
    def _design(dose, group_size):
        return (np.ascontiguousarray(dose, dtype=np.float64),
                np.ascontiguousarray(group_size, dtype=np.uint32))

    def bioassay_log_likelihood(self, beta, dose, group_size, deaths):
        b = np.ascontiguousarray(beta, dtype=np.float64).reshape(-1, 2)
        d, g = self._design(dose, group_size)
        y = np.ascontiguousarray(deaths, dtype=np.uint32)
        out = np.zeros(b.shape[0])
        self._check(self.lib.vxb_bioassay_log_likelihood(self.handle, _ptr(b), u64(b.shape[0]),
                                                         u32(d.size), _ptr(d), _ptr(g), _ptr(y),
                                                         _ptr(out)))
        return out

    def bioassay_sample(self, lam, seeds, dose, group_size):
        lam = np.ascontiguousarray(lam, dtype=np.float64).reshape(-1, 2)
        seeds = np.ascontiguousarray(seeds, dtype=np.uint64)
        d, g = self._design(dose, group_size)
        theta = np.zeros_like(lam)
        deaths = np.zeros((lam.shape[0], d.size), dtype=np.uint32)
        self._check(self.lib.vxb_bioassay_sample(self.handle, u64(lam.shape[0]), u32(d.size),
                                                 _ptr(d), _ptr(g), _ptr(lam), _ptr(seeds),
                                                 _ptr(theta), _ptr(deaths)))
        return theta, deaths

    def smc_bioassay(self, dose, group_size, deaths, lam, seeds, particles, block_width=4, c=0.01,
                     scale=1.6828427124746189, trace_rows=0):
        """Batch of independent annealed-SMC evidence estimates (one CTA per run)."""
        d, g = self._design(dose, group_size)
        y = np.ascontiguousarray(deaths, dtype=np.uint32).reshape(-1, d.size)
        lam = np.ascontiguousarray(lam, dtype=np.float64).reshape(-1, 2)
        seeds = np.ascontiguousarray(seeds, dtype=np.uint64)
        n = y.shape[0]
        ev, it, st = np.zeros(n), np.zeros(n, dtype=np.uint32), np.zeros(n, dtype=np.uint8)
        tr = np.zeros((n, trace_rows, 6)) if trace_rows else None
        self._check(self.lib.vxb_smc_bioassay(self.handle, u64(n), u32(d.size), _ptr(d), _ptr(g),
                                              _ptr(y), _ptr(lam), _ptr(seeds), u64(particles),
                                              u64(block_width), f64(c), f64(scale), _ptr(ev),
                                              _ptr(it), _ptr(st), _ptr(tr), u32(trace_rows)))
        return dict(log_evidence=ev, iterations=it, status=st, trace=tr)

    def smc_bioassay_ensemble(self, dose, group_size, deaths, lam, seed, particles, block_width=4,
                              c=0.01, scale=1.6828427124746189, trace_rows=16, esjd_scales=None):
        """One run with its final ensemble (the reference's SmcResult).  esjd_scales: the
        scale grid of SmcConfig::esjd = true (None: fixed-scale sampler)."""
        d, g = self._design(dose, group_size)
        y = np.ascontiguousarray(deaths, dtype=np.uint32)
        lam = np.ascontiguousarray(lam, dtype=np.float64)
        ev, it = f64(), u32()
        ens = np.zeros((5, particles))
        tr = np.zeros((trace_rows, 6))
        sc = None if esjd_scales is None else np.ascontiguousarray(esjd_scales, dtype=np.float64)
        self._check(self.lib.vxb_smc_bioassay_ensemble(
            self.handle, u32(d.size), _ptr(d), _ptr(g), _ptr(y), _ptr(lam), u64(seed), u64(particles),
            u64(block_width), f64(c), f64(scale), C.byref(ev), C.byref(it), _ptr(ens), _ptr(tr),
            u32(trace_rows), _ptr(sc), u32(0 if sc is None else sc.size)))
        return dict(log_evidence=ev.value, iterations=it.value, particles=ens[:2].T.copy(),
                    log_weights=ens[2], log_liks=ens[3], log_priors=ens[4], trace=tr[:it.value])

    def weak_info_test(self, cfg, want_evidence=False):
        k = cfg.hyper_count + 1
        lam, gamma = np.zeros((k, 2)), np.zeros(k)
        weakly, completed = np.zeros(k, dtype=np.uint8), np.zeros(k, dtype=np.uint64)
        ev = np.zeros((k, cfg.datasets, 2)) if want_evidence else None
        self._check(self.lib.vxb_weak_info_test(self.handle, C.byref(cfg), _ptr(lam), _ptr(gamma),
                                                _ptr(weakly), _ptr(completed), _ptr(ev)))
        return dict(lambda_=lam, gamma=gamma, weakly=weakly, completed=completed, evidence=ev)

    def weak_info_lambdas(self, cfg):
        lam = np.zeros((cfg.hyper_count + 1, 2))
        self._check(self.lib.vxb_weak_info_lambdas(self.handle, C.byref(cfg), _ptr(lam)))
        return lam

    def weak_info_evidence(self, cfg, lam, first_row, n_rows, out=None):
        """Evidences of rows [first_row, first_row + n_rows): n_rows x N x 2."""
        lam = np.ascontiguousarray(lam, dtype=np.float64)
        if out is None:
            out = np.zeros((n_rows, cfg.datasets, 2))
        self._check(self.lib.vxb_weak_info_evidence(self.handle, C.byref(cfg), _ptr(lam),
                                                    u64(first_row), u64(n_rows), _ptr(out)))
        return out

    # ---- tau-leap
    def mlmc_level(self, model, cfg, level, first, count, want_y=False):
        sums = np.zeros(4, dtype=np.int64)
        y = np.zeros(count, dtype=np.int32) if want_y else None
        self._check(self.lib.vxb_mlmc_level(self.handle, C.byref(model), C.byref(cfg), u32(level),
                                            u64(first), u64(count), _ptr(sums), _ptr(y)))
        return sums, y

    def mlmc_tauleap(self, model, cfg):
        L = cfg.levels
        res = dict(level_mean=np.zeros(L), level_var=np.zeros(L), level_cost=np.zeros(L))
        out = A.vxb_mlmc_out(res["level_mean"].ctypes.data, res["level_var"].ctypes.data,
                             res["level_cost"].ctypes.data, 0.0, 0.0)
        self._check(self.lib.vxb_mlmc_tauleap(self.handle, C.byref(model), C.byref(cfg),
                                              C.byref(out)))
        res["estimate"], res["std_error"] = out.estimate, out.std_error
        return res
