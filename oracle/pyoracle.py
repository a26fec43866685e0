"""ctypes front-ends of the two CPU checkers.  TEST INFRASTRUCTURE ONLY.

* ``Oracle`` -> oracle/libvxb_oracle.so  (vxb_oracle.cpp, own CPU restatement)
* ``Ref``    -> oracle/_ref/libvxb_ref.so (ref_driver.cpp + the unmodified
  reference translation units; present only where oracle/Makefile could build
  it or where the prebuilt file travelled)

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline / --impl
reference) may import this module; the product package never does.
"""
import ctypes as C
import os
import subprocess

import numpy as np

from paper_1902_09046_b200 import _abi as A

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "libvxb_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libvxb_ref.so")

u64, u32, f64, i32 = C.c_uint64, C.c_uint32, C.c_double, C.c_int32
P = C.c_void_p


def build(verbose=False):
    """Compile the checkers (oracle always; _ref when /root/reference exists)."""
    out = subprocess.run(["make", "-C", HERE, "all"], capture_output=True, text=True)
    if verbose or out.returncode:
        print(out.stdout, out.stderr)
    if out.returncode:
        raise RuntimeError("oracle build failed")


def _ptr(a):
    if a is None:
        return None
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(P)


def _f64(x):
    return np.ascontiguousarray(x, dtype=np.float64)


class OracleError(RuntimeError):
    def __init__(self, text):
        super().__init__(text)
        self.code = text.split(":", 1)[0]


class _Base:
    prefix = ""

    def _check(self, rc):
        if rc != 0:
            fn = getattr(self.lib, self.prefix + "last_error")
            fn.restype = C.c_char_p
            raise OracleError(fn().decode())

    def _call(self, name, *args):
        self._check(getattr(self.lib, self.prefix + name)(*args))

    # ---- likelihood-annealed SMC / weak-informativity test
    @staticmethod
    def _design(dose, group_size, deaths=None):
        d = _f64(dose)
        g = np.ascontiguousarray(group_size, dtype=np.uint32)
        y = None if deaths is None else np.ascontiguousarray(deaths, dtype=np.uint32)
        return d, g, y

    def bioassay_ll(self, beta, dose, group_size, deaths):
        b = _f64(beta).reshape(-1, 2)
        d, g, y = self._design(dose, group_size, deaths)
        out = np.zeros(b.shape[0])
        self._call("bioassay_ll", _ptr(b), u64(b.shape[0]), _ptr(d), _ptr(g), _ptr(y), u32(d.size),
                   _ptr(out))
        return out

    def bioassay_sample(self, lambda1, lambda2, dose, group_size, seed):
        d, g, _ = self._design(dose, group_size)
        theta, deaths = np.zeros(2), np.zeros(d.size, dtype=np.uint32)
        self._call("bioassay_sample", f64(lambda1), f64(lambda2), _ptr(d), _ptr(g), u32(d.size),
                   u64(seed), _ptr(theta), _ptr(deaths))
        return theta, deaths

    def weak_info_test(self, hyper_count, datasets, particles, alpha=0.05, c=0.01,
                       scale=1.6828427124746189, workers=1, block_width=4, seed=0,
                       redraw_base=False, csv_path=None):
        k = hyper_count + 1
        lam, gamma = np.zeros((k, 2)), np.zeros(k)
        weakly, completed = np.zeros(k, dtype=np.uint8), np.zeros(k, dtype=np.uint64)
        self._call("weak_info_test", u64(hyper_count), u64(datasets), u64(particles), f64(alpha),
                   f64(c), f64(scale), u64(workers), u64(block_width), u64(seed),
                   C.c_int(1 if redraw_base else 0), _ptr(lam), _ptr(gamma), _ptr(weakly),
                   _ptr(completed), C.c_char_p(os.fsencode(csv_path)) if csv_path else None)
        return dict(lambda_=lam, gamma=gamma, weakly=weakly, completed=completed)

    # ---- TB Gillespie ABC
    def tb_simulate(self, theta, initial, horizon, target, seed, sid, pos, block_width=4):
        th = _f64(theta)
        out, after, n = np.zeros(5), u64(), u64()
        counts = np.zeros(1 << 16)
        self._call("tb_simulate", _ptr(th), u64(initial), f64(horizon), f64(target), u64(seed),
                   self._sid(sid), u64(pos), u64(block_width), _ptr(out), C.byref(after), _ptr(counts),
                   u64(counts.size), C.byref(n))
        return dict(time=out[0], total=out[1], genotypes=int(out[2]), summaries=out[3:5].copy(),
                    pos_after=after.value, counts=counts[:n.value].copy())

    def tb_abc_particle(self, initial, horizon, target, first, count, seed, observed, threads=None):
        obs = _f64(observed)
        params, summ = np.zeros((count, 3)), np.zeros((count, 2))
        rho, failed = np.zeros(count), np.zeros(count, dtype=np.uint8)
        self._call("tb_abc_particle", u64(initial), f64(horizon), f64(target), u64(first), u64(count),
                   u64(seed), _ptr(obs), _ptr(params), _ptr(summ), _ptr(rho), _ptr(failed),
                   C.c_uint(threads or os.cpu_count() or 1))
        return params, summ, rho, failed

    def tb_observed(self, initial, horizon, target, seed, block_width=4):
        out = np.zeros(2)
        self._call("tb_observed", u64(initial), f64(horizon), f64(target), u64(seed), u64(block_width),
                   _ptr(out))
        return out


class Oracle(_Base):
    _sid = staticmethod(u64)
    prefix = "vxo_"

    def __init__(self, threads=None):
        if not os.path.exists(ORACLE_SO):
            build()
        self.lib = C.CDLL(ORACLE_SO)
        self.threads = threads or os.cpu_count() or 1
        self.lib.vxo_splitmix64.restype = u64
        self.lib.vxo_splitmix64.argtypes = [u64]
        self.lib.vxo_derive_seed.restype = u64
        self.lib.vxo_derive_seed.argtypes = [u64, P, C.c_size_t]
        self.lib.vxo_discrepancy.restype = f64
        self.lib.vxo_canon_sum.restype = f64

    # ---- substrate
    def smc_bioassay(self, dose, group_size, deaths, lambda1, lambda2, particles, block_width, c,
                     scale, seed, want_trace=False):
        """trace columns: temperature, ess, steps (R_n), pilot acceptance."""
        d, g, y = self._design(dose, group_size, deaths)
        ev, it = f64(), u64()
        tr = np.zeros((1000, 4)) if want_trace else None
        self._call("smc_bioassay", _ptr(d), _ptr(g), _ptr(y), u32(d.size), f64(lambda1),
                   f64(lambda2), u64(particles), u64(block_width), f64(c), f64(scale), u64(seed),
                   C.byref(ev), C.byref(it), _ptr(tr), u64(1000))
        if not want_trace:
            return ev.value, it.value
        return ev.value, it.value, tr[:it.value]

    def smc_bioassay_ensemble(self, dose, group_size, deaths, lambda1, lambda2, particles,
                              block_width, c, scale, seed, esjd_scales=None):
        """SmcResult of one run; trace columns: temperature, ess, steps, p_acc, log evidence,
        proposal scale.  esjd_scales: the scale grid of the ESJD adaptation (None: fixed scale)."""
        d, g, y = self._design(dose, group_size, deaths)
        ev, it = f64(), u64()
        ens, tr = np.zeros((5, particles)), np.zeros((1000, 6))
        sc = None if esjd_scales is None else np.ascontiguousarray(esjd_scales, dtype=np.float64)
        self._call("smc_bioassay_ensemble", _ptr(d), _ptr(g), _ptr(y), u32(d.size), f64(lambda1),
                   f64(lambda2), u64(particles), u64(block_width), f64(c), f64(scale), u64(seed),
                   C.byref(ev), C.byref(it), _ptr(ens), _ptr(tr), u64(1000), _ptr(sc),
                   u64(0 if sc is None else sc.size))
        return dict(log_evidence=ev.value, iterations=it.value, particles=ens[:2].T.copy(),
                    log_weights=ens[2], log_liks=ens[3], log_priors=ens[4], trace=tr[:it.value])

    def splitmix64(self, z):
        return int(self.lib.vxo_splitmix64(z))

    def derive_seed(self, seed, path):
        a = np.asarray(path, dtype=np.uint64)
        return int(self.lib.vxo_derive_seed(seed, _ptr(a), len(a)))

    def stream_u64(self, seed, sid, pos, n):
        out = np.zeros(n, dtype=np.uint64)
        self._call("stream_u64", u64(seed), u64(sid), u64(pos), u64(n), _ptr(out))
        return out

    def fill_uniform(self, seed, sid, pos, n, a=0.0, b=1.0):
        out = np.zeros(n)
        self._call("fill_uniform", u64(seed), u64(sid), u64(pos), u64(n), f64(a), f64(b), _ptr(out))
        return out

    def fill_gaussian(self, seed, sid, pos, n, mu=0.0, sigma=1.0):
        out = np.zeros(n)
        self._call("fill_gaussian", u64(seed), u64(sid), u64(pos), u64(n), f64(mu), f64(sigma),
                   _ptr(out))
        return out

    def fastmath(self, fn, x, y=None):
        x = _f64(x)
        y = _f64(y) if y is not None else np.zeros_like(x)
        out = np.zeros_like(x)
        self._call("fastmath", i32(fn), _ptr(x), _ptr(y), u64(x.size), _ptr(out))
        return out

    def quantile(self, sample, level):
        s = _f64(sample)
        out = f64()
        self._call("quantile", _ptr(s), u64(s.size), f64(level), C.byref(out))
        return out.value

    def logsumexp(self, x):
        x = _f64(x)
        out = f64()
        self._call("logsumexp", _ptr(x), u64(x.size), C.byref(out))
        return out.value

    def sample_covariance(self, data):
        d = _f64(data)
        cov = np.zeros((d.shape[1], d.shape[1]))
        self._call("sample_covariance", _ptr(d), u64(d.shape[0]), u64(d.shape[1]), _ptr(cov))
        return cov

    def cholesky(self, a):
        a = _f64(a).copy()
        rc = self.lib.vxo_cholesky(_ptr(a), u64(a.shape[0]))
        return rc == 0, a

    def partition(self, total, workers, width):
        r = np.zeros((workers, 2), dtype=np.uint64)
        self._call("partition", u64(total), u64(workers), u64(width), _ptr(r))
        return r

    def discrepancy(self, sim, obs):
        s, o = _f64(sim), _f64(obs)
        return float(self.lib.vxo_discrepancy(_ptr(s), _ptr(o), u64(s.size)))

    # ---- ABC
    def abc_prior_predictive(self, model, key, n_total, first, count, observed, noise=None,
                             want_summaries=True, threads=None):
        d, sd = model.dim, model.summary_dim
        obs = _f64(observed)
        params = np.zeros((count, d))
        summ = np.zeros((count, sd)) if want_summaries else None
        rho = np.zeros(count)
        failed = np.zeros(count, dtype=np.uint8)
        nz = _f64(noise) if noise is not None else None
        self._call("abc_prior_predictive", C.byref(model), C.byref(key), u64(n_total), u64(first),
                   u64(count), _ptr(obs), _ptr(params), _ptr(summ), _ptr(rho), _ptr(failed),
                   _ptr(nz), C.c_uint(threads or self.threads))
        return params, summ, rho, failed

    def simulate_at(self, model, theta, seed, sid, pos):
        th = _f64(theta)
        out = np.zeros(model.summary_dim)
        self._call("simulate_at", C.byref(model), _ptr(th), u64(seed), u64(sid), u64(pos), _ptr(out))
        return out

    def select_epsilon(self, rho, failed, q):
        rho = _f64(rho)
        n = rho.size
        f = np.ascontiguousarray(failed, dtype=np.uint8) if failed is not None else None
        eps, nacc = f64(), u64()
        idx = np.zeros(n, dtype=np.uint64)
        self._call("select_epsilon", _ptr(rho), _ptr(f), u64(n), f64(q), C.byref(eps), u64(n),
                   C.byref(nacc), _ptr(idx))
        return eps.value, idx[: nacc.value].copy()

    # ---- p-values
    def ppp_pvalues(self, model, lam, log_norm, m_total, first, count, seed, ybar_obs,
                    want_ybar=False, threads=None):
        lam, ln = _f64(lam), _f64(log_norm)
        counts = np.zeros(lam.size, dtype=np.uint64)
        pv = np.zeros(lam.size)
        yb = np.zeros((lam.size, count)) if want_ybar else None
        self._call("ppp_pvalues", C.byref(model), _ptr(lam), _ptr(ln), u32(lam.size), u64(m_total),
                   u64(first), u64(count), u64(seed), f64(ybar_obs), _ptr(counts), _ptr(pv),
                   _ptr(yb), C.c_uint(threads or self.threads))
        return counts, pv, yb

    def estimate_pvalues(self, base, k):
        b, k = _f64(base), _f64(k)
        out = np.zeros(b.size)
        self._call("estimate_pvalues", _ptr(b), u64(b.size), _ptr(k), u64(k.size), _ptr(out))
        return out

    def compute_cutoff(self, p, alpha):
        p = _f64(p)
        out = f64()
        self._call("compute_cutoff", _ptr(p), u64(p.size), f64(alpha), C.byref(out))
        return out.value

    # ---- the restatement of the host libm's exp (pins csrc/vxb_libmexp.cuh)
    def exp_restated(self, x, plain_build=False):
        """(restated exp, live std::exp) of every x.  plain_build: the library's build
        without FMA contraction (what its ifunc selects on CPUs without FMA + AVX2)."""
        x = _f64(x)
        out, live = np.zeros_like(x), np.zeros_like(x)
        self._call("exp_restated", _ptr(x), u64(x.size), _ptr(out), _ptr(live), i32(1 if plain_build else 0))
        return out, live

    def exp_restated_sweep(self, seed, n, lo, hi, threads=None, plain_build=False):
        """Number of pseudo-random arguments in [lo, hi) on which the restatement and
        the live std::exp differ bitwise, and the first such argument (NaN if none)."""
        m, first = u64(), f64(float("nan"))
        self._call("exp_restated_sweep", u64(seed), u64(n), f64(lo), f64(hi),
                   C.c_uint(threads or (os.cpu_count() or 1)), C.byref(m), C.byref(first),
                   i32(1 if plain_build else 0))
        return m.value, first.value

    # ---- SMC pieces
    def ess(self, lw):
        lw = _f64(lw)
        out = f64()
        self._call("ess", _ptr(lw), u64(lw.size), C.byref(out))
        return out.value

    def resample_multinomial(self, log_w, particles, seed, sid):
        lw, p = _f64(log_w), _f64(particles)
        n, d = p.shape
        out = np.zeros_like(p)
        anc = np.zeros(n, dtype=np.uint64)
        self._call("resample_multinomial", u64(n), u32(d), _ptr(lw), _ptr(p), u64(seed), u64(sid),
                   _ptr(out), _ptr(anc))
        return out, anc

    def weighted_moments(self, theta, w):
        th, w = _f64(theta), _f64(w)
        n, d = th.shape
        mean, cov, s2 = np.zeros(d), np.zeros((d, d)), f64()
        self._call("weighted_moments", _ptr(th), _ptr(w), u64(n), u32(d), _ptr(mean), _ptr(cov),
                   C.byref(s2))
        return mean, cov, s2.value

    def canon_cumsum(self, w):
        w = _f64(w)
        out = np.zeros_like(w)
        self._call("canon_cumsum", _ptr(w), u64(w.size), _ptr(out))
        return out

    def canon_sum(self, w):
        w = _f64(w)
        return float(self.lib.vxo_canon_sum(_ptr(w), u64(w.size)))

    def make_kernel(self, cov, scale, jitter=1e-10):
        cov = _f64(cov)
        chol = np.zeros_like(cov)
        self._call("make_kernel", _ptr(cov), u32(cov.shape[0]), f64(scale), f64(jitter), _ptr(chol))
        return chol

    def abcsmc_propose(self, model, seed, gen, first, count, theta_prev, cum_prev, chol, observed,
                       eps, threads=None):
        tp, cp, ch, obs = _f64(theta_prev), _f64(cum_prev), _f64(chol), _f64(observed)
        th = np.zeros((count, 3))
        rho = np.zeros(count)
        flag = np.zeros(count, dtype=np.uint8)
        self._call("abcsmc_propose", C.byref(model), u64(seed), u32(gen), u64(first), u64(count),
                   u64(tp.shape[0]), _ptr(tp), _ptr(cp), _ptr(ch), _ptr(obs), f64(eps), _ptr(th),
                   _ptr(rho), _ptr(flag), C.c_uint(threads or self.threads))
        return th, rho, flag

    def abcsmc_weights(self, theta_new, theta_prev, w_prev, chol, threads=None):
        tn, tp, wp, ch = _f64(theta_new), _f64(theta_prev), _f64(w_prev), _f64(chol)
        out = np.zeros(tn.shape[0])
        self._call("abcsmc_weights", u32(tn.shape[1]), u64(tn.shape[0]), _ptr(tn), u64(tp.shape[0]),
                   _ptr(tp), _ptr(wp), _ptr(ch), _ptr(out), C.c_uint(threads or self.threads))
        return out

    def abcsmc_run(self, model, cfg, observed, threads=None):
        n, g, d = cfg.particles, cfg.generations, 3
        obs = _f64(observed)
        res = dict(theta=np.zeros((n, d)), weight=np.zeros(n), rho=np.zeros(n),
                   epsilon=np.zeros(g), ess=np.zeros(g), accept_rate=np.zeros(g),
                   proposals=np.zeros(g, dtype=np.uint64), mean=np.zeros((g, d)),
                   cov=np.zeros((g, d, d)))
        out = A.vxb_abcsmc_out(*[res[k].ctypes.data for k in
                                 ("theta", "weight", "rho", "epsilon", "ess", "accept_rate",
                                  "proposals", "mean", "cov")])
        self._call("abcsmc_run", C.byref(model), C.byref(cfg), _ptr(obs), C.byref(out),
                   C.c_uint(threads or self.threads))
        return res

    # ---- tau-leap
    def mlmc_level(self, model, cfg, level, first, count, want_y=False, threads=None):
        sums = np.zeros(4, dtype=np.int64)
        y = np.zeros(count, dtype=np.int32) if want_y else None
        self._call("mlmc_level", C.byref(model), C.byref(cfg), u32(level), u64(first), u64(count),
                   _ptr(sums), _ptr(y), C.c_uint(threads or self.threads))
        return sums, y

    def mlmc_tauleap(self, model, cfg, threads=None):
        L = cfg.levels
        res = dict(level_mean=np.zeros(L), level_var=np.zeros(L), level_cost=np.zeros(L))
        out = A.vxb_mlmc_out(res["level_mean"].ctypes.data, res["level_var"].ctypes.data,
                             res["level_cost"].ctypes.data, 0.0, 0.0)
        self._call("mlmc_tauleap", C.byref(model), C.byref(cfg), C.byref(out),
                   C.c_uint(threads or self.threads))
        res["estimate"], res["std_error"] = out.estimate, out.std_error
        return res

    def mm_gillespie(self, model, t_end, paths, seed, threads=None):
        mean, var = f64(), f64()
        self._call("mm_gillespie", C.byref(model), f64(t_end), u64(paths), u64(seed),
                   C.byref(mean), C.byref(var), C.c_uint(threads or self.threads))
        return mean.value, var.value


class Ref(_Base):
    _sid = staticmethod(u32)
    """The unmodified reference library behind ref_driver.cpp."""
    prefix = "ref_"

    @staticmethod
    def available():
        return os.path.exists(REF_SO)

    def __init__(self):
        if not os.path.exists(REF_SO):
            raise FileNotFoundError(REF_SO)
        self.lib = C.CDLL(REF_SO)
        self.lib.ref_splitmix64.restype = u64
        self.lib.ref_splitmix64.argtypes = [u64]
        self.lib.ref_derive_seed.restype = u64
        self.lib.ref_derive_seed.argtypes = [u64, P, C.c_size_t]
        self.lib.ref_discrepancy.restype = f64

    def smc_bioassay(self, dose, group_size, deaths, lambda1, lambda2, particles, block_width, c,
                     scale, seed, want_trace=False):
        d, g, y = self._design(dose, group_size, deaths)
        ev, it = f64(), u64()
        buf = C.create_string_buffer(1 << 16) if want_trace else None
        self._call("smc_bioassay", _ptr(d), _ptr(g), _ptr(y), u32(d.size), f64(lambda1),
                   f64(lambda2), u64(particles), u64(block_width), f64(c), f64(scale), u64(seed),
                   C.byref(ev), C.byref(it), buf, u64(len(buf) if buf else 0))
        if not want_trace:
            return ev.value, it.value
        rows = [ln.split(",") for ln in buf.value.decode().strip().splitlines()[1:]]
        full = np.array([[float(x) for x in r] for r in rows])  # n,t_n,ess,log_evidence,R_n,p_acc,h
        return ev.value, it.value, full[:, [1, 2, 4, 5]]       # temperature, ess, steps, p_acc

    def smc_bioassay_ensemble(self, dose, group_size, deaths, lambda1, lambda2, particles,
                              block_width, c, scale, seed, esjd_scales=None):
        d, g, y = self._design(dose, group_size, deaths)
        ev, it = f64(), u64()
        ens = np.zeros((5, particles))
        buf = C.create_string_buffer(1 << 16)
        sc = None if esjd_scales is None else np.ascontiguousarray(esjd_scales, dtype=np.float64)
        self._call("smc_bioassay_ensemble", _ptr(d), _ptr(g), _ptr(y), u32(d.size), f64(lambda1),
                   f64(lambda2), u64(particles), u64(block_width), f64(c), f64(scale), u64(seed),
                   C.byref(ev), C.byref(it), _ptr(ens), buf, u64(len(buf)), _ptr(sc),
                   u64(0 if sc is None else sc.size))
        rows = [ln.split(",") for ln in buf.value.decode().strip().splitlines()[1:]]
        full = np.array([[float(x) for x in r] for r in rows])  # n,t_n,ess,log_evidence,R_n,p_acc,h
        return dict(log_evidence=ev.value, iterations=it.value, particles=ens[:2].T.copy(),
                    log_weights=ens[2], log_liks=ens[3], log_priors=ens[4],
                    trace=full[:, [1, 2, 4, 5, 3, 6]], trace_text=buf.value.decode())

    def splitmix64(self, z):
        return int(self.lib.ref_splitmix64(z))

    def derive_seed(self, seed, path):
        a = np.asarray(path, dtype=np.uint64)
        return int(self.lib.ref_derive_seed(seed, _ptr(a), len(a)))

    def stream_u64(self, seed, sid, pos, n):
        out = np.zeros(n, dtype=np.uint64)
        self._call("stream_u64", u64(seed), u32(sid), u64(pos), u64(n), _ptr(out))
        return out

    def fill_uniform(self, seed, sid, pos, n, a=0.0, b=1.0):
        out = np.zeros(n)
        self._call("fill_uniform", u64(seed), u32(sid), u64(pos), u64(n), f64(a), f64(b),
                   _ptr(out), None)
        return out

    def fill_gaussian(self, seed, sid, pos, n, mu=0.0, sigma=1.0):
        out = np.zeros(n)
        self._call("fill_gaussian", u64(seed), u32(sid), u64(pos), u64(n), f64(mu), f64(sigma),
                   _ptr(out))
        return out

    def fastmath(self, fn, x, y=None):
        x = _f64(x)
        y = _f64(y) if y is not None else np.zeros_like(x)
        out = np.zeros_like(x)
        self._call("fastmath", i32(fn), _ptr(x), _ptr(y), u64(x.size), _ptr(out))
        return out

    def quantile(self, sample, level):
        s = _f64(sample)
        out = f64()
        self._call("quantile", _ptr(s), u64(s.size), f64(level), C.byref(out))
        return out.value

    def logsumexp(self, x):
        x = _f64(x)
        out = f64()
        self._call("logsumexp", _ptr(x), u64(x.size), C.byref(out))
        return out.value

    def sample_covariance(self, data):
        d = _f64(data)
        cov = np.zeros((d.shape[1], d.shape[1]))
        self._call("sample_covariance", _ptr(d), u64(d.shape[0]), u64(d.shape[1]), _ptr(cov))
        return cov

    def cholesky(self, a):
        a = _f64(a).copy()
        rc = self.lib.ref_cholesky(_ptr(a), u64(a.shape[0]))
        return rc == 0, a

    def partition(self, total, workers, width):
        r = np.zeros((workers, 2), dtype=np.uint64)
        self._call("partition", u64(total), u64(workers), u64(width), _ptr(r))
        return r

    def discrepancy(self, sim, obs):
        s, o = _f64(sim), _f64(obs)
        return float(self.lib.ref_discrepancy(_ptr(s), _ptr(o), u64(s.size)))

    def logistic_abc(self, model, n, workers, block_width, seed, observed):
        d, sd = model.dim, model.summary_dim
        obs = _f64(observed)
        params, summ = np.zeros((n, d)), np.zeros((n, sd))
        rho, failed = np.zeros(n), np.zeros(n, dtype=np.uint8)
        self._call("logistic_abc", C.byref(model), u64(n), u64(workers), u64(block_width),
                   u64(seed), _ptr(obs), _ptr(params), _ptr(summ), _ptr(rho), _ptr(failed))
        return params, summ, rho, failed

    def logistic_abc_csv(self, model, n, workers, block_width, seed, observed, path):
        """abc::write_csv of the reference's own run_prior_predictive result."""
        obs = _f64(observed)
        self._call("logistic_abc_csv", C.byref(model), u64(n), u64(workers), u64(block_width),
                   u64(seed), _ptr(obs), C.c_char_p(os.fsencode(path)))

    def bench_csv(self, records, path):
        """bench::write_csv of (experiment, mode, threads, width, replicate, runtime, failed)."""
        cols = list(zip(*records))
        e, m = np.array(cols[0], dtype=np.int32), np.array(cols[1], dtype=np.int32)
        t, w, r = (np.array(cols[k], dtype=np.uint64) for k in (2, 3, 4))
        rt, f = np.array(cols[5], dtype=np.float64), np.array(cols[6], dtype=np.uint8)
        self._call("bench_csv", u64(len(records)), _ptr(e), _ptr(m), _ptr(t), _ptr(w), _ptr(r),
                   _ptr(rt), _ptr(f), C.c_char_p(os.fsencode(path)))

    def amdahl_bound(self, serial, parallel, units):
        out = f64()
        self._call("amdahl_bound", f64(serial), f64(parallel), f64(units), C.byref(out))
        return out.value

    def logistic_abc_particle(self, model, first, count, seed, observed, threads=None,
                              want_summaries=True):
        d, sd = model.dim, model.summary_dim
        obs = _f64(observed)
        params = np.zeros((count, d))
        summ = np.zeros((count, sd)) if want_summaries else None
        rho, failed = np.zeros(count), np.zeros(count, dtype=np.uint8)
        self._call("logistic_abc_particle", C.byref(model), u64(first), u64(count), u64(seed),
                   _ptr(obs), _ptr(params), _ptr(summ), _ptr(rho), _ptr(failed),
                   C.c_uint(threads or os.cpu_count() or 1))
        return params, summ, rho, failed

    def logistic_simulate(self, model, theta, seed, sid, pos):
        th = _f64(theta)
        out = np.zeros(model.summary_dim)
        self._call("logistic_simulate", C.byref(model), _ptr(th), u64(seed), u32(sid), u64(pos),
                   _ptr(out))
        return out

    def select_epsilon(self, rho, failed, q):
        rho = _f64(rho)
        n = rho.size
        f = np.ascontiguousarray(failed, dtype=np.uint8) if failed is not None else None
        eps, nacc = f64(), u64()
        idx = np.zeros(n, dtype=np.uint64)
        self._call("select_epsilon", _ptr(rho), _ptr(f), u64(n), f64(q), C.byref(eps), u64(n),
                   C.byref(nacc), _ptr(idx))
        return eps.value, idx[: nacc.value].copy()

    def toggle_abc(self, steps, cells, n, workers, width, seed):
        obs = np.zeros(19)
        params, summ = np.zeros((n, 7)), np.zeros((n, 19))
        rho, failed = np.zeros(n), np.zeros(n, dtype=np.uint8)
        self._call("toggle_abc", u64(steps), u64(cells), u64(n), u64(workers), u64(width),
                   u64(seed), _ptr(obs), _ptr(params), _ptr(summ), _ptr(rho), _ptr(failed))
        return obs, params, summ, rho, failed

    def toggle_simulate(self, theta7, steps, cells, seed, sid, pos, width):
        th = _f64(theta7)
        y = np.zeros(cells)
        end = u64()
        self._call("toggle_simulate", _ptr(th), u64(steps), u64(cells), u64(seed), u32(sid),
                   u64(pos), u64(width), _ptr(y), C.byref(end))
        return y, end.value

    def estimate_pvalues(self, base, k):
        b, k = _f64(base), _f64(k)
        out = np.zeros(b.size)
        self._call("estimate_pvalues", _ptr(b), u64(b.size), _ptr(k), u64(k.size), _ptr(out))
        return out

    def compute_cutoff(self, p, alpha):
        p = _f64(p)
        out = f64()
        self._call("compute_cutoff", _ptr(p), u64(p.size), f64(alpha), C.byref(out))
        return out.value

    def normal_mean_logm(self, seed, k, lam, log_norm, n_data, first, count):
        yb, lm = np.zeros(count), np.zeros(count)
        self._call("normal_mean_logm", u64(seed), u64(k), f64(lam), f64(log_norm), u64(n_data),
                   u64(first), u64(count), _ptr(yb), _ptr(lm))
        return yb, lm

    def ess(self, lw):
        lw = _f64(lw)
        out = f64()
        self._call("ess", _ptr(lw), u64(lw.size), C.byref(out))
        return out.value

    def resample_multinomial(self, log_w, particles, seed, sid):
        lw, p = _f64(log_w), _f64(particles)
        n, d = p.shape
        out = np.zeros_like(p)
        anc = np.zeros(n, dtype=np.uint64)
        self._call("resample_multinomial", u64(n), u32(d), _ptr(lw), _ptr(p), u64(seed), u32(sid),
                   _ptr(out), _ptr(anc))
        return out, anc
