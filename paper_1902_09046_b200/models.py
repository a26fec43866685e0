"""POD model descriptors for the BASELINE.json workloads (host side, no compute).

Each constructor fills a ``vxb_model`` (include/vexbayes_cuda.h); it plays the
role of the reference's ``make_abc_model`` factories (toggle_switch.cpp:135-152)
with the closures replaced by a plain descriptor the device can read.
"""
import math

from . import _abi as A


def logistic_model(steps=2000, obs_stride=100, dt=0.01, x0=10.0,
                   prior_lo=(0.0, 50.0, 0.0), prior_hi=(1.0, 150.0, 0.2),
                   precision=A.VXB_F64, rng=A.VXB_RNG_REF, arith=A.VXB_ARITH_EXACT):
    """Stochastic logistic growth dX = rX(1-X/K)dt + sigma X dW (configs 0/1/3)."""
    m = A.vxb_model()
    m.model = A.VXB_MODEL_LOGISTIC_SDE
    m.precision, m.rng, m.arith = precision, rng, arith
    m.dim = 3
    m.steps, m.obs_stride = steps, obs_stride
    m.summary_dim = steps // obs_stride if obs_stride else 0
    m.dt, m.x0 = dt, x0
    for k in range(3):
        m.prior_lo[k] = prior_lo[k]
        m.prior_hi[k] = prior_hi[k]
    m.consts[0] = math.sqrt(dt)
    return m


TOGGLE_PRIOR_LO = (250.0, 0.05, 0.05, 0.0, 0.0, 0.0, 0.0)
TOGGLE_PRIOR_HI = (400.0, 0.5, 0.35, 50.0, 50.0, 7.0, 7.0)
TOGGLE_MIDPOINT = (325.0, 0.275, 0.2, 25.0, 25.0, 3.5, 3.5)  # bench.cpp:72 "true" parameters


def toggle_model(steps=600, cells=8000, rng=A.VXB_RNG_REF):
    """The reference's toggle-switch SDE (toggle_switch.hpp:16-82): theta =
    (mu, sigma, gamma, alpha_u, alpha_v, beta_u, beta_v), C cells, T time points,
    summaries = 19 quantiles of the noisy terminal observations."""
    m = A.vxb_model()
    m.model = A.VXB_MODEL_TOGGLE
    m.precision, m.rng, m.arith = A.VXB_F64, rng, A.VXB_ARITH_EXACT
    m.dim, m.summary_dim = 7, 19
    m.steps, m.obs_stride = steps, steps
    m.x0 = 10.0
    for k in range(7):
        m.prior_lo[k] = TOGGLE_PRIOR_LO[k]
        m.prior_hi[k] = TOGGLE_PRIOR_HI[k]
    m.consts[1] = float(cells)
    return m


def normal_mean_model(n_data=100, rng=A.VXB_RNG_REF, arith=A.VXB_ARITH_EXACT):
    """y_i ~ N(theta, 1), theta ~ N(0, lambda^2) (config 2)."""
    m = A.vxb_model()
    m.model = A.VXB_MODEL_NORMAL_MEAN
    m.precision, m.rng, m.arith = A.VXB_F64, rng, arith
    m.dim, m.summary_dim = 1, 1
    m.steps, m.obs_stride = n_data, n_data
    return m


def mm_tauleap_model(x0=(100, 20, 0, 0), rates=(1e-3, 1e-4, 0.1), rng=A.VXB_RNG_REF,
                     precision=A.VXB_F64):
    """Michaelis-Menten network S+E->C, C->S+E, C->E+P (config 4).  precision VXB_F32:
    rates and the Poisson inversion in float (throughput generator only)."""
    m = A.vxb_model()
    m.model = A.VXB_MODEL_MM_TAULEAP
    m.precision, m.rng, m.arith = precision, rng, A.VXB_ARITH_EXACT
    m.dim, m.summary_dim = 3, 1
    for k in range(4):
        m.consts[k] = float(x0[k])
    for k in range(3):
        m.consts[4 + k] = float(rates[k])
    return m


def keying(seed, mode=A.VXB_KEY_PARTICLE, workers=1, block_width=1):
    k = A.vxb_keying()
    k.mode, k.workers, k.block_width, k.reserved, k.seed = mode, workers, block_width, 0, seed
    return k


def lambda_grid(n=64, lo=0.1, hi=100.0):
    """Config 2 hyperparameter grid: n values log-spaced in [lo, hi]."""
    a, b = math.log10(lo), math.log10(hi)
    return [10.0 ** (a + (b - a) * k / (n - 1)) for k in range(n)]


DEFAULT_DOSE = (-0.86, -0.3, -0.05, -0.75)   # default_design, weak_info.cpp:62-64
DEFAULT_GROUP_SIZE = (5, 5, 5, 5)


def weakinfo_config(hyper_count=400, datasets=400, particles=500, alpha=0.05, c=0.01,
                    scale=1.6828427124746189, block_width=4, seed=0, redraw_base=False,
                    base=(10.0, 2.5), dose=DEFAULT_DOSE, group_size=DEFAULT_GROUP_SIZE,
                    arith=A.VXB_ARITH_EXACT, rng=A.VXB_RNG_REF):
    """WeakInfoConfig (weak_info.hpp:62-75) with the reference defaults.  arith: the
    sampler's arithmetic (VXB_ARITH_FMA: throughput mode, same random numbers)."""
    cfg = A.vxb_weakinfo_cfg()
    cfg.hyper_count, cfg.datasets, cfg.particles = hyper_count, datasets, particles
    cfg.block_width, cfg.seed = block_width, seed
    cfg.alpha, cfg.c, cfg.scale = alpha, c, scale
    cfg.base[0], cfg.base[1] = base
    cfg.redraw_base, cfg.groups = int(redraw_base), len(dose)
    cfg.arith, cfg.rng = arith, rng
    for g in range(len(dose)):
        cfg.dose[g], cfg.group_size[g] = dose[g], group_size[g]
    return cfg


TB_TRUE_THETA = (0.2, 0.1, 0.05)   # bench.cpp:81 "true" parameters of the synthetic observation


def tb_model(initial_cases=10, time_horizon=50.0, case_target=10000.0, attempts=1):
    """The reference's TB transmission model (tb_model.hpp:12-76): theta = (alpha,
    delta, tau), exact Gillespie simulation, summaries (G, H).  StopRule defaults as
    tb_model.hpp:41-44."""
    m = A.vxb_model()
    m.model = A.VXB_MODEL_TB
    m.precision, m.rng, m.arith = A.VXB_F64, A.VXB_RNG_REF, A.VXB_ARITH_EXACT
    m.dim, m.summary_dim = 3, 2
    m.consts[0], m.consts[1], m.consts[2], m.consts[3] = initial_cases, time_horizon, case_target, attempts
    m.prior_hi[0], m.prior_hi[2] = 2.0, 1.0
    return m
