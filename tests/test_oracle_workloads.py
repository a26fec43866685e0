"""CPU tests of the oracle's definitions of the workloads the reference does not
contain (configs 2-4: "parity unpinned" -- anchored analytically)."""
import math

import numpy as np
import pytest

from paper_1902_09046_b200 import _abi as A, models as M


def mm_cfg(levels=3, paths=20000, seed=1337):
    c = A.vxb_mlmc_cfg()
    c.levels, c.refine, c.tau0, c.t_end, c.paths, c.seed = levels, 4, 1.0, 30.0, paths, seed
    return c


def smc_cfg(n=1500, gens=4, seed=1337):
    c = A.vxb_abcsmc_cfg()
    c.particles, c.generations, c.quantile, c.kernel_scale = n, gens, 0.5, 2.0
    c.jitter, c.round_size, c.max_rounds, c.seed = 1e-10, 0, 0, seed
    return c


# ----------------------------------------------------------------- config 2
def test_ppp_pvalues_match_the_closed_form(oracle):
    """ybar ~ N(0, lambda^2 + 1/n) under the prior predictive, so
    p(lambda) = erfc(|ybar_obs| / sqrt(2 (lambda^2 + 1/n)))."""
    n, m_total = 100, 40000
    mdl = M.normal_mean_model(n)
    lam = np.array(M.lambda_grid(8))
    ln = np.array([-0.5 * math.log(2.0 * math.pi * (l * l + 1.0 / n)) for l in lam])
    y_obs = 3.0 + oracle.fill_gaussian(oracle.derive_seed(2, [90]), 0, 0, n)
    ybar_obs = float(y_obs.mean())
    counts, pv, _ = oracle.ppp_pvalues(mdl, lam, ln, m_total, 0, m_total, 1337, ybar_obs)
    for k, l in enumerate(lam):
        exact = math.erfc(abs(ybar_obs) / math.sqrt(2.0 * (l * l + 1.0 / n)))
        se = math.sqrt(max(exact * (1 - exact), 1e-12) / m_total)
        assert abs(pv[k] - exact) < 5 * se + 2.0 / m_total
    # shards add up (integer counters)
    c1, _, _ = oracle.ppp_pvalues(mdl, lam, ln, m_total, 0, 15000, 1337, ybar_obs)
    c2, _, _ = oracle.ppp_pvalues(mdl, lam, ln, m_total, 15000, 25000, 1337, ybar_obs)
    assert np.array_equal(c1 + c2, counts)


# ----------------------------------------------------------------- config 3
def test_weighted_moments_and_canonical_sums(oracle):
    rs = np.random.RandomState(3)
    th = rs.normal(size=(1000, 3)) * [0.1, 20.0, 0.05] + [0.5, 100.0, 0.05]
    w = np.full(1000, 1e-3)
    mean, cov, s2 = oracle.weighted_moments(th, w)
    assert np.allclose(mean, th.mean(0), rtol=1e-12)
    assert np.allclose(cov, oracle.sample_covariance(th), rtol=1e-9)  # equal weights -> n-1 divisor
    w = rs.uniform(size=1000)
    w /= w.sum()
    mean, cov, s2 = oracle.weighted_moments(th, w)
    assert np.allclose(mean, (w[:, None] * th).sum(0), rtol=1e-12)
    d = th - mean
    assert np.allclose(cov, (w[:, None, None] * d[:, :, None] * d[:, None, :]).sum(0) / (1 - (w * w).sum()), rtol=1e-10)
    cum = oracle.canon_cumsum(w)
    assert (np.diff(cum) >= 0).all() and abs(cum[-1] - 1.0) < 1e-12
    assert abs(oracle.canon_sum(w) - 1.0) < 1e-12
    chol = oracle.make_kernel(cov, 2.0)
    assert np.allclose(chol @ chol.T, 2.0 * cov, rtol=1e-12)


def test_abcsmc_weights_are_the_gaussian_kernel_sum(oracle):
    rs = np.random.RandomState(5)
    prev = rs.normal(size=(300, 3))
    new = rs.normal(size=(50, 3))
    w = rs.uniform(size=300)
    w /= w.sum()
    cov = np.cov(prev.T) * 2.0
    chol = np.linalg.cholesky(cov)
    got = oracle.abcsmc_weights(new, prev, w, chol)
    inv = np.linalg.inv(cov)
    for i in range(50):
        d = new[i] - prev
        q = np.einsum("ij,jk,ik->i", d, inv, d)
        assert abs(got[i] * (w * np.exp(-0.5 * q)).sum() - 1.0) < 1e-10


@pytest.mark.timeout(600)
def test_abcsmc_run_invariants(oracle, golden):
    m = M.logistic_model()
    obs = golden["logistic_observed"]
    cfg = smc_cfg(n=1500, gens=4)
    res = oracle.abcsmc_run(m, cfg, obs)
    assert math.isinf(res["epsilon"][0]) and res["accept_rate"][0] == 1.0
    assert (np.diff(res["epsilon"][1:]) < 0).all()                 # thresholds tighten
    assert abs(res["weight"].sum() - 1.0) < 1e-12                   # sum w = 1
    assert ((res["ess"] >= 1.0) & (res["ess"] <= cfg.particles + 1e-6)).all()  # ESS in [1, N]
    assert (res["rho"] <= res["epsilon"][-1]).all()
    lo, hi = np.array([0.0, 50.0, 0.0]), np.array([1.0, 150.0, 0.2])
    assert ((res["theta"] >= lo) & (res["theta"] < hi)).all()       # prior support
    # generation 0 equals the config-0 machinery (run_prior_predictive rows)
    key = M.keying(oracle.derive_seed(cfg.seed, [0]))
    p, s, rho, f = oracle.abc_prior_predictive(m, key, 1500, 0, 1500, obs, want_summaries=False)
    cfg0 = smc_cfg(n=1500, gens=1)
    r0 = oracle.abcsmc_run(m, cfg0, obs)
    assert np.array_equal(r0["theta"], p) and np.array_equal(r0["rho"], rho)
    # the posterior concentrates around the data-generating K = 100
    k_mean = (res["weight"] * res["theta"][:, 1]).sum()
    assert 90.0 < k_mean < 110.0
    # determinism, thread-count independence
    res2 = oracle.abcsmc_run(m, cfg, obs, threads=1)
    assert np.array_equal(res["theta"], res2["theta"]) and np.array_equal(res["weight"], res2["weight"])


# ----------------------------------------------------------------- config 4
def test_tauleap_conservation_and_telescoping(oracle):
    m = M.mm_tauleap_model()
    cfg = mm_cfg(levels=4, paths=3000)
    for level in range(4):
        sums, y = oracle.mlmc_level(m, cfg, level, 0, 3000, want_y=True)
        assert sums[0] == y.sum() and sums[1] == (y.astype(np.int64) ** 2).sum()
        # shard-independence of the integer sums
        s1, _ = oracle.mlmc_level(m, cfg, level, 0, 1000)
        s2, _ = oracle.mlmc_level(m, cfg, level, 1000, 2000)
        assert np.array_equal(s1 + s2, sums)
    # level 0 is a plain tau-leap: P(T) in [0, 100] up to leap overshoot, mean near the SSA mean
    sums0, y0 = oracle.mlmc_level(m, cfg, 0, 0, 3000, want_y=True)
    assert y0.min() >= 0 and y0.max() <= 110


def test_tauleap_level_variance_decays_and_estimate_matches_ssa(oracle):
    m = M.mm_tauleap_model()
    cfg = mm_cfg(levels=5, paths=20000)
    res = oracle.mlmc_tauleap(m, cfg)
    v = res["level_var"]
    assert v[2] < v[1] and v[3] < v[2] and v[4] < v[3]             # coupling tightens with tau
    ssa_mean, ssa_var = oracle.mm_gillespie(m, 30.0, 20000, 7)
    se = math.sqrt(res["std_error"] ** 2 + ssa_var / 20000)
    # remaining bias at tau = 4^-4 is small against the Monte-Carlo error bar used here
    assert abs(res["estimate"] - ssa_mean) < 5 * se + 0.15
    assert np.allclose(res["level_cost"], [30, 150, 600, 2400, 9600])


def test_poisson_inversion_moments(oracle):
    """Level-0 firing counts are Poisson: with k2 = k3 = 0 and S,E frozen by a
    huge pool, one step's K1 has mean = variance = a1 * tau."""
    m = M.mm_tauleap_model(x0=(1000000, 1, 0, 0), rates=(3e-6, 0.0, 0.0))
    cfg = mm_cfg(levels=1, paths=200000)
    cfg.tau0, cfg.t_end = 1.0, 1.0
    # P never fires; C = K1 after one step; read it through S: not exposed -> use k3 trick instead
    m2 = M.mm_tauleap_model(x0=(0, 0, 30, 0), rates=(0.0, 0.0, 0.1))
    sums, y = oracle.mlmc_level(m2, cfg, 0, 0, 200000, want_y=True)  # P(1) ~ Poisson(0.1*30*1)
    lam = 3.0
    assert abs(y.mean() - lam) < 5 * math.sqrt(lam / 200000)
    assert abs(y.var() - lam) < 0.05
    pmf0 = (y == 0).mean()
    assert abs(pmf0 - math.exp(-lam)) < 5 * math.sqrt(math.exp(-lam) / 200000)
