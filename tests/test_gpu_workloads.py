"""GPU parity tests for configs 2-4 and the SMC building blocks, through the C
ABI, against the oracle (bit-exact for counts, indices and the canonical-order
fp64 reductions; stated tolerances where the reference calls libm)."""
import math

import numpy as np
import pytest

from paper_1902_09046_b200 import _abi as A, lib, models as M

pytestmark = pytest.mark.gpu


def eq(a, b):
    return np.array_equal(np.asarray(a), np.asarray(b), equal_nan=True)


def mm_cfg(levels=3, paths=20000, seed=1337):
    c = A.vxb_mlmc_cfg()
    c.levels, c.refine, c.tau0, c.t_end, c.paths, c.seed = levels, 4, 1.0, 30.0, paths, seed
    return c


def smc_cfg(n=1500, gens=4, seed=1337, round_size=0):
    c = A.vxb_abcsmc_cfg()
    c.particles, c.generations, c.quantile, c.kernel_scale = n, gens, 0.5, 2.0
    c.jitter, c.round_size, c.max_rounds, c.seed = 1e-10, round_size, 0, seed
    return c


# ----------------------------------------------------------------- config 2
def test_ppp_pvalues_parity(ctx, oracle, golden):
    n, m_total = 100, 20000
    mdl = M.normal_mean_model(n)
    lam = np.array(M.lambda_grid(64))
    ln = np.array([-0.5 * math.log(2.0 * math.pi * (l * l + 1.0 / n)) for l in lam])
    y_obs = 3.0 + oracle.fill_gaussian(oracle.derive_seed(2, [90]), 0, 0, n)
    ybar_obs = float(y_obs.mean())
    want_c, want_p, want_y = oracle.ppp_pvalues(mdl, lam, ln, m_total, 0, m_total, 1337, ybar_obs, want_ybar=True)
    got_c, got_p, got_y = ctx.ppp_pvalues(mdl, lam, ln, m_total, 0, m_total, 1337, ybar_obs, want_ybar=True)
    assert eq(got_y, want_y)                       # every dataset mean bit-identical
    assert eq(got_c, want_c) and eq(got_p, want_p)
    # golden: reference-drawn datasets (weak_info.cpp draw order)
    lam6, ln6 = np.full(6, 0.7), np.full(6, golden["nm_lognorm"][0])
    _, _, yb = ctx.ppp_pvalues(mdl, lam6, ln6, 1000, 10, 40, 1337, 0.3, want_ybar=True)
    assert eq(yb[5], golden["nm_ybar"])
    # shards add up; odd n; error codes
    c1, _, _ = ctx.ppp_pvalues(mdl, lam, ln, m_total, 0, 7001, 1337, ybar_obs)
    c2, _, _ = ctx.ppp_pvalues(mdl, lam, ln, m_total, 7001, m_total - 7001, 1337, ybar_obs)
    assert eq(c1 + c2, want_c)
    m7 = M.normal_mean_model(7)
    a = oracle.ppp_pvalues(m7, lam[:5], ln[:5], 500, 0, 500, 3, 0.2, want_ybar=True)
    b = ctx.ppp_pvalues(m7, lam[:5], ln[:5], 500, 0, 500, 3, 0.2, want_ybar=True)
    assert eq(a[0], b[0]) and eq(a[2], b[2])
    with pytest.raises(lib.VxbError) as e:
        ctx.ppp_pvalues(mdl, -lam, ln, 10, 0, 10, 1, 0.0)
    assert e.value.code == "invalid-argument"


def test_ppp_fast_generator_matches_closed_form(ctx):
    n, m_total = 100, 400000
    mdl = M.normal_mean_model(n, rng=A.VXB_RNG_FAST)
    lam = np.array(M.lambda_grid(16))
    ln = np.array([-0.5 * math.log(2.0 * math.pi * (l * l + 1.0 / n)) for l in lam])
    ybar_obs = 2.95
    counts, pv, _ = ctx.ppp_pvalues(mdl, lam, ln, m_total, 0, m_total, 99, ybar_obs)
    for k, l in enumerate(lam):
        exact = math.erfc(abs(ybar_obs) / math.sqrt(2.0 * (l * l + 1.0 / n)))
        se = math.sqrt(max(exact * (1 - exact), 1e-12) / m_total)
        assert abs(pv[k] - exact) < 5 * se + 2.0 / m_total


# ------------------------------------------------------------- SMC pieces
def test_device_exp_is_the_host_libm_exp(ctx, oracle):
    """fn 9 of vxb_fastmath_eval = csrc/vxb_libmexp.cuh: bit-identical to the oracle's
    restatement AND to the live std::exp of this box (what the reference calls)."""
    rs = np.random.RandomState(5)
    x = np.concatenate([-rs.exponential(8.0, 3_000_000), rs.uniform(-760, -690, 500_000),
                        rs.uniform(-1100, 800, 500_000), rs.uniform(-1e-3, 1e-3, 200_000),
                        rs.normal(size=200_000) * 1e-16, rs.uniform(700, 712, 100_000),
                        [0.0, -0.0, np.inf, -np.inf, -745.13321910194122, -5e-324, 709.79,
                         -1024.0, 512.0, -512.0, 2.0 ** -54, -(2.0 ** -55)]])
    dev = ctx.fastmath(9, x)
    restated, live = oracle.exp_restated(x)
    assert np.array_equal(dev.view(np.uint64), live.view(np.uint64))
    assert np.array_equal(dev.view(np.uint64), restated.view(np.uint64))
    assert np.isnan(ctx.fastmath(9, np.array([np.nan]))[0])
    # the library's other build (CPUs without FMA): fn 11 against its own restatement
    assert ctx.host_exp_variant() == 0
    assert np.array_equal(ctx.fastmath(10, x).view(np.uint64), dev.view(np.uint64))
    plain, _ = oracle.exp_restated(x, plain_build=True)
    dev_plain = ctx.fastmath(11, x)
    assert np.array_equal(dev_plain.view(np.uint64), plain.view(np.uint64))
    assert 100 < (dev_plain.view(np.uint64) != dev.view(np.uint64)).sum() < 50_000


def test_resample_follows_the_host_libm_build(golden):
    """A host whose libm runs the PLAIN build of exp (no FMA: simulated with
    GLIBC_TUNABLES in a subprocess): vxb_init detects it and resample_multinomial / ess /
    logsumexp stay bit-identical to that host's reference arithmetic."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = """
import sys
sys.path.insert(0, %r)
import numpy as np
from oracle.pyoracle import Oracle
from paper_1902_09046_b200 import lib
ctx, o = lib.Context(0), Oracle()
assert ctx.host_exp_variant() == 1, ctx.host_exp_variant()
rs = np.random.RandomState(9)
for n, spread in ((100000, 3.0), (40001, 40.0)):
    lw, parts = rs.normal(size=n) * spread, rs.normal(size=(n, 3))
    g, h = ctx.resample_multinomial(lw, parts, 77, 9), o.resample_multinomial(lw, parts, 77, 9)
    assert np.array_equal(g[1], h[1]) and np.array_equal(g[0], h[0])
    assert ctx.ess(lw) == o.ess(lw) and ctx.logsumexp(lw) == o.logsumexp(lw)
print("plain host ok")
""" % root
    run = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600,
                         env=dict(os.environ, GLIBC_TUNABLES="glibc.cpu.hwcaps=-AVX2,-FMA"))
    assert run.returncode == 0 and "plain host ok" in run.stdout, run.stdout[-800:] + run.stderr[-1500:]


def test_ess_logsumexp_resample(ctx, oracle, golden):
    """ess / logsumexp / resample_multinomial are bit-exact: the device evaluates the
    host libm's exp and adds in the reference's sequential order."""
    lw = golden["smc_lw"]
    assert ctx.ess(lw) == golden["smc_ess"][0] == oracle.ess(lw)
    assert abs(ctx.ess(np.log([1.0, 1.0, 2.0])) - 16.0 / 6.0) < 1e-12
    assert ctx.logsumexp(lw) == oracle.logsumexp(lw)
    assert ctx.logsumexp(np.array([-np.inf, -np.inf])) == -np.inf
    with pytest.raises(lib.VxbError) as e:
        ctx.ess(np.array([-np.inf, -np.inf]))
    assert e.value.code == "degenerate-ensemble"
    out, anc = ctx.resample_multinomial(lw, golden["smc_particles"], 2718, 3 | (5 << 16))
    assert eq(anc, golden["smc_ancestors"]) and eq(out, golden["smc_resampled"])
    rs = np.random.RandomState(9)
    for n, spread in ((100000, 3.0), (100001, 40.0), (4097, 300.0), (1, 1.0), (2049, 0.0)):
        lw = rs.normal(size=n) * spread
        if n > 4000:
            lw[rs.randint(0, n, 50)] = -np.inf     # zero-weight particles are never drawn
        parts = rs.normal(size=(n, 3))
        o_out, o_anc = oracle.resample_multinomial(lw, parts, 77, 9)
        g_out, g_anc = ctx.resample_multinomial(lw, parts, 77, 9)
        assert eq(g_anc, o_anc) and eq(g_out, o_out), n
        assert ctx.ess(lw) == oracle.ess(lw), n
        assert ctx.logsumexp(lw) == oracle.logsumexp(lw), n
    n = 100000
    lw = rs.normal(size=n) * 3
    parts = rs.normal(size=(n, 3))
    g_out, g_anc = ctx.resample_multinomial(lw, parts, 77, 9)
    # point mass: every draw picks it
    lw0 = np.full(1000, -np.inf)
    lw0[123] = 0.0
    _, anc0 = ctx.resample_multinomial(lw0, parts[:1000], 1, 0)
    assert (anc0 == 123).all()
    # unbiasedness: ancestor frequencies follow the weights
    w = np.exp(lw - lw.max())
    w /= w.sum()
    top = np.argsort(w)[-5:]
    cnt = np.bincount(g_anc.astype(np.int64), minlength=lw.size)
    for i in top:
        assert abs(cnt[i] - lw.size * w[i]) < 6 * math.sqrt(lw.size * w[i]) + 3


# ----------------------------------------------------------------- config 3
def test_abcsmc_stages_parity(ctx, oracle, golden):
    m = M.logistic_model()
    obs = golden["logistic_observed"]
    n = 3000
    key = M.keying(oracle.derive_seed(5, [0]))
    theta, _, rho, f = oracle.abc_prior_predictive(m, key, n, 0, n, obs, want_summaries=False)
    rs = np.random.RandomState(1)
    w = rs.uniform(0.5, 1.5, size=n)
    w /= oracle.canon_sum(w)
    mean, cov, s2 = oracle.weighted_moments(theta, w)
    chol = oracle.make_kernel(cov, 2.0)
    cum = oracle.canon_cumsum(w)
    eps = oracle.quantile(rho, 0.5)
    want = oracle.abcsmc_propose(m, 5, 1, 100, 4000, theta, cum, chol, obs, eps)
    got = ctx.abcsmc_propose(m, 5, 1, 100, 4000, theta, cum, chol, obs, eps)
    assert eq(got[2], want[2]) and eq(got[0], want[0]) and eq(got[1], want[1])
    assert set(np.unique(want[2])) >= {0, 1, 2}      # accepted, rejected and outside-prior rows
    new = want[0][want[2] == 1][:500]
    w_o = oracle.abcsmc_weights(new, theta, w, chol)
    w_g = ctx.abcsmc_weights(new, theta, w, chol)
    assert eq(w_g, w_o)                               # sequential-order sum reproduced exactly


@pytest.mark.timeout(900)
def test_abcsmc_run_parity(ctx, oracle, golden):
    m = M.logistic_model()
    obs = golden["logistic_observed"]
    for cfg in (smc_cfg(n=2000, gens=5), smc_cfg(n=777, gens=3, seed=9, round_size=300)):
        want = oracle.abcsmc_run(m, cfg, obs)
        got = ctx.abcsmc_run(m, cfg, obs)
        for k in ("epsilon", "proposals", "accept_rate", "theta", "rho", "weight", "ess", "mean", "cov"):
            assert eq(got[k], want[k]), k
        assert abs(got["weight"].sum() - 1.0) < 1e-12


@pytest.mark.timeout(900)
def test_sharded_abcsmc_driver_on_device(ctx, oracle, golden):
    """The multi-GPU ABC-SMC host driver (dist.sharded_abcsmc) with the device
    stages, run as one rank: bit-identical to the native one-GPU driver
    (vxb_abcsmc_run) and to the oracle; also the stage entry points it uses."""
    import torch
    from paper_1902_09046_b200 import dist as D
    m = M.logistic_model()
    obs = golden["logistic_observed"]
    for cfg in (smc_cfg(n=2000, gens=4), smc_cfg(n=777, gens=3, seed=9, round_size=300)):
        native = ctx.abcsmc_run(m, cfg, obs)
        got = D.sharded_abcsmc(D.DeviceStages(ctx), m, cfg, obs)
        for k in ("epsilon", "proposals", "accept_rate", "theta", "rho", "weight", "ess", "mean", "cov"):
            assert eq(got[k], native[k]), k
    want = oracle.abcsmc_run(m, cfg, obs)
    assert eq(got["theta"], want["theta"]) and eq(got["weight"], want["weight"])
    # throughput generator: the sharded driver must take the throughput form of the
    # weights too (vxb_abcsmc_weights rng argument), or it drifts from the native run
    mf = M.logistic_model(rng=A.VXB_RNG_FAST)
    cfg = smc_cfg(n=1500, gens=4, seed=21)
    native = ctx.abcsmc_run(mf, cfg, obs)
    got = D.sharded_abcsmc(D.DeviceStages(ctx), mf, cfg, obs)
    for k in ("epsilon", "proposals", "accept_rate", "theta", "rho", "weight", "ess", "mean", "cov"):
        assert eq(got[k], native[k]), k
    # stage entry points against the oracle (host and device buffers)
    rs = np.random.RandomState(3)
    theta = rs.normal(size=(1000, 3))
    w = rs.uniform(0.1, 1.0, size=1000)
    w /= oracle.canon_sum(w)
    mean, cov, s2 = ctx.weighted_moments(theta, w)
    mo, co, so = oracle.weighted_moments(theta, w)
    assert eq(mean, mo) and eq(cov, co) and s2 == so
    assert eq(ctx.canon_cumsum(w), oracle.canon_cumsum(w))
    cs = ctx.canon_chunk_sums(w)
    assert eq(cs, [oracle.canon_sum(w[i:i + 256]) for i in range(0, 1000, 256)])
    assert ctx.quantile(w, 0.37) == oracle.quantile(w, 0.37)
    assert eq(lib.make_kernel(cov, 2.0), oracle.make_kernel(cov, 2.0))
    w_dev = torch.from_numpy(w).cuda()
    assert eq(ctx.canon_cumsum(w_dev, torch.empty_like(w_dev)).cpu().numpy(), oracle.canon_cumsum(w))


def test_sharded_select_on_device(ctx, oracle, golden):
    """dist.sharded_select as one rank equals select_epsilon over the whole job."""
    from paper_1902_09046_b200 import dist as D
    m = M.logistic_model(steps=200, obs_stride=10)
    obs = oracle.simulate_at(m, [0.5, 100.0, 0.05], 5, 0, 0)
    n = 20000
    p, _, rho, f = oracle.abc_prior_predictive(m, M.keying(1337), n, 0, n, obs, want_summaries=False)
    eps_o, idx_o = oracle.select_epsilon(rho, f, 0.01)
    eps, idx, th, r = D.sharded_select(ctx, m, M.keying(1337), n, obs, 0.01)
    assert eps == eps_o and eq(idx.cpu().numpy(), idx_o)
    assert eq(th.cpu().numpy(), p[idx_o]) and eq(r.cpu().numpy(), rho[idx_o])


@pytest.mark.timeout(900)
def test_abcsmc_fast_generator_statistics(ctx, golden):
    """Throughput mode (Philox4x32, FMA, whitened weights with table-based exp2)
    against the exact mode: same epsilon schedule, ESS and posterior moments
    within Monte-Carlo error; weights normalised; support respected."""
    obs = golden["logistic_observed"]
    cfg = smc_cfg(n=40000, gens=6)
    ref = ctx.abcsmc_run(M.logistic_model(), cfg, obs)
    fast = ctx.abcsmc_run(M.logistic_model(rng=A.VXB_RNG_FAST), cfg, obs)
    assert abs(fast["weight"].sum() - 1.0) < 1e-12
    assert (fast["rho"] <= fast["epsilon"][-1]).all()
    lo, hi = np.array([0.0, 50.0, 0.0]), np.array([1.0, 150.0, 0.2])
    assert ((fast["theta"] >= lo) & (fast["theta"] < hi)).all()
    # median-distance schedule: relative sampling error of a median of 4e4 values ~ 1%
    assert np.allclose(fast["epsilon"][1:], ref["epsilon"][1:], rtol=0.05)
    assert np.allclose(fast["ess"][1:], ref["ess"][1:], rtol=0.05)
    assert np.allclose(fast["accept_rate"][1:], ref["accept_rate"][1:], rtol=0.1)
    for g in range(1, 6):
        sd = np.sqrt(np.diag(ref["cov"][g]))
        assert (np.abs(fast["mean"][g] - ref["mean"][g]) < 6 * sd / math.sqrt(ref["ess"][g])).all()
        assert np.allclose(np.diag(fast["cov"][g]), np.diag(ref["cov"][g]), rtol=0.1)


# ----------------------------------------------------------------- config 4
def test_tauleap_parity(ctx, oracle):
    m = M.mm_tauleap_model()
    cfg = mm_cfg(levels=5, paths=4000)
    for level in range(5):
        s_o, y_o = oracle.mlmc_level(m, cfg, level, 0, 4000, want_y=True)
        s_g, y_g = ctx.mlmc_level(m, cfg, level, 0, 4000, want_y=True)
        assert eq(y_g, y_o) and eq(s_g, s_o)          # every coupled path identical, exact sums
        a, _ = ctx.mlmc_level(m, cfg, level, 0, 1234)
        b, _ = ctx.mlmc_level(m, cfg, level, 1234, 4000 - 1234)
        assert eq(a + b, s_o)
    res_o = oracle.mlmc_tauleap(m, cfg)
    res_g = ctx.mlmc_tauleap(m, cfg)
    for k in ("level_mean", "level_var", "level_cost"):
        assert eq(res_g[k], res_o[k])
    assert res_g["estimate"] == res_o["estimate"] and res_g["std_error"] == res_o["std_error"]
    # other networks / rates through the same kernel
    m2 = M.mm_tauleap_model(x0=(40, 7, 3, 1), rates=(5e-3, 2e-2, 0.3))
    cfg2 = mm_cfg(levels=3, paths=1000, seed=5)
    cfg2.refine, cfg2.tau0, cfg2.t_end = 3, 0.5, 6.0
    for level in range(3):
        s_o, y_o = oracle.mlmc_level(m2, cfg2, level, 0, 1000, want_y=True)
        s_g, y_g = ctx.mlmc_level(m2, cfg2, level, 0, 1000, want_y=True)
        assert eq(y_g, y_o) and eq(s_g, s_o)
    with pytest.raises(lib.VxbError) as e:
        ctx.mlmc_level(m, cfg, 7, 0, 10)
    assert e.value.code == "invalid-argument"


def test_tauleap_full_level_properties(ctx):
    """BASELINE size for one level (1e6 paths): integer sums are shard-additive
    and the level mean sits where the small-sample oracle runs put it."""
    m = M.mm_tauleap_model()
    cfg = mm_cfg(levels=6, paths=1_000_000)
    whole, _ = ctx.mlmc_level(m, cfg, 2, 0, 1_000_000)
    parts = [ctx.mlmc_level(m, cfg, 2, b, 250_000)[0] for b in range(0, 1_000_000, 250_000)]
    assert eq(sum(parts), whole)
    mean = whole[0] / 1e6
    var = (whole[1] - whole[0] * mean) / (1e6 - 1)
    assert abs(mean) < 1.0 and 0.0 < var < 10.0


def test_tauleap_fast_generator_statistics(ctx):
    """The throughput generator (Philox4x32, FMA exp) agrees with the exact-RNG
    run level by level within Monte-Carlo error, and is shard independent."""
    cfg = mm_cfg(levels=5, paths=400000)
    ref = ctx.mlmc_tauleap(M.mm_tauleap_model(), cfg)
    fast_model = M.mm_tauleap_model(rng=A.VXB_RNG_FAST)
    fast = ctx.mlmc_tauleap(fast_model, cfg)
    n = cfg.paths
    for l in range(5):
        se = math.sqrt((ref["level_var"][l] + fast["level_var"][l]) / n)
        assert abs(ref["level_mean"][l] - fast["level_mean"][l]) < 4.5 * se
        assert abs(fast["level_var"][l] / ref["level_var"][l] - 1.0) < 0.05
    a, _ = ctx.mlmc_level(fast_model, cfg, 3, 0, 1000)
    b, _ = ctx.mlmc_level(fast_model, cfg, 3, 1000, 3000)
    c, _ = ctx.mlmc_level(fast_model, cfg, 3, 0, 4000)
    assert eq(a + b, c)


# ------------------------------------------- toggle switch
@pytest.mark.timeout(600)
def test_tauleap_fp32_instance_statistics(ctx):
    """The fp32 throughput instance of the tau-leap kernel (float propensities and CDF
    inversion, exp by one MUFU, 23-bit midpoint uniforms): level means and variances
    agree with the reference-exact fp64 instance within Monte-Carlo error (Bonferroni over
    6 levels), the estimate too; counts are integers, so shard sums add exactly; the
    REF + fp32 combination is refused."""
    cfg = mm_cfg(levels=6, paths=400000, seed=77)
    e = ctx.mlmc_tauleap(M.mm_tauleap_model(), cfg)
    mf = M.mm_tauleap_model(rng=A.VXB_RNG_FAST, precision=A.VXB_F32)
    f = ctx.mlmc_tauleap(mf, cfg)
    for l in range(6):
        z = (f["level_mean"][l] - e["level_mean"][l]) / math.sqrt((f["level_var"][l] + e["level_var"][l]) / cfg.paths)
        assert abs(z) < 3.9, (l, z)
        assert abs(math.log(f["level_var"][l] / e["level_var"][l])) < 0.1, l
    assert abs(f["estimate"] - e["estimate"]) < 4.0 * math.hypot(f["std_error"], e["std_error"])
    whole, _ = ctx.mlmc_level(mf, cfg, 3, 0, 20000)
    a, _ = ctx.mlmc_level(mf, cfg, 3, 0, 7001)
    b, ys = ctx.mlmc_level(mf, cfg, 3, 7001, 12999, want_y=True)
    assert eq(whole[:3], (a + b)[:3]) and int(ys.sum()) == int(b[0])
    with pytest.raises(lib.VxbError) as err:
        ctx.mlmc_tauleap(M.mm_tauleap_model(rng=A.VXB_RNG_REF, precision=A.VXB_F32), cfg)
    assert err.value.code == "invalid-argument"


def test_toggle_switch_parity(ctx, oracle, golden):
    """The reference's own SDE, through the reference's own sampler keying:
    bit-identical summaries, distances and selection (KAT of SURVEY.md 8c)."""
    m = M.toggle_model(100, 256)
    obs = ctx.simulate_at(m, M.TOGGLE_MIDPOINT, lib.derive_seed(1337, [90]), 0, 0)
    assert eq(obs, golden["toggle_observed"])
    key = M.keying(1337, A.VXB_KEY_WORKER, 1, 4)
    p, s, rho, f = ctx.abc_prior_predictive_host(m, key, 256, 0, 256, obs)
    assert rho[0] == 445.69940013687017
    assert eq(rho, golden["toggle_rho"]) and eq(s[0], golden["toggle_summ0"])
    eps, idx, nacc = ctx.select_epsilon(rho, f, 0.01)
    assert eps == 208.44209220565364 and idx.tolist() == [120, 208, 239]
    # other (workers, block width) layouts and particle keying against the oracle
    m2 = M.toggle_model(37, 250)     # cells not a multiple of V: padded stream positions
    obs2 = oracle.simulate_at(m2, M.TOGGLE_MIDPOINT, 5, 2, 7)
    assert eq(ctx.simulate_at(m2, M.TOGGLE_MIDPOINT, 5, 2, 7), obs2)
    for key in (M.keying(3, A.VXB_KEY_WORKER, 3, 16), M.keying(3, A.VXB_KEY_WORKER, 5, 1), M.keying(3)):
        want = oracle.abc_prior_predictive(m2, key, 97, 10, 80, obs2)
        got = ctx.abc_prior_predictive_host(m2, key, 97, 10, 80, obs2)
        for g, w in zip(got, want):
            assert eq(g, w)
    # rows the reference flags: too few cells for 19 quantiles / a single time point
    for bad in (M.toggle_model(50, 10), M.toggle_model(1, 64)):
        want = oracle.abc_prior_predictive(bad, M.keying(1), 8, 0, 8, np.zeros(19))
        got = ctx.abc_prior_predictive_host(bad, M.keying(1), 8, 0, 8, np.zeros(19))
        assert (got[3] == 1).all() and np.isnan(got[2]).all() and (got[1] == 0).all()
        for g, w in zip(got, want):
            assert eq(g, w)


# ------------------------------------------- TB Gillespie ABC
@pytest.mark.timeout(900)
def test_tb_gillespie_parity(ctx, oracle):
    """The reference's exact-simulation model, one warp per path: summaries,
    distances and failure flags bit-identical to tb::gillespie_simulate run row by
    row on RngStream(seed, row) (oracle pinned to the unmodified reference in
    tests/test_oracle_pins.py)."""
    m = M.tb_model(10, 10.0, 10000.0)                      # bench.hpp:39-42 sizes
    for theta, seed, sid, pos in [((0.2, 0.1, 0.05), 5, 2, 3), ((1.5, 0.3, 0.9), 6, 0, 0),
                                  ((0.4, 0.39, 0.2), 7, 1, 8), ((0.3, 0.0, 0.0), 9, 0, 1),
                                  ((0.0, 0.0, 0.0), 8, 0, 0)]:
        want = oracle.tb_simulate(theta, 10, 10.0, 10000.0, seed, sid, pos)
        assert eq(ctx.simulate_at(m, theta, seed, sid, pos), want["summaries"]), theta
    # the synthetic observation of the harness: retries while the population dies out
    obs = ctx.simulate_at(M.tb_model(10, 10.0, 10000.0, attempts=64), M.TB_TRUE_THETA,
                          lib.derive_seed(1337, [91]), 0, 0)
    assert eq(obs, oracle.tb_observed(10, 10.0, 10000.0, 1337))
    with pytest.raises(lib.VxbError) as e:                 # certain extinction: delta >> alpha, long horizon
        ctx.simulate_at(M.tb_model(1, 1e6, 100.0), (0.0, 5.0, 0.0), 3, 0, 0)
    assert e.value.code == "extinct-population"
    with pytest.raises(lib.VxbError) as e:
        ctx.simulate_at(m, (-0.1, 0.1, 0.1), 3, 0, 0)
    assert e.value.code == "invalid-argument"
    n = 300
    want = oracle.tb_abc_particle(10, 10.0, 10000.0, 0, n, 1337, obs)
    got = ctx.abc_prior_predictive_host(m, M.keying(1337), n, 0, n, obs)
    for g, w in zip(got, want):
        assert eq(g, w)
    assert got[3].any() and not got[3].all()               # extinct rows are flagged, not fatal
    assert got[1][:, 0].max() > 1000                       # paths that reach thousands of genotypes
    # shards reproduce the job; other stop rules and small targets (slot array refills)
    part = ctx.abc_prior_predictive_host(m, M.keying(1337), n, 100, 50, obs)
    for g, w in zip(part, want):
        assert eq(g, w[100:150])
    for initial, horizon, target in ((10, 50.0, 10000.0), (3, 25.0, 400.0), (500, 4.0, 700.0)):
        mm = M.tb_model(initial, horizon, target)
        want = oracle.tb_abc_particle(initial, horizon, target, 0, 96, 77, [50.0, 0.9])
        got = ctx.abc_prior_predictive_host(mm, M.keying(77), 96, 0, 96, np.array([50.0, 0.9]))
        for g, w in zip(got, want):
            assert eq(g, w), (initial, horizon, target)
    with pytest.raises(lib.VxbError) as e:
        ctx.abc_prior_predictive_host(m, M.keying(1, A.VXB_KEY_WORKER, 2, 4), 8, 0, 8, obs)
    assert e.value.code == "invalid-argument"


def test_tb_gillespie_edge_cases(ctx, oracle):
    """Stop rules that end a path before its first event, an unbounded horizon with a
    small case target, and a target at the device limit."""
    inf = float("inf")
    for initial, horizon, target, n in ((50, 10.0, 20.0, 32), (5, inf, 300.0, 64), (1, 0.0, 1000.0, 16),
                                        (20, 3.0, 60000.0, 24)):
        mm = M.tb_model(initial, horizon, target)
        want = oracle.tb_abc_particle(initial, horizon, target, 3, n, 2024, [5.0, 0.5])
        got = ctx.abc_prior_predictive_host(mm, M.keying(2024), n + 3, 3, n, np.array([5.0, 0.5]))
        for g, w in zip(got, want):
            assert eq(g, w), (initial, horizon, target)
    with pytest.raises(lib.VxbError) as e:
        ctx.abc_prior_predictive_host(M.tb_model(10, 10.0, 1e6), M.keying(1), 4, 0, 4, np.zeros(2))
    assert e.value.code == "invalid-argument"
    with pytest.raises(lib.VxbError) as e:
        ctx.abc_prior_predictive_host(M.tb_model(0, 10.0, 100.0), M.keying(1), 4, 0, 4, np.zeros(2))
    assert e.value.code == "invalid-shape"


@pytest.mark.timeout(900)
def test_toggle_throughput_mode_statistics(ctx):
    """The toggle model's throughput mode (packed Philox4x32 normals, table-based
    log2 / 2^z, FMA arithmetic) against its bit-exact mode: distances and the 19
    quantile summaries agree in distribution (two-sample KS at 1 %, means within
    Monte-Carlo error)."""
    n = 3000
    m_ref, m_fast = M.toggle_model(100, 256), M.toggle_model(100, 256, rng=A.VXB_RNG_FAST)
    obs = ctx.simulate_at(m_ref, M.TOGGLE_MIDPOINT, lib.derive_seed(1337, [90]), 0, 0)
    p0, s0, r0, f0 = ctx.abc_prior_predictive_host(m_ref, M.keying(11), n, 0, n, obs)
    p1, s1, r1, f1 = ctx.abc_prior_predictive_host(m_fast, M.keying(12), n, 0, n, obs)
    assert not f0.any() and not f1.any() and np.isfinite(s1).all() and (s1 >= 1.0).all()

    def ks(a, b):
        xs = np.sort(np.concatenate([a, b]))
        return np.abs(np.searchsorted(np.sort(a), xs, side="right") / len(a)
                      - np.searchsorted(np.sort(b), xs, side="right") / len(b)).max()
    crit = 1.628 * math.sqrt(2.0 / n)
    assert ks(r0, r1) < crit
    for k in (0, 9, 18):
        assert ks(s0[:, k], s1[:, k]) < crit, k
        se = math.sqrt(s0[:, k].var() / n + s1[:, k].var() / n)
        assert abs(s0[:, k].mean() - s1[:, k].mean()) < 4.5 * se, k
    for k in range(7):   # the prior box
        assert p1[:, k].min() >= M.TOGGLE_PRIOR_LO[k] and p1[:, k].max() < M.TOGGLE_PRIOR_HI[k]
        assert ks(p0[:, k], p1[:, k]) < crit
    # same parameters, same model: a cell ensemble simulated by both modes at fixed theta
    # has the same summaries up to the spread over 4096 cells
    part = ctx.abc_prior_predictive_host(m_fast, M.keying(12), n, 100, 50, obs)
    assert eq(part[2], r1[100:150])                      # shard independence of the throughput mode
