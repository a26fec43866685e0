"""CPU tests: pin the oracle (oracle/vxb_oracle.cpp) before anything trusts it.

1. against the golden vectors generated from the unmodified reference
   (tests/golden/golden.npz, made by tests/golden/make_golden.py) -- always;
2. against oracle/_ref (the reference compiled here) on fresh seeded inputs --
   when that library is present;
3. against the properties the reference's own tests pin (test_rng.cpp,
   test_fastmath.cpp, test_numeric.cpp, test_blocked.cpp) and the SPEC.md
   examples for the pieces whose reference tests are empty.
"""
import math
import os

import numpy as np
import pytest

from paper_1902_09046_b200 import _abi as A, models as M


def eq(a, b):
    return np.array_equal(np.asarray(a), np.asarray(b), equal_nan=True)


# ----------------------------------------------------------------- golden
def test_rng_known_answers(oracle, golden):
    assert oracle.splitmix64(0) == 0xE220A8397B1DCDAF == int(golden["splitmix64_0"])
    assert oracle.derive_seed(42, [1, 2, 3]) == 0x3FB96077DA5807FD == int(golden["derive_seed_42_123"])
    w = oracle.stream_u64(1337, 0, 0, 64)
    assert [hex(x) for x in w[:4]] == ["0xfe78345bef749875", "0x77013bd4b5221611",
                                       "0xa5f809b9395f05e5", "0x66b9e7b9a087a139"]
    assert eq(w, golden["words_1337_0"])
    assert eq(oracle.stream_u64(7, 3, 1001, 33), golden["words_7_3_pos1001"])
    gz = oracle.fill_gaussian(1337, 0, 0, 64)
    assert [repr(float(x)) for x in gz[:4]] == ["-3.1222123110592097", "0.7007283101377776",
                                                "-1.1763603487266563", "0.8403694724866424"]
    assert eq(gz, golden["gauss_1337_0"])
    assert eq(oracle.fill_gaussian(555, 9, 13, 41, 1.5, 2.0), golden["gauss_555_9_pos13"])
    assert eq(oracle.fill_uniform(4242, 1, 0, 64, 250.0, 400.0), golden["unif_4242_1"])
    assert eq(oracle.fill_uniform(4242, 1, 5, 64, 1e16, 1e16 + 4.0), golden["unif_big"])


def test_fastmath_golden(oracle, golden):
    assert eq(oracle.fastmath(0, golden["fm_x_log"]), golden["fm_log2"])
    assert eq(oracle.fastmath(1, golden["fm_x_log"]), golden["fm_ln"])
    assert eq(oracle.fastmath(2, golden["fm_x_exp"]), golden["fm_exp2"])
    assert eq(oracle.fastmath(3, golden["fm_x_ang"]), golden["fm_sinpi"])
    assert eq(oracle.fastmath(4, golden["fm_x_ang"]), golden["fm_cospi"])
    assert eq(oracle.fastmath(5, golden["fm_pow_b"], golden["fm_pow_e"]), golden["fm_pow"])


def test_numeric_golden(oracle, golden):
    s = golden["num_sample"]
    qs = [oracle.quantile(s, q) for q in (0.0, 0.05, 0.5, 0.55, 0.999, 1.0)]
    assert eq(qs, golden["num_quantiles"])
    assert oracle.logsumexp(s) == golden["num_logsumexp"][0]
    cov = oracle.sample_covariance(golden["num_data"])
    assert eq(cov, golden["num_cov"])
    ok, chol = oracle.cholesky(cov)
    assert ok and eq(chol, golden["num_chol"])
    assert eq(oracle.partition(8064, 16, 4), golden["partition_8064_16_4"])
    assert eq(oracle.partition(1003, 7, 8), golden["partition_1003_7_8"])


def test_logistic_abc_golden(oracle, golden):
    m = M.logistic_model()
    obs = oracle.simulate_at(m, [0.5, 100.0, 0.05], int(golden["derive_seed_1_90"]), 0, 0)
    assert eq(obs, golden["logistic_observed"])
    p, s, rho, f = oracle.abc_prior_predictive(m, M.keying(1337, A.VXB_KEY_WORKER, 3, 4), 96, 0, 96, obs)
    assert eq(p, golden["abc_w_params"]) and eq(s, golden["abc_w_summ"])
    assert eq(rho, golden["abc_w_rho"]) and eq(f, golden["abc_w_failed"])
    p, s, rho, f = oracle.abc_prior_predictive(m, M.keying(1337), 5000, 1000, 32, obs)
    assert eq(p, golden["abc_p_params"]) and eq(s, golden["abc_p_summ"]) and eq(rho, golden["abc_p_rho"])
    m32 = M.logistic_model(precision=A.VXB_F32)
    p, s, rho, f = oracle.abc_prior_predictive(m32, M.keying(1337), 5000, 1000, 32, obs)
    assert eq(p, golden["abc32_p_params"]) and eq(s, golden["abc32_p_summ"]) and eq(rho, golden["abc32_p_rho"])
    p, s, rho, f = oracle.abc_prior_predictive(m32, M.keying(7, A.VXB_KEY_WORKER, 2, 1), 48, 0, 48, obs)
    assert eq(p, golden["abc32_w_params"]) and eq(s, golden["abc32_w_summ"]) and eq(rho, golden["abc32_w_rho"])


def test_logistic_edge_cases_golden(oracle, golden):
    mo = M.logistic_model(steps=37, obs_stride=5)
    oo = oracle.simulate_at(mo, [0.5, 100.0, 0.05], 99, 4, 3)
    assert eq(oo, golden["odd_observed"])
    p, s, rho, f = oracle.abc_prior_predictive(mo, M.keying(11, A.VXB_KEY_WORKER, 4, 2), 50, 0, 50, oo)
    assert eq(p, golden["odd_w_params"]) and eq(s, golden["odd_w_summ"]) and eq(rho, golden["odd_w_rho"])
    mb = M.logistic_model(steps=400, obs_stride=100, prior_hi=(4000.0, 150.0, 0.2))
    p, s, rho, f = oracle.abc_prior_predictive(mb, M.keying(21), 64, 0, 64, golden["bad_observed"])
    assert eq(f, golden["bad_failed"]) and f.any()
    assert eq(p, golden["bad_params"]) and eq(s, golden["bad_summ"]) and eq(rho, golden["bad_rho"])
    assert np.isnan(rho[f == 1]).all() and (s[f == 1] == 0).all()  # abc.cpp:57-60


def test_select_epsilon_golden(oracle, golden):
    rho = golden["sel_rho"]
    for q in (0.001, 0.01, 0.5, 1.0):
        eps, idx = oracle.select_epsilon(rho, None, q)
        assert eps == golden[f"sel_eps_{q}"][0] and eq(idx, golden[f"sel_idx_{q}"])
        assert len(idx) >= math.ceil(q * len(rho))
    eps, idx = oracle.select_epsilon(golden["bad_rho"], golden["bad_failed"], 0.25)
    assert eps == golden["sel_bad_eps"][0] and eq(idx, golden["sel_bad_idx"])


def test_smc_pieces_golden(oracle, golden):
    assert oracle.ess(golden["smc_lw"]) == golden["smc_ess"][0]
    assert oracle.ess(np.log([1.0, 1.0, 2.0])) == golden["smc_ess"][1]
    out, anc = oracle.resample_multinomial(golden["smc_lw"], golden["smc_particles"], 2718, 3 | (5 << 16))
    assert eq(anc, golden["smc_ancestors"]) and eq(out, golden["smc_resampled"])


def test_pvalues_golden(oracle, golden):
    assert eq(oracle.estimate_pvalues([2.0, 5.0], [1.0, 3.0, 4.0, 6.0]), golden["pv_spec"])
    assert oracle.compute_cutoff(np.linspace(0.1, 1.0, 10), 0.5) == golden["pv_cutoff"][0]
    lam, n = 0.7, 100
    ln = golden["nm_lognorm"][0]
    assert ln == -0.5 * math.log(2.0 * math.pi * (lam * lam + 1.0 / n))
    m = M.normal_mean_model(n)
    # dataset stream = (derive_seed(seed,{k}), j): run lambda index 5 by padding the grid
    lam_grid = np.full(6, lam)
    counts, pv, yb = oracle.ppp_pvalues(m, lam_grid, np.full(6, ln), 1000, 10, 40, 1337, 0.3, want_ybar=True)
    assert eq(yb[5], golden["nm_ybar"])
    v = lam * lam + 1.0 / n
    logm_obs = ln - ((0.5 * 0.3) * 0.3) / v
    assert counts[5] == int((golden["nm_logm"] <= logm_obs).sum())


# ------------------------------------------------------------ live vs _ref
def test_oracle_matches_reference_library(oracle, ref):
    rs = np.random.RandomState(7)
    for seed, sid, pos, n in [(1, 0, 0, 257), (20240518, 1, 12345678901, 64), (99, 4000000000, 3, 31)]:
        assert eq(oracle.stream_u64(seed, sid, pos, n), ref.stream_u64(seed, sid, pos, n))
        assert eq(oracle.fill_gaussian(seed, sid, pos, n, -1.0, 0.5), ref.fill_gaussian(seed, sid, pos, n, -1.0, 0.5))
        assert eq(oracle.fill_uniform(seed, sid, pos, n, -3.0, 7.5), ref.fill_uniform(seed, sid, pos, n, -3.0, 7.5))
    x = np.exp(rs.uniform(-600, 600, 5000))
    for fn in (0, 1):
        assert eq(oracle.fastmath(fn, x), ref.fastmath(fn, x))
    z = rs.uniform(-1100, 1100, 5000)
    assert eq(oracle.fastmath(2, z), ref.fastmath(2, z))
    a = rs.uniform(-4, 4, 5000)
    for fn in (3, 4):
        assert eq(oracle.fastmath(fn, a), ref.fastmath(fn, a))
    b, e = rs.uniform(1, 2000, 5000), rs.uniform(-8, 8, 5000)
    assert eq(oracle.fastmath(5, b, e), ref.fastmath(5, b, e))
    m = M.logistic_model(steps=200, obs_stride=20)
    obs = ref.logistic_simulate(m, [0.4, 80.0, 0.1], 5, 1, 7)
    assert eq(obs, oracle.simulate_at(m, [0.4, 80.0, 0.1], 5, 1, 7))
    for workers, width in [(1, 1), (3, 4), (5, 16), (7, 2)]:
        want = ref.logistic_abc(m, 333, workers, width, 42, obs)
        got = oracle.abc_prior_predictive(m, M.keying(42, A.VXB_KEY_WORKER, workers, width), 333, 0, 333, obs)
        for g, w in zip(got, want):
            assert eq(g, w)
        e1, i1 = ref.select_epsilon(want[2], want[3], 0.07)
        e2, i2 = oracle.select_epsilon(got[2], got[3], 0.07)
        assert e1 == e2 and eq(i1, i2)
    lw = rs.normal(size=2000) * 3
    parts = rs.normal(size=(2000, 3))
    assert oracle.ess(lw) == ref.ess(lw)
    o1, a1 = ref.resample_multinomial(lw, parts, 77, 9)
    o2, a2 = oracle.resample_multinomial(lw, parts, 77, 9)
    assert eq(a1, a2) and eq(o1, o2)
    base, k = rs.normal(size=50), rs.normal(size=400)
    assert eq(oracle.estimate_pvalues(base, k), ref.estimate_pvalues(base, k))


def test_ppp_counts_match_reference_counting(oracle, ref):
    """Config 2 on a small grid: the oracle's fused count equals the reference's
    estimate_pvalues applied to reference-drawn log densities."""
    n, m_total = 100, 300
    mdl = M.normal_mean_model(n)
    lam = np.array(M.lambda_grid(5))
    ln = np.array([-0.5 * math.log(2.0 * math.pi * (l * l + 1.0 / n)) for l in lam])
    ybar_obs = 2.9
    counts, pv, _ = oracle.ppp_pvalues(mdl, lam, ln, m_total, 0, m_total, 1337, ybar_obs)
    for k in range(lam.size):
        _, logm = ref.normal_mean_logm(1337, k, lam[k], ln[k], n, 0, m_total)
        v = lam[k] * lam[k] + 1.0 / n
        logm_obs = ln[k] - ((0.5 * ybar_obs) * ybar_obs) / v
        assert pv[k] == ref.estimate_pvalues([logm_obs], logm)[0]
        assert counts[k] == round(pv[k] * m_total)


# ------------------------------- properties pinned by the reference tests
def test_rng_properties(oracle):
    # test_rng.cpp:12-26 replay / divergence
    assert eq(oracle.fill_uniform(1337, 0, 0, 1000), oracle.fill_uniform(1337, 0, 0, 1000))
    assert not eq(oracle.fill_uniform(1337, 0, 0, 16), oracle.fill_uniform(1337, 1, 0, 16))
    # :28-49 cross-stream correlation
    x, y = oracle.fill_uniform(20240518, 0, 0, 100000), oracle.fill_uniform(20240518, 1, 0, 100000)
    assert abs(np.corrcoef(x, y)[0, 1]) < 0.02
    # :51-56 degenerate range exact
    assert (oracle.fill_uniform(7, 3, 0, 100, 3.0, 3.0) == 3.0).all()
    # :58-66 mean, :91-101 variance
    assert abs(oracle.fill_uniform(99, 0, 0, 100000).mean() - 0.5) < 0.005
    assert abs(oracle.fill_gaussian(31337, 2, 0, 100000).var(ddof=1) - 1.0) < 0.03
    # :68-77 half-open ranges
    for a, b in [(0.0, 1.0), (-3.0, 7.5), (1e16, 1e16 + 4.0), (250.0, 400.0)]:
        u = oracle.fill_uniform(4242, 1, 0, 4096, a, b)
        assert u.min() >= a and u.max() < b
    # :79-83, :112-118 error codes
    from oracle.pyoracle import OracleError
    with pytest.raises(OracleError) as e:
        oracle.fill_uniform(1, 1, 0, 4, 2.0, 1.0)
    assert e.value.code == "invalid-range"
    with pytest.raises(OracleError) as e:
        oracle.fill_gaussian(0, 0, 0, 4, 0.0, -1.0)
    assert e.value.code == "invalid-scale"
    # :85-89 zero sigma exact
    assert (oracle.fill_gaussian(8, 0, 0, 100, 5.0, 0.0) == 5.0).all()
    # :120-156 purity in the counter
    whole = oracle.fill_gaussian(777, 5, 0, 40)
    assert eq(np.concatenate([oracle.fill_gaussian(777, 5, 0, 16), oracle.fill_gaussian(777, 5, 16, 24)]), whole)
    assert oracle.fill_gaussian(777, 5, 21, 1)[0] == whole[21]
    assert oracle.fill_gaussian(777, 5, 20, 1)[0] == whole[20]
    wu = oracle.fill_uniform(123456789, 17, 0, 256, -1.0, 1.0)
    for off in (1, 7, 128, 255):
        assert eq(oracle.fill_uniform(123456789, 17, off, 256 - off, -1.0, 1.0), wu[off:])
    # :158-175 KS screen
    n, crit, passed = 10000, 1.62762 / math.sqrt(10000), 0
    for seed in range(100):
        xs = np.sort(oracle.fill_uniform(seed, 0, 0, n))
        i = np.arange(n)
        d = max(((i + 1) / n - xs).max(), (xs - i / n).max())
        passed += d < crit
    assert passed >= 95
    # :177-184 derive_seed path sensitivity
    s1 = oracle.derive_seed(42, [1, 2, 3])
    assert s1 != oracle.derive_seed(42, [1, 2, 4]) and s1 != oracle.derive_seed(42, [1, 2])


def test_fastmath_properties(oracle):
    def rel(got, want):
        return np.abs(got - want) / np.abs(want)
    x = np.array([1e-6, 0.001, 0.3, 0.9999, 1.0000001, 1.5, 2.0, 10.0, 325.0, 1650.0, 1e8])
    lg = oracle.fastmath(0, x)
    assert (rel(lg[x != 1.0], np.log2(x[x != 1.0])) < 1e-14).all()  # test_fastmath.cpp:19-25
    assert oracle.fastmath(0, [1.0, 2.0]).tolist() == [0.0, 1.0]
    z = np.array([-700.0, -30.0, -1.25, -0.4999, 0.0, 0.5, 1.0, 13.7, 100.0, 900.0])
    assert (rel(oracle.fastmath(2, z), np.exp2(z)) < 1e-14).all()  # :27-32
    b = np.repeat([1.0, 1.01, 2.5, 10.0, 42.0, 400.0, 1650.0], 8)
    e = np.tile([0.0, 0.05, 0.2, 0.35, 1.0, 3.5, 6.999, 7.0], 7)
    assert (rel(oracle.fastmath(5, b, e), np.power(b, e)) < 5e-13).all()  # :34-42
    assert oracle.fastmath(5, [10.0, 1650.0, 1.0, 1.0], [0.0, 0.0, 6.3, 0.0]).tolist() == [1.0] * 4
    a = 2.0 * np.arange(2000) / 2000.0
    assert np.abs(oracle.fastmath(3, a) - np.sin(np.pi * a)).max() < 1e-13  # :51-61
    assert np.abs(oracle.fastmath(4, a) - np.cos(np.pi * a)).max() < 1e-13
    xl = np.array([1e-300, 2.2e-16, 0.5, 1.0 - 2.0 ** -53, 3.7, 1e10])
    assert (rel(oracle.fastmath(1, xl), np.log(xl)) < 1e-13).all()  # :63-71
    assert oracle.fastmath(1, [1.0])[0] == 0.0


def test_numeric_and_partition_properties(oracle):
    from oracle.pyoracle import OracleError
    assert oracle.quantile(np.arange(1.0, 101.0), 0.5) == 50.5  # test_numeric.cpp:20-29
    assert oracle.quantile([1.0, 2.0, 3.0], 0.0) == 1.0 and oracle.quantile([1.0, 2.0, 3.0], 1.0) == 3.0
    assert abs(oracle.quantile(np.linspace(0.1, 1.0, 10), 0.5) - 0.55) < 1e-15
    ok, L = oracle.cholesky([[4.0, 2.0], [2.0, 3.0]])  # :31-42
    assert ok and np.allclose(L, [[2.0, 0.0], [1.0, math.sqrt(2.0)]])
    assert not oracle.cholesky([[1.0, 2.0], [2.0, 4.0]])[0]
    cov = oracle.sample_covariance([[0.0, 0.0], [1.0, 0.0], [0.0, 1.0], [1.0, 1.0]])  # :44-51
    assert np.allclose(cov, [[1 / 3, 0.0], [0.0, 1 / 3]])
    assert abs(oracle.logsumexp([0.0, 0.0]) - math.log(2.0)) < 1e-15  # :12-18
    r = oracle.partition(8064, 16, 4)  # test_blocked.cpp:38-48
    assert (r[:, 1] - r[:, 0] == 504).all()
    for total, workers, width in [(1003, 7, 8), (5, 9, 1), (100, 3, 16), (17, 4, 4)]:  # :63-84
        r = oracle.partition(total, workers, width).astype(np.int64)
        assert r[0, 0] == 0 and r[-1, 1] == total
        assert (r[1:, 0] == r[:-1, 1]).all()
        inner = r[:-1, 1][r[:-1, 1] < total]
        assert (inner % width == 0).all()
    with pytest.raises(OracleError) as e:
        oracle.partition(0, 1, 1)
    assert e.value.code == "invalid-shape"
    # SPEC.md examples for the untested pieces
    assert oracle.discrepancy([0.0, 0.0], [3.0, 4.0]) == 5.0
    eps, idx = oracle.select_epsilon([1.0, 2.0, 3.0, 4.0], None, 0.5)
    assert idx.tolist() == [0, 1]
    assert abs(oracle.ess(np.log([1.0, 1.0, 2.0])) - 16.0 / 6.0) < 1e-14
    assert oracle.estimate_pvalues([2.0, 5.0], [1.0, 3.0, 4.0, 6.0]).tolist() == [0.25, 0.75]
    with pytest.raises(OracleError) as e:
        oracle.select_epsilon([np.nan], [1], 0.5)
    assert e.value.code == "empty-set"
    with pytest.raises(OracleError) as e:
        oracle.select_epsilon([1.0], None, 0.0)
    assert e.value.code == "invalid-argument"


def test_logistic_analytic_anchors(oracle):
    """sigma = 0 => the deterministic Euler iterate of the logistic ODE (the
    hand-evaluable anchor in the style of test_toggle.cpp:95-113)."""
    m = M.logistic_model(steps=300, obs_stride=100, prior_lo=(0.5, 100.0, 0.0), prior_hi=(0.5, 100.0, 0.0))
    p, s, rho, f = oracle.abc_prior_predictive(m, M.keying(3), 4, 0, 4, [0.0, 0.0, 0.0])
    assert (p == [0.5, 100.0, 0.0]).all()
    x, want = 10.0, []
    a, inv_k = 0.5 * 0.01, 1.0 / 100.0
    for j in range(300):
        x = (x + (a * x) * (1.0 - x * inv_k)) + (0.0 * x) * 0.0
        if (j + 1) % 100 == 0:
            want.append(x)
    assert eq(s[0], want) and eq(s[3], want)
    assert rho[0] == math.sqrt(sum(v * v for v in want))
    # long horizon: X settles near K
    m2 = M.logistic_model(prior_lo=(0.9, 120.0, 0.01), prior_hi=(0.9, 120.0, 0.01))
    p, s, rho, f = oracle.abc_prior_predictive(m2, M.keying(3), 8, 0, 8, np.zeros(20))
    assert np.abs(s[:, -1] - 120.0).max() < 5.0
    # sharding / thread count do not change results (particle keying)
    m3 = M.logistic_model(steps=100, obs_stride=10)
    a = oracle.abc_prior_predictive(m3, M.keying(5), 1000, 0, 1000, np.ones(10), threads=1)
    b1 = oracle.abc_prior_predictive(m3, M.keying(5), 1000, 0, 400, np.ones(10), threads=3)
    b2 = oracle.abc_prior_predictive(m3, M.keying(5), 1000, 400, 600, np.ones(10), threads=8)
    for x0, x1, x2 in zip(a, b1, b2):
        assert eq(x0, np.concatenate([x1, x2]))


def test_tb_gillespie_restatement_equals_reference(oracle, ref):
    """tb::gillespie_simulate / tb_summaries / sample_prior / tb_observed_summaries:
    the oracle's restatement against the unmodified reference, bit for bit (state,
    summaries and the stream position a path stops at)."""
    for theta, seed in [((0.2, 0.1, 0.05), 5), ((1.5, 0.3, 0.9), 6), ((0.4, 0.39, 0.2), 7),
                        ((0.0, 0.0, 0.0), 8), ((0.3, 0.0, 0.0), 9), ((0.1, 1.9, 0.5), 10)]:
        a = ref.tb_simulate(theta, 10, 10.0, 10000.0, seed, 2, 3)
        b = oracle.tb_simulate(theta, 10, 10.0, 10000.0, seed, 2, 3)
        for k in a:
            assert np.array_equal(a[k], b[k], equal_nan=True), (theta, k)
    assert np.array_equal(ref.tb_observed(10, 10.0, 10000.0, 1337), oracle.tb_observed(10, 10.0, 10000.0, 1337))
    obs = [10.0, 0.7]
    for initial, horizon, target in ((10, 10.0, 10000.0), (3, 25.0, 400.0)):
        a = ref.tb_abc_particle(initial, horizon, target, 5, 64, 1337, obs)
        b = oracle.tb_abc_particle(initial, horizon, target, 5, 64, 1337, obs)
        for x, y in zip(a, b):
            assert np.array_equal(x, y, equal_nan=True)
        assert a[3].any()


def test_libm_exp_restatement_equals_live_libm(oracle):
    """The exp algorithm csrc/vxb_libmexp.cuh runs on the device (glibc's N = 128 table
    scheme, FMA build) restated on the CPU: identical, bit for bit, to this machine's
    std::exp -- the function the reference's weight algebra calls (smc.cpp:214,278,299,
    numeric.cpp:16-17).  Sweeps cover the weight domain (x <= 0), the subnormal and
    underflow range, overflow, tiny arguments and the special values."""
    for lo, hi, n in ((-50.0, 0.0, 6_000_000), (-760.0, -690.0, 2_000_000),
                      (-1100.0, 800.0, 2_000_000), (-1e-3, 1e-3, 1_000_000),
                      (700.0, 712.0, 500_000), (-1e-15, 1e-15, 200_000)):
        bad, first = oracle.exp_restated_sweep(20240 + int(n), n, lo, hi)
        assert bad == 0, (lo, hi, first)
    x = np.array([0.0, -0.0, 1e-300, -1e-300, 1e-17, -745.2, -745.13321910194122, -746.0,
                  -708.4, -709.0, 709.78, 709.79, 710.0, np.inf, -np.inf, np.nan, -1023.9,
                  -1024.0, -5e-324, 2.0 ** -54, -(2.0 ** -55), 512.0, -512.0, -511.99999,
                  1.0, -1.0, 0.5 * math.log(2.0), -math.log(2.0) / 256.0])
    got, live = oracle.exp_restated(x)
    assert np.array_equal(got.view(np.uint64), live.view(np.uint64))
    assert np.array_equal(live[:11].view(np.uint64),
                          np.array([math.exp(v) for v in x[:11]]).view(np.uint64))
    # the two builds of the library differ (about one argument in 10^3): this process
    # runs the FMA build, so the plain restatement must NOT match everywhere ...
    bad_plain, _ = oracle.exp_restated_sweep(1, 2_000_000, -50.0, 0.0, plain_build=True)
    assert 100 < bad_plain < 20_000


def test_libm_exp_plain_build_restatement_equals_live_libm_without_fma():
    """... and in a process whose libm is told to ignore FMA / AVX2 (GLIBC_TUNABLES, the
    ifunc then picks the plain build -- what a host CPU without FMA runs), the PLAIN
    restatement equals the live std::exp bit for bit and the FMA one does not."""
    import subprocess
    import sys
    code = """
import sys
sys.path.insert(0, %r)
from oracle.pyoracle import Oracle
o = Oracle()
for lo, hi, n in ((-50.0, 0.0, 4000000), (-760.0, -690.0, 1000000), (-1100.0, 800.0, 1000000), (-1e-3, 1e-3, 500000)):
    bad, first = o.exp_restated_sweep(77 + n, n, lo, hi, plain_build=True)
    assert bad == 0, (lo, hi, first)
bad_fma, _ = o.exp_restated_sweep(1, 2000000, -50.0, 0.0, plain_build=False)
assert 100 < bad_fma < 20000, bad_fma
print("plain build ok", bad_fma)
""" % os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, GLIBC_TUNABLES="glibc.cpu.hwcaps=-AVX2,-FMA")
    run = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600, env=env)
    assert run.returncode == 0 and "plain build ok" in run.stdout, run.stdout[-800:] + run.stderr[-1500:]


def test_libm_exp_table_is_what_the_generator_emits():
    """csrc/vxb_libm_exp_entries.inc is generated (exact integer arithmetic); the committed
    file must be exactly the generator's output, and entry 0 / 64 are 1 and sqrt(2)."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, os.path.join(root, "scripts", "gen_libm_exp_table.py")],
                         capture_output=True, text=True, check=True).stdout
    committed = open(os.path.join(root, "paper_1902_09046_b200", "csrc", "vxb_libm_exp_entries.inc")).read()
    assert out == committed
    rows = [l for l in committed.splitlines() if l.startswith("VXB_EXP_PAIR")]
    assert len(rows) == 128 and "0x3ff0000000000000ull" in rows[0]
    h64 = int(rows[64].split(",")[1].strip(" )ull").replace("ull", ""), 16) + ((64 << 52) // 128)
    assert np.array([h64], dtype=np.uint64).view(np.float64)[0] == math.sqrt(2.0)
