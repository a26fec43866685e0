"""Likelihood-annealed SMC on the bioassay model and the weak-informativity test
(SURVEY.md 8f-3).  CPU: the oracle restatement against golden values of the
unmodified reference (tests/golden/make_golden_anneal.py) and, where
oracle/_ref is present, against the live reference -- bit for bit.  GPU: the
one-CTA-per-run device sampler against the oracle: model evaluations and
datasets bit-exact; evidences to 1e-9 (the device calls exp/log where the
reference calls libm and sums in a fixed tree order) with identical iteration
counts, step counts and acceptance rates; the cut-off table identical."""
import os
import sys

import numpy as np
import pytest

from paper_1902_09046_b200 import lib, models as M

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
import make_golden_anneal as G  # noqa: E402


@pytest.fixture(scope="module")
def gold():
    return np.load(os.path.join(ROOT, "tests", "golden", "anneal.npz"))


def test_oracle_matches_reference_golden(oracle, gold):
    assert np.array_equal(oracle.bioassay_ll(gold["ll_beta"], G.DOSE, G.SIZE, [0, 2, 5, 1]), gold["ll_values"])
    for j, (l1, l2, ds, ss, npart) in enumerate(G.RUNS):
        th, y = oracle.bioassay_sample(l1, l2, G.DOSE, G.SIZE, ds)
        assert np.array_equal(th, gold["run_theta"][j]) and np.array_equal(y, gold["run_deaths"][j])
        ev, it, tr = oracle.smc_bioassay(G.DOSE, G.SIZE, y, l1, l2, npart, 4, 0.01, G.H, ss, True)
        assert ev == gold["run_evidence"][j] and it == gold["run_iterations"][j]
        # the reference prints its trace with 17 significant digits
        assert np.allclose(tr, gold["run_trace"][j][:it], rtol=1e-15, atol=0)
        assert np.array_equal(tr[:, 2:], gold["run_trace"][j][:it, 2:])
    # the whole SmcResult of one run: final ensemble and the trace's evidence column
    l1, l2, ds, ss, npart = G.RUNS[G.ENSEMBLE_RUN]
    e = oracle.smc_bioassay_ensemble(G.DOSE, G.SIZE, gold["run_deaths"][G.ENSEMBLE_RUN], l1, l2, npart, 4,
                                     0.01, G.H, ss)
    assert e["log_evidence"] == gold["run_evidence"][G.ENSEMBLE_RUN]
    assert np.array_equal(e["particles"], gold["ens_particles"])
    assert np.array_equal(np.stack([e["log_weights"], e["log_liks"], e["log_priors"]]), gold["ens_rows"])
    assert np.allclose(e["trace"], gold["ens_trace"], rtol=1e-15, atol=0)
    # SmcConfig::esjd = true: scale adaptation (sweeps until half the ensemble has moved)
    for j, (l1, l2, ds, ss, npart, scales) in enumerate(G.ESJD_RUNS):
        e = oracle.smc_bioassay_ensemble(G.DOSE, G.SIZE, gold[f"esjd{j}_deaths"], l1, l2, npart, 4, 0.01, 0.0,
                                         ss, esjd_scales=scales)
        assert e["log_evidence"] == gold[f"esjd{j}_evidence"][0], j
        assert np.array_equal(e["particles"], gold[f"esjd{j}_particles"]), j
        assert np.array_equal(e["trace"][:, [2, 3]], gold[f"esjd{j}_trace"][:, [2, 3]]), j   # sweeps, acceptance
        assert np.allclose(e["trace"], gold[f"esjd{j}_trace"], rtol=1e-15, atol=0), j
    for redraw in (0, 1):
        t = oracle.weak_info_test(G.TABLE["hyper_count"], G.TABLE["datasets"], G.TABLE["particles"],
                                  seed=G.TABLE["seed"], redraw_base=bool(redraw), workers=4)
        for k, v in t.items():
            assert np.array_equal(v, gold[f"table{redraw}_{k}"]), (redraw, k)


def test_oracle_matches_live_reference(oracle, ref):
    rs = np.random.RandomState(11)
    for trial in range(4):
        l1, l2 = rs.uniform(0.1, 10.0), rs.uniform(0.1, 20.0)
        th, y = ref.bioassay_sample(l1, l2, G.DOSE, G.SIZE, 1000 + trial)
        th2, y2 = oracle.bioassay_sample(l1, l2, G.DOSE, G.SIZE, 1000 + trial)
        assert np.array_equal(th, th2) and np.array_equal(y, y2)
        a = ref.smc_bioassay(G.DOSE, G.SIZE, y, l1, l2, 300, 8, 0.05, 0.9, 7 * trial)
        b = oracle.smc_bioassay(G.DOSE, G.SIZE, y, l1, l2, 300, 8, 0.05, 0.9, 7 * trial)
        assert a == b
        ea = ref.smc_bioassay_ensemble(G.DOSE, G.SIZE, y, l1, l2, 300, 8, 0.05, 0.9, 7 * trial)
        eb = oracle.smc_bioassay_ensemble(G.DOSE, G.SIZE, y, l1, l2, 300, 8, 0.05, 0.9, 7 * trial)
        for k in ("particles", "log_weights", "log_liks", "log_priors"):
            assert np.array_equal(ea[k], eb[k]), k
        for scales in ((0.3, 0.6, 0.9, 1.2), (6.0, 12.0)):
            ea = ref.smc_bioassay_ensemble(G.DOSE, G.SIZE, y, l1, l2, 301, 8, 0.05, 0.0, 7 * trial, esjd_scales=scales)
            eb = oracle.smc_bioassay_ensemble(G.DOSE, G.SIZE, y, l1, l2, 301, 8, 0.05, 0.0, 7 * trial,
                                              esjd_scales=scales)
            assert ea["log_evidence"] == eb["log_evidence"] and ea["iterations"] == eb["iterations"]
            assert np.array_equal(ea["particles"], eb["particles"]) and np.array_equal(ea["trace"], eb["trace"])
    a = ref.weak_info_test(2, 6, 100, seed=5)
    b = oracle.weak_info_test(2, 6, 100, seed=5)
    for k in a:
        assert np.array_equal(a[k], b[k], equal_nan=True), k
    # argument errors of the sampler (smc.cpp:356-364)
    from oracle.pyoracle import OracleError
    for o in (ref, oracle):
        with pytest.raises(OracleError) as e:
            o.smc_bioassay(G.DOSE, G.SIZE, [1, 1, 1, 1], 1.0, 1.0, 7, 4, 0.01, 1.0, 1)
        assert str(e.value).startswith("invalid-shape")
        with pytest.raises(OracleError) as e:
            o.smc_bioassay(G.DOSE, G.SIZE, [1, 1, 1, 1], 1.0, 1.0, 64, 3, 0.01, 1.0, 1)
        assert str(e.value).startswith("invalid-shape")


# ------------------------------------------------------------------ device
@pytest.mark.gpu
def test_device_model_and_datasets_bit_exact(ctx, oracle, gold):
    assert np.array_equal(ctx.bioassay_log_likelihood(gold["ll_beta"], G.DOSE, G.SIZE, [0, 2, 5, 1]),
                          gold["ll_values"])
    rs = np.random.RandomState(2)
    n = 500
    lam = np.stack([rs.uniform(0.1, 10.0, n), rs.uniform(0.1, 20.0, n)], axis=1)
    seeds = rs.randint(0, 2 ** 62, size=n).astype(np.uint64)
    theta, deaths = ctx.bioassay_sample(lam, seeds, G.DOSE, G.SIZE)
    for j in range(0, n, 7):
        th, y = oracle.bioassay_sample(lam[j, 0], lam[j, 1], G.DOSE, G.SIZE, int(seeds[j]))
        assert np.array_equal(theta[j], th) and np.array_equal(deaths[j], y)
    assert deaths.max() == 5 and deaths.min() == 0
    # a design with large groups uses the device-side binomial table
    dose, size = (-1.0, 0.0, 0.5), (40, 12, 9)
    beta = rs.normal(size=(32, 2)) * 3
    assert np.array_equal(ctx.bioassay_log_likelihood(beta, dose, size, [17, 0, 9]),
                          oracle.bioassay_ll(beta, dose, size, [17, 0, 9]))


@pytest.mark.gpu
def test_device_sampler_matches_oracle(ctx, oracle, gold):
    lam = np.array([[r[0], r[1]] for r in G.RUNS])
    seeds = np.array([r[3] for r in G.RUNS], dtype=np.uint64)
    for npart in sorted({r[4] for r in G.RUNS}):
        sel = [j for j, r in enumerate(G.RUNS) if r[4] == npart]
        res = ctx.smc_bioassay(G.DOSE, G.SIZE, gold["run_deaths"][sel], lam[sel], seeds[sel], npart,
                               trace_rows=8)
        assert (res["status"] == 0).all()
        assert np.array_equal(res["iterations"], gold["run_iterations"][sel])
        assert np.allclose(res["log_evidence"], gold["run_evidence"][sel], rtol=0, atol=1e-9)
        want = gold["run_trace"][sel]
        assert np.array_equal(res["trace"][:, :, 2:4], want[:, :, 2:])          # R_n and p_acc: identical
        assert np.allclose(res["trace"][:, :, :2], want[:, :, :2], rtol=1e-9, atol=1e-9)
    # a larger random batch against the oracle, other tuning constants and widths
    rs = np.random.RandomState(5)
    n = 96
    lam = np.stack([rs.uniform(0.1, 10.0, n), rs.uniform(0.1, 20.0, n)], axis=1)
    seeds = rs.randint(0, 2 ** 62, size=n).astype(np.uint64)
    _, deaths = ctx.bioassay_sample(lam, seeds ^ np.uint64(0xABCDEF), G.DOSE, G.SIZE)
    res = ctx.smc_bioassay(G.DOSE, G.SIZE, deaths, lam, seeds, 250, block_width=8, c=0.05, scale=0.9)
    for j in range(n):
        ev, it = oracle.smc_bioassay(G.DOSE, G.SIZE, deaths[j], lam[j, 0], lam[j, 1], 250, 8, 0.05, 0.9,
                                     int(seeds[j]))
        assert res["iterations"][j] == it and abs(res["log_evidence"][j] - ev) < 1e-9, j
    # argument errors mirror the reference sampler
    for kwargs, code in ((dict(particles=7), "invalid-shape"), (dict(particles=64, block_width=3), "invalid-shape"),
                         (dict(particles=64, c=1.5), "invalid-argument")):
        with pytest.raises(lib.VxbError) as e:
            ctx.smc_bioassay(G.DOSE, G.SIZE, deaths[:2], lam[:2], seeds[:2], **kwargs)
        assert e.value.code == code
    with pytest.raises(lib.VxbError) as e:
        ctx.smc_bioassay(G.DOSE, G.SIZE, [[9, 0, 0, 0]], lam[:1], seeds[:1], 64)
    assert e.value.code == "invalid-argument"


@pytest.mark.gpu
def test_device_run_smc_result(ctx, oracle, gold):
    """vxb_smc_bioassay_ensemble = smc::run_smc's SmcResult: same accept/resample decisions,
    so the final ensemble agrees to rounding (the proposal factor differs by ulps)."""
    l1, l2, ds, ss, npart = G.RUNS[G.ENSEMBLE_RUN]
    e = ctx.smc_bioassay_ensemble(G.DOSE, G.SIZE, gold["run_deaths"][G.ENSEMBLE_RUN], [l1, l2], ss, npart,
                                  scale=G.H)
    assert e["iterations"] == gold["run_iterations"][G.ENSEMBLE_RUN]
    assert abs(e["log_evidence"] - gold["run_evidence"][G.ENSEMBLE_RUN]) < 1e-9
    assert np.allclose(e["particles"], gold["ens_particles"], rtol=1e-9, atol=1e-9)
    assert np.allclose(np.stack([e["log_weights"], e["log_liks"], e["log_priors"]]), gold["ens_rows"],
                       rtol=1e-9, atol=1e-9)
    assert np.array_equal(e["trace"][:, 2:4], gold["ens_trace"][:, 2:4])
    assert np.allclose(e["trace"], gold["ens_trace"], rtol=1e-9, atol=1e-9)
    rs = np.random.RandomState(21)
    for trial, (npart, bw) in enumerate(((1000, 4), (250, 8), (2000, 4), (96, 16))):
        l1, l2 = rs.uniform(0.1, 10.0), rs.uniform(0.1, 20.0)
        _, y = oracle.bioassay_sample(l1, l2, G.DOSE, G.SIZE, 50 + trial)
        want = oracle.smc_bioassay_ensemble(G.DOSE, G.SIZE, y, l1, l2, npart, bw, 0.01, 0.0, 900 + trial)
        got = ctx.smc_bioassay_ensemble(G.DOSE, G.SIZE, y, [l1, l2], 900 + trial, npart, block_width=bw,
                                        scale=0.0)
        assert got["iterations"] == want["iterations"]
        assert abs(got["log_evidence"] - want["log_evidence"]) < 1e-9
        for k in ("particles", "log_weights", "log_liks", "log_priors", "trace"):
            assert np.allclose(got[k], want[k], rtol=1e-9, atol=1e-9), (trial, k)
        # the batched entry point runs the same sampler
        one = ctx.smc_bioassay(G.DOSE, G.SIZE, [y], [[l1, l2]], [900 + trial], npart, block_width=bw, scale=0.0)
        assert one["log_evidence"][0] == got["log_evidence"]
    # sampler failures are errors here, as in the reference (status codes in the batched call)
    with pytest.raises(lib.VxbError) as err:
        ctx.smc_bioassay_ensemble(G.DOSE, G.SIZE, [0, 0, 0, 0], [1.0, 1.0], 1, 7)
    assert err.value.code == "invalid-shape"


@pytest.mark.gpu
def test_device_run_smc_esjd(ctx, oracle, gold):
    """SmcConfig::esjd = true on the device (esjd_core, smc.cpp:156-204): the same trial
    acceptance, chosen scale and number of sweeps per iteration as the reference, the
    same accept decisions, evidences and ensembles to rounding."""
    for j, (l1, l2, ds, ss, npart, scales) in enumerate(G.ESJD_RUNS):
        e = ctx.smc_bioassay_ensemble(G.DOSE, G.SIZE, gold[f"esjd{j}_deaths"], [l1, l2], ss, npart, scale=0.0,
                                      esjd_scales=scales)
        want = gold[f"esjd{j}_trace"]
        assert e["iterations"] == len(want)
        assert abs(e["log_evidence"] - gold[f"esjd{j}_evidence"][0]) < 1e-9, j
        assert np.array_equal(e["trace"][:, [2, 3, 5]], want[:, [2, 3, 5]]), j   # sweeps, acceptance, scale
        assert np.allclose(e["trace"], want, rtol=1e-9, atol=1e-9), j
        assert np.allclose(e["particles"], gold[f"esjd{j}_particles"], rtol=1e-9, atol=1e-9), j
    rs = np.random.RandomState(31)
    many_sweeps = 0
    for trial, (npart, scales) in enumerate(((1000, G.GRID), (255, (5.0, 10.0, 15.0)), (96, (0.4,)),
                                             (2000, G.GRID), (501, (8.0,)), (128, tuple(0.05 * k for k in range(1, 17))))):
        l1, l2 = rs.uniform(0.1, 10.0), rs.uniform(0.1, 20.0)
        _, y = oracle.bioassay_sample(l1, l2, G.DOSE, G.SIZE, 70 + trial)
        want = oracle.smc_bioassay_ensemble(G.DOSE, G.SIZE, y, l1, l2, npart, 4, 0.01, 0.0, 500 + trial,
                                            esjd_scales=scales)
        got = ctx.smc_bioassay_ensemble(G.DOSE, G.SIZE, y, [l1, l2], 500 + trial, npart, scale=0.0,
                                        esjd_scales=scales)
        assert got["iterations"] == want["iterations"]
        assert abs(got["log_evidence"] - want["log_evidence"]) < 1e-9
        assert np.array_equal(got["trace"][:, [2, 3, 5]], want["trace"][:, [2, 3, 5]]), trial
        for k in ("particles", "log_weights", "log_liks", "log_priors"):
            assert np.allclose(got[k], want[k], rtol=1e-9, atol=1e-9), (trial, k)
        many_sweeps += int((want["trace"][:, 2] >= 3).any())
    assert many_sweeps >= 1                                # the repeated-sweep loop was exercised
    with pytest.raises(lib.VxbError) as err:               # the device carries at most 16 scales
        ctx.smc_bioassay_ensemble(G.DOSE, G.SIZE, [0, 1, 2, 3], [1.0, 1.0], 1, 64, esjd_scales=[0.1] * 17)
    assert err.value.code == "invalid-argument"
    with pytest.raises(lib.VxbError) as err:
        ctx.smc_bioassay_ensemble(G.DOSE, G.SIZE, [0, 1, 2, 3], [1.0, 1.0], 1, 64, esjd_scales=[0.5, -1.0])
    assert err.value.code == "invalid-scale"


@pytest.mark.gpu
def test_device_weak_info_table_equals_reference(ctx, oracle, gold):
    for redraw in (0, 1):
        cfg = M.weakinfo_config(seed=G.TABLE["seed"], redraw_base=bool(redraw),
                                **{k: G.TABLE[k] for k in ("hyper_count", "datasets", "particles")})
        t = ctx.weak_info_test(cfg, want_evidence=True)
        assert np.array_equal(t["lambda_"], gold[f"table{redraw}_lambda_"])
        assert np.array_equal(t["gamma"], gold[f"table{redraw}_gamma"])
        assert np.array_equal(t["weakly"], gold[f"table{redraw}_weakly"])
        assert np.array_equal(t["completed"], gold[f"table{redraw}_completed"])
        assert np.isfinite(t["evidence"]).all()
    # a somewhat larger table against the oracle run here
    cfg = M.weakinfo_config(hyper_count=6, datasets=40, particles=128, seed=77, alpha=0.1)
    t = ctx.weak_info_test(cfg)
    o = oracle.weak_info_test(6, 40, 128, alpha=0.1, seed=77, workers=8)
    for k in ("lambda_", "gamma", "weakly", "completed"):
        assert np.array_equal(t[k], o[k]), k


@pytest.mark.gpu
def test_device_weak_info_fma_mode(ctx):
    """VXB_ARITH_FMA: the same random numbers and polynomials with contracted multiply-adds.
    Evidences agree with the reference-exact mode to rounding, the cut-off table is the same."""
    from paper_1902_09046_b200 import _abi as A
    kw = dict(hyper_count=6, datasets=40, particles=300, seed=77)
    for redraw in (False, True):
        exact = ctx.weak_info_test(M.weakinfo_config(redraw_base=redraw, **kw), want_evidence=True)
        fused = ctx.weak_info_test(M.weakinfo_config(redraw_base=redraw, arith=A.VXB_ARITH_FMA, **kw),
                                   want_evidence=True)
        assert np.allclose(exact["evidence"], fused["evidence"], rtol=0, atol=1e-9, equal_nan=True)
        assert not np.array_equal(exact["evidence"], fused["evidence"])      # it is a different instance
        for k in ("gamma", "weakly", "completed", "lambda_"):
            assert np.array_equal(exact[k], fused[k]), k
    with pytest.raises(lib.VxbError) as err:
        ctx.weak_info_test(M.weakinfo_config(arith=7, **kw))
    assert err.value.code == "invalid-argument"


@pytest.mark.gpu
def test_device_weak_info_throughput_generator(ctx):
    """VXB_RNG_FAST instance of the sampler (Philox4x32, table-based normals / log / softplus,
    FMA): other random numbers, so the check is statistical -- on the same datasets the
    evidence estimates are unbiased against the reference-exact instance (paired difference
    within 5 standard errors, of the size two independent N_p = 300 estimates differ by),
    equally distributed (two-sample KS at 1 %), and the p-value estimates move by Monte-Carlo
    noise only."""
    from paper_1902_09046_b200 import _abi as A
    kw = dict(hyper_count=8, datasets=150, particles=300, seed=2024)
    exact = ctx.weak_info_test(M.weakinfo_config(**kw), want_evidence=True)
    fast = ctx.weak_info_test(M.weakinfo_config(rng=A.VXB_RNG_FAST, **kw), want_evidence=True)
    a, b = exact["evidence"].ravel(), fast["evidence"].ravel()
    assert np.isfinite(b).all() and (fast["completed"] == kw["datasets"]).all()
    assert np.array_equal(exact["lambda_"], fast["lambda_"])         # same hyperparameters and datasets
    d = b - a
    assert abs(d.mean()) < 5.0 * d.std() / np.sqrt(d.size)
    assert 0.02 < d.std() < 0.5                                      # noise of two sampler runs, not a shift
    assert abs(b.std() / a.std() - 1.0) < 0.02
    xs = np.sort(np.concatenate([a, b]))
    ks = np.abs(np.searchsorted(np.sort(a), xs, side="right") / a.size
                - np.searchsorted(np.sort(b), xs, side="right") / b.size).max()
    assert ks < 1.628 * np.sqrt(2.0 / a.size)
    assert np.abs(exact["gamma"] - fast["gamma"]).max() < 0.06        # alpha-quantiles of 150 p-values each
    again = ctx.weak_info_test(M.weakinfo_config(rng=A.VXB_RNG_FAST, **kw), want_evidence=True)
    assert np.array_equal(again["evidence"], fast["evidence"])        # deterministic in the seed
    with pytest.raises(lib.VxbError) as err:
        ctx.weak_info_test(M.weakinfo_config(rng=5, **kw))
    assert err.value.code == "invalid-argument"


@pytest.mark.gpu
def test_device_weak_info_row_shards(ctx, gold):
    """Evidences of row ranges equal the rows of the whole table (seeds are keyed by
    row and dataset), so sharding hyperparameters over GPUs cannot change it."""
    from paper_1902_09046_b200 import dist as D
    for redraw in (False, True):
        cfg = M.weakinfo_config(hyper_count=5, datasets=9, particles=128, seed=3, redraw_base=redraw)
        whole = ctx.weak_info_test(cfg, want_evidence=True)
        lam = ctx.weak_info_lambdas(cfg)
        assert np.array_equal(lam, whole["lambda_"])
        parts = [ctx.weak_info_evidence(cfg, lam, a, b - a) for a, b in ((0, 2), (2, 3), (3, 6))]
        assert np.array_equal(np.concatenate(parts), whole["evidence"])
        t = D.sharded_weak_info(ctx, cfg)
        for k in ("gamma", "weakly", "completed"):
            assert np.array_equal(t[k], whole[k])


@pytest.mark.gpu
def test_device_sampler_other_designs_and_sizes(ctx, oracle):
    """Designs with large groups (device-side binomial table), other group counts,
    particle counts that are not multiples of the CTA size, near-degenerate priors."""
    rs = np.random.RandomState(12)
    for dose, size, npart in (((-1.0, 0.0, 0.5), (40, 12, 9), 333), ((0.2,), (7,), 64),
                              ((-2.0, -1.0, 0.0, 1.0, 2.0, 3.0), (3, 3, 3, 3, 3, 3), 1000)):
        n = 10
        lam = np.stack([rs.uniform(0.05, 10.0, n), rs.uniform(0.05, 20.0, n)], axis=1)
        seeds = rs.randint(0, 2 ** 62, size=n).astype(np.uint64)
        theta, deaths = ctx.bioassay_sample(lam, seeds, dose, size)
        res = ctx.smc_bioassay(dose, size, deaths, lam, seeds + np.uint64(1), npart, trace_rows=6)
        for j in range(n):
            th, y = oracle.bioassay_sample(lam[j, 0], lam[j, 1], dose, size, int(seeds[j]))
            assert np.array_equal(theta[j], th) and np.array_equal(deaths[j], y)
            ev, it, tr = oracle.smc_bioassay(dose, size, y, lam[j, 0], lam[j, 1], npart, 4, 0.01, G.H,
                                             int(seeds[j]) + 1, True)
            assert res["status"][j] == 0 and res["iterations"][j] == it
            assert abs(res["log_evidence"][j] - ev) < 1e-9
            k = min(it, 6)
            assert np.array_equal(res["trace"][j, :k, 2:4], tr[:k, 2:])
    # the whole test on a non-default design
    cfg = M.weakinfo_config(hyper_count=3, datasets=10, particles=96, seed=5, dose=(-1.0, 0.0, 0.5),
                            group_size=(8, 4, 6))
    t = ctx.weak_info_test(cfg)
    assert np.isfinite(t["gamma"]).all() and (t["completed"] == 10).all()
