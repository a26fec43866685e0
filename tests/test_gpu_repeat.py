"""Repeatability of the kernels with shared-memory hand-offs and atomics (SURVEY.md
section 5, "race detection": compute-sanitizer's racecheck is closed on this pool).
A data race shows up as a result that depends on scheduling; every one of these
kernels is therefore launched many times on identical inputs -- alone and with a
second context keeping the SMs busy on another stream -- and its output must be
bit-identical every time (and, elsewhere in the suite, identical to the oracle)."""
import threading

import numpy as np
import pytest

from paper_1902_09046_b200 import _abi as A, lib, models as M

pytestmark = pytest.mark.gpu
REPS = 12


def same(results):
    first = results[0]
    for r in results[1:]:
        for a, b in zip(first, r):
            if not np.array_equal(np.asarray(a), np.asarray(b), equal_nan=True):
                return False
    return True


def early(c, call):
    c.set_early_reject(True)
    try:
        return call()
    finally:
        c.set_early_reject(False)


@pytest.mark.timeout(900)
def test_kernels_with_shared_memory_or_atomics_are_repeatable(ctx, golden):
    obs = golden["logistic_observed"]
    m = M.logistic_model(steps=200, obs_stride=10)
    o = obs[:20]
    n = 30011
    p, s, rho, f = ctx.abc_prior_predictive_host(m, M.keying(5), n, 0, n, o)
    rs = np.random.RandomState(2)
    lw = rs.normal(size=20001) * 4
    parts = rs.normal(size=(20001, 3))
    mc = A.vxb_mlmc_cfg()
    mc.levels, mc.refine, mc.tau0, mc.t_end, mc.paths, mc.seed = 3, 4, 1.0, 30.0, 3001, 7
    tbm = M.tb_model(10, 3.0, 300.0)
    tb_obs = ctx.simulate_at(M.tb_model(10, 3.0, 300.0, attempts=64), M.TB_TRUE_THETA, lib.derive_seed(1337, [91]), 0, 0)
    tm = M.toggle_model(40, 512)
    tobs = ctx.simulate_at(tm, M.TOGGLE_MIDPOINT, lib.derive_seed(1337, [90]), 0, 0)
    wcfg = M.weakinfo_config(hyper_count=3, datasets=7, particles=100, seed=11)
    cfg = A.vxb_abcsmc_cfg()
    cfg.particles, cfg.generations, cfg.quantile, cfg.kernel_scale = 900, 3, 0.5, 2.0
    cfg.jitter, cfg.round_size, cfg.max_rounds, cfg.seed = 1e-10, 400, 0, 3
    cases = {
        "select_epsilon (radix_hist / pick, accept_count / scan / write)":
            lambda c: c.select_epsilon(rho, f, 0.013)[:2],
        "order_statistics": lambda c: (c.order_statistics(rho, f, [0, 17, n // 3, n - 200])[0],),
        "abc_reject (compaction + gather)": lambda c: c.abc_reject(m, M.keying(5), n, 0, n, o, 40.0, cap=n)[1:],
        "abc_reject with early rejection (survivor queues filled through warp-aggregated atomics)":
            lambda c: early(c, lambda: c.abc_reject(m, M.keying(5), 90011, 0, 90011, o, 40.0, cap=90011)[1:]),
        "resample / ess (sequential exp-sum hand-off between warps)":
            lambda c: c.resample_multinomial(lw, parts, 77, 9) + (np.array([c.ess(lw), c.logsumexp(lw)]),),
        "tauleap (shared sums, atomics)": lambda c: tuple(c.mlmc_tauleap(M.mm_tauleap_model(), mc)[k]
                                                          for k in ("level_mean", "level_var")),
        "tb_abc (three-level counts, persistent CTAs)":
            lambda c: c.abc_prior_predictive_host(tbm, M.keying(3), 257, 0, 257, tb_obs),
        "toggle (in-CTA sort)": lambda c: c.abc_prior_predictive_host(tm, M.keying(3), 9, 0, 9, tobs),
        "anneal (one CTA per run)": lambda c: (c.weak_info_test(wcfg, want_evidence=True)["evidence"],),
        "abcsmc (canonical reductions, pack / append)": lambda c: tuple(
            c.sharded_abcsmc_run(None, M.logistic_model(steps=200, obs_stride=10), cfg, o)[k]
            for k in ("theta", "weight", "rho")),
    }
    # a second context hammering the device from another host thread changes the scheduling
    other = lib.Context(0)
    stop = threading.Event()

    def noise():
        big = M.logistic_model(steps=400, obs_stride=20, rng=A.VXB_RNG_FAST)
        while not stop.is_set():
            other.abc_reject(big, M.keying(1), 200000, 0, 200000, np.zeros(20), 1.0, cap=16)

    failures = []
    for name, fn in cases.items():
        quiet = [fn(ctx) for _ in range(REPS)]
        t = threading.Thread(target=noise)
        stop.clear()
        t.start()
        try:
            busy = [fn(ctx) for _ in range(REPS)]
        finally:
            stop.set()
            t.join()
        if not same(quiet + busy):
            failures.append(name)
    other.close()
    assert not failures, failures
