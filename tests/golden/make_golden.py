"""Generates tests/golden/golden.npz from the UNMODIFIED reference library.

Run in the build container (needs /root/reference):

    make -C oracle ref && python tests/golden/make_golden.py

Every array below is an output of reference code reached through
oracle/ref_driver.cpp (RngStream, fastmath, numeric, partition,
abc::run_prior_predictive, abc::select_epsilon, smc::ess,
smc::resample_multinomial, weakinfo::estimate_pvalues, toggle::*).  The
fixtures travel to the GPU box, where /root/reference does not exist.
"""
import math
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle.pyoracle import Ref  # noqa: E402
from paper_1902_09046_b200 import _abi as A, models as M  # noqa: E402


def main():
    r = Ref()
    g = {}
    # ---- RNG known answers
    g["splitmix64_0"] = np.uint64(r.splitmix64(0))
    g["derive_seed_42_123"] = np.uint64(r.derive_seed(42, [1, 2, 3]))
    g["derive_seed_1_90"] = np.uint64(r.derive_seed(1, [90]))
    g["words_1337_0"] = r.stream_u64(1337, 0, 0, 64)
    g["words_7_3_pos1001"] = r.stream_u64(7, 3, 1001, 33)
    g["gauss_1337_0"] = r.fill_gaussian(1337, 0, 0, 64)
    g["gauss_555_9_pos13"] = r.fill_gaussian(555, 9, 13, 41, 1.5, 2.0)
    g["unif_4242_1"] = r.fill_uniform(4242, 1, 0, 64, 250.0, 400.0)
    g["unif_big"] = r.fill_uniform(4242, 1, 5, 64, 1e16, 1e16 + 4.0)

    # ---- fastmath on grids (fn ids: 0 log2, 1 ln, 2 exp2, 3 sinpi, 4 cospi, 5 pow)
    rs = np.random.RandomState(20240518)
    xs_log = np.concatenate([np.exp(rs.uniform(-700, 700, 200)), [1.0, 2.0, 1e-300, 5e-324,
                             1.0 - 2.0 ** -53, 1.4142135623730951, 0.5]])
    xs_exp = np.concatenate([rs.uniform(-1100, 1100, 200), [0.0, 0.5, -0.4999, 1023.0, -1022.0]])
    xs_ang = np.concatenate([rs.uniform(0, 2, 200), [0.0, 0.5, 1.0, 1.5, 0.25, 1.999999]])
    pb = rs.uniform(1.0, 1650.0, 200)
    pe = rs.uniform(0.0, 7.0, 200)
    g["fm_x_log"], g["fm_x_exp"], g["fm_x_ang"], g["fm_pow_b"], g["fm_pow_e"] = \
        xs_log, xs_exp, xs_ang, pb, pe
    g["fm_log2"] = r.fastmath(0, xs_log)
    g["fm_ln"] = r.fastmath(1, xs_log)
    g["fm_exp2"] = r.fastmath(2, xs_exp)
    g["fm_sinpi"] = r.fastmath(3, xs_ang)
    g["fm_cospi"] = r.fastmath(4, xs_ang)
    g["fm_pow"] = r.fastmath(5, pb, pe)

    # ---- numeric
    sample = rs.normal(size=101)
    g["num_sample"] = sample
    g["num_quantiles"] = np.array([r.quantile(sample, q) for q in (0.0, 0.05, 0.5, 0.55, 0.999, 1.0)])
    g["num_logsumexp"] = np.array([r.logsumexp(sample)])
    data = rs.normal(size=(50, 3)) @ np.array([[1.0, 0.2, 0.0], [0.0, 0.5, 0.1], [0.0, 0.0, 2.0]])
    g["num_data"] = data
    g["num_cov"] = r.sample_covariance(data)
    ok, chol = r.cholesky(g["num_cov"])
    assert ok
    g["num_chol"] = chol
    g["partition_8064_16_4"] = r.partition(8064, 16, 4)
    g["partition_1003_7_8"] = r.partition(1003, 7, 8)

    # ---- logistic ABC through the reference sampler (worker keying)
    m = M.logistic_model()
    theta_true = [0.5, 100.0, 0.05]
    obs = r.logistic_simulate(m, theta_true, r.derive_seed(1, [90]), 0, 0)
    g["logistic_observed"] = obs
    p, s, rho, f = r.logistic_abc(m, 96, 3, 4, 1337, obs)
    g["abc_w_params"], g["abc_w_summ"], g["abc_w_rho"], g["abc_w_failed"] = p, s, rho, f
    # particle keying, rows 1000..1031 (per-row sequence of abc.cpp:51-60)
    p, s, rho, f = r.logistic_abc_particle(m, 1000, 32, 1337, obs)
    g["abc_p_params"], g["abc_p_summ"], g["abc_p_rho"], g["abc_p_failed"] = p, s, rho, f
    m32 = M.logistic_model(precision=A.VXB_F32)
    p, s, rho, f = r.logistic_abc_particle(m32, 1000, 32, 1337, obs)
    g["abc32_p_params"], g["abc32_p_summ"], g["abc32_p_rho"] = p, s, rho
    p, s, rho, f = r.logistic_abc(m32, 48, 2, 1, 7, obs)
    g["abc32_w_params"], g["abc32_w_summ"], g["abc32_w_rho"] = p, s, rho
    # a short-horizon model with odd sizes
    mo = M.logistic_model(steps=37, obs_stride=5)
    oo = r.logistic_simulate(mo, theta_true, 99, 4, 3)
    g["odd_observed"] = oo
    p, s, rho, f = r.logistic_abc(mo, 50, 4, 2, 11, oo)
    g["odd_w_params"], g["odd_w_summ"], g["odd_w_rho"] = p, s, rho
    # a prior box that blows up (failed rows)
    mb = M.logistic_model(steps=400, obs_stride=100, prior_lo=(0.0, 50.0, 0.0),
                          prior_hi=(4000.0, 150.0, 0.2))
    ob = r.logistic_simulate(M.logistic_model(steps=400, obs_stride=100), theta_true, 5, 0, 0)
    p, s, rho, f = r.logistic_abc_particle(mb, 0, 64, 21, ob)
    g["bad_observed"], g["bad_params"], g["bad_summ"], g["bad_rho"], g["bad_failed"] = ob, p, s, rho, f
    assert f.any() and not f.all()

    # ---- select_epsilon on 2000 reference rows
    p, s, rho, f = r.logistic_abc_particle(m, 0, 2000, 1337, obs, want_summaries=False)
    g["sel_rho"] = rho
    for q in (0.001, 0.01, 0.5, 1.0):
        eps, idx = r.select_epsilon(rho, f, q)
        g[f"sel_eps_{q}"] = np.array([eps])
        g[f"sel_idx_{q}"] = idx
    eps, idx = r.select_epsilon(g["bad_rho"], g["bad_failed"], 0.25)
    g["sel_bad_eps"], g["sel_bad_idx"] = np.array([eps]), idx

    # ---- toggle switch known answers
    tobs, tp, ts, trho, tf = r.toggle_abc(100, 256, 256, 1, 4, 1337)
    g["toggle_observed"], g["toggle_rho"], g["toggle_summ0"] = tobs, trho, ts[0]
    eps, idx = r.select_epsilon(trho, tf, 0.01)
    g["toggle_eps"], g["toggle_idx"] = np.array([eps]), idx
    y, end = r.toggle_simulate([325.0, 0.275, 0.2, 25.0, 25.0, 3.5, 3.5], 80, 64, 2024, 1, 0, 4)
    g["toggle_y"], g["toggle_end"] = y, np.uint64(end)

    # ---- SMC pieces
    lw = rs.normal(size=500) * 2.0
    g["smc_lw"] = lw
    g["smc_ess"] = np.array([r.ess(lw), r.ess(np.log([1.0, 1.0, 2.0]))])
    parts = rs.normal(size=(500, 3))
    out, anc = r.resample_multinomial(lw, parts, 2718, 3 | (5 << 16))
    g["smc_particles"], g["smc_resampled"], g["smc_ancestors"] = parts, out, anc

    # ---- p-values
    g["pv_spec"] = r.estimate_pvalues([2.0, 5.0], [1.0, 3.0, 4.0, 6.0])
    g["pv_cutoff"] = np.array([r.compute_cutoff(np.linspace(0.1, 1.0, 10), 0.5)])
    lam, n = 0.7, 100
    ln = -0.5 * math.log(2.0 * math.pi * (lam * lam + 1.0 / n))
    yb, lm = r.normal_mean_logm(1337, 5, lam, ln, n, 10, 40)
    g["nm_ybar"], g["nm_logm"], g["nm_lognorm"] = yb, lm, np.array([ln])

    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.npz")
    np.savez_compressed(path, **g)
    print(path, os.path.getsize(path), "bytes,", len(g), "arrays")


if __name__ == "__main__":
    main()
