"""The smallest launch of every kernel family with shared-memory hand-offs or atomics,
for compute-sanitizer (ONE tool per gpurun call, profiling guide):

    compute-sanitizer --tool memcheck  python scripts/sanitize_small.py
    compute-sanitizer --tool racecheck python scripts/sanitize_small.py
    VXB_GUARD=1 python scripts/sanitize_small.py    # the library's own canary check

Covers vxb_select.cu (radix_hist / pick, accept_count / scan_blocks / accept_write),
vxb_smc.cu (canonical reductions, sequential exp-sum, resample, pack / append rounds,
weights), vxb_tauleap.cu (shared sums), vxb_tb.cu (three-level counts), vxb_anneal.cu
(one CTA per run), vxb_toggle.cu (in-CTA sort), vxb_logistic.cu and vxb_ppp.cu."""
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch

from paper_1902_09046_b200 import _abi as A, dist as D, lib, models as M

ctx = lib.Context(0)
m = M.logistic_model(steps=200, obs_stride=10)
obs = ctx.simulate_at(m, [0.5, 100.0, 0.05], lib.derive_seed(1, [90]), 0, 0)
n = 20000
# simulate + select (radix select, compaction) with host and device buffers
p, s, rho, f = ctx.abc_prior_predictive_host(m, M.keying(1337), n, 0, n, obs)
print("select", ctx.select_epsilon(rho, f, 0.01)[0])
print("order", ctx.order_statistics(rho, f, [0, 5, n // 2])[0])
for prec, rng in ((A.VXB_F64, A.VXB_RNG_FAST), (A.VXB_F32, A.VXB_RNG_FAST), (A.VXB_F64, A.VXB_RNG_REF)):
    mv = M.logistic_model(steps=200, obs_stride=10, precision=prec, rng=rng)
    print("reject", ctx.abc_reject(mv, M.keying(7), n, 0, n, obs, 30.0, cap=n)[0])
ctx.set_early_reject(True)   # segment launches with survivor queues (70 001 rows: above the threshold)
for prec, rng in ((A.VXB_F64, A.VXB_RNG_FAST), (A.VXB_F32, A.VXB_RNG_FAST), (A.VXB_F64, A.VXB_RNG_REF)):
    mv = M.logistic_model(steps=200, obs_stride=10, precision=prec, rng=rng)
    print("early reject", ctx.abc_reject(mv, M.keying(7), 70001, 0, 70001, obs, 30.0, cap=70001)[0])
ctx.set_early_reject(False)
idx, params, r, n_dev = D.sharded_reject(ctx, m, M.keying(3), n, obs, 30.0, cap_fraction=0.5)
ctx.synchronize()
print("sharded_reject", int(n_dev.item()))
lb = lib.Multi(loopback_ranks=3)   # all-reduced digit histograms (vxb_sharded_select_epsilon)
print("multi select", lb.select_epsilon(rho, f, 0.01)[0])
lb.close()
# config 2
lam = np.array(M.lambda_grid(4))
ln = np.array([-0.5 * math.log(2.0 * math.pi * (l * l + 0.01)) for l in lam])
for rng in (A.VXB_RNG_REF, A.VXB_RNG_FAST):
    print("ppp", ctx.ppp_pvalues(M.normal_mean_model(100, rng=rng), lam, ln, 3000, 0, 3000, 1337, 2.9)[0])
# SMC pieces: sequential exp-sum, resample, canonical reductions, ABC-SMC incl. the
# multi-GPU host driver (pack / append rounds) as one rank
rs = np.random.RandomState(1)
lw = rs.normal(size=5000) * 3
print("ess", ctx.ess(lw), ctx.logsumexp(lw))
print("resample", ctx.resample_multinomial(lw, rs.normal(size=(5000, 3)), 77, 9)[1][:3])
cfg = A.vxb_abcsmc_cfg()
cfg.particles, cfg.generations, cfg.quantile, cfg.kernel_scale = 1200, 3, 0.5, 2.0
cfg.jitter, cfg.round_size, cfg.max_rounds, cfg.seed = 1e-10, 500, 0, 1337
for rng in (A.VXB_RNG_REF, A.VXB_RNG_FAST):
    mm = M.logistic_model(steps=200, obs_stride=10, rng=rng)
    a = ctx.abcsmc_run(mm, cfg, obs)
    b = D.sharded_abcsmc(D.DeviceStages(ctx), mm, cfg, obs)
    print("abcsmc", a["epsilon"][-1], bool(np.array_equal(a["theta"], b["theta"])))
# config 4
mc = A.vxb_mlmc_cfg()
mc.levels, mc.refine, mc.tau0, mc.t_end, mc.paths, mc.seed = 3, 4, 1.0, 30.0, 1000, 1337
for rng in (A.VXB_RNG_REF, A.VXB_RNG_FAST):
    print("mlmc", ctx.mlmc_tauleap(M.mm_tauleap_model(rng=rng), mc)["estimate"])
# toggle (in-CTA sort), both instances
for rng in (A.VXB_RNG_REF, A.VXB_RNG_FAST):
    tm = M.toggle_model(40, 512, rng=rng)
    tobs = ctx.simulate_at(M.toggle_model(40, 512), M.TOGGLE_MIDPOINT, lib.derive_seed(1337, [90]), 0, 0)
    print("toggle", ctx.abc_prior_predictive_host(tm, M.keying(1337), 8, 0, 8, tobs)[2][:2])
# annealed SMC (one CTA per run), exact / FMA / throughput instances and the ESJD run
for kw in ({}, {"arith": A.VXB_ARITH_FMA}, {"rng": A.VXB_RNG_FAST}):
    wcfg = M.weakinfo_config(hyper_count=2, datasets=6, particles=100, seed=1337, **kw)
    print("weakinfo", ctx.weak_info_test(wcfg)["gamma"][:2])
print("esjd", ctx.smc_bioassay_ensemble(M.DEFAULT_DOSE, M.DEFAULT_GROUP_SIZE, [0, 1, 3, 5], [10.0, 2.5], 5, 100,
                                        esjd_scales=[0.5, 1.0, 2.0])["log_evidence"])
# TB Gillespie (three-level running counts, persistent CTAs)
tbm = M.tb_model(10, 3.0, 300.0)
tb_obs = ctx.simulate_at(M.tb_model(10, 3.0, 300.0, attempts=64), M.TB_TRUE_THETA, lib.derive_seed(1337, [91]), 0, 0)
print("tb", ctx.abc_prior_predictive_host(tbm, M.keying(1337), 300, 0, 300, tb_obs)[2][:2])
if os.environ.get("VXB_GUARD"):
    print("guard", ctx.guard_report(selftest=True), ctx.guard_report())
ctx.close()
print("sanitize_small done")
