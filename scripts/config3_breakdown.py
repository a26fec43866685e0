"""Config 3 (N = 1e5 x 10 generations), both generator modes: wall time against the sum of
the kernel times, per kernel family (proposals / weights / selection / ...)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1902_09046_b200 import _abi as A, lib, models as M
ctx = lib.Context(0)
obs = ctx.simulate_at(M.logistic_model(), [0.5, 100.0, 0.05], lib.derive_seed(1, [90]), 0, 0)
cfg = A.vxb_abcsmc_cfg()
cfg.particles, cfg.generations, cfg.quantile, cfg.kernel_scale = 100000, 10, 0.5, 2.0
cfg.jitter, cfg.round_size, cfg.max_rounds, cfg.seed = 1e-10, 0, 0, 1337
for rng in (A.VXB_RNG_FAST, A.VXB_RNG_REF):
    m = M.logistic_model(rng=rng)
    ctx.abcsmc_run(m, cfg, obs)
    t0 = time.perf_counter(); ctx.abcsmc_run(m, cfg, obs); wall = time.perf_counter() - t0
    ctx.profile_enable(True); ctx.profile_reset()
    ctx.abcsmc_run(m, cfg, obs)
    prof = ctx.profile_read(); ctx.profile_enable(False)
    tot = sum(v["total_ms"] for v in prof.values())
    print("rng", rng, "wall ms", round(1e3 * wall, 1), "kernel ms", round(tot, 1), {k: (v["launches"], round(v["total_ms"], 1)) for k, v in prof.items() if v["launches"]})
