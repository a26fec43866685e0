"""BASELINE config 3 (ABC-SMC, N = 1e5, 10 generations) once, both generator modes
(for launch lists:  ncu --metrics gpu__time_duration.sum ... python scripts/run_config3.py)."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1902_09046_b200 import _abi as A, lib, models as M
ctx = lib.Context(0)
n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 100000
obs = ctx.simulate_at(M.logistic_model(), [0.5, 100.0, 0.05], lib.derive_seed(1, [90]), 0, 0)
cfg = A.vxb_abcsmc_cfg()
cfg.particles, cfg.generations, cfg.quantile, cfg.kernel_scale, cfg.jitter, cfg.round_size, cfg.max_rounds, cfg.seed = n, 10, 0.5, 2.0, 1e-10, 0, 0, 1337
for rng in (A.VXB_RNG_REF, A.VXB_RNG_FAST):
    m = M.logistic_model(rng=rng)
    t0 = time.perf_counter()
    r = ctx.abcsmc_run(m, cfg, obs)
    print("rng", rng, "seconds", round(time.perf_counter() - t0, 4), "eps", r["epsilon"][-1], "ess", r["ess"][-1])
