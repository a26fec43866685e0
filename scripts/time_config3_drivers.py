import sys, time
sys.path.insert(0, '/root/repo')
import numpy as np, torch
from paper_1902_09046_b200 import _abi as A, dist as D, lib, models as M
ctx = lib.Context(0)
m = M.logistic_model()
obs = ctx.simulate_at(m, [0.5, 100.0, 0.05], lib.derive_seed(1, [90]), 0, 0)
cfg = A.vxb_abcsmc_cfg()
cfg.particles, cfg.generations, cfg.quantile, cfg.kernel_scale = 100000, 10, 0.5, 2.0
cfg.jitter, cfg.round_size, cfg.max_rounds, cfg.seed = 1e-10, 0, 0, 1337
for rng in (A.VXB_RNG_FAST, A.VXB_RNG_REF):
    mm = M.logistic_model(rng=rng)
    st = D.DeviceStages(ctx)
    for name, fn in (("native", lambda: ctx.abcsmc_run(mm, cfg, obs)), ("spmd-native", lambda: ctx.sharded_abcsmc_run(None, mm, cfg, obs)), ("python-host", lambda: D.sharded_abcsmc(st, mm, cfg, obs))):
        fn(); torch.cuda.synchronize()
        t0 = time.perf_counter(); r = fn(); torch.cuda.synchronize(); dt = time.perf_counter() - t0
        print(rng, name, round(dt * 1e3, 1), "ms", r["epsilon"][-1], int(r["proposals"].sum()))
