"""One launch of each kernel added in round 2 (for the ncu capture of profile_r2.sh):
the bit-exact sequential exp-sum + resampling draw at N = 1e5, and the round kernels of
the multi-GPU ABC-SMC host (gated propose, pack, append, chunk-total normalisation)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np

from paper_1902_09046_b200 import _abi as A, dist as D, lib, models as M

ctx = lib.Context(0)
rs = np.random.RandomState(9)
n = 100_000
lw, parts = rs.normal(size=n) * 3, rs.normal(size=(n, 3))
out, anc = ctx.resample_multinomial(lw, parts, 77, 9)
print("resample", anc[:4], ctx.ess(lw))
m = M.logistic_model()
obs = ctx.simulate_at(m, [0.5, 100.0, 0.05], lib.derive_seed(1, [90]), 0, 0)
cfg = A.vxb_abcsmc_cfg()
cfg.particles, cfg.generations, cfg.quantile, cfg.kernel_scale = 20000, 3, 0.5, 2.0
cfg.jitter, cfg.round_size, cfg.max_rounds, cfg.seed = 1e-10, 0, 0, 1337
res = D.sharded_abcsmc(D.DeviceStages(ctx), m, cfg, obs)
print("sharded_abcsmc", res["epsilon"], res["proposals"])
ctx.close()
