import sys, math
sys.path.insert(0, '/root/repo')
import numpy as np
from paper_1902_09046_b200 import _abi as A, lib, models as M
ctx = lib.Context(0)
def cfg(seed, paths=1_000_000, levels=6):
    c = A.vxb_mlmc_cfg(); c.levels, c.refine, c.tau0, c.t_end, c.paths, c.seed = levels, 4, 1.0, 30.0, paths, seed
    return c
seeds = [1337, 11, 12, 13, 14, 15, 16, 17]
for name, rng in (("ref", A.VXB_RNG_REF), ("fast", A.VXB_RNG_FAST)):
    runs = [ctx.mlmc_tauleap(M.mm_tauleap_model(rng=rng), cfg(s)) for s in seeds]
    est = np.array([r["estimate"] for r in runs]); l0 = np.array([r["level_mean"][0] for r in runs])
    print(name, "estimates", np.round(est, 4), "mean", est.mean().round(4), "sd", est.std(ddof=1).round(4), "(se per run", round(runs[0]["std_error"], 4), ")")
    print(name, "level0   ", np.round(l0, 4))
