"""All six levels of config 4 at a small path count, the three tau-leap instances (for ncu)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1902_09046_b200 import _abi as A, lib, models as M
ctx = lib.Context(0)
mc = A.vxb_mlmc_cfg()
mc.levels, mc.refine, mc.tau0, mc.t_end, mc.paths, mc.seed = 6, 4, 1.0, 30.0, int(float(sys.argv[1])) if len(sys.argv) > 1 else 40000, 1337
for kw in ({}, {"rng": A.VXB_RNG_FAST}, {"rng": A.VXB_RNG_FAST, "precision": A.VXB_F32}):
    print(ctx.mlmc_tauleap(M.mm_tauleap_model(**kw), mc)["estimate"])
