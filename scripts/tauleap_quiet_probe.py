"""Config 4 with the reaction rates as they are and scaled to ~zero (every fine step quiet):
the second run is what the generator alone costs, the difference is the inversion path."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1902_09046_b200 import _abi as A, lib, models as M
ctx = lib.Context(0)
c = A.vxb_mlmc_cfg()
c.levels, c.refine, c.tau0, c.t_end, c.paths, c.seed = 6, 4, 1.0, 30.0, 1_000_000, 1337
for scale in (1.0, 1e-9):
    for name, kw in (("exact", {}), ("fast", {"rng": A.VXB_RNG_FAST}), ("fast_f32", {"rng": A.VXB_RNG_FAST, "precision": A.VXB_F32})):
        m = M.mm_tauleap_model(rates=(1e-3 * scale, 1e-4 * scale, 0.1 * scale), **kw)
        ctx.mlmc_tauleap(m, c)
        t0 = time.perf_counter(); r = ctx.mlmc_tauleap(m, c); t = time.perf_counter() - t0
        print(scale, name, round(1e3 * t, 1), r["estimate"])
