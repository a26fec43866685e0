"""Config 4 (6 levels x 1e6 paths) through vxb_mlmc_tauleap: wall time of the exact, throughput
and fp32 instances (three passes each after a warm-up) and the estimate, for A/B runs of the
tau-leap kernels (VXB_LIBRARY selects the build)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1902_09046_b200 import _abi as A, lib, models as M

ctx = lib.Context(0)
c = A.vxb_mlmc_cfg()
c.levels, c.refine, c.tau0, c.t_end, c.paths, c.seed = 6, 4, 1.0, 30.0, 1_000_000, 1337
for name, kw in (("exact", {}), ("fast", {"rng": A.VXB_RNG_FAST}), ("fast_f32", {"rng": A.VXB_RNG_FAST, "precision": A.VXB_F32})):
    m = M.mm_tauleap_model(**kw)
    ctx.mlmc_tauleap(m, c)
    t = []
    for _ in range(3):
        t0 = time.perf_counter()
        r = ctx.mlmc_tauleap(m, c)
        t.append(time.perf_counter() - t0)
    print(name, "ms", [round(1e3 * x, 1) for x in t], "estimate", repr(r["estimate"]), "level_cost", r["level_cost"].tolist()[:2])
