"""8 020 annealed-SMC runs (K = 9, N = 401, N_p = 500) in the three instances of the
kernel (for ncu captures): reference-exact, FMA, throughput generator."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1902_09046_b200 import _abi as A, lib, models as M
ctx = lib.Context(0)
kw = dict(hyper_count=9, datasets=401, particles=500, seed=1337)
for name, extra in (("exact", {}), ("fma", {"arith": A.VXB_ARITH_FMA}), ("throughput", {"rng": A.VXB_RNG_FAST})):
    print(name, ctx.weak_info_test(M.weakinfo_config(**kw, **extra))["gamma"][:3])
