"""vxb_abc_reject with and without VXB_OPT_EARLY_REJECT: same accepted set (indices, parameters,
distances, bit for bit) and the time of both, for the three instances of the fused kernel."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1902_09046_b200 import _abi as A, lib, models as M

n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 20_000_000
eps_arg = float(sys.argv[2]) if len(sys.argv) > 2 else None   # default: the 0.1 % epsilon of config 0
ctx = lib.Context(0)
obs = ctx.simulate_at(M.logistic_model(), [0.5, 100.0, 0.05], lib.derive_seed(1, [90]), 0, 0)
eps = eps_arg if eps_arg is not None else 19.47051606010851
cap = n if eps_arg is not None else n // 100   # host buffers for the accepted rows
for name, kw in (("f64_fast", {"rng": A.VXB_RNG_FAST}), ("f32_fast", {"rng": A.VXB_RNG_FAST, "precision": A.VXB_F32}),
                 ("f64_ref", {})):
    m = M.logistic_model(**kw)
    res = []
    for early in (False, True):
        ctx.set_early_reject(early)
        ctx.abc_reject(m, M.keying(1337), n, 0, n, obs, eps, cap=cap)
        t0 = time.perf_counter()
        out = ctx.abc_reject(m, M.keying(1337), n, 0, n, obs, eps, cap=cap)
        res.append((time.perf_counter() - t0, out))
    (t0, a), (t1, b) = res
    same = a[0] == b[0] and all(np.array_equal(x, y) for x, y in zip(a[1:], b[1:]))
    print(name, "rows", n, "accepted", a[0], "identical", same, "ms full", round(1e3 * t0, 1), "early", round(1e3 * t1, 1),
          "speed-up", round(t0 / t1, 2))
ctx.set_early_reject(False)
