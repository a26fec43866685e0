import sys, json, math
sys.path.insert(0, '/root/repo')
from paper_1902_09046_b200 import _abi as A, lib
ctx = lib.Context(0)
thr = [3, 4, 5, 5.5, 5.65, 6, 6.5, 7]
for prec, rows in ((A.VXB_F32, 5_000_000), (A.VXB_F64, 2_000_000)):
    import time
    ctx.rng_fast_stats(prec, 1, 0, 1000, 2000, thr)
    t0 = time.time()
    s = ctx.rng_fast_stats(prec, 2024, 0, rows, 2000, thr)
    dt = time.time() - t0
    n = s["n"]
    exp = [n * math.erfc(t / math.sqrt(2)) for t in thr]
    print(prec, n, round(dt, 3), "s")
    print(" tails", [int(x) for x in s["tails"]], [round(e, 1) for e in exp])
    print(" mean %.3e var-1 %.3e skew %.3e kurt-3 %.3e max %.4f" % (s["mean"], s["var"] - 1, s["skew"], s["kurt"] - 3, s["max_abs"]))
    print(" err_max %.3e err_max_tail %.3e err_rms %.3e" % (s["err_max"], s["err_max_tail"], s["err_rms"]))
