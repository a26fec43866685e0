"""Device-side statistics of the throughput generator (vxb_rng_fast_stats): tail counts
against the normal tail, moments, the largest |z| and the fp32 MUFU error, at 1e10 (fp32)
and 4e10 (fp64) samples per seed.

    python scripts/fast_stats_probe.py > profiles/r2_fast_generator_stats.json
"""
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1902_09046_b200 import _abi as A, lib

ctx = lib.Context(0)
thr = [3, 4, 5, 5.5, 5.65, 6, 6.5, 7]
out = {"thresholds": thr, "runs": []}
for name, prec, rows in (("f32", A.VXB_F32, 5_000_000), ("f64", A.VXB_F64, 20_000_000)):
    ctx.rng_fast_stats(prec, 1, 0, 1000, 2000, thr)
    for seed in (2024, 7, 99):
        t0 = time.time()
        s = ctx.rng_fast_stats(prec, seed, 0, rows, 2000, thr)
        dt = time.time() - t0
        n = s["n"]
        exp = [n * math.erfc(t / math.sqrt(2)) for t in thr]
        z = [(int(c) - e) / math.sqrt(e) if e > 5 else None for c, e in zip(s["tails"], exp)]
        out["runs"].append({"precision": name, "seed": seed, "samples": n, "seconds": dt,
                            "tail_counts": [int(x) for x in s["tails"]], "tail_expected": exp,
                            "tail_z": z, "mean": s["mean"], "var_minus_1": s["var"] - 1,
                            "third_moment": s["skew"], "fourth_moment_minus_3": s["kurt"] - 3,
                            "max_abs": s["max_abs"], "f32_err_max": s["err_max"],
                            "f32_err_max_beyond_4sigma": s["err_max_tail"], "f32_err_rms": s["err_rms"]})
print(json.dumps(out))
