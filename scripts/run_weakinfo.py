"""The paper's case study 1 at its published size: weak-informativity test with
K = 400 hyperparameters, N = 400 datasets, N_p = 500 particles:
2 (K+1) N = 320 800 annealed-SMC runs.  Published best: 90 s on 16 AVX-512 cores
(PAPER.md:742-746)."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
from paper_1902_09046_b200 import _abi as A, lib, models as M

ctx = lib.Context(0)
k = int(sys.argv[1]) if len(sys.argv) > 1 else 400
n = int(sys.argv[2]) if len(sys.argv) > 2 else 400
cfg = M.weakinfo_config(hyper_count=k, datasets=n, particles=500, seed=1337)
ctx.weak_info_test(M.weakinfo_config(hyper_count=4, datasets=16, particles=500, seed=1))  # warm-up
times = []
for rep in range(3):
    t0 = time.perf_counter()
    t = ctx.weak_info_test(cfg, want_evidence=True)
    times.append(time.perf_counter() - t0)
runs = 2 * (k + 1) * n
ev = t["evidence"]
out = {"hyper_count": k, "datasets": n, "particles": 500, "sampler_runs": runs,
       "seconds": times, "runs_per_s": runs / min(times), "published_best_s": 90.0,
       "weakly_informative": int(t["weakly"].sum()), "gamma0": float(t["gamma"][0]),
       "completed_min": int(t["completed"].min()), "evidence_mean": float(np.nanmean(ev)),
       "failed_runs": int(np.isnan(ev).sum())}
# the same test with contracted multiply-adds (VXB_ARITH_FMA: same random numbers)
cfg_fma = M.weakinfo_config(hyper_count=k, datasets=n, particles=500, seed=1337, arith=A.VXB_ARITH_FMA)
ctx.weak_info_test(cfg_fma)
fma_times = []
for rep in range(3):
    t0 = time.perf_counter()
    tf = ctx.weak_info_test(cfg_fma, want_evidence=True)
    fma_times.append(time.perf_counter() - t0)
out["fma_mode"] = {"seconds": fma_times, "max_abs_evidence_difference": float(np.nanmax(np.abs(tf["evidence"] - ev))),
                   "table_identical": bool(np.array_equal(tf["gamma"], t["gamma"]) and
                                           np.array_equal(tf["weakly"], t["weakly"]))}
# the throughput generator (VXB_RNG_FAST: other random numbers, statistically validated)
cfg_fast = M.weakinfo_config(hyper_count=k, datasets=n, particles=500, seed=1337, rng=A.VXB_RNG_FAST)
ctx.weak_info_test(cfg_fast)
fast_times = []
for rep in range(3):
    t0 = time.perf_counter()
    tg = ctx.weak_info_test(cfg_fast, want_evidence=True)
    fast_times.append(time.perf_counter() - t0)
dv = (tg["evidence"] - ev).ravel()
out["throughput_generator"] = {"seconds": fast_times, "weakly_informative": int(tg["weakly"].sum()),
                               "gamma0": float(tg["gamma"][0]),
                               "evidence_mean_difference": float(np.nanmean(dv)),
                               "evidence_mean_difference_se": float(np.nanstd(dv) / np.sqrt(dv.size)),
                               "flags_agree": float((tg["weakly"] == t["weakly"]).mean())}
print(json.dumps(out))
