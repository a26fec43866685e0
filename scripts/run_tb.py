"""Throughput of the exact-Gillespie TB ABC at the reference's
bench sizes (bench.hpp:39-42: 10 initial cases, horizon 10, case target 10000),
with the reference's CPU path timed beside it on a small sample."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
from paper_1902_09046_b200 import bench_harness as B, lib, models as M

ctx = lib.Context(0)
n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 100000
m = M.tb_model(10, 10.0, 10000.0)
obs = B.tb_observed_summaries(ctx, 10, 10.0, 10000.0, 1337, 4)
ctx.abc_prior_predictive_host(m, M.keying(1), 2000, 0, 2000, obs)
ctx.profile_enable(True)
ctx.profile_reset()
t0 = time.perf_counter()
p, s, rho, f = ctx.abc_prior_predictive_host(m, M.keying(1337), n, 0, n, obs)
dt = time.perf_counter() - t0
kernel_ms = ctx.profile_read()["simulate"]["total_ms"]
ctx.profile_enable(False)
out = {"rows": n, "seconds": dt, "rows_per_s": n / dt, "kernel_ms": kernel_ms, "failed": int(f.sum()),
       "mean_genotypes": float(s[f == 0, 0].mean()), "max_genotypes": float(s[:, 0].max())}
try:
    from oracle.pyoracle import Ref
    r = Ref()
    k = min(n, int(sys.argv[2]) if len(sys.argv) > 2 else 8192)
    t0 = time.perf_counter()
    ref_rows = r.tb_abc_particle(10, 10.0, 10000.0, 0, k, 1337, obs)
    out["cpu_reference"] = {"rows": k, "seconds": time.perf_counter() - t0, "cores": os.cpu_count(),
                            "rows_per_s": k / (time.perf_counter() - t0)}
    out["parity_on_sample"] = all(np.array_equal(a[:k], b, equal_nan=True)
                                  for a, b in zip((p, s, rho, f), ref_rows))
except Exception as e:  # the reference library travels with the repo when built
    out["cpu_reference"] = repr(e)
print(json.dumps(out))
