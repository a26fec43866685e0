"""Record of the Philox4x32-7 opt-in build (python -m paper_1902_09046_b200.build
--rounds7; run with VXB_LIBRARY=paper_1902_09046_b200/libvexbayes_cuda_rounds7.so):
generator statistics on the device (tails, moments; 1e10 fp32 / 4e10 fp64 samples),
serial / within-batch correlations and KS on 8.2e6 host-side samples, the config-1
acceptance count against the 10-round build's, and the kernel rate.

    VXB_LIBRARY=... python scripts/philox7_record.py > profiles/r2_philox7.json
"""
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch

from paper_1902_09046_b200 import _abi as A, lib, models as M

ctx = lib.Context(0)
out = {"philox4x32_rounds": int(lib.load().vxb_fast_generator_rounds()), "library": lib.LIB_PATH}
thr = [3, 4, 5, 5.5, 6]
for name, prec, rows in (("f32", A.VXB_F32, 5_000_000), ("f64", A.VXB_F64, 20_000_000)):
    s = ctx.rng_fast_stats(prec, 2024, 0, rows, 2000, thr)
    n = s["n"]
    exp = [n * math.erfc(t / math.sqrt(2)) for t in thr]
    out[f"device_stats_{name}"] = {
        "samples": n, "tail_counts": [int(x) for x in s["tails"]], "tail_expected": exp,
        "tail_z": [(int(c) - e) / math.sqrt(e) for c, e in zip(s["tails"], exp)],
        "mean_z": s["mean"] * math.sqrt(n), "var_z": (s["var"] - 1) / math.sqrt(2.0 / n),
        "third_moment_z": s["skew"] / math.sqrt(15.0 / n),
        "fourth_moment_z": (s["kurt"] - 3) / math.sqrt(96.0 / n), "max_abs": s["max_abs"]}
    # host-side: KS and correlations (lags up to two batches, values and squares)
    rows_h, per = 4096, 2000
    z = ctx.rng_fill_gaussian_fast(prec, 99, 0, rows_h, per).astype(np.float64)
    sub = np.sort(z.ravel()[::20])
    cdf = 0.5 * (1.0 + np.vectorize(math.erf)(sub / math.sqrt(2.0)))
    k = np.arange(1, sub.size + 1) / sub.size
    ks = max(np.abs(cdf - k).max(), np.abs(cdf - (k - 1.0 / sub.size)).max())
    batch = 16 if prec == A.VXB_F32 else 8
    zc = z - z.mean()
    corr = {}
    for lag in list(range(1, batch + 1)) + [2 * batch]:
        nn = rows_h * (per - lag)
        corr[lag] = {"r_z": float((zc[:, :-lag] * zc[:, lag:]).mean() * math.sqrt(nn)),
                     "r2_z": float(((z[:, :-lag] ** 2 - 1) * (z[:, lag:] ** 2 - 1)).mean() / 2.0 * math.sqrt(nn))}
    out[f"host_stats_{name}"] = {"ks_statistic_times_sqrt_n": float(ks * math.sqrt(sub.size)),
                                 "ks_critical_0.001": 1.95, "correlation_z_by_lag": corr,
                                 "row_to_row_z": float((zc[:-1] * zc[1:]).mean() * math.sqrt(z.size))}
# config 1 at 2e7 rows: accepted count and kernel time
m = M.logistic_model()
obs = ctx.simulate_at(m, [0.5, 100.0, 0.05], lib.derive_seed(1, [90]), 0, 0)
eps = 19.712058377057488
for name, prec in (("f64_fast", A.VXB_F64), ("f32_fast", A.VXB_F32)):
    mv = M.logistic_model(precision=prec, rng=A.VXB_RNG_FAST)
    n = 20_000_000
    real = torch.float32 if prec == A.VXB_F32 else torch.float64
    bufs = dict(idx=torch.empty(400000, dtype=torch.int64, device="cuda"),
                params=torch.empty((400000, 3), dtype=real, device="cuda"),
                rho=torch.empty(400000, dtype=real, device="cuda"),
                n_accepted=torch.zeros(1, dtype=torch.int64, device="cuda"))
    ms = []
    for rep in range(4):
        ctx.profile_enable(True)
        ctx.profile_reset()
        ctx.abc_reject(mv, M.keying(1337 + rep), n, 0, n, obs, eps, 400000, **bufs)
        ms.append(ctx.profile_read()["simulate"]["total_ms"])
        ctx.profile_enable(False)
    acc = int(bufs["n_accepted"].item())
    out[f"config1_{name}"] = {"rows": n, "kernel_ms": min(ms[1:]), "sims_per_s": n / (min(ms[1:]) * 1e-3),
                              "accepted_last_step": acc, "accept_rate": acc / n}
print(json.dumps(out))
