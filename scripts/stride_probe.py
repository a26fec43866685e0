"""Does the BASELINE observation stride (100 steps, not a multiple of the 8- / 16-normal
batches of the throughput generator) cost anything against strides that take the
regular-grid path of logistic_path (csrc/vxb_logistic.cuh)?  Same 2000 steps, fixed
epsilon, N rows; event-timed through the library's profiler.

    python scripts/stride_probe.py [rows]
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch

from paper_1902_09046_b200 import _abi as A, lib, models as M

ctx = lib.Context(0)
n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 20_000_000
out = {"rows": n, "steps": 2000, "cases": []}
dev_n = torch.zeros(1, dtype=torch.int64, device="cuda")
for name, prec, rng in (("f64_fast", A.VXB_F64, A.VXB_RNG_FAST), ("f32_fast", A.VXB_F32, A.VXB_RNG_FAST),
                        ("f64_ref", A.VXB_F64, A.VXB_RNG_REF)):
    for stride in (100, 80, 200, 400):
        m = M.logistic_model(steps=2000, obs_stride=stride, precision=prec, rng=rng)
        obs = np.full(2000 // stride, 50.0)
        rows = n if rng == A.VXB_RNG_FAST else n // 4
        ms = []
        for rep in range(4):
            ctx.profile_enable(True)
            ctx.profile_reset()
            ctx.abc_reject(m, M.keying(1337 + rep), rows, 0, rows, obs, 1.0, 1024, idx=None if False else torch.empty(1024, dtype=torch.int64, device="cuda"),
                           params=torch.empty((1024, 3), dtype=torch.float32 if prec == A.VXB_F32 else torch.float64, device="cuda"),
                           rho=torch.empty(1024, dtype=torch.float32 if prec == A.VXB_F32 else torch.float64, device="cuda"),
                           n_accepted=dev_n)
            ms.append(ctx.profile_read()["simulate"]["total_ms"])
            ctx.profile_enable(False)
        best = min(ms[1:])
        out["cases"].append({"variant": name, "obs_stride": stride, "rows": rows, "kernel_ms": best,
                             "sims_per_s": rows / (best * 1e-3)})
print(json.dumps(out))
