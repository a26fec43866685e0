"""select_epsilon at large N (radix select + compaction), device-resident rho."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
from paper_1902_09046_b200 import _abi as A, lib, models as M
ctx = lib.Context(0)
m = M.logistic_model(rng=A.VXB_RNG_FAST)
obs = ctx.simulate_at(M.logistic_model(), [0.5, 100.0, 0.05], lib.derive_seed(1, [90]), 0, 0)
for n in (1_000_000, 100_000_000):
    rho = torch.empty(n, dtype=torch.float64, device="cuda")
    failed = torch.empty(n, dtype=torch.uint8, device="cuda")
    ctx.abc_prior_predictive(m, M.keying(7), n, 0, n, obs, rho=rho, failed=failed)
    idx = torch.empty(max(1024, n // 500), dtype=torch.int64, device="cuda")
    ctx.select_epsilon(rho, failed, 1e-3, cap=idx.numel(), precision=A.VXB_F64, n=n, idx=idx)
    ctx.profile_enable(True); ctx.profile_reset()
    t0 = time.perf_counter()
    eps, _, nacc = ctx.select_epsilon(rho, failed, 1e-3, cap=idx.numel(), precision=A.VXB_F64, n=n, idx=idx)
    dt = time.perf_counter() - t0
    p = ctx.profile_read(); ctx.profile_enable(False)
    print(n, f"wall {dt*1e3:.2f} ms eps {eps:.6f} acc {nacc}", {k: (v['launches'], round(v['total_ms'], 3)) for k, v in p.items() if v['launches']})
