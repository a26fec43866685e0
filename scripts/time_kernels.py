"""Quick kernel timing (one GPU): sims/s of the fused logistic kernel per variant."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from paper_1902_09046_b200 import _abi as A, lib as L, models as M

n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 4_000_000
ctx = L.Context(0)
obs = ctx.simulate_at(M.logistic_model(), [0.5, 100.0, 0.05], 5, 0, 0)
rho = torch.empty(n, dtype=torch.float64, device="cuda")
peak = {A.VXB_F64: 37.22, A.VXB_F32: 74.45}
for name, prec, rng in (("f64_fast", A.VXB_F64, A.VXB_RNG_FAST), ("f64_ref", A.VXB_F64, A.VXB_RNG_REF),
                        ("f32_fast", A.VXB_F32, A.VXB_RNG_FAST), ("f32_ref", A.VXB_F32, A.VXB_RNG_REF)):
    m = M.logistic_model(precision=prec, rng=rng)
    ctx.abc_prior_predictive(m, M.keying(1), n, 0, n, obs, rho=rho)
    ctx.synchronize()
    t0 = time.perf_counter()
    for s in range(3):
        ctx.abc_prior_predictive(m, M.keying(2 + s), n, 0, n, obs, rho=rho)
    ctx.synchronize()
    dt = (time.perf_counter() - t0) / 3
    print(f"{name}: {n / dt:.4e} sims/s  {n / dt * 110070 / 1e12 / peak[prec] * 100:.1f}% of nominal peak", flush=True)
