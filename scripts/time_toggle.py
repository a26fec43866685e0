"""Paper-size toggle-switch ABC (N = 8064, C = 8000, T = 600), both generator modes: kernel ms."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from paper_1902_09046_b200 import _abi as A, lib, models as M
ctx = lib.Context(0)
n, c, t = 8064, 8000, 600
out = {}
for name, rng in (("exact", A.VXB_RNG_REF), ("throughput", A.VXB_RNG_FAST)):
    m = M.toggle_model(t, c, rng=rng)
    obs = ctx.simulate_at(M.toggle_model(t, c), M.TOGGLE_MIDPOINT, lib.derive_seed(1337, [90]), 0, 0)
    rho = torch.empty(n, dtype=torch.float64, device="cuda")
    ctx.abc_prior_predictive(m, M.keying(1337), 296, 0, 296, obs, rho=rho)
    ctx.synchronize()
    ctx.profile_enable(True); ctx.profile_reset()
    ctx.abc_prior_predictive(m, M.keying(1337), n, 0, n, obs, rho=rho)
    ctx.synchronize()
    out[name] = ctx.profile_read()["simulate"]["total_ms"]
    ctx.profile_enable(False)
print(out)
