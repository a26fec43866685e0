import sys; sys.path.insert(0, "/root/repo")
import numpy as np
from paper_1902_09046_b200 import _abi as A, lib, models as M
ctx = lib.Context(0)
m = M.logistic_model(rng=A.VXB_RNG_FAST)
obs = ctx.simulate_at(M.logistic_model(), [0.5, 100.0, 0.05], lib.derive_seed(1, [90]), 0, 0)
n = 1_000_000
p, s, rho, f = ctx.abc_prior_predictive_host(m, M.keying(1337), n, 0, n, obs)
eps = np.quantile(rho[~np.isnan(rho)], 1e-3)
print("eps", eps)
cum = np.cumsum((s - obs[None, :]) ** 2, axis=1)
alive = cum <= eps * eps
print("alive after obs k:", [round(float(alive[:, k].mean()), 4) for k in range(20)])
# warp-level: fraction of warps (32 consecutive rows) with any lane alive
w = alive.reshape(-1, 32, 20).any(axis=1)
print("warps alive:", [round(float(w[:, k].mean()), 4) for k in range(20)])
