"""One small launch of every kernel family (for ncu captures of the non-headline kernels)."""
import math, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
from paper_1902_09046_b200 import _abi as A, lib, models as M

ctx = lib.Context(0)
m = M.logistic_model()
obs = ctx.simulate_at(m, [0.5, 100.0, 0.05], lib.derive_seed(1, [90]), 0, 0)
# config 0 shape: simulate + select + compact at 1e6
n = 1_000_000
rho = torch.empty(n, dtype=torch.float64, device="cuda")
failed = torch.empty(n, dtype=torch.uint8, device="cuda")
ctx.abc_prior_predictive(m, M.keying(1337), n, 0, n, obs, rho=rho, failed=failed)
print("config0", ctx.select_epsilon(rho, failed, 1e-3, cap=2000, precision=A.VXB_F64, n=n)[::2])
# config 2: 64 lambdas x 1e5 datasets
lam = np.array(M.lambda_grid(64)); nd = 100
ln = np.array([-0.5 * math.log(2.0 * math.pi * (l * l + 1.0 / nd)) for l in lam])
for rng in (A.VXB_RNG_REF, A.VXB_RNG_FAST):
    print("config2", ctx.ppp_pvalues(M.normal_mean_model(nd, rng=rng), lam, ln, 100000, 0, 100000, 1337, 2.9)[1][:3])
# config 3: N = 20000 x 3 generations
cfg = A.vxb_abcsmc_cfg()
cfg.particles, cfg.generations, cfg.quantile, cfg.kernel_scale, cfg.jitter, cfg.round_size, cfg.max_rounds, cfg.seed = 20000, 3, 0.5, 2.0, 1e-10, 0, 0, 1337
print("config3", ctx.abcsmc_run(m, cfg, obs)["epsilon"])
# config 4: levels 0..3, 1e5 paths
mc = A.vxb_mlmc_cfg(); mc.levels, mc.refine, mc.tau0, mc.t_end, mc.paths, mc.seed = 4, 4, 1.0, 30.0, 100000, 1337
for rng in (A.VXB_RNG_REF, A.VXB_RNG_FAST):
    print("config4", ctx.mlmc_tauleap(M.mm_tauleap_model(rng=rng), mc)["estimate"])
print("config4 f32", ctx.mlmc_tauleap(M.mm_tauleap_model(rng=A.VXB_RNG_FAST, precision=A.VXB_F32), mc)["estimate"])
# toggle: 296 samples x 8000 cells x 600 steps (two CTAs per SM)
tm = M.toggle_model(600, 8000)
tobs = ctx.simulate_at(tm, M.TOGGLE_MIDPOINT, lib.derive_seed(1337, [90]), 0, 0)
trho = torch.empty(296, dtype=torch.float64, device="cuda")
ctx.abc_prior_predictive(tm, M.keying(1337), 296, 0, 296, tobs, rho=trho)
ctx.synchronize()
print("toggle", float(trho[0]))
tmf = M.toggle_model(600, 8000, rng=A.VXB_RNG_FAST)   # throughput instance, same sizes
ctx.abc_prior_predictive(tmf, M.keying(1337), 296, 0, 296, tobs, rho=trho)
ctx.synchronize()
print("toggle throughput mode", float(trho[0]))
# annealed SMC: 8 020 sampler runs (K = 9, N = 401) of 500 particles
wcfg = M.weakinfo_config(hyper_count=9, datasets=401, particles=500, seed=1337)
print("weakinfo", ctx.weak_info_test(wcfg)["gamma"][:3])
# TB Gillespie ABC: 4 000 paths at the reference's bench sizes
tbm = M.tb_model(10, 10.0, 10000.0)
tb_obs = ctx.simulate_at(M.tb_model(10, 10.0, 10000.0, attempts=64), M.TB_TRUE_THETA, lib.derive_seed(1337, [91]), 0, 0)
print("tb", ctx.abc_prior_predictive_host(tbm, M.keying(1337), 4000, 0, 4000, tb_obs)[2][:2])
