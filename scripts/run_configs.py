"""Runs all five BASELINE.json configs at full size on one GPU and prints one
JSON object with timings (CUDA-event kernel times from the library profiler
plus wall time per call) and the headline results of each config.

    python scripts/run_configs.py [--quick]
"""
import json
import math
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1902_09046_b200 import _abi as A, lib, models as M  # noqa: E402


def timed(ctx, fn, reps=1):
    ctx.profile_reset()
    ctx.profile_enable(True)
    ctx.synchronize()
    t0 = time.perf_counter()
    out = None
    for _ in range(reps):
        out = fn()
    ctx.synchronize()
    wall = (time.perf_counter() - t0) / reps
    prof = {k: v for k, v in ctx.profile_read().items() if v["launches"]}
    for v in prof.values():
        v["total_ms"] /= reps
        v["launches"] //= reps
    ctx.profile_enable(False)
    return out, wall, prof


def main():
    quick = "--quick" in sys.argv
    import torch
    ctx = lib.Context(0)
    res = {"device": ctx.device_info()["name"]}
    m = M.logistic_model()
    obs = ctx.simulate_at(m, [0.5, 100.0, 0.05], lib.derive_seed(1, [90]), 0, 0)

    # ---- config 0: N = 1e6, accept the 0.1% nearest
    n0 = 1_000_000
    rho = torch.empty(n0, dtype=torch.float64, device="cuda")
    failed = torch.empty(n0, dtype=torch.uint8, device="cuda")

    def c0():
        ctx.abc_prior_predictive(m, M.keying(1337), n0, 0, n0, obs, rho=rho, failed=failed)
        return ctx.select_epsilon(rho, failed, 1e-3, cap=2000, precision=A.VXB_F64, n=n0)
    c0()
    (eps, idx, nacc), wall, prof = timed(ctx, c0, 3)
    res["config0"] = {"n": n0, "epsilon": eps, "accepted": nacc, "wall_ms": wall * 1e3,
                      "sims_per_s": n0 / wall, "kernels": prof, "rng": "reference-exact"}

    # ---- config 2: 64 lambdas x 1e6 datasets x n = 100
    nl, mt, nd = 64, (100_000 if quick else 1_000_000), 100
    lam = np.array(M.lambda_grid(nl))
    ln = np.array([-0.5 * math.log(2.0 * math.pi * (l * l + 1.0 / nd)) for l in lam])
    y_obs = 3.0 + ctx.rng_fill_gaussian(lib.derive_seed(2, [90]), 0, 0, nd)
    ybar = float(y_obs.mean())
    for name, rng in (("ref", A.VXB_RNG_REF), ("fast", A.VXB_RNG_FAST)):
        mdl = M.normal_mean_model(nd, rng=rng)
        ctx.ppp_pvalues(mdl, lam, ln, mt, 0, mt, 1337, ybar)
        (counts, pv, _), wall, prof = timed(ctx, lambda: ctx.ppp_pvalues(mdl, lam, ln, mt, 0, mt, 1337, ybar))
        exact = np.array([math.erfc(abs(ybar) / math.sqrt(2.0 * (l * l + 1.0 / nd))) for l in lam])
        res[f"config2_{name}"] = {"datasets": nl * mt, "wall_ms": wall * 1e3,
                                  "datasets_per_s": nl * mt / wall,
                                  "max_abs_err_vs_closed_form": float(np.abs(pv - exact).max()),
                                  "kernels": prof}

    # ---- config 3: ABC-SMC N = 1e5 x 10 generations
    cfg = A.vxb_abcsmc_cfg()
    cfg.particles, cfg.generations = (20_000 if quick else 100_000), 10
    cfg.quantile, cfg.kernel_scale, cfg.jitter, cfg.round_size, cfg.max_rounds, cfg.seed = 0.5, 2.0, 1e-10, 0, 0, 1337
    out, wall, prof = timed(ctx, lambda: ctx.abcsmc_run(m, cfg, obs))
    res["config3"] = {"particles": cfg.particles, "generations": 10, "wall_ms": wall * 1e3,
                      "epsilon": out["epsilon"].tolist(), "ess": out["ess"].tolist(),
                      "accept_rate": out["accept_rate"].tolist(),
                      "proposals": out["proposals"].tolist(),
                      "posterior_mean": out["mean"][-1].tolist(), "kernels": prof}

    mfast = M.logistic_model(rng=A.VXB_RNG_FAST)
    outf, wall, prof = timed(ctx, lambda: ctx.abcsmc_run(mfast, cfg, obs))
    res["config3_fast"] = {"particles": cfg.particles, "generations": 10, "wall_ms": wall * 1e3,
                           "epsilon": outf["epsilon"].tolist(), "ess": outf["ess"].tolist(),
                           "accept_rate": outf["accept_rate"].tolist(),
                           "proposals": outf["proposals"].tolist(),
                           "posterior_mean": outf["mean"][-1].tolist(), "kernels": prof}

    # ---- config 4: MLMC tau-leap, 6 levels x 1e6 paths
    mm = M.mm_tauleap_model()
    mc = A.vxb_mlmc_cfg()
    mc.levels, mc.refine, mc.tau0, mc.t_end, mc.paths, mc.seed = 6, 4, 1.0, 30.0, (100_000 if quick else 1_000_000), 1337
    out, wall, prof = timed(ctx, lambda: ctx.mlmc_tauleap(mm, mc))
    steps = sum(mc.paths * c for c in out["level_cost"])
    res["config4"] = {"paths_per_level": mc.paths, "wall_ms": wall * 1e3, "estimate": out["estimate"],
                      "std_error": out["std_error"], "level_mean": out["level_mean"].tolist(),
                      "level_var": out["level_var"].tolist(), "path_steps_per_s": steps / wall,
                      "kernels": prof}
    mmf = M.mm_tauleap_model(rng=A.VXB_RNG_FAST)
    ctx.mlmc_level(mmf, mc, 0, 0, 1000)
    outf, wall, prof = timed(ctx, lambda: ctx.mlmc_tauleap(mmf, mc))
    res["config4_fast"] = {"paths_per_level": mc.paths, "wall_ms": wall * 1e3,
                           "estimate": outf["estimate"], "std_error": outf["std_error"],
                           "level_var": outf["level_var"].tolist(),
                           "path_steps_per_s": steps / wall, "kernels": prof,
                           "z_vs_exact_rng": (outf["estimate"] - out["estimate"]) /
                           math.sqrt(outf["std_error"] ** 2 + out["std_error"] ** 2)}
    # ---- the paper's toggle-switch workload: N = 8064, C = 8000, T = 600
    n_t, c_t, t_t = (512 if quick else 8064), 8000, 600
    tm = M.toggle_model(t_t, c_t)
    tobs = ctx.simulate_at(tm, M.TOGGLE_MIDPOINT, lib.derive_seed(1337, [90]), 0, 0)
    trho = torch.empty(n_t, dtype=torch.float64, device="cuda")
    tkey = M.keying(1337, A.VXB_KEY_WORKER, 16, 4)   # the layout of the published 16-thread run
    _, wall, prof = timed(ctx, lambda: ctx.abc_prior_predictive(tm, tkey, n_t, 0, n_t, tobs, rho=trho))
    cell_steps = n_t * c_t * (t_t - 1)
    res["toggle_paper"] = {"samples": n_t, "cells": c_t, "steps": t_t, "wall_ms": wall * 1e3,
                           "cell_steps_per_s": cell_steps / wall, "sims_per_s": n_t / wall,
                           "published_best_s": 69.0, "kernels": prof}
    rho_exact = trho.cpu().numpy().copy()
    tmf = M.toggle_model(t_t, c_t, rng=A.VXB_RNG_FAST)
    fkey = M.keying(1337)
    ctx.abc_prior_predictive(tmf, fkey, n_t, 0, n_t, tobs, rho=trho)
    _, wall, prof = timed(ctx, lambda: ctx.abc_prior_predictive(tmf, fkey, n_t, 0, n_t, tobs, rho=trho))
    rho_fast = trho.cpu().numpy()
    xs = np.sort(np.concatenate([rho_exact, rho_fast]))
    ks = float(np.abs(np.searchsorted(np.sort(rho_exact), xs, side="right") / n_t
                      - np.searchsorted(np.sort(rho_fast), xs, side="right") / n_t).max())
    res["toggle_paper_fast"] = {"samples": n_t, "cells": c_t, "steps": t_t, "wall_ms": wall * 1e3,
                                "cell_steps_per_s": cell_steps / wall, "sims_per_s": n_t / wall,
                                "published_best_s": 69.0, "kernels": prof,
                                "ks_rho_vs_exact": ks, "ks_critical_1pct": 1.628 * math.sqrt(2.0 / n_t)}
    print(json.dumps(res))


if __name__ == "__main__":
    main()
