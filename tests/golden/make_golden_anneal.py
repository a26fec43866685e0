"""Golden values of the annealed-SMC / weak-informativity path from the UNMODIFIED
reference (smc::run_smc on the bioassay model, run_weak_info_test):

    make -C oracle ref && python tests/golden/make_golden_anneal.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
HERE = os.path.dirname(os.path.abspath(__file__))

from oracle.pyoracle import Ref  # noqa: E402

DOSE = (-0.86, -0.3, -0.05, -0.75)
SIZE = (5, 5, 5, 5)
H = 1.6828427124746189
RUNS = [  # (lambda1, lambda2, data seed, sampler seed, particles)
    (10.0, 2.5, 1234, 3702, 500), (0.3, 15.0, 77, 231, 500), (4.0, 0.2, 5, 15, 64),
    (9.5, 19.0, 42, 4242, 500), (0.11, 0.13, 8, 88, 200), (2.0, 2.0, 9, 99, 1000),
]
ENSEMBLE_RUN = 2
GRID = (0.1, 0.2, 0.3, 0.4, 0.5, 0.6, 0.7, 0.8, 0.9, 1.0)   # SmcConfig::esjd_scales default (smc.hpp:119)
ESJD_RUNS = [  # (lambda1, lambda2, data seed, sampler seed, particles, scale grid)
    (10.0, 2.5, 1234, 3702, 500, GRID), (4.0, 0.2, 5, 15, 333, GRID),
    (9.5, 19.0, 42, 4242, 200, (4.0, 9.0, 20.0)), (2.0, 2.0, 9, 99, 127, (0.05,)),
]
TABLE = dict(hyper_count=3, datasets=12, particles=200, seed=1337)


def main():
    r = Ref()
    g = {}
    theta, deaths, ev, it, traces = [], [], [], [], []
    for l1, l2, ds, ss, npart in RUNS:
        th, y = r.bioassay_sample(l1, l2, DOSE, SIZE, ds)
        e, n, tr = r.smc_bioassay(DOSE, SIZE, y, l1, l2, npart, 4, 0.01, H, ss, True)
        theta.append(th)
        deaths.append(y)
        ev.append(e)
        it.append(n)
        traces.append(np.pad(tr, ((0, 8 - len(tr)), (0, 0))))
    g["run_theta"], g["run_deaths"] = np.array(theta), np.array(deaths, dtype=np.uint32)
    g["run_evidence"], g["run_iterations"] = np.array(ev), np.array(it, dtype=np.uint64)
    g["run_trace"] = np.array(traces)  # temperature, ess, steps, p_acc per iteration
    # the SmcResult of the third run (64 particles): final ensemble and evidence column
    l1, l2, ds, ss, npart = RUNS[ENSEMBLE_RUN]
    e = r.smc_bioassay_ensemble(DOSE, SIZE, deaths[ENSEMBLE_RUN], l1, l2, npart, 4, 0.01, H, ss)
    g["ens_particles"], g["ens_trace"] = e["particles"], e["trace"]
    g["ens_rows"] = np.stack([e["log_weights"], e["log_liks"], e["log_priors"]])
    # SmcConfig::esjd = true (scale adaptation): evidence, iterations, trace per case
    for j, (l1, l2, ds, ss, npart, scales) in enumerate(ESJD_RUNS):
        _, y = r.bioassay_sample(l1, l2, DOSE, SIZE, ds)
        e = r.smc_bioassay_ensemble(DOSE, SIZE, y, l1, l2, npart, 4, 0.01, 0.0, ss, esjd_scales=scales)
        g[f"esjd{j}_deaths"] = np.array(y, dtype=np.uint32)
        g[f"esjd{j}_evidence"] = np.array([e["log_evidence"]])
        g[f"esjd{j}_trace"] = e["trace"]
        g[f"esjd{j}_particles"] = e["particles"]
    beta = np.random.RandomState(3).normal(size=(64, 2)) * np.array([8.0, 12.0])
    g["ll_beta"] = beta
    g["ll_values"] = r.bioassay_ll(beta, DOSE, SIZE, [0, 2, 5, 1])
    for redraw in (0, 1):
        t = r.weak_info_test(TABLE["hyper_count"], TABLE["datasets"], TABLE["particles"],
                             seed=TABLE["seed"], redraw_base=bool(redraw))
        for k, v in t.items():
            g[f"table{redraw}_{k}"] = v
    np.savez(os.path.join(HERE, "anneal.npz"), **g)
    print("wrote anneal.npz:", {k: v.shape for k, v in g.items()})
    print(g["run_evidence"], g["run_iterations"], g["table0_gamma"], g["table1_gamma"])


if __name__ == "__main__":
    main()
