"""Generates the reference-format CSV fixtures from the UNMODIFIED reference:

    make -C oracle ref && python tests/golden/make_golden_csv.py

* logistic_set.csv   abc::write_csv (abc.cpp:99-124) of the set the reference's
                     run_prior_predictive returns for the logistic hooks with a
                     prior box that makes some rows fail (NaN rho, failed = 1);
                     (n, workers, block_width, seed) = (24, 3, 2, 21).
* weakinfo_table.csv weakinfo::write_csv of the reference's run_weak_info_test.
* bench_records.csv  bench::write_csv (bench.cpp:215-230) of the synthetic
                     records below (a failed replicate included).
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
HERE = os.path.dirname(os.path.abspath(__file__))

from oracle.pyoracle import Ref  # noqa: E402
from paper_1902_09046_b200 import models as M  # noqa: E402

SET_CASE = dict(n=24, workers=3, block_width=2, seed=21)


def set_model():
    return M.logistic_model(steps=400, obs_stride=100, prior_lo=(0.0, 50.0, 0.0),
                            prior_hi=(4000.0, 150.0, 0.2))


def bench_records():
    # (experiment, mode, threads, block_width, replicate, runtime_seconds, failed)
    rec = []
    rs = np.random.RandomState(7)
    for width in (1, 4, 8):
        for threads in (1, 2, 16):
            for rep in range(3):
                t = 10.0 / threads / (1.0 + 0.3 * (width > 1)) * (1.0 + 0.01 * rs.normal())
                rec.append((0, 0 if width == 1 else 1, threads, width, rep, float(t), 0))
    rec[5] = rec[5][:5] + (float("nan"), 1)
    rec.append((3, 0, 1, 1, 0, 1.0 / 3.0, 0))
    return rec


def main():
    r = Ref()
    obs = np.load(os.path.join(HERE, "golden.npz"))["bad_observed"]
    r.logistic_abc_csv(set_model(), SET_CASE["n"], SET_CASE["workers"], SET_CASE["block_width"],
                       SET_CASE["seed"], obs, os.path.join(HERE, "logistic_set.csv"))
    r.bench_csv(bench_records(), os.path.join(HERE, "bench_records.csv"))
    # weakinfo::write_csv (weak_info.cpp:279-293) of run_weak_info_test(K=3, N=12, N_p=200, seed 1337)
    r.weak_info_test(3, 12, 200, seed=1337, csv_path=os.path.join(HERE, "weakinfo_table.csv"))
    text = open(os.path.join(HERE, "logistic_set.csv")).read()
    assert ",1\n" in text and ",0\n" in text, "want failed and good rows in the fixture"
    print("wrote logistic_set.csv", len(text), "bytes; bench_records.csv")


if __name__ == "__main__":
    main()
