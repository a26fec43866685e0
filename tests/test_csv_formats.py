"""Reference-format outputs: the CSV writers of the host layer
produce the bytes the reference's own writers produce (fixtures generated from
the unmodified reference by tests/golden/make_golden_csv.py)."""
import io
import math
import os
import subprocess

import numpy as np
import pytest

from paper_1902_09046_b200 import _abi as A, abc, bench_harness as B, lib, models as M

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")


def golden_text(name):
    with open(os.path.join(GOLD, name), newline="") as fh:
        return fh.read()


def test_prior_predictive_set_csv_roundtrip():
    text = golden_text("logistic_set.csv")
    pps = abc.read_csv(text)
    assert (pps.rows, pps.dim, pps.summary_dim) == (24, 3, 4)
    assert pps.failed.any() and not pps.failed.all()
    assert np.isnan(pps.discrepancies[pps.failed == 1]).all()
    out = io.StringIO()
    abc.write_csv(pps, out)
    assert out.getvalue() == text


def test_bench_csv_matches_reference_bytes(tmp_path):
    text = golden_text("bench_records.csv")
    records = B.parse_csv(text)
    assert len(records) == 28 and records[5].failed and math.isnan(records[5].runtime_seconds)
    assert records[-1].experiment == "tb" and records[9].mode == "blocked"
    # runtimes in the file carry 6 digits; rebuilding the file from the generator's
    # full-precision records must give the reference's bytes (records + summary)
    import sys
    sys.path.insert(0, GOLD)
    import make_golden_csv as G
    full = [B.BenchmarkRecord(B.EXPERIMENTS[e], B.MODES[m], t, w, r, rt, bool(f))
            for e, m, t, w, r, rt, f in G.bench_records()]
    out = io.StringIO()
    B.write_csv(full, out)
    assert out.getvalue() == text
    path = tmp_path / "b.csv"
    B.write_csv(full, str(path))
    assert open(path, newline="").read() == text
    rows = B.summarize(full)
    assert rows[0].speedup_vs_baseline == 1.0 and len(rows) == 10


def test_bench_harness_argument_errors(ref):
    for args in [(1.0, 9.0, 4.0), (0.0, 3.0, 16.0), (2.5, 0.0, 1.0)]:
        assert B.amdahl_bound(*args) == ref.amdahl_bound(*args)
    for args, code in [((-1.0, 1.0, 2.0), "invalid-input"), ((0.0, 0.0, 2.0), "invalid-input"),
                       ((1.0, 1.0, 0.5), "invalid-input")]:
        with pytest.raises(lib.VxbError) as e:
            B.amdahl_bound(*args)
        assert e.value.code == code
    with pytest.raises(lib.VxbError):
        B.parse_csv("nonsense\n")
    with pytest.raises(lib.VxbError):
        B.experiment_from_string("toggle")
    with pytest.raises(lib.VxbError):
        B.run_benchmark(None, B.BenchConfig(replicates=0))


@pytest.mark.gpu
def test_gpu_set_csv_equals_reference_file(ctx, golden, tmp_path):
    """run_prior_predictive on the GPU with the reference keying, written with the
    host layer's write_csv: byte-identical to the file the reference wrote."""
    import sys
    sys.path.insert(0, GOLD)
    import make_golden_csv as G
    c = G.SET_CASE
    pps = abc.run_prior_predictive(ctx, G.set_model(), c["n"], c["workers"], c["block_width"],
                                   c["seed"], golden["bad_observed"])
    path = tmp_path / "set.csv"
    abc.write_csv(pps, str(path))
    assert open(path, newline="").read() == golden_text("logistic_set.csv")


@pytest.mark.gpu
def test_gpu_bench_harness_runs_the_toggle_experiment(ctx, golden):
    cfg = B.BenchConfig(threads=[1, 3], block_widths=[1, 4], replicates=2,
                        sizes=B.ExperimentSizes(samples=32, cells=256, steps=100))
    records = B.run_benchmark(ctx, cfg)
    assert [(r.block_width, r.threads, r.replicate) for r in records] == \
        [(v, p, k) for v in (1, 4) for p in (1, 3) for k in (0, 1)]
    assert not any(r.failed for r in records) and all(r.runtime_seconds > 0 for r in records)
    out = io.StringIO()
    B.write_csv(records, out)
    again = B.parse_csv(out.getvalue())
    assert [(r.mode, r.threads, r.failed) for r in again] == [(r.mode, r.threads, r.failed) for r in records]
    # the body is the reference's experiment: same observed summaries as the KAT
    assert np.array_equal(B.toggle_observed_summaries(ctx, 100, 256, 1337, 4), golden["toggle_observed"])
    p, s, rho, f = B.run_experiment_once(ctx, "toggle-abc", cfg.sizes, 1, 4, 1337)
    assert rho[0] == 445.69940013687017
    with pytest.raises(lib.VxbError) as e:
        B.run_experiment_once(ctx, "bege", cfg.sizes, 1, 1, 1)
    assert e.value.code == "unsupported-model"


@pytest.mark.gpu
def test_gpu_weak_info_csv_equals_reference_file(ctx, tmp_path):
    from paper_1902_09046_b200 import weak_info as W
    table = W.run_weak_info_test(ctx, W.WeakInfoConfig(hyper_count=3, datasets=12, particles=200, seed=1337))
    out = io.StringIO()
    W.write_csv(table, out)
    assert out.getvalue() == golden_text("weakinfo_table.csv")
    assert [r.weakly_informative for r in table.rows][0] is False
    recs = B.run_benchmark(ctx, B.BenchConfig(experiment="weakinfo", threads=[1], block_widths=[4], replicates=1))
    assert len(recs) == 1 and not recs[0].failed
    assert np.array_equal(W.estimate_pvalues([2.0, 5.0], [1.0, 3.0, 4.0, 6.0]), [0.25, 0.75])
