"""Host-side mirror of the reference benchmark harness (bench.hpp / bench.cpp).

Same record and summary layout, same CSV bytes (records section, then the
summary section; times with six significant digits, bench.cpp:22-31,215-230),
same timing protocol (one discarded warm-up per cell, wall clock around the
experiment body only, failures recorded as NaN + flag, bench.cpp:140-172) -- so
that files written here diff against files written by the reference.  The
experiment body runs on the GPU through the C ABI: `threads` and `block_width`
keep their meaning as the (P, V) of the reference keying (VXB_KEY_WORKER), which
makes the produced samples identical to the CPU run of the same cell.

Only the experiments on the GPU path are runnable (toggle-abc, weakinfo, tb); bege is
kept as a name so that reference files parse.
"""
import math
import time
from dataclasses import dataclass, field

import numpy as np

from . import _abi as A, models as M
from .lib import VxbError, derive_seed

EXPERIMENTS = ("toggle-abc", "weakinfo", "bege", "tb")   # bench.cpp:33-41
MODES = ("scalar", "blocked")                            # bench.cpp:43
RECORD_HEADER = "experiment,mode,threads,block_width,replicate,runtime_seconds,failed"
SUMMARY_HEADER = "experiment,mode,threads,block_width,mean_runtime,speedup_vs_baseline"


def _c_g(value, digits):
    """printf("%.<digits>g") -- Python's % formatting follows C for finite values;
    non-finite values are spelled the way glibc spells them."""
    if math.isnan(value):
        return "-nan" if math.copysign(1.0, value) < 0 else "nan"
    if math.isinf(value):
        return "-inf" if value < 0 else "inf"
    return "%.*g" % (digits, value)


def format_time(seconds):
    return _c_g(seconds, 6)


def experiment_from_string(name):
    if name not in EXPERIMENTS:
        raise VxbError("invalid-input: unknown experiment: " + name)
    return name


def mode_from_string(name):
    if name not in MODES:
        raise VxbError("invalid-input: unknown mode: " + name)
    return name


@dataclass
class BenchmarkRecord:          # bench.hpp:22-30
    experiment: str
    mode: str
    threads: int
    block_width: int
    replicate: int
    runtime_seconds: float
    failed: bool


@dataclass
class ExperimentSizes:          # bench.hpp:32-43
    samples: int = 64
    cells: int = 256
    steps: int = 100
    particles: int = 200  # SMC N_p
    hypers: int = 2       # weak-info K
    datasets: int = 8     # weak-info N
    tb_initial: int = 10
    tb_horizon: float = 10.0
    tb_target: float = 10000.0


@dataclass
class BenchConfig:              # bench.hpp:45-53
    experiment: str = "toggle-abc"
    threads: list = field(default_factory=lambda: [1, 2, 4, 8, 16])
    block_widths: list = field(default_factory=lambda: [1, 4, 8])
    replicates: int = 4
    seed: int = 1337
    sizes: ExperimentSizes = field(default_factory=ExperimentSizes)
    warmup: bool = True


@dataclass
class SummaryRow:               # bench.hpp:76-83
    experiment: str
    mode: str
    threads: int
    block_width: int
    mean_runtime: float
    speedup_vs_baseline: float


def amdahl_bound(serial_seconds, parallel_seconds, units):
    """(C_S + C_P) / (C_S + C_P / P), bench.cpp:58-67."""
    if not (serial_seconds >= 0.0 and parallel_seconds >= 0.0):
        raise VxbError("invalid-input: runtimes must be nonnegative")
    if not serial_seconds + parallel_seconds > 0.0:
        raise VxbError("invalid-input: total runtime must be positive")
    if not units >= 1.0:
        raise VxbError("invalid-input: need at least one processing unit")
    return (serial_seconds + parallel_seconds) / (serial_seconds + parallel_seconds / units)


def toggle_observed_summaries(ctx, steps, cells, seed, block_width):
    """bench.cpp:69-77: one simulation at the prior midpoints from
    RngStream(derive_seed(seed,{90}), 0), reduced to the 19 quantiles."""
    # cell c owns stream positions [c*2T, (c+1)*2T) (toggle_switch.hpp:52-57), so a
    # single simulation from position 0 does not depend on the block width
    del block_width
    return ctx.simulate_at(M.toggle_model(steps, cells), M.TOGGLE_MIDPOINT,
                           derive_seed(seed, [90]), 0, 0)


def tb_observed_summaries(ctx, initial_cases, horizon, target, seed, block_width):
    """bench.cpp:79-92: theta = (0.2, 0.1, 0.05) from RngStream(derive_seed(seed,{91}), 0),
    retried off the same stream while the population dies out."""
    del block_width
    return ctx.simulate_at(M.tb_model(initial_cases, horizon, target, attempts=64),
                           M.TB_TRUE_THETA, derive_seed(seed, [91]), 0, 0)


def run_experiment_once(ctx, experiment, sizes, threads, block_width, seed):
    """bench.cpp:94-137, the toggle-abc body on the GPU."""
    if experiment_from_string(experiment) == "weakinfo":   # bench.cpp:113-123
        cfg = M.weakinfo_config(hyper_count=sizes.hypers, datasets=sizes.datasets,
                                particles=sizes.particles, block_width=block_width, seed=seed)
        return ctx.weak_info_test(cfg)
    if experiment == "tb":                                 # bench.cpp:104-111; particle keying
        observed = tb_observed_summaries(ctx, sizes.tb_initial, sizes.tb_horizon, sizes.tb_target,
                                         seed, block_width)
        model = M.tb_model(sizes.tb_initial, sizes.tb_horizon, sizes.tb_target)
        return ctx.abc_prior_predictive_host(model, M.keying(seed), sizes.samples, 0, sizes.samples,
                                             observed)
    if experiment != "toggle-abc":
        raise VxbError("unsupported-model: experiment " + experiment + " has no device path")
    observed = toggle_observed_summaries(ctx, sizes.steps, sizes.cells, seed, block_width)
    key = M.keying(seed, A.VXB_KEY_WORKER, threads, block_width)
    return ctx.abc_prior_predictive_host(M.toggle_model(sizes.steps, sizes.cells), key,
                                         sizes.samples, 0, sizes.samples, observed)


def run_benchmark(ctx, config):
    """bench.cpp:140-172: every (block width, threads, replicate) cell in the
    reference's order; a failing cell is recorded, not raised."""
    if config.replicates < 1:
        raise VxbError("invalid-input: need at least one replicate")
    if not config.threads or not config.block_widths:
        raise VxbError("invalid-input: thread and block-width lists must not be empty")
    records = []
    for v in config.block_widths:
        mode = "scalar" if v == 1 else "blocked"
        for p in config.threads:
            if config.warmup:
                try:
                    run_experiment_once(ctx, config.experiment, config.sizes, p, v, config.seed)
                except Exception:
                    pass
            for rep in range(config.replicates):
                rec = BenchmarkRecord(config.experiment, mode, p, v, rep, 0.0, False)
                start = time.perf_counter()
                try:
                    run_experiment_once(ctx, config.experiment, config.sizes, p, v, config.seed)
                    rec.runtime_seconds = time.perf_counter() - start
                except Exception:
                    rec.runtime_seconds, rec.failed = float("nan"), True
                records.append(rec)
    return records


def summarize(records):
    """bench.cpp:174-213: per-cell mean over the non-failed replicates and the
    speed-up against the first (scalar, threads = 1) cell."""
    rows, cells = [], {}
    for r in records:
        cell = (r.experiment, r.mode, r.threads, r.block_width)
        if cell not in cells:
            cells[cell] = [0.0, 0]
            rows.append(SummaryRow(*cell, 0.0, 0.0))
        if not r.failed:
            cells[cell][0] += r.runtime_seconds
            cells[cell][1] += 1
    baseline = float("nan")
    for row in rows:
        total, n = cells[(row.experiment, row.mode, row.threads, row.block_width)]
        row.mean_runtime = total / n if n else float("nan")
    for row in rows:
        if row.mode == "scalar" and row.threads == 1:
            baseline = row.mean_runtime
            break
    for row in rows:
        row.speedup_vs_baseline = baseline / row.mean_runtime
    return rows


def write_csv(records, out):
    """bench.cpp:215-230.  `out` is a path or a text file object."""
    lines = [RECORD_HEADER]
    for r in records:
        lines.append(f"{r.experiment},{r.mode},{r.threads},{r.block_width},{r.replicate},"
                     f"{format_time(r.runtime_seconds)},{1 if r.failed else 0}")
    lines.append(SUMMARY_HEADER)
    for s in summarize(records):
        lines.append(f"{s.experiment},{s.mode},{s.threads},{s.block_width},"
                     f"{format_time(s.mean_runtime)},{format_time(s.speedup_vs_baseline)}")
    text = "\n".join(lines) + "\n"
    if hasattr(out, "write"):
        out.write(text)
        return
    try:
        with open(out, "w", newline="") as fh:
            fh.write(text)
    except OSError:
        raise VxbError(f"io-error: cannot open {out} for writing")


def parse_csv(text):
    """bench.cpp:239-269: the records section (up to the summary header)."""
    lines = text.split("\n")
    if not lines or (len(lines) == 1 and lines[0] == ""):
        raise VxbError("io-error: empty benchmark file")
    header = lines[0].rstrip("\r")
    if header != RECORD_HEADER:
        raise VxbError("io-error: unexpected benchmark header: " + header)
    records = []
    for line in lines[1:]:
        line = line.rstrip("\r")
        if not line:
            continue
        if line == SUMMARY_HEADER:
            break
        f = line.split(",")
        if len(f) < 7:
            raise VxbError("io-error: malformed benchmark row: " + line)
        records.append(BenchmarkRecord(experiment_from_string(f[0]), mode_from_string(f[1]),
                                       int(f[2]), int(f[3]), int(f[4]), float(f[5]),
                                       int(f[6]) != 0))
    return records
