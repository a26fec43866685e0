"""Host-side mirror of the reference weak-informativity interface
(weak_info.hpp:13-104); every sampler run executes on the GPU (one CTA per run,
``vxb_weak_info_test``).  The C++ form lives in ``cpp/vexbayes/weak_info.hpp``."""
from dataclasses import dataclass, field

import numpy as np

from . import models as M
from .bench_harness import _c_g
from .lib import VxbError

BASE_PRIOR = (10.0, 2.5)                      # kBasePrior, weak_info.hpp:21


@dataclass
class WeakInfoConfig:                         # weak_info.hpp:62-75
    hyper_count: int = 400
    datasets: int = 400
    particles: int = 500
    alpha: float = 0.05
    c: float = 0.01
    scale: float = 1.6828427124746189
    workers: int = 1                          # accepted; no device meaning
    block_width: int = 4
    seed: int = 0
    redraw_base: bool = False
    base: tuple = BASE_PRIOR
    dose: tuple = M.DEFAULT_DOSE
    group_size: tuple = M.DEFAULT_GROUP_SIZE


@dataclass
class CutoffRow:                              # weak_info.hpp:77-83
    index: int
    lambda1: float
    lambda2: float
    gamma: float
    weakly_informative: bool
    completed: int


@dataclass
class CutoffTable:
    alpha: float = 0.0
    rows: list = field(default_factory=list)


def estimate_pvalues(evidences_base, evidences_k):
    """weak_info.cpp:108-120: p_i = #{j : k_j <= base_i} / N (ties count)."""
    k = np.sort(np.asarray(evidences_k, dtype=np.float64))
    if k.size == 0:
        raise VxbError("invalid-argument: need at least one comparison evidence")
    return np.searchsorted(k, np.asarray(evidences_base, dtype=np.float64), side="right") / k.size


def run_weak_info_test(ctx, config):
    """weak_info.cpp:163-277 on the GPU."""
    if config.datasets < 1:
        raise VxbError("invalid-argument: need at least one dataset per prior")
    if config.workers < 1:
        raise VxbError("invalid-argument: need at least one worker")
    cfg = M.weakinfo_config(config.hyper_count, config.datasets, config.particles, config.alpha,
                            config.c, config.scale, config.block_width, config.seed,
                            config.redraw_base, config.base, config.dose, config.group_size)
    t = ctx.weak_info_test(cfg)
    table = CutoffTable(config.alpha)
    for k in range(config.hyper_count + 1):
        table.rows.append(CutoffRow(k, float(t["lambda_"][k, 0]), float(t["lambda_"][k, 1]),
                                    float(t["gamma"][k]), bool(t["weakly"][k]),
                                    int(t["completed"][k])))
    return table


def write_csv(table, out):
    """weak_info.cpp:279-293: k,lambda1,lambda2,gamma_alpha,weakly_informative."""
    lines = ["k,lambda1,lambda2,gamma_alpha,weakly_informative"]
    for r in table.rows:
        lines.append(f"{r.index},{_c_g(r.lambda1, 17)},{_c_g(r.lambda2, 17)},{_c_g(r.gamma, 17)},"
                     f"{1 if r.weakly_informative else 0}")
    text = "\n".join(lines) + "\n"
    if hasattr(out, "write"):
        out.write(text)
    else:
        with open(out, "w", newline="") as fh:
            fh.write(text)
