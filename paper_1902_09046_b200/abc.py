"""Host-side mirror of the reference ABC sampler interface (abc.hpp:16-58).

Same names, argument meaning and error behaviour as ``vexbayes::abc``; every
call runs on the GPU through the C ABI (``lib.Context``).  The C++ form of the
same shim lives in ``cpp/vexbayes/abc.hpp``.
"""
from dataclasses import dataclass

import numpy as np

from . import _abi as A, models as M
from .lib import VxbError


@dataclass
class PriorPredictiveSet:
    """abc.hpp:16-31 -- rows x dim params, rows x summary_dim summaries, rho, failed."""
    rows: int
    dim: int
    summary_dim: int
    params: np.ndarray
    summaries: np.ndarray
    discrepancies: np.ndarray
    failed: np.ndarray

    def param_row(self, r):
        return self.params[r]

    def summary_row(self, r):
        return self.summaries[r]


@dataclass
class EpsilonSelection:
    """abc.hpp:45-48"""
    epsilon: float
    accepted: np.ndarray  # ascending row indices with rho <= epsilon


def discrepancy(sim, obs):
    """abc::discrepancy (abc.cpp:16-24): Euclidean, left-to-right accumulation."""
    sim, obs = np.asarray(sim, dtype=np.float64), np.asarray(obs, dtype=np.float64)
    if sim.shape != obs.shape:
        raise VxbError("invalid-summary: summary vector lengths differ")
    ss = 0.0
    for s, o in zip(sim.tolist(), obs.tolist()):
        d = s - o
        ss += d * d
    return float(np.sqrt(ss))


def run_prior_predictive(ctx, model, n, workers, block_width, seed, observed):
    """abc::run_prior_predictive (abc.cpp:26-73) on the GPU.

    ``model`` is a ``vxb_model`` descriptor (models.logistic_model).  Results
    are bit-identical to the reference for the same (seed, workers,
    block_width): the device reproduces the reference's per-worker stream
    consumption (VXB_KEY_WORKER).  ``ctx`` may be a ``lib.Context`` (one GPU) or a
    ``lib.Multi`` (rows split over its devices by partition(n, G, 1); same rows)."""
    if n < 1:
        raise VxbError("invalid-shape: need at least one prior predictive sample")
    if workers < 1:
        raise VxbError("invalid-shape: need at least one worker")
    observed = np.asarray(observed, dtype=np.float64)
    if observed.size != model.summary_dim:
        raise VxbError("invalid-summary: observed summary length differs from the model "
                       "summary dimension")
    key = M.keying(seed, A.VXB_KEY_WORKER, workers, block_width)
    if hasattr(ctx, "abc_prior_predictive_host"):
        p, s, rho, f = ctx.abc_prior_predictive_host(model, key, n, 0, n, observed)
    else:  # lib.Multi
        p, s, rho, f = ctx.abc_prior_predictive(model, key, n, observed)
    return PriorPredictiveSet(n, model.dim, model.summary_dim, p, s, rho, f)


def select_epsilon(ctx, pps, accept_fraction):
    """abc::select_epsilon (abc.cpp:75-97) on the GPU."""
    eps, idx, _ = ctx.select_epsilon(pps.discrepancies, pps.failed, accept_fraction)
    return EpsilonSelection(eps, idx)


def write_csv(pps, out):
    """abc::write_csv (abc.cpp:99-124): header ``row,theta_*,s_*,rho,failed``,
    every real with ``%.17g``.  `out` is a path or a text file object."""
    from .bench_harness import _c_g
    head = ["row"] + [f"theta_{k + 1}" for k in range(pps.dim)] + \
           [f"s_{k + 1}" for k in range(pps.summary_dim)] + ["rho", "failed"]
    lines = [",".join(head)]
    params = np.asarray(pps.params, dtype=np.float64).reshape(pps.rows, pps.dim)
    summ = np.asarray(pps.summaries, dtype=np.float64).reshape(pps.rows, pps.summary_dim)
    rho = np.asarray(pps.discrepancies, dtype=np.float64)
    for r in range(pps.rows):
        cells = [str(r)] + [_c_g(v, 17) for v in params[r].tolist()] + \
                [_c_g(v, 17) for v in summ[r].tolist()] + [_c_g(float(rho[r]), 17),
                                                          str(int(pps.failed[r]))]
        lines.append(",".join(cells))
    text = "\n".join(lines) + "\n"
    if hasattr(out, "write"):
        out.write(text)
        return
    try:
        with open(out, "w", newline="") as fh:
            fh.write(text)
    except OSError:
        raise VxbError(f"io-error: cannot open {out} for writing")


def read_csv(text):
    """Inverse of write_csv (``%.17g`` round-trips every double)."""
    lines = [ln for ln in text.split("\n") if ln]
    head = lines[0].split(",")
    dim = sum(h.startswith("theta_") for h in head)
    sd = sum(h.startswith("s_") for h in head)
    body = np.array([[float(c) for c in ln.split(",")] for ln in lines[1:]], dtype=np.float64)
    body = body.reshape(len(lines) - 1, len(head))
    return PriorPredictiveSet(body.shape[0], dim, sd, body[:, 1:1 + dim].copy(),
                              body[:, 1 + dim:1 + dim + sd].copy(), body[:, 1 + dim + sd].copy(),
                              body[:, -1].astype(np.uint8))
