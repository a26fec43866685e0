"""CPU tests of the multi-GPU host logic (gloo, world_size 2).

The data path has no collective: ranks simulate contiguous row ranges keyed by
global row index.  What needs testing without GPUs is the host side: the shard
rule (the reference's partition), the variable-length gather of accepted sets in
ascending global order, and the counter all-reduce.  The per-rank compute is
played by the oracle here (tests may use it); on the GPU box the same gather
code moves CUDA tensors over NCCL.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1902_09046_b200 import dist as D, models as M


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, n_total, eps, obs, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle.pyoracle import Oracle
    o = Oracle(threads=2)
    m = M.logistic_model(steps=200, obs_stride=10)
    begin, end = D.shard_range(n_total, world, rank)
    p, s, rho, f = o.abc_prior_predictive(m, M.keying(1337), n_total, begin, end - begin, obs,
                                          want_summaries=False)
    keep = (rho <= eps) & (f == 0)
    idx = torch.from_numpy((np.nonzero(keep)[0] + begin).astype(np.int64))
    g_idx, g_p, g_rho, counts = D.gather_accepted(idx, torch.from_numpy(p[keep]),
                                                  torch.from_numpy(rho[keep]))
    total = D.allreduce_sum(torch.tensor([int(keep.sum())], dtype=torch.int64))
    # asynchronous form: this rank's fixed-capacity packed block (count | idx | theta |
    # rho, include/vexbayes_cuda.h vxb_accept_layout) and ONE all_gather_into_tensor
    from paper_1902_09046_b200 import _abi as A, lib
    cap, k = 400, int(keep.sum())
    lay = lib.accept_layout(A.VXB_F64, 3, cap)
    block = torch.zeros(int(lay.stride), dtype=torch.uint8)
    b_idx, b_p, b_rho, b_n = D.packed_views(block, lay, A.VXB_F64, 3)
    b_idx[0].fill_(-1)
    b_idx[0, :k], b_p[0, :k], b_rho[0, :k], b_n[0] = idx, torch.from_numpy(p[keep]), torch.from_numpy(rho[keep]), k
    gathered = D.gather_packed(block, world)
    pi, pp, pr, pc = D.packed_views(gathered, lay, A.VXB_F64, 3, world)
    ci, cp, cr, cc = D.compact_gathered(pi, pp, pr, pc)
    # the C-ABI's host-side unpacking of the same gathered bytes agrees
    n_acc, u_idx, u_p, u_rho, over = lib.accept_unpack(lay, A.VXB_F64, 3, world, gathered.numpy())
    assert n_acc == sum(cc) and not over
    assert np.array_equal(u_idx.astype(np.int64), ci.numpy()) and np.array_equal(u_p, cp.numpy())
    assert np.array_equal(u_rho, cr.numpy())
    assert torch.equal(ci, g_idx) and torch.equal(cp, g_p) and torch.equal(cr, g_rho) and cc == counts
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), idx=g_idx.numpy(), p=g_p.numpy(),
             rho=g_rho.numpy(), counts=np.array(counts), total=total.numpy())
    dist.destroy_process_group()


def _counter_worker(rank, world, port, out_dir):
    """Configs 2 and 4: ranks own disjoint dataset / path ranges; one
    all-reduce(SUM) of integer counters gives the job's result."""
    import math
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle.pyoracle import Oracle
    from paper_1902_09046_b200 import _abi as A
    o = Oracle(threads=2)
    n_data, m_total = 20, 1001
    lam = np.array(M.lambda_grid(4))
    ln = np.array([-0.5 * math.log(2.0 * math.pi * (l * l + 1.0 / n_data)) for l in lam])
    b, e = D.shard_range(m_total, world, rank)
    counts, _, _ = o.ppp_pvalues(M.normal_mean_model(n_data), lam, ln, m_total, b, e - b, 7, 0.4)
    t = D.allreduce_sum(torch.from_numpy(counts.astype(np.int64)))
    cfg = A.vxb_mlmc_cfg()
    cfg.levels, cfg.refine, cfg.tau0, cfg.t_end, cfg.paths, cfg.seed = 3, 4, 1.0, 10.0, 501, 3
    b, e = D.shard_range(cfg.paths, world, rank)
    sums, _ = o.mlmc_level(M.mm_tauleap_model(), cfg, 2, b, e - b)
    s = D.allreduce_sum(torch.from_numpy(sums.copy()))
    np.savez(os.path.join(out_dir, f"c{rank}.npz"), counts=t.numpy(), sums=s.numpy())
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_rank_counter_allreduce(tmp_path, oracle):
    import math
    from paper_1902_09046_b200 import _abi as A
    mp.spawn(_counter_worker, args=(2, free_port(), str(tmp_path)), nprocs=2, join=True)
    n_data, m_total = 20, 1001
    lam = np.array(M.lambda_grid(4))
    ln = np.array([-0.5 * math.log(2.0 * math.pi * (l * l + 1.0 / n_data)) for l in lam])
    counts, _, _ = oracle.ppp_pvalues(M.normal_mean_model(n_data), lam, ln, m_total, 0, m_total, 7, 0.4)
    cfg = A.vxb_mlmc_cfg()
    cfg.levels, cfg.refine, cfg.tau0, cfg.t_end, cfg.paths, cfg.seed = 3, 4, 1.0, 10.0, 501, 3
    sums, _ = oracle.mlmc_level(M.mm_tauleap_model(), cfg, 2, 0, 501)
    for r in range(2):
        z = np.load(tmp_path / f"c{r}.npz")
        assert np.array_equal(z["counts"], counts.astype(np.int64))
        assert np.array_equal(z["sums"], sums)


def test_shard_rule_is_the_reference_partition(oracle):
    for total, world in [(100_000_000, 8), (1_000_003, 4), (7, 8), (1, 2), (1000, 3)]:
        want = oracle.partition(total, world, 1)
        got = np.array([D.shard_range(total, world, r) for r in range(world)], dtype=np.uint64)
        assert np.array_equal(got, want)
    want = oracle.partition(1003, 7, 8)
    got = np.array([D.shard_range(1003, 7, r, 8) for r in range(7)], dtype=np.uint64)
    assert np.array_equal(got, want)


@pytest.mark.timeout(300)
def test_two_rank_gather_equals_single_rank(tmp_path, oracle):
    n_total, world = 3001, 2
    m = M.logistic_model(steps=200, obs_stride=10)
    obs = oracle.simulate_at(m, [0.5, 100.0, 0.05], 5, 0, 0)
    p, s, rho, f = oracle.abc_prior_predictive(m, M.keying(1337), n_total, 0, n_total, obs,
                                               want_summaries=False)
    eps, idx = oracle.select_epsilon(rho, f, 0.05)
    mp.spawn(_worker, args=(world, free_port(), n_total, eps, obs, str(tmp_path)), nprocs=world,
             join=True)
    for r in range(world):
        z = np.load(tmp_path / f"rank{r}.npz")
        assert np.array_equal(z["idx"], idx.astype(np.int64))      # ascending global order
        assert np.array_equal(z["p"], p[idx]) and np.array_equal(z["rho"], rho[idx])
        assert z["counts"].sum() == len(idx) == z["total"][0]


# ---------------------------------------------------------------- ABC-SMC
class OracleStages:
    """Test stand-in for dist.DeviceStages: the same stage interface, computed by
    the CPU oracle on torch CPU tensors (so the gloo run exercises exactly the
    host logic that moves CUDA tensors over NCCL on the GPU box), including the
    device-resident round state: state[0] rows filled, [1] accepted, [2] rounds used."""

    def __init__(self, oracle):
        self.o = oracle
        self.device = torch.device("cpu")

    def scope(self):
        import contextlib
        return contextlib.nullcontext()

    @staticmethod
    def _pack(theta, rho, mask, layout, block, state, n):
        from paper_1902_09046_b200 import _abi as A
        idx, p, r, count = D.packed_views(block, layout, A.VXB_F64, theta.shape[1] if theta.ndim == 2 else 3)
        if int(state[0]) >= n or rho.size == 0:      # the gate of pack_rows_kernel
            count[0] = 0
            return
        k = int(mask.sum())
        assert k <= int(layout.cap)
        p[0, :k] = torch.from_numpy(np.ascontiguousarray(theta[mask]))
        r[0, :k] = torch.from_numpy(np.ascontiguousarray(rho[mask]))
        count[0] = k

    def prior_round(self, model, seed0, n_total, first, count, observed, layout, block, state, n):
        if count == 0:
            return self._pack(np.zeros((0, 3)), np.zeros(0), np.zeros(0, bool), layout, block, state, n)
        p, _, rho, f = self.o.abc_prior_predictive(model, M.keying(seed0), n_total, first, count,
                                                   observed, want_summaries=False)
        self._pack(p, rho, f == 0, layout, block, state, n)

    def propose_round(self, model, seed, gen, first, count, theta_prev, cum_prev, chol, observed, eps,
                      layout, block, state, n):
        if count == 0 or int(state[0]) >= n:         # the gate of the propose kernel
            return self._pack(np.zeros((0, 3)), np.zeros(0), np.zeros(0, bool), layout, block, state, n)
        th, rho, flag = self.o.abcsmc_propose(model, seed, gen, first, count, theta_prev.numpy(),
                                              cum_prev.numpy(), chol, observed, eps)
        self._pack(th, rho, flag == 1, layout, block, state, n)

    def append_round(self, blocks, world, layout, pop_theta, pop_rho, n, state):
        from paper_1902_09046_b200 import _abi as A
        got = int(state[0])
        if got >= n:
            return
        idx, p, r, count = D.packed_views(blocks, layout, A.VXB_F64, pop_theta.shape[1], world)
        total = 0
        for q in range(world):
            c = min(int(count[q]), int(layout.cap))
            take = max(0, min(c, n - (got + total)))
            pop_theta[got + total:got + total + take] = p[q, :take]
            pop_rho[got + total:got + total + take] = r[q, :take]
            total += c
        state[1] += total
        state[2] += 1
        state[0] = min(n, got + total)

    def weights(self, theta_new, theta_prev, w_prev, chol, rng=0):
        if theta_new.shape[0] == 0:
            return torch.zeros(0, dtype=torch.float64)
        return torch.from_numpy(self.o.abcsmc_weights(theta_new.numpy(), theta_prev.numpy(),
                                                      w_prev.numpy(), chol))

    def quantile(self, values, level):
        return self.o.quantile(values.numpy(), level)

    def moments(self, theta, w):
        return self.o.weighted_moments(theta.numpy(), w.numpy())

    def cumsum(self, w):
        return torch.from_numpy(self.o.canon_cumsum(w.numpy()))

    def chunk_sums(self, v):
        v = v.numpy()
        return torch.tensor([self.o.canon_sum(v[i:i + D.CHUNK]) for i in range(0, v.size, D.CHUNK)],
                            dtype=torch.float64)

    def normalise_by_totals(self, w_raw, totals):
        total = 0.0
        for v in totals.tolist():  # chunk totals, left to right
            total += v
        return torch.from_numpy(w_raw.numpy() / total)

    def make_kernel(self, cov, scale, jitter):
        return self.o.make_kernel(cov, scale, jitter)


def smc_case():
    from paper_1902_09046_b200 import _abi as A
    m = M.logistic_model(steps=100, obs_stride=10)
    cfg = A.vxb_abcsmc_cfg()
    cfg.particles, cfg.generations, cfg.quantile = 700, 3, 0.5
    cfg.kernel_scale, cfg.jitter, cfg.round_size, cfg.max_rounds, cfg.seed = 2.0, 1e-10, 900, 200, 11
    return m, cfg


def _smc_worker(rank, world, port, obs, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle.pyoracle import Oracle
    m, cfg = smc_case()
    res = D.sharded_abcsmc(OracleStages(Oracle(threads=2)), m, cfg, obs)
    np.savez(os.path.join(out_dir, f"smc{rank}.npz"), **res)
    dist.destroy_process_group()


@pytest.mark.timeout(600)
@pytest.mark.parametrize("world", [2, 3, 4])
def test_sharded_abcsmc_equals_single_run(tmp_path, oracle, world):
    """Proposals and new particles sharded over ranks; the packed blocks of accepted
    rows all-gathered once per round (rounds issued ahead of the host, state on the
    "device"), chunk totals of the weights all-reduced: bit-identical to the
    one-process run (oracle.abcsmc_run) for every world size.  With 4 ranks the 700
    particles make 3 canonical chunks: one rank owns an EMPTY weight shard."""
    m, cfg = smc_case()
    obs = oracle.simulate_at(m, [0.5, 100.0, 0.05], 5, 0, 0)
    want = oracle.abcsmc_run(m, cfg, obs)
    mp.spawn(_smc_worker, args=(world, free_port(), obs, str(tmp_path)), nprocs=world, join=True)
    for r in range(world):
        z = np.load(tmp_path / f"smc{r}.npz")
        for k, v in want.items():
            assert np.array_equal(z[k], v), (k, r)
    # one rank, no process group: same driver, same result
    got = D.sharded_abcsmc(OracleStages(oracle), m, cfg, obs)
    for k, v in want.items():
        assert np.array_equal(got[k], v), k


# -------------------------------------------------- weak-informativity test
def _fake_evidence(cfg):
    """A deterministic stand-in for the device sampler: evidence of (row, dataset,
    which) as a pure function of its indices, a few NaN (failed runs)."""
    rows, n = cfg.hyper_count + 1, cfg.datasets
    k, i, w = np.meshgrid(np.arange(rows), np.arange(n), np.arange(2), indexing="ij")
    ev = np.sin(1.0 + 0.37 * k + 0.11 * i + 1.3 * w) * (1.0 + 0.05 * k)
    ev[(k * 7 + i * 3 + w) % 23 == 0] = np.nan
    return ev


def _weakinfo_worker(rank, world, port, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = M.weakinfo_config(hyper_count=10, datasets=17, particles=64, alpha=0.1)
    full = _fake_evidence(cfg)
    t = D.sharded_weak_info(None, cfg, evidence_fn=lambda first, count: full[first:first + count])
    np.savez(os.path.join(out_dir, f"wi{rank}.npz"), gamma=t["gamma"], weakly=t["weakly"],
             completed=t["completed"], evidence=t["evidence"])
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_sharded_weak_info_rows(tmp_path, oracle):
    """Rows sharded over 3 ranks, evidences all-gathered, cut-offs computed by the
    library's host stage: equal to the unsharded table and to the oracle's
    estimate_pvalues / compute_cutoff on the same evidences."""
    from paper_1902_09046_b200 import lib
    mp.spawn(_weakinfo_worker, args=(3, free_port(), str(tmp_path)), nprocs=3, join=True)
    cfg = M.weakinfo_config(hyper_count=10, datasets=17, particles=64, alpha=0.1)
    full = _fake_evidence(cfg)
    gamma, weakly, completed = lib.weak_info_cutoffs(cfg, full)
    for r in range(3):
        z = np.load(tmp_path / f"wi{r}.npz")
        assert np.array_equal(z["evidence"], full, equal_nan=True)
        assert np.array_equal(z["gamma"], gamma) and np.array_equal(z["weakly"], weakly)
        assert np.array_equal(z["completed"], completed)
    for k in range(cfg.hyper_count + 1):
        b, h = full[k, :, 0], full[k, :, 1]
        pv = oracle.estimate_pvalues(b[~np.isnan(b)], h[~np.isnan(h)])
        assert gamma[k] == oracle.compute_cutoff(pv, 0.1)
        assert completed[k] == int((~np.isnan(b) & ~np.isnan(h)).sum())
    assert np.array_equal(weakly, (np.arange(11) != 0) & (gamma > gamma[0]))
