"""GPU tests of the multi-GPU layer behind the C ABI (include/vexbayes_cuda.h, section
"multi-GPU"), run with however many GPUs the box has: vxb_multi_* over every visible
device against the oracle and against the one-context calls, and the library's own NCCL
communicator (vxb_comm_*) -- with one GPU a real 1-rank communicator, so NCCL is
loaded, initialised and runs its collectives on the device."""
import math

import numpy as np
import pytest

from paper_1902_09046_b200 import _abi as A, dist as D, lib, models as M

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def multi():
    m = lib.Multi()
    yield m
    m.close()


def test_multi_drivers_equal_one_context_and_oracle(ctx, multi, oracle, golden):
    import torch
    assert multi.size == torch.cuda.device_count() == lib.device_count()
    obs = golden["logistic_observed"]
    m = M.logistic_model()
    # run_prior_predictive, reference keying (workers = stream layout, not devices)
    key = M.keying(1337, A.VXB_KEY_WORKER, 5, 4)
    got = multi.abc_prior_predictive(m, key, 2003, obs)
    want = oracle.abc_prior_predictive(m, key, 2003, 0, 2003, obs)
    for g, w in zip(got, want):
        assert np.array_equal(g, w, equal_nan=True)
    from paper_1902_09046_b200 import abc
    pps = abc.run_prior_predictive(multi, m, 2003, 5, 4, 1337, obs)       # the Python mirror over Multi
    assert np.array_equal(pps.discrepancies, want[2], equal_nan=True) and np.array_equal(pps.params, want[0])
    # fused rejection + gather of the accepted samples
    p, _, rho, f = oracle.abc_prior_predictive(m, M.keying(7), 40000, 0, 40000, obs, want_summaries=False)
    eps, idx_o = oracle.select_epsilon(rho, f, 0.02)
    nacc, idx, params, rho_acc = multi.abc_reject(m, M.keying(7), 40000, obs, eps, cap=40000)
    assert nacc == len(idx_o) and np.array_equal(idx, idx_o)
    assert np.array_equal(params, p[idx_o]) and np.array_equal(rho_acc, rho[idx_o])
    nacc2, idx2, _, _ = multi.abc_reject(m, M.keying(7), 40000, obs, eps, cap=9)
    assert nacc2 == nacc and np.array_equal(idx2, idx_o[:9])
    # fp32 throughput variant: equal to the one-context call
    mf = M.logistic_model(precision=A.VXB_F32, rng=A.VXB_RNG_FAST)
    a = multi.abc_reject(mf, M.keying(7), 40000, obs, eps, cap=4000)
    b = ctx.abc_reject(mf, M.keying(7), 40000, 0, 40000, obs, eps, cap=4000)
    assert a[0] == b[0] and all(np.array_equal(x, y) for x, y in zip(a[1:], b[1:]))
    # configs 2 and 4: integer counters of disjoint ranges
    lam = np.array(M.lambda_grid(8))
    ln = np.array([-0.5 * math.log(2.0 * math.pi * (l * l + 0.01)) for l in lam])
    mdl = M.normal_mean_model(100)
    c1, p1, _ = ctx.ppp_pvalues(mdl, lam, ln, 30001, 0, 30001, 1337, 2.9)
    c2, p2 = multi.ppp_pvalues(mdl, lam, ln, 30001, 1337, 2.9)
    assert np.array_equal(c1, c2) and np.array_equal(p1, p2)
    mc = A.vxb_mlmc_cfg()
    mc.levels, mc.refine, mc.tau0, mc.t_end, mc.paths, mc.seed = 3, 4, 1.0, 30.0, 20001, 1337
    r1, r2 = ctx.mlmc_tauleap(M.mm_tauleap_model(), mc), multi.mlmc_tauleap(M.mm_tauleap_model(), mc)
    for k in ("level_mean", "level_var", "level_cost"):
        assert np.array_equal(r1[k], r2[k])
    assert r1["estimate"] == r2["estimate"] and r1["std_error"] == r2["std_error"]


def test_library_nccl_communicator_one_rank(ctx, oracle, golden):
    """vxb_comm_* with n_ranks = 1: NCCL is dlopen'ed, a communicator is created on the
    context's stream and its all-gather / all-reduce run on the GPU; the SPMD entry point
    vxb_sharded_abc_reject through dist.sharded_reject(comm=...) equals the plain path."""
    import torch
    assert lib.comm_version() >= 21800
    comm = lib.Comm(ctx, lib.comm_unique_id(), 0, 1)
    assert (comm.rank, comm.size) == (0, 1)
    dev = torch.device("cuda", ctx.device_info()["device"])
    with torch.cuda.stream(torch.cuda.ExternalStream(ctx.stream(), device=dev)):
        a = torch.arange(1000, dtype=torch.float64, device=dev)
        b = torch.empty_like(a)
        comm.allgather(a, b, a.numel() * 8)
        comm.allreduce(b, b.numel(), A.VXB_DT_F64, A.VXB_OP_SUM)
        c = torch.arange(64, dtype=torch.int64, device=dev)
        comm.allreduce(c, 64, A.VXB_DT_I64, A.VXB_OP_MAX)
    ctx.synchronize()
    assert torch.equal(a, b) and torch.equal(c, torch.arange(64, dtype=torch.int64, device=dev))
    obs = golden["logistic_observed"]
    m = M.logistic_model()
    _, _, rho, f = oracle.abc_prior_predictive(m, M.keying(3), 20000, 0, 20000, obs, want_summaries=False)
    eps, idx_o = oracle.select_epsilon(rho, f, 0.03)
    for kw in ({}, {"comm": comm}):
        idx, params, r, n_dev = D.sharded_reject(ctx, m, M.keying(3), 20000, obs, eps, cap_fraction=0.1, **kw)
        ctx.synchronize()
        k = int(n_dev.item())
        assert k == len(idx_o) and np.array_equal(idx[:k].cpu().numpy(), idx_o.astype(np.int64))
        assert np.array_equal(r[:k].cpu().numpy(), rho[idx_o])
    # the SPMD selection over this (real, one-rank) NCCL communicator: the all-reduces of the
    # valid counts (int64) and of the digit histograms (uint32) and the gather of the index
    # block run through NCCL; same epsilon bits and indices as the oracle
    cap = 2000
    blk = torch.zeros(16 + 8 * cap, dtype=torch.uint8, device=dev)
    blks = torch.zeros_like(blk)
    e, n_acc = ctx.sharded_select_epsilon(comm, rho, f, 0, 0.03, cap=cap, block_local=blk, blocks_all=blks)
    ctx.synchronize()
    got = blks.cpu().numpy()
    assert e == eps and n_acc == len(idx_o) == int(got[:8].view(np.uint64)[0])
    assert np.array_equal(got[16:16 + 8 * n_acc].view(np.uint64), idx_o.astype(np.uint64))
    # configs 2 and 4 through the same communicator (int64 all-reduce of the counters)
    lam = np.array(M.lambda_grid(8))
    ln = np.array([-0.5 * math.log(2.0 * math.pi * (l * l + 0.01)) for l in lam])
    c1, p1, _ = ctx.ppp_pvalues(M.normal_mean_model(100), lam, ln, 20001, 0, 20001, 1337, 2.9)
    c2, p2 = ctx.sharded_ppp_pvalues(comm, M.normal_mean_model(100), lam, ln, 20001, 1337, 2.9)
    assert np.array_equal(c1, c2) and np.array_equal(p1, p2)
    mc = A.vxb_mlmc_cfg()
    mc.levels, mc.refine, mc.tau0, mc.t_end, mc.paths, mc.seed = 3, 4, 1.0, 30.0, 5001, 1337
    r1, r2 = ctx.mlmc_tauleap(M.mm_tauleap_model(), mc), ctx.sharded_mlmc_tauleap(comm, M.mm_tauleap_model(), mc)
    assert all(np.array_equal(r1[k], r2[k]) for k in ("level_mean", "level_var")) and r1["estimate"] == r2["estimate"]
    h = torch.arange(5000, dtype=torch.int32, device=dev)
    with torch.cuda.stream(torch.cuda.ExternalStream(ctx.stream(), device=dev)):
        comm.allreduce(h, h.numel(), A.VXB_DT_U32, A.VXB_OP_SUM)
    ctx.synchronize()
    assert torch.equal(h, torch.arange(5000, dtype=torch.int32, device=dev))
    comm.close()


def test_native_sharded_abcsmc_equals_one_gpu_driver(ctx, multi, golden):
    """vxb_sharded_abcsmc_run (SPMD, NCCL inside the library) and vxb_multi_abcsmc_run:
    bit-identical to vxb_abcsmc_run in both generator modes, with rounds smaller than
    the population (several rounds per generation, issued ahead of the host); as one
    rank without a communicator, as one rank WITH a real NCCL communicator, and over
    every visible device."""
    obs = golden["logistic_observed"]
    comm = lib.Comm(ctx, lib.comm_unique_id(), 0, 1)
    for rng, n, gens, round_size, seed in ((A.VXB_RNG_REF, 2000, 4, 0, 1337), (A.VXB_RNG_REF, 777, 3, 300, 9),
                                           (A.VXB_RNG_FAST, 1500, 4, 0, 21)):
        m = M.logistic_model(rng=rng)
        cfg = A.vxb_abcsmc_cfg()
        cfg.particles, cfg.generations, cfg.quantile, cfg.kernel_scale = n, gens, 0.5, 2.0
        cfg.jitter, cfg.round_size, cfg.max_rounds, cfg.seed = 1e-10, round_size, 0, seed
        want = ctx.abcsmc_run(m, cfg, obs)
        for got in (ctx.sharded_abcsmc_run(None, m, cfg, obs), ctx.sharded_abcsmc_run(comm, m, cfg, obs),
                    multi.abcsmc_run(m, cfg, obs)):
            for k, v in want.items():
                assert np.array_equal(got[k], v), (k, rng, n)
    comm.close()


def test_guard_mode_finds_no_out_of_bounds_write():
    """compute-sanitizer is closed on this pool, so the library carries its own check:
    with VXB_GUARD=1 every library-owned device buffer is bracketed by canaries that are
    verified on release.  scripts/sanitize_small.py launches every kernel family on small
    ragged sizes; the guard must (a) catch a provoked one-byte overrun and (b) report zero
    violations for the real kernels."""
    import os
    import re
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, VXB_GUARD="1")
    run = subprocess.run([sys.executable, os.path.join(root, "scripts", "sanitize_small.py")],
                         capture_output=True, text=True, timeout=900, env=env)
    assert run.returncode == 0, run.stdout[-1500:] + run.stderr[-1500:]
    assert "guard (0, True) (0, None)" in run.stdout          # self-test detected, nothing else
    lines = [l for l in run.stderr.splitlines() if l.startswith("vxb guard:")]
    assert len([l for l in lines if "out-of-bounds" in l]) == 1  # the provoked one
    assert all(re.search(r"\b0 violation", l) for l in lines if "violation(s)" in l)


@pytest.mark.timeout(900)
@pytest.mark.parametrize("comm", ["torch", "native"])
def test_bench_walks_the_multi_rank_path_with_one_rank(comm):
    """bench.py under the launcher with VXB_FORCE_GATHER=1: ONE rank executes exactly the
    code of N > 1 -- NCCL process group, the packed all_gather_into_tensor (or the
    library's communicator with --comm native), barrier and max-over-ranks timing."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, VXB_FORCE_GATHER="1")
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK"):
        env.pop(k, None)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=1",
           "--master-addr", "127.0.0.1", "--master-port", "29611" if comm == "torch" else "29612",
           os.path.join(root, "bench.py"), "--gpus", "1", "--steps", "2", "--warmup", "3",
           "--particles", "2e6", "--no-extras", "--comm", comm]
    run = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env)
    assert run.returncode == 0, run.stdout[-1500:] + run.stderr[-3000:]
    line = json.loads([l for l in run.stdout.splitlines() if l.startswith("{")][-1])
    assert line["n_gpus"] == 1 and line["value"] > 1e8
    assert line["config"]["accepted_per_step"] > 1500
    want = "library NCCL" if comm == "native" else "torch.distributed NCCL"
    assert want in line["config"]["exchange"], line["config"]["exchange"]


@pytest.mark.timeout(900)
@pytest.mark.parametrize("ranks", [2, 3, 4])
def test_multi_rank_drivers_on_one_gpu_through_the_loopback_group(ctx, oracle, golden, ranks):
    """The multi-rank native code -- row sharding, the packed accepted-set gather,
    vxb_sharded_abcsmc_run's rounds (gated propose, pack, gather, append in rank order),
    the padded weight gather and the all-reduce of the chunk totals -- executed for real
    with 2, 3 and 4 ranks: `ranks` contexts on this one GPU joined by the library's
    loopback group (host rendezvous + device-to-device copies in place of NCCL; no kernel
    waits for another rank).  Everything must equal the one-context result bit for bit.
    With 4 ranks the 600-particle ABC-SMC run has 3 canonical chunks: one rank owns an
    empty weight shard; round_size 250 gives ragged slices (63/63/62/62)."""
    multi = lib.Multi(loopback_ranks=ranks)
    assert multi.size == ranks
    obs = golden["logistic_observed"]
    m = M.logistic_model()
    key = M.keying(1337, A.VXB_KEY_WORKER, 5, 4)
    got = multi.abc_prior_predictive(m, key, 2003, obs)
    want = oracle.abc_prior_predictive(m, key, 2003, 0, 2003, obs)
    for g, w in zip(got, want):
        assert np.array_equal(g, w, equal_nan=True)
    p, _, rho, f = oracle.abc_prior_predictive(m, M.keying(7), 40001, 0, 40001, obs, want_summaries=False)
    eps, idx_o = oracle.select_epsilon(rho, f, 0.02)
    nacc, idx, params, rho_acc = multi.abc_reject(m, M.keying(7), 40001, obs, eps, cap=40001)
    assert nacc == len(idx_o) and np.array_equal(idx, idx_o)
    assert np.array_equal(params, p[idx_o]) and np.array_equal(rho_acc, rho[idx_o])
    # early rejection on every rank (segment launches per shard): the same gathered set
    multi.set_early_reject(True)
    big = multi.abc_reject(m, M.keying(7), 300007, obs, eps, cap=300007)
    multi.set_early_reject(False)
    ref = multi.abc_reject(m, M.keying(7), 300007, obs, eps, cap=300007)
    assert big[0] == ref[0] > 1000 and all(np.array_equal(a, b) for a, b in zip(big[1:], ref[1:]))
    # config 0's selection over a sharded distance vector: all-reduced digit histograms.
    # Same epsilon bits and the same indices as the oracle / one context, with failed rows
    # (flag-only, NaN-only, both), ties, fp32 keys, a capacity below the accepted count,
    # and fewer rows than ranks
    rs = np.random.RandomState(ranks)
    for q in (0.02, 0.5, 1.0, 1e-6):
        e, idx_s, n_s = multi.select_epsilon(rho, f, q)
        e_o, i_o = oracle.select_epsilon(rho, f, q)
        assert e == e_o and n_s == len(i_o) and np.array_equal(idx_s, i_o), q
    e0, idx0, n0 = multi.select_epsilon(rho, f, 0.02, cap=0)          # epsilon and count only
    assert e0 == oracle.select_epsilon(rho, f, 0.02)[0] and idx0.size == 0 and n0 == len(oracle.select_epsilon(rho, f, 0.02)[1])
    r2, f2 = np.round(rs.gamma(2.0, 3.0, 30011), 1), (rs.uniform(size=30011) < 0.05).astype(np.uint8)
    r2[rs.uniform(size=30011) < 0.03] = np.nan          # NaN rows, some of them unflagged
    for arr in (r2, r2.astype(np.float32)):
        e, idx_s, n_s = multi.select_epsilon(arr, f2, 0.1)
        e_1, idx_1, n_1 = ctx.select_epsilon(arr, f2, 0.1)
        e_o, i_o = oracle.select_epsilon(arr.astype(np.float64), f2 | np.isnan(arr).astype(np.uint8), 0.1)
        assert e == e_1 == e_o and n_s == n_1 == len(i_o)
        assert np.array_equal(idx_s, idx_1) and np.array_equal(idx_s, i_o)
        e, idx_s, n_s = multi.select_epsilon(arr, None, 0.1, cap=100)     # NaN-only failures, small cap
        e_1, idx_1, n_1 = ctx.select_epsilon(arr, None, 0.1)
        assert e == e_1 and n_s == n_1 > 100 and np.array_equal(idx_s, idx_1[:100])
    small = np.array([3.0, 1.0][:max(1, ranks - 2)])
    e, idx_s, n_s = multi.select_epsilon(small, None, 0.5)
    assert (e, idx_s.tolist(), n_s) == ((2.0, [1], 1) if small.size == 2 else (3.0, [0], 1))
    with pytest.raises(lib.VxbError) as err:
        multi.select_epsilon(np.full(5, np.nan), None, 0.5)
    assert err.value.code == "empty-set"
    for rng, n, gens, round_size, seed in ((A.VXB_RNG_REF, 600, 3, 250, 9), (A.VXB_RNG_FAST, 1500, 4, 0, 21),
                                           (A.VXB_RNG_REF, 2000, 3, 0, 1337)):
        mm = M.logistic_model(rng=rng)
        cfg = A.vxb_abcsmc_cfg()
        cfg.particles, cfg.generations, cfg.quantile, cfg.kernel_scale = n, gens, 0.5, 2.0
        cfg.jitter, cfg.round_size, cfg.max_rounds, cfg.seed = 1e-10, round_size, 0, seed
        one, many = ctx.abcsmc_run(mm, cfg, obs), multi.abcsmc_run(mm, cfg, obs)
        for k, v in one.items():
            assert np.array_equal(many[k], v), (k, rng, n, ranks)
    lam = np.array(M.lambda_grid(8))
    ln = np.array([-0.5 * math.log(2.0 * math.pi * (l * l + 0.01)) for l in lam])
    c1, p1, _ = ctx.ppp_pvalues(M.normal_mean_model(100), lam, ln, 30001, 0, 30001, 1337, 2.9)
    c2, p2 = multi.ppp_pvalues(M.normal_mean_model(100), lam, ln, 30001, 1337, 2.9)
    assert np.array_equal(c1, c2) and np.array_equal(p1, p2)
    mc = A.vxb_mlmc_cfg()
    mc.levels, mc.refine, mc.tau0, mc.t_end, mc.paths, mc.seed = 3, 4, 1.0, 30.0, 10001, 1337
    for mm in (M.mm_tauleap_model(), M.mm_tauleap_model(rng=A.VXB_RNG_FAST, precision=A.VXB_F32)):
        r1, r2 = ctx.mlmc_tauleap(mm, mc), multi.mlmc_tauleap(mm, mc)   # all-reduce of int64 sums
        for k in ("level_mean", "level_var", "level_cost"):
            assert np.array_equal(r1[k], r2[k]), k
        assert r1["estimate"] == r2["estimate"] and r1["std_error"] == r2["std_error"]
    # the weak-informativity test: hyperparameter rows over the ranks
    wcfg = M.weakinfo_config(hyper_count=6, datasets=9, particles=100, seed=1337)
    w1, w2 = ctx.weak_info_test(wcfg, want_evidence=True), multi.weak_info_test(wcfg, want_evidence=True)
    for k in ("lambda_", "gamma", "weakly", "completed", "evidence"):
        assert np.array_equal(w1[k], w2[k], equal_nan=True), k
    # fewer rows than ranks: some ranks own EMPTY shards
    tiny = multi.abc_prior_predictive(m, M.keying(7), ranks - 1, obs)
    for g, w in zip(tiny, oracle.abc_prior_predictive(m, M.keying(7), ranks - 1, 0, ranks - 1, obs)):
        assert np.array_equal(g, w, equal_nan=True)
    nacc, idx, _, _ = multi.abc_reject(m, M.keying(7), ranks - 1, obs, 1e9, cap=16)
    assert nacc == ranks - 1 and idx.tolist() == list(range(ranks - 1))
    c3, _ = multi.ppp_pvalues(M.normal_mean_model(100), lam, ln, ranks - 1, 1337, 2.9)
    assert np.array_equal(c3, ctx.ppp_pvalues(M.normal_mean_model(100), lam, ln, ranks - 1, 0, ranks - 1, 1337, 2.9)[0])
    multi.close()


@pytest.mark.timeout(600)
def test_loopback_group_releases_its_ranks_when_one_fails():
    """A rank that fails never arrives at the next collective.  The loopback group must
    release the ranks waiting for it -- the call returns the root cause instead of hanging
    -- and stay usable (the group is reset after the join).  The failure is injected once,
    on rank 1 of 3, by VXB_LOOPBACK_FAIL_RANK (read by vxb_multi_init_loopback)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = f"""
import sys; sys.path.insert(0, {root!r})
import numpy as np
from paper_1902_09046_b200 import lib, models as M
obs = np.load({os.path.join(root, 'tests', 'golden', 'golden.npz')!r})["logistic_observed"]
multi = lib.Multi(loopback_ranks=3)
for attempt in range(2):                      # the second call finds a clean group
    try:
        n = multi.abc_reject(M.logistic_model(), M.keying(7), 5000, obs, 30.0, cap=5000)[0]
        print("no error", n)
    except lib.VxbError as e:
        print("error", e.code, "|", e)
multi.close()
"""
    run = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300,
                         env=dict(os.environ, VXB_LOOPBACK_FAIL_RANK="1"))
    assert run.returncode == 0, run.stdout[-800:] + run.stderr[-800:]
    lines = run.stdout.splitlines()
    assert len(lines) == 2 and lines[0].startswith("error internal") and "injected failure" in lines[0], run.stdout
    assert "device rank 1" in lines[0] and lines[1].startswith("no error") and int(lines[1].split()[-1]) > 0
