"""GPU test of the C++ shim (paper_1902_09046_b200/cpp/vexbayes): a program
written against the reference's own API names is compiled with g++, linked to
libvexbayes_cuda.so and its output compared with the oracle / reference."""
import io
import math
import os
import struct
import subprocess

import numpy as np
import pytest

from paper_1902_09046_b200 import _abi as A, lib, models as M

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def parse(out):
    res = {}
    for line in out.strip().splitlines():
        name, *rest = line.split()
        res[name] = rest
    return res


def hexd(tokens):
    return np.array([struct.unpack("<d", bytes.fromhex(t)[::-1])[0] for t in tokens[1:]])


def test_cpp_shim_matches_oracle(tmp_path, oracle, golden):
    exe = tmp_path / "test_shim"
    pkg = os.path.join(ROOT, "paper_1902_09046_b200")
    cmd = ["g++", "-std=c++20", "-O1", "-I", os.path.join(pkg, "cpp"),
           os.path.join(ROOT, "tests", "cpp", "test_shim.cpp"), "-o", str(exe),
           "-L", pkg, "-lvexbayes_cuda", f"-Wl,-rpath,{pkg}"]
    subprocess.run(cmd, check=True)
    run = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert run.returncode == 0, run.stdout + run.stderr
    r = parse(run.stdout)
    m = M.logistic_model()
    obs = hexd(r["observed"])
    assert np.array_equal(obs, golden["logistic_observed"])
    key = M.keying(1337, A.VXB_KEY_WORKER, 3, 4)
    p, s, rho, f = oracle.abc_prior_predictive(m, key, 500, 0, 500, obs)
    assert np.array_equal(hexd(r["params"]), p.ravel())
    assert np.array_equal(hexd(r["summaries"]), s.ravel())
    assert np.array_equal(hexd(r["rho"]), rho)
    eps, idx = oracle.select_epsilon(rho, f, 0.05)
    assert hexd(r["epsilon"])[0] == eps
    assert [int(t) for t in r["accepted"][1:]] == idx.tolist()
    assert float(r["discrepancy"][0]) == 5.0
    p2, _, rho2, f2 = oracle.abc_prior_predictive(m, M.keying(1337), 20000, 0, 20000, obs, want_summaries=False)
    want = np.nonzero((rho2 <= eps) & (f2 == 0))[0]
    assert int(r["reject"][0]) == len(want) and [int(t) for t in r["reject"][1:]] == want.tolist()
    assert r["early_reject_identical"] == ["1"]      # cuda::set_early_reject: same accepted set
    assert r["errors"] == ["6"]
    g = oracle.fill_gaussian(7, 1, 0, 768)
    assert float(r["ess"][0]) == oracle.ess(g[512:])          # bit-exact: host-libm exp, sequential sums
    out, anc = oracle.resample_multinomial(g[512:], g[:512].reshape(256, 2), 2718, 3)
    assert np.array_equal(hexd(r["resampled"]), out.ravel())
    lam = np.array([0.1, 1.0, 10.0, 100.0])
    ln = np.array([-0.5 * math.log(2.0 * math.pi * (l * l + 1.0 / 100)) for l in lam])
    counts, _, _ = oracle.ppp_pvalues(M.normal_mean_model(100), lam, ln, 20000, 0, 20000, 1337, 2.9)
    assert [int(t) for t in r["counts"]] == counts.tolist()
    assert [float(t) for t in r["pvalues"]] == [0.25, 0.75]


def test_cpp_shim_reference_format_outputs(tmp_path, golden, oracle):
    """abc::write_csv and the bench harness of the C++ shim: the set file equals
    the file the reference wrote; the bench file survives parse -> write."""
    from paper_1902_09046_b200 import bench_harness as B
    exe = tmp_path / "test_shim"
    pkg = os.path.join(ROOT, "paper_1902_09046_b200")
    subprocess.run(["g++", "-std=c++20", "-O1", "-I", os.path.join(pkg, "cpp"),
                    os.path.join(ROOT, "tests", "cpp", "test_shim.cpp"), "-o", str(exe),
                    "-L", pkg, "-lvexbayes_cuda", f"-Wl,-rpath,{pkg}"], check=True)
    gold = os.path.join(ROOT, "tests", "golden")
    run = subprocess.run([str(exe), "csv", os.path.join(gold, "bench_records.csv"), str(tmp_path)],
                         capture_output=True, text=True, timeout=300)
    assert run.returncode == 0, run.stdout + run.stderr
    r = parse(run.stdout)
    assert r["sweep"] == ["8", "0"]
    assert r["bench_errors"][0] == "3" and float(r["bench_errors"][2]) == B.amdahl_bound(1.0, 9.0, 4.0)
    read = lambda p: open(p, newline="").read()
    assert read(tmp_path / "set.csv") == read(os.path.join(gold, "logistic_set.csv"))
    text = read(os.path.join(gold, "bench_records.csv"))
    want = io.StringIO()
    B.write_csv(B.parse_csv(text), want)
    assert read(tmp_path / "bench_rewritten.csv") == want.getvalue()
    cut = text.index(B.SUMMARY_HEADER)
    assert read(tmp_path / "bench_rewritten.csv")[:cut] == text[:cut]   # records section: reference bytes
    assert read(tmp_path / "weakinfo_table.csv") == read(os.path.join(gold, "weakinfo_table.csv"))
    anneal = np.load(os.path.join(gold, "anneal.npz"))
    assert abs(float(r["evidence"][0]) - anneal["run_evidence"][0]) < 1e-9
    assert int(r["evidence"][1]) == anneal["run_iterations"][0]
    assert r["evidence"][2] == "".join(str(v) for v in anneal["run_deaths"][0])
    k = 2  # make_golden_anneal.ENSEMBLE_RUN: (4.0, 0.2, data seed 5, sampler seed 15, 64 particles)
    assert abs(float(r["run_smc"][0]) - anneal["run_evidence"][k]) < 1e-9
    assert [int(t) for t in r["run_smc"][1:4]] == [int(anneal["run_iterations"][k]), 64, 2]
    assert float(r["run_smc"][4]) == 1.0
    assert np.allclose(hexd(r["run_smc_particles"]).reshape(64, 2), anneal["ens_particles"], rtol=1e-9, atol=1e-9)
    assert np.allclose(hexd(r["run_smc_log_liks"]), anneal["ens_rows"][1], rtol=1e-9, atol=1e-9)
    lines = read(tmp_path / "smc_trace.csv").strip().splitlines()
    assert lines[0] == "n,t_n,ess,log_evidence,R_n,p_acc,h"
    rows = np.array([[float(x) for x in ln.split(",")] for ln in lines[1:]])
    assert rows[:, 0].tolist() == [1.0, 2.0]
    assert np.allclose(rows[:, [1, 2, 4, 5, 3, 6]], anneal["ens_trace"], rtol=1e-9, atol=1e-9)
    assert r["run_smc_refused"] == ["3"]
    # SmcConfig::esjd = true through the shim = golden case 1 (same data, prior, seed, 333 particles)
    want = anneal["esjd1_trace"]
    assert abs(float(r["run_smc_esjd"][0]) - anneal["esjd1_evidence"][0]) < 1e-9
    assert int(r["run_smc_esjd"][1]) == len(want)
    rows = np.array([[float(x) for x in ln.split(",")]
                     for ln in read(tmp_path / "smc_trace_esjd.csv").strip().splitlines()[1:]])
    assert np.array_equal(rows[:, [4, 5, 6]], want[:, [2, 3, 5]])      # sweeps, trial acceptance, scale
    tb_obs = oracle.tb_observed(10, 10.0, 10000.0, 1337)
    tb_rows = oracle.tb_abc_particle(10, 10.0, 10000.0, 0, 40, 1337, tb_obs)
    assert [float(t) for t in r["tb"][:4]] == [tb_obs[0], tb_obs[1], tb_rows[1][0, 0], tb_rows[2][1]]
    assert int(r["tb"][4]) == int(tb_rows[3][0]) + int(tb_rows[3][1])
    sweep = B.parse_csv(read(tmp_path / "sweep.csv"))
    assert [(x.block_width, x.threads, x.replicate) for x in sweep] == \
        [(v, p, k) for v in (1, 4) for p in (1, 3) for k in (0, 1)]


def test_cpp_multi_gpu_drivers(tmp_path, oracle):
    """tests/cpp/test_multi.cpp: the shim's drivers over every visible GPU (vxb_multi_*),
    the library's own NCCL communicator (a real 1-rank communicator on one GPU; the SPMD
    per-device form on two or more), the packed accepted-set exchange.  The C++ side
    checks G devices == 1 device itself; here its output is compared with the oracle."""
    exe = tmp_path / "test_multi"
    pkg = os.path.join(ROOT, "paper_1902_09046_b200")
    subprocess.run(["g++", "-std=c++20", "-O1", "-pthread", "-I", os.path.join(pkg, "cpp"),
                    os.path.join(ROOT, "tests", "cpp", "test_multi.cpp"), "-o", str(exe),
                    "-L", pkg, "-lvexbayes_cuda", f"-Wl,-rpath,{pkg}"], check=True)
    run = subprocess.run([str(exe)], capture_output=True, text=True, timeout=600)
    assert run.returncode == 0, run.stdout[-2000:] + run.stderr[-2000:]
    r = parse(run.stdout)
    import torch
    assert int(r["devices"][0]) == torch.cuda.device_count() == int(r["in_use"][0])
    assert r["nccl_one_rank"] == ["ok"] and int(r["nccl_version"][0]) >= 21800
    assert r["loopback_three_ranks"] == ["ok"]
    if torch.cuda.device_count() >= 2:
        assert r["multi_gpu"][0] == "ok"
    m = M.logistic_model()
    obs = oracle.simulate_at(m, [0.5, 100.0, 0.05], 0x9b1d6f0c5a3e7c21, 0, 0)
    assert np.array_equal(hexd(r["observed"]), obs)
    p, s, rho, f = oracle.abc_prior_predictive(m, M.keying(1337, A.VXB_KEY_WORKER, 3, 4), 1003, 0, 1003, obs)
    assert np.array_equal(hexd(r["rho"]), rho) and np.array_equal(hexd(r["params"]), p.ravel())
    eps, _ = oracle.select_epsilon(rho, f, 0.05)
    assert float(r["epsilon"][1]) == eps
    p2, _, rho2, f2 = oracle.abc_prior_predictive(m, M.keying(1337), 30001, 0, 30001, obs, want_summaries=False)
    want = np.nonzero((rho2 <= eps) & (f2 == 0))[0]
    assert int(r["reject_total"][0]) == len(want)
    assert [int(t) for t in r["reject_rows"][1:]] == want.tolist()
    assert np.array_equal(hexd(r["reject_rho"]), rho2[want])
    assert np.array_equal(hexd(r["reject_params"]), p2[want].ravel())
    cfg = A.vxb_abcsmc_cfg()
    cfg.particles, cfg.generations, cfg.quantile, cfg.kernel_scale = 1500, 3, 0.5, 2.0
    cfg.jitter, cfg.round_size, cfg.max_rounds, cfg.seed = 1e-10, 700, 0, 77
    pop = oracle.abcsmc_run(m, cfg, obs)
    assert np.array_equal(hexd(r["smc_particles"]), pop["theta"].ravel())
    assert np.array_equal(hexd(r["smc_weights"]), pop["weight"])
    assert np.array_equal(hexd(r["smc_epsilon"]), pop["epsilon"])
