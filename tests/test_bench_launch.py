"""CPU tests of bench.py's launch path: `--gpus N` without a launcher must start N
ranks itself, a mismatch with WORLD_SIZE must fail loudly, and the reference arm under
a launcher prints on rank 0 only.  The ranks run bench.py's gloo self-test (one packed
all_gather_into_tensor of accepted blocks); no GPU is touched."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BENCH = os.path.join(ROOT, "bench.py")


def run(args, env=None, timeout=300):
    e = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK"):
        e.pop(k, None)
    e.update(env or {})
    return subprocess.run([sys.executable, BENCH] + args, capture_output=True, text=True,
                          timeout=timeout, env=e)


@pytest.mark.timeout(600)
def test_gpus_n_spawns_n_ranks():
    r = run(["--gpus", "2", "--selftest-dist"])
    assert r.returncode == 0, r.stdout + r.stderr[-2000:]
    lines = [json.loads(l) for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1                     # rank 0 alone prints
    assert lines[0]["ok"] and lines[0]["n_gpus"] == 2 and lines[0]["accepted"] == 5 + 6
    assert lines[0]["launched_by"] == "torch.distributed.run"
    r1 = run(["--gpus", "1", "--selftest-dist"])
    assert r1.returncode == 0 and json.loads(r1.stdout.splitlines()[-1])["launched_by"] == "direct"


def test_world_size_mismatch_is_an_error():
    r = run(["--gpus", "2", "--selftest-dist"], env={"WORLD_SIZE": "3", "RANK": "0", "LOCAL_RANK": "0"})
    assert r.returncode != 0 and "WORLD_SIZE=3" in r.stderr


@pytest.mark.timeout(600)
def test_reference_arm_under_a_launcher_prints_once():
    """`bench.py --impl reference` launched like the GPU arm (torchrun, N = 2): rank 0 alone
    runs the reference's CPU path and prints the line; the other rank exits 0 silently."""
    env = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK"):
        env.pop(k, None)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", "29621", BENCH, "--impl", "reference",
           "--gpus", "2", "--steps", "1", "--warmup", "0", "--cpu-sample", "2000"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=500, env=env)
    assert r.returncode == 0, r.stdout + r.stderr[-2000:]
    lines = [json.loads(l) for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1 and lines[0]["impl"] == "reference" and lines[0]["n_gpus"] == 2
    assert lines[0]["value"] > 0 and lines[0]["cpu_baseline"]["kind"] in ("reference", "port")
    assert lines[0]["e2e"]["h2d_bytes_per_step"] == 0
