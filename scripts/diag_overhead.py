"""Per-step wall time vs event-timed kernel time (is the jitter on the GPU or on the host?)."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from paper_1902_09046_b200 import _abi as A, dist as D, lib, models as M

torch.cuda.set_device(0)
ctx = lib.Context(0)
m = M.logistic_model(rng=A.VXB_RNG_FAST)
obs = ctx.simulate_at(M.logistic_model(), [0.5, 100.0, 0.05], lib.derive_seed(1, [90]), 0, 0)
n, eps = 100_000_000, 19.712058377057488
ctx.profile_enable(True)
import pynvml
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
for s in range(14):
    ctx.profile_reset()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    D.sharded_reject(ctx, m, M.keying(1337 + s), n, obs, eps)
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) * 1e3
    p = ctx.profile_read()
    clk = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
    pw = pynvml.nvmlDeviceGetPowerUsage(h) / 1000
    print(f"step {s}: wall {wall:.1f} ms  simulate {p['simulate']['total_ms']:.1f} ms  compact {p['compact']['total_ms']:.2f} ms  clk_after={clk} MHz  power={pw:.0f} W", flush=True)
