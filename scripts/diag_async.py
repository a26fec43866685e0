"""Where does the asynchronous device-resident step lose time against the host-buffer step?"""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
from paper_1902_09046_b200 import _abi as A, dist as D, lib, models as M

torch.cuda.set_device(0)
ctx = lib.Context(0)
m = M.logistic_model(rng=A.VXB_RNG_FAST)
obs = ctx.simulate_at(M.logistic_model(), [0.5, 100.0, 0.05], lib.derive_seed(1, [90]), 0, 0)
n, eps = 100_000_000, 19.712058377057488
ext = torch.cuda.ExternalStream(ctx.stream(), device=torch.device("cuda", 0))
cap = 1_000_000

def timed(fn, steps=4, warm=2):
    with torch.cuda.stream(ext):
        for s in range(warm):
            fn(s)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(ext)
        t0 = time.perf_counter()
        for s in range(steps):
            fn(warm + s)
        t_enq = time.perf_counter() - t0
        e1.record(ext)
        torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps, t_enq * 1e3 / steps

print("A sharded_reject       ", timed(lambda s: D.sharded_reject(ctx, m, M.keying(1337 + s), n, obs, eps)))
with torch.cuda.stream(ext):
    idx = torch.empty(cap, dtype=torch.int64, device="cuda")
    par = torch.empty((cap, 3), dtype=torch.float64, device="cuda")
    rho = torch.empty(cap, dtype=torch.float64, device="cuda")
    nd = torch.empty(1, dtype=torch.int64, device="cuda")
print("B async, preallocated  ", timed(lambda s: ctx.abc_reject(m, M.keying(1337 + s), n, 0, n, obs, eps, cap, idx=idx, params=par, rho=rho, n_accepted=nd)))
print("C host buffers (sync)  ", timed(lambda s: ctx.abc_reject(m, M.keying(1337 + s), n, 0, n, obs, eps, cap)))
rho_all = torch.empty(n, dtype=torch.float64, device="cuda")
print("D simulate only        ", timed(lambda s: ctx.abc_prior_predictive(m, M.keying(1337 + s), n, 0, n, obs, rho=rho_all)))
ctx.profile_enable(True); ctx.profile_reset()
print("B again, profiled      ", timed(lambda s: ctx.abc_reject(m, M.keying(1337 + s), n, 0, n, obs, eps, cap, idx=idx, params=par, rho=rho, n_accepted=nd)))
p = ctx.profile_read()
print({k: (v["launches"], round(v["total_ms"] / max(v["launches"], 1), 3)) for k, v in p.items() if v["launches"]})
