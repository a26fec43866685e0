"""Per-step device time of the asynchronous loop (events after every step), repeated."""
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
ext = torch.cuda.ExternalStream(ctx.stream(), device=torch.device("cuda", 0))
for rep in range(4):
    with torch.cuda.stream(ext):
        for s in range(3):
            D.sharded_reject(ctx, m, M.keying(1337 + s), n, obs, eps)
        torch.cuda.synchronize()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
        ev[0].record(ext)
        outs = []
        for s in range(5):
            out = D.sharded_reject(ctx, m, M.keying(1340 + s), n, obs, eps)
            ev[s + 1].record(ext)
        torch.cuda.synchronize()
    print(rep, [round(ev[i].elapsed_time(ev[i + 1]), 1) for i in range(5)], flush=True)
