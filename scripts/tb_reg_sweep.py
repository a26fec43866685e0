import os, sys, time, subprocess
code = r'''
import sys, time
sys.path.insert(0, ".")
import torch
from paper_1902_09046_b200 import bench_harness as B, lib, models as M
ctx = lib.Context(0)
n = 1000000
tbm = M.tb_model(10, 10.0, 10000.0)
obs = B.tb_observed_summaries(ctx, 10, 10.0, 10000.0, 1337, 4)
rho = torch.empty(n, dtype=torch.float64, device="cuda"); f = torch.empty(n, dtype=torch.uint8, device="cuda")
ctx.abc_prior_predictive(tbm, M.keying(1), 20000, 0, 20000, obs, rho=rho[:20000], failed=f[:20000]); ctx.synchronize()
t0 = time.perf_counter(); ctx.abc_prior_predictive(tbm, M.keying(1337), n, 0, n, obs, rho=rho, failed=f); ctx.synchronize()
print("rows/s %.4g" % (n / (time.perf_counter() - t0)), float(rho[:1000].nan_to_num().sum()))
'''
for lib_path in [None] + [f"build_variants/libvxb_tb{r}.so" for r in (72, 76, 84, 88)]:
    env = dict(os.environ)
    if lib_path: env["VXB_LIBRARY"] = os.path.abspath(lib_path)
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env)
    print(lib_path or "default(96)", out.stdout.strip(), out.stderr[-300:])
