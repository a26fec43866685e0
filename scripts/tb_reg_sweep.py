"""Register-cap sweep of the TB Gillespie kernel (one-warp CTAs: the cap decides how many
paths are resident per SM).  Build the variants first, here (nvcc cross-compiles):

    python - <<'PY'
    from paper_1902_09046_b200 import build
    for r in (64, 72, 76, 80, 84, 88, 128):
        build.build_library(force=True, extra=[f"-DVXB_TB_REGS={r}"], out=f"build_variants/libvxb_tb{r}.so")
    PY

then on the GPU box: python scripts/tb_reg_sweep.py  (each variant is loaded through
VXB_LIBRARY in its own process; 1e6 rows at the reference bench sizes).  Round-2 result:
64 -> 5.18e5 rows/s, 72 -> 4.90e5, 76 -> 5.57e5, 80 -> 6.19e5, 84 -> 5.85e5, 88 -> 5.96e5,
96 -> 5.89e5, 128 -> 5.56e5."""
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
for lib_path in [None] + sorted(p for p in (f"build_variants/libvxb_tb{r}.so" for r in (64, 72, 76, 80, 84, 88, 128)) if os.path.exists(p)):
    env = dict(os.environ)
    if lib_path: env["VXB_LIBRARY"] = os.path.abspath(lib_path)
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env)
    print(lib_path or "default (80)", out.stdout.strip(), out.stderr[-300:])
