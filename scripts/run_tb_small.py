"""One launch of the TB Gillespie ABC kernel (for ncu captures): 20 000 paths."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1902_09046_b200 import bench_harness as B, lib, models as M
ctx = lib.Context(0)
n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 20000
m = M.tb_model(10, 10.0, 10000.0)
obs = B.tb_observed_summaries(ctx, 10, 10.0, 10000.0, 1337, 4)
p, s, rho, f = ctx.abc_prior_predictive_host(m, M.keying(1337), n, 0, n, obs)
print("tb", n, int(f.sum()), float(s[:, 0].mean()))
