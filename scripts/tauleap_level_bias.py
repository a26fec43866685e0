"""Per-level means of the tau-leap instances at very large path counts: the fp32 and fp64
throughput instances against the exact one (independent streams), level by level.

    python scripts/tauleap_level_bias.py [paths_level0] [paths_fine]
"""
import json, math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1902_09046_b200 import _abi as A, lib, models as M

n0 = int(float(sys.argv[1])) if len(sys.argv) > 1 else 1_000_000_000
nf = int(float(sys.argv[2])) if len(sys.argv) > 2 else 100_000_000
ctx = lib.Context(0)
cfg = A.vxb_mlmc_cfg()
cfg.levels, cfg.refine, cfg.tau0, cfg.t_end, cfg.paths, cfg.seed = 6, 4, 1.0, 30.0, 1, 1337
models = {"exact": M.mm_tauleap_model(), "fast_f64": M.mm_tauleap_model(rng=A.VXB_RNG_FAST),
          "fast_f32": M.mm_tauleap_model(rng=A.VXB_RNG_FAST, precision=A.VXB_F32)}
out = {"paths": {}, "levels": {}}
for level in range(6):
    n = n0 if level == 0 else max(nf // 4 ** (level - 1), 10_000_000)
    chunk = 100_000_000
    stats = {}
    for name, m in models.items():
        s = np.zeros(4, dtype=object)
        for first in range(0, n, chunk):
            sums, _ = ctx.mlmc_level(m, cfg, level, first, min(chunk, n - first))
            s = s + np.array([int(v) for v in sums], dtype=object)
        mean = float(s[0]) / n
        var = (float(s[1]) - float(s[0]) ** 2 / n) / (n - 1)
        stats[name] = (mean, var)
    row = {"paths": n}
    for name in ("fast_f64", "fast_f32"):
        d = stats[name][0] - stats["exact"][0]
        se = math.sqrt((stats[name][1] + stats["exact"][1]) / n)
        row[name] = {"mean": stats[name][0], "diff": d, "z": d / se, "rel": d / 22.72}
    row["exact_mean"] = stats["exact"][0]
    out["levels"][level] = row
    print(level, json.dumps(row), flush=True)
print(json.dumps(out))
