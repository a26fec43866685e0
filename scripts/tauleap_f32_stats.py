"""fp32 throughput instance of the tau-leap kernel against the reference-exact fp64
instance: per-level and pooled z-scores of the level means at --paths paths per level
over several seeds (the same protocol as scripts/fastmode_stats.py for config 4).

    python scripts/tauleap_f32_stats.py > profiles/r2_tauleap_f32_stats.json
"""
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np

from paper_1902_09046_b200 import _abi as A, lib, models as M

paths = int(float(sys.argv[1])) if len(sys.argv) > 1 else 10_000_000
seeds = [1337, 2337, 3337, 4337]
ctx = lib.Context(0)


def run(rng, prec, seed):
    mc = A.vxb_mlmc_cfg()
    mc.levels, mc.refine, mc.tau0, mc.t_end, mc.paths, mc.seed = 6, 4, 1.0, 30.0, paths, seed
    return ctx.mlmc_tauleap(M.mm_tauleap_model(rng=rng, precision=prec), mc)


out = {"paths_per_level": paths, "seeds": seeds, "per_seed": []}
d_sum, v_sum = np.zeros(6), np.zeros(6)
zs = []
for s in seeds:
    e, f = run(A.VXB_RNG_REF, A.VXB_F64, s), run(A.VXB_RNG_FAST, A.VXB_F32, s)
    d = f["level_mean"] - e["level_mean"]
    v = (f["level_var"] + e["level_var"]) / paths
    zs.append((d / np.sqrt(v)).tolist())
    d_sum += d
    v_sum += v
    out["per_seed"].append({"seed": s, "exact_estimate": e["estimate"], "f32_estimate": f["estimate"],
                            "std_error": e["std_error"], "z_level": zs[-1],
                            "var_ratio_level": (f["level_var"] / e["level_var"]).tolist()})
out["z_level_pooled"] = (d_sum / np.sqrt(v_sum)).tolist()
out["z_estimate_pooled"] = float(d_sum.sum() / math.sqrt(v_sum.sum()))
out["p_estimate_pooled"] = math.erfc(abs(out["z_estimate_pooled"]) / math.sqrt(2.0))
out["chi2_all_levels"] = float((np.array(zs) ** 2).sum())
out["chi2_dof"] = 6 * len(seeds)
out["relative_difference_of_pooled_estimate"] = float(d_sum.sum() / len(seeds) / 22.72)
print(json.dumps(out))
