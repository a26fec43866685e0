"""Build tuning variants of the library (CPU side) or time them (GPU side).

    python scripts/variant_bench.py build     # here: nvcc, one .so per variant
    python scripts/variant_bench.py run       # on the GPU box: time each variant
"""
import ctypes as C
import glob
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
OUT = os.path.join(ROOT, "build_variants")

VARIANTS = {
    "base": [],
    "minblk3": ["-DVXB_SIM_MIN_BLOCKS=3"],
    "block128_min5": ["-DVXB_SIM_BLOCK=128", "-DVXB_SIM_MIN_BLOCKS=5"],
    "block128_min6": ["-DVXB_SIM_BLOCK=128", "-DVXB_SIM_MIN_BLOCKS=6"],
    "block128_min3": ["-DVXB_SIM_BLOCK=128", "-DVXB_SIM_MIN_BLOCKS=3"],
    "block64_min8": ["-DVXB_SIM_BLOCK=64", "-DVXB_SIM_MIN_BLOCKS=8"],
}


def build():
    from paper_1902_09046_b200 import build as B
    os.makedirs(OUT, exist_ok=True)
    for name, flags in VARIANTS.items():
        lib = os.path.join(OUT, f"lib_{name}.so")
        cmd = ["nvcc"] + B.NVCC_FLAGS + flags + ["-o", lib] + B.sources()
        subprocess.run(cmd, check=True, cwd=B.CSRC)
        print("built", lib)


def run():
    import numpy as np
    import torch
    from paper_1902_09046_b200 import _abi as A, lib as L, models as M
    n = 4_000_000
    for path in sorted(glob.glob(os.path.join(OUT, "lib_*.so"))):
        L._lib = None
        L.LIB_PATH = path
        ctx = L.Context(0)
        obs = ctx.simulate_at(M.logistic_model(), [0.5, 100.0, 0.05], 5, 0, 0)
        rho = torch.empty(n, dtype=torch.float64, device="cuda")
        res = []
        for variant, prec, rng in (("f64_fast", A.VXB_F64, A.VXB_RNG_FAST), ("f64_ref", A.VXB_F64, A.VXB_RNG_REF),
                                   ("f32_fast", A.VXB_F32, A.VXB_RNG_FAST)):
            m = M.logistic_model(precision=prec, rng=rng)
            ctx.abc_prior_predictive(m, M.keying(1), n, 0, n, obs, rho=rho)
            ctx.synchronize()
            t0 = time.perf_counter()
            for s in range(3):
                ctx.abc_prior_predictive(m, M.keying(2 + s), n, 0, n, obs, rho=rho)
            ctx.synchronize()
            dt = (time.perf_counter() - t0) / 3
            res.append(f"{variant} {n / dt:.3e} sims/s")
        print(os.path.basename(path), " | ".join(res), flush=True)
        ctx.close()


if __name__ == "__main__":
    {"build": build, "run": run}[sys.argv[1]]()
