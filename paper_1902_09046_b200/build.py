"""In-tree build of libvexbayes_cuda.so (nvcc, sm_100a only).

``python -m paper_1902_09046_b200.build`` or ``build_library()``.  The shared
object lands next to this file so that it travels with the repository snapshot
to the GPU box; it is git-ignored.
"""
import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libvexbayes_cuda.so")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-lineinfo", "-O3", "-std=c++17", "--threads", "0",   # one nvcc job per source file
    "-Xcompiler", "-fPIC", "-shared",
    # IEEE division / square root / no flush-to-zero (the defaults, stated):
    "-prec-div=true", "-prec-sqrt=true", "-ftz=false",
]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def needs_build():
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + [
        os.path.join(HERE, "..", "include", "vexbayes_cuda.h")]
    return any(os.path.getmtime(d) > t for d in deps)


LIB_ROUNDS7 = os.path.join(HERE, "libvexbayes_cuda_rounds7.so")


def build_library(force=False, verbose=False, extra=(), out=None):
    """out=None: the product library.  out=LIB_ROUNDS7 with extra=["-DVXB_FAST_ROUNDS=7"]:
    the documented opt-in whose throughput generator runs Philox4x32-7 (load it with the
    environment variable VXB_LIBRARY; profiles/r2_philox7_*.json is its record)."""
    if out is None:
        if not force and not needs_build():
            return LIB
        out = LIB
    nvcc = os.environ.get("NVCC", "nvcc")
    cmd = [nvcc] + NVCC_FLAGS + list(extra) + ["-o", out] + sources()
    res = subprocess.run(cmd, capture_output=True, text=True, cwd=CSRC)
    if verbose or res.returncode:
        sys.stderr.write(res.stdout + res.stderr)
    out = res
    if out.returncode:
        raise RuntimeError("nvcc failed building libvexbayes_cuda.so")
    return cmd[cmd.index("-o") + 1]


if __name__ == "__main__":
    if "--rounds7" in sys.argv:
        print(build_library(force=True, verbose=True, extra=["-DVXB_FAST_ROUNDS=7"], out=LIB_ROUNDS7))
    else:
        build_library(force=True, verbose=True, extra=["-Xptxas", "-v"] if "-v" in sys.argv else [])
        print(LIB)
