"""CPU tests of the drop-in boundary: the C-ABI library loads and exports every
symbol include/vexbayes_cuda.h declares; the ctypes mirror matches the header;
host-only entry points (no GPU needed) behave like the reference."""
import ctypes
import os
import re

import numpy as np
import pytest

from paper_1902_09046_b200 import _abi as A, build, lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "vexbayes_cuda.h")


@pytest.fixture(scope="module")
def so():
    build.build_library()  # nvcc cross-compiles sm_100a without a GPU
    return lib.load()


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(vxb_[a-z0-9_]+)\s*\(", text)))


def test_header_and_python_mirror_agree():
    assert declared_functions() == sorted(A.EXPORTED_SYMBOLS)
    text = open(HEADER).read()
    assert f"#define VXB_ABI_VERSION {A.VXB_ABI_VERSION}" in text
    # struct sizes follow from the header's field lists
    assert ctypes.sizeof(A.vxb_model) == 4 * 4 + 4 * 4 + 2 * 8 + 8 * 8 + 8 * 8 + 16 * 8
    assert ctypes.sizeof(A.vxb_keying) == 24
    assert ctypes.sizeof(A.vxb_abcsmc_cfg) == 64
    assert ctypes.sizeof(A.vxb_mlmc_cfg) == 40
    assert ctypes.sizeof(A.vxb_profile) == 16 * A.VXB_K_COUNT
    assert ctypes.sizeof(A.vxb_weakinfo_cfg) == 5 * 8 + 5 * 8 + 2 * 4 + 16 * 4 + 16 * 8 + 2 * 4
    assert ctypes.sizeof(A.vxb_accept_layout) == 48


def test_struct_sizes_match_the_c_compiler(tmp_path):
    """The ctypes mirrors against sizeof() as gcc sees the header (plain C)."""
    import subprocess
    names = ["vxb_model", "vxb_keying", "vxb_abcsmc_cfg", "vxb_mlmc_cfg", "vxb_weakinfo_cfg", "vxb_profile",
             "vxb_accept_layout"]
    src = tmp_path / "sizes.c"
    src.write_text('#include <stdio.h>\n#include "vexbayes_cuda.h"\nint main(void) {\n' +
                   "".join(f'    printf("{n} %zu\\n", sizeof({n}));\n' for n in names) + "    return 0;\n}\n")
    exe = tmp_path / "sizes"
    subprocess.run(["gcc", "-std=c11", "-I", os.path.dirname(HEADER), str(src), "-o", str(exe)], check=True)
    out = dict(line.split() for line in subprocess.run([str(exe)], capture_output=True, text=True,
                                                        check=True).stdout.splitlines())
    for n in names:
        assert int(out[n]) == ctypes.sizeof(getattr(A, n)), n


def test_library_exports_every_declared_symbol(so):
    for name in declared_functions():
        assert hasattr(so, name), f"libvexbayes_cuda.so does not export {name}"
    assert so.vxb_abi_version() == A.VXB_ABI_VERSION


def test_host_side_entry_points(so, oracle, golden):
    assert lib.splitmix64(0) == 0xE220A8397B1DCDAF
    assert lib.derive_seed(42, [1, 2, 3]) == 0x3FB96077DA5807FD
    assert lib.derive_seed(1, [90]) == oracle.derive_seed(1, [90])
    assert np.array_equal(lib.partition(8064, 16, 4), golden["partition_8064_16_4"])
    assert np.array_equal(lib.partition(1003, 7, 8), golden["partition_1003_7_8"])
    for total, workers, width in [(5, 9, 1), (100, 3, 16), (17, 4, 4), (1, 1, 1)]:
        assert np.array_equal(lib.partition(total, workers, width), oracle.partition(total, workers, width))
    with pytest.raises(lib.VxbError) as e:
        lib.partition(0, 1, 1)
    assert e.value.code == "invalid-shape"


def test_no_cpu_fallback_without_gpu(so):
    """vxb_init must fail loudly (device-error) when no CUDA device exists."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(lib.VxbError) as e:
        lib.Context(0)
    assert e.value.code == "device-error"


def test_cpp_shim_compiles_and_links(so, tmp_path):
    """The C++ shim that keeps the vexbayes:: signatures builds against the C ABI."""
    import subprocess
    pkg = os.path.join(ROOT, "paper_1902_09046_b200")
    exe = tmp_path / "test_shim"
    for name in ("test_shim", "test_multi"):
        exe = tmp_path / name
        subprocess.run(["g++", "-std=c++20", "-O1", "-Wall", "-Wextra", "-pthread",
                        "-I", os.path.join(pkg, "cpp"),
                        os.path.join(ROOT, "tests", "cpp", name + ".cpp"), "-o", str(exe),
                        "-L", pkg, "-lvexbayes_cuda", f"-Wl,-rpath,{pkg}"], check=True)
        assert exe.exists()
    # without a GPU the multi-GPU program stops at its first check, loudly
    import torch
    if not torch.cuda.is_available():
        run = subprocess.run([str(tmp_path / "test_multi")], capture_output=True, text=True)
        assert run.returncode != 0 and "devices 0" in run.stdout


def test_product_package_never_imports_the_oracle():
    """The oracle is a checker: the product may mention it in comments, but must
    never import, include, link or dlopen anything under oracle/."""
    pkg = os.path.join(ROOT, "paper_1902_09046_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            path = os.path.join(dirpath, f)
            if f.endswith(".py"):
                for line in open(path, errors="ignore"):
                    code = line.split("#", 1)[0]
                    assert not re.search(r"\b(import|from)\s+oracle\b|pyoracle|libvxb_oracle|libvxb_ref", code), (f, line)
            elif f.endswith((".cu", ".cuh", ".hpp", ".cpp", ".h")):
                for line in open(path, errors="ignore"):
                    code = line.split("//", 1)[0]
                    assert not re.search(r"#\s*include.*oracle|libvxb_oracle|libvxb_ref|vxo_", code), (f, line)
    # and the built library has no dependency on the checker
    import subprocess
    deps = subprocess.run(["ldd", lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "vxb_oracle" not in deps and "vxb_ref" not in deps


def test_multi_gpu_entry_points_argument_errors(so):
    """Host-side behaviour of the multi-GPU section of the ABI (no GPU needed): the
    packed accepted-set layout and its unpacking, argument checks, and the loud failure
    of vxb_multi_init without a CUDA device."""
    import torch
    lay = lib.accept_layout(A.VXB_F64, 3, 1000)
    assert (lay.off_count, lay.off_idx) == (0, 16) and lay.off_params == 16 + 8000
    assert lay.off_rho == lay.off_params + 24000 and lay.stride == lay.off_rho + 8000
    lay32 = lib.accept_layout(A.VXB_F32, 3, 7)           # every field stays 16-byte aligned
    assert all(v % 16 == 0 for v in (lay32.off_idx, lay32.off_params, lay32.off_rho, lay32.stride))
    for bad in ((A.VXB_F64, 0, 10), (A.VXB_F64, 3, 0), (5, 3, 10)):
        with pytest.raises(lib.VxbError) as e:
            lib.accept_layout(*bad)
        assert e.value.code in ("invalid-shape", "invalid-argument")
    # unpack: two blocks, the second one over capacity -> only `cap` rows, flagged
    buf = np.zeros(2 * lay32.stride, dtype=np.uint8)
    for r, count in enumerate((3, 9)):
        base = r * lay32.stride
        buf[base:base + 8].view(np.uint64)[0] = count
        buf[base + lay32.off_idx:base + lay32.off_idx + 56].view(np.uint64)[:] = np.arange(7) + 100 * r
        buf[base + lay32.off_rho:base + lay32.off_rho + 28].view(np.float32)[:] = r + 0.5
    n_acc, idx, params, rho, over = lib.accept_unpack(lay32, A.VXB_F32, 3, 2, buf)
    assert n_acc == 12 and over and idx.tolist() == [0, 1, 2, 100, 101, 102, 103, 104, 105, 106]
    assert rho.tolist() == [0.5] * 3 + [1.5] * 7
    n_acc, idx, _, _, _ = lib.accept_unpack(lay32, A.VXB_F32, 3, 2, buf, cap_out=4)
    assert n_acc == 12 and idx.tolist() == [0, 1, 2, 100]
    assert lib.device_count() == (torch.cuda.device_count() if torch.cuda.is_available() else 0)
    if not torch.cuda.is_available():
        with pytest.raises(lib.VxbError) as e:
            lib.Multi()
        assert e.value.code == "device-error"
    # the library finds NCCL by itself (dlopen); the version is the loaded library's
    assert lib.comm_version() >= 21800


def test_host_libm_exp_probe(so):
    """vxb_init probes which build of glibc's exp this process runs so that the device can
    reproduce it (csrc/vxb_libmexp.cuh).  Here: the FMA build; with the ifunc told to
    ignore FMA / AVX2 (GLIBC_TUNABLES -- a host CPU without FMA) the plain build."""
    import subprocess
    import sys
    assert lib.host_exp_variant() == 0
    code = "import sys; sys.path.insert(0, %r); from paper_1902_09046_b200 import lib; print('variant', lib.host_exp_variant())" % ROOT
    run = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300,
                         env=dict(os.environ, GLIBC_TUNABLES="glibc.cpu.hwcaps=-AVX2,-FMA"))
    assert run.returncode == 0 and "variant 1" in run.stdout, run.stdout + run.stderr[-800:]
