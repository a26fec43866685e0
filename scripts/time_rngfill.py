"""Kernel 1 alone: device-resident fills of N(0,1) variates, reference-exact stream
(Philox2x64-10 + the reference's polynomial Box-Muller) and throughput generator."""
import ctypes as C, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from paper_1902_09046_b200 import _abi as A, lib
ctx = lib.Context(0)
u64, u32, f64, i32 = C.c_uint64, C.c_uint32, C.c_double, C.c_int32
n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 400_000_000
out = torch.empty(n, dtype=torch.float64, device="cuda")
ptr = C.c_void_p(out.data_ptr())
res = {}
def timed(name, call, count, bytes_):
    call(); ctx.synchronize()
    ctx.profile_enable(True); ctx.profile_reset()
    call(); ctx.synchronize()
    ms = sum(v["total_ms"] for v in ctx.profile_read().values())
    ctx.profile_enable(False)
    res[name] = {"normals": count, "ms": ms, "normals_per_s": count / ms * 1e3, "write_GBps": bytes_ / ms / 1e6}
timed("exact_f64", lambda: ctx._check(ctx.lib.vxb_rng_fill_gaussian(ctx.handle, u64(7), u32(0), u64(0), u64(n), f64(0.0), f64(1.0), ptr)), n, 8 * n)
rows, per = n // 2000, 2000
timed("fast_f64", lambda: ctx._check(ctx.lib.vxb_rng_fill_gaussian_fast(ctx.handle, i32(A.VXB_F64), u64(7), u64(0), u64(rows), u32(per), ptr)), rows * per, 8 * rows * per)
timed("fast_f32", lambda: ctx._check(ctx.lib.vxb_rng_fill_gaussian_fast(ctx.handle, i32(A.VXB_F32), u64(7), u64(0), u64(rows), u32(per), ptr)), rows * per, 4 * rows * per)
import json
print(json.dumps(res))
