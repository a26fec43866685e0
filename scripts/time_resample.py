import sys, time
sys.path.insert(0, '/root/repo')
import numpy as np, torch
from paper_1902_09046_b200 import lib
ctx = lib.Context(0)
rs = np.random.RandomState(9)
for n in (100000, 1000003):
    lw = torch.from_numpy(rs.normal(size=n) * 3).cuda(); parts = torch.from_numpy(rs.normal(size=(n, 3))).cuda()
    out = torch.empty_like(parts); anc = torch.empty(n, dtype=torch.int64, device="cuda")
    def f():
        ctx._check(ctx.lib.vxb_resample_multinomial(ctx.handle, lib.u64(n), lib.u32(3), lib._ptr(lw), lib._ptr(parts), lib.u64(77), lib.u32(9), lib._ptr(out), lib._ptr(anc)))
    f(); torch.cuda.synchronize()
    ctx.profile_enable(True); ctx.profile_reset()
    t0=time.perf_counter()
    for _ in range(20): f()
    torch.cuda.synchronize(); dt=(time.perf_counter()-t0)/20
    print(n, "wall ms", dt*1e3, "kernels ms", ctx.profile_read()["resample"]["total_ms"]/20)
    ctx.profile_enable(False)
