"""GPU tests of the device-resident / asynchronous forms of the C ABI: buffers
passed as device memory (torch tensors) and the fused fixed-epsilon path whose
accepted count stays on the device (no host round trip per step)."""
import numpy as np
import pytest

from paper_1902_09046_b200 import _abi as A, dist as D, lib, models as M

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("precision", [A.VXB_F64, A.VXB_F32])
def test_async_reject_equals_synchronous(ctx, oracle, golden, precision):
    import torch
    obs = golden["logistic_observed"]
    m = M.logistic_model(precision=precision)
    n = 40000
    p, s, rho, f = oracle.abc_prior_predictive(m, M.keying(1337), n, 0, n, obs, want_summaries=False)
    eps, idx_o = oracle.select_epsilon(rho, f, 0.02)
    # synchronous, host buffers
    nacc, idx, params, rho_acc = ctx.abc_reject(m, M.keying(1337), n, 0, n, obs, eps, cap=n)
    assert nacc == len(idx_o) and np.array_equal(idx, idx_o)
    # asynchronous, everything device resident (several steps queued back to back)
    outs = [D.sharded_reject(ctx, m, M.keying(1337), n, obs, eps, cap_fraction=0.1) for _ in range(3)]
    ctx.synchronize()
    for d_idx, d_params, d_rho, d_n in outs:
        k = int(d_n.item())
        assert k == len(idx_o)
        assert np.array_equal(d_idx[:k].cpu().numpy(), idx_o.astype(np.int64))
        assert np.array_equal(d_params[:k].cpu().numpy().astype(np.float64), p[idx_o])
        assert np.array_equal(d_rho[:k].cpu().numpy().astype(np.float64), rho[idx_o])
    # a capped asynchronous call reports the full count and fills only `cap` rows
    dt = torch.float32 if precision == A.VXB_F32 else torch.float64
    cap = 7
    d_idx = torch.full((cap + 3,), -1, dtype=torch.int64, device="cuda")
    d_par = torch.zeros((cap, 3), dtype=dt, device="cuda")
    d_rho = torch.zeros(cap, dtype=dt, device="cuda")
    d_n = torch.zeros(1, dtype=torch.int64, device="cuda")
    ctx.abc_reject(m, M.keying(1337), n, 0, n, obs, eps, cap, idx=d_idx, params=d_par, rho=d_rho, n_accepted=d_n)
    ctx.synchronize()
    assert int(d_n.item()) == len(idx_o)
    assert np.array_equal(d_idx.cpu().numpy()[:cap], idx_o[:cap].astype(np.int64))
    assert (d_idx.cpu().numpy()[cap:] == -1).all()
    # host outputs cannot be combined with a device-resident count
    with pytest.raises(lib.VxbError) as e:
        ctx.abc_reject(m, M.keying(1337), n, 0, n, obs, eps, cap, idx=np.zeros(cap, dtype=np.uint64),
                       params=d_par, rho=d_rho, n_accepted=d_n)
    assert e.value.code == "invalid-argument"


def test_device_buffers_for_prior_predictive_and_select(ctx, oracle, golden):
    import torch
    obs = golden["logistic_observed"]
    m = M.logistic_model()
    n = 5000
    d_rho = torch.empty(n, dtype=torch.float64, device="cuda")
    d_failed = torch.empty(n, dtype=torch.uint8, device="cuda")
    d_params = torch.empty((n, 3), dtype=torch.float64, device="cuda")
    ctx.abc_prior_predictive(m, M.keying(7), n, 0, n, obs, params=d_params, rho=d_rho, failed=d_failed)
    ctx.synchronize()
    p, s, rho, f = oracle.abc_prior_predictive(m, M.keying(7), n, 0, n, obs, want_summaries=False)
    assert np.array_equal(d_rho.cpu().numpy(), rho) and np.array_equal(d_params.cpu().numpy(), p)
    d_idx = torch.empty(n, dtype=torch.int64, device="cuda")
    eps, _, nacc = ctx.select_epsilon(d_rho, d_failed, 0.05, cap=n, precision=A.VXB_F64, n=n, idx=d_idx)
    eps_o, idx_o = oracle.select_epsilon(rho, f, 0.05)
    assert eps == eps_o and nacc == len(idx_o)
    assert np.array_equal(d_idx[:nacc].cpu().numpy(), idx_o.astype(np.int64))
