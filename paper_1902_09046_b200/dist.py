"""Multi-GPU host layer: one process per GPU, torch.distributed for the exchange.

The hot path shards by construction: rows are keyed by
their global index, so rank r simulating rows [begin_r, end_r) of the job
produces exactly the rows a single GPU would.  The data path needs no
collective; only results are exchanged:

* accepted sets (config 0/1): all_gather of the per-rank counts, then a padded
  all_gather of (index, theta, rho); concatenation in rank order is ascending
  in the global row index because the shards are contiguous and ordered.
* counters (config 2) / level sums (config 4): one all_reduce(SUM).

On CUDA ranks the exchange runs over NCCL (NVLink); the same code runs over
gloo with CPU tensors for the world_size-2 tests.
"""
import numpy as np


def shard_range(total, world, rank, block=1):
    """The reference's static partition (blocked.cpp:34-63) as the shard rule."""
    blocks = (total + block - 1) // block
    base, extra = divmod(blocks, world)
    begin_block = rank * base + min(rank, extra)
    nblocks = base + (1 if rank < extra else 0)
    begin = min(total, begin_block * block)
    end = min(total, (begin_block + nblocks) * block)
    return begin, end


def gather_accepted(idx, params, rho, group=None):
    """All-gather variable-length accepted sets; returns the concatenation in
    rank order (ascending global row index).  Inputs are torch tensors on the
    rank's device (CUDA -> NCCL, CPU -> gloo), trimmed to the local count."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    n_local = torch.tensor([idx.shape[0]], dtype=torch.int64, device=idx.device)
    counts = [torch.zeros_like(n_local) for _ in range(world)]
    dist.all_gather(counts, n_local, group=group)
    counts = [int(c.item()) for c in counts]
    cap = max(max(counts), 1)

    def padded(t):
        out = torch.zeros((cap,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
        out[: t.shape[0]] = t
        return out

    outs = []
    for t in (idx, params, rho):
        buf = [torch.empty((cap,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
               for _ in range(world)]
        dist.all_gather(buf, padded(t), group=group)
        outs.append(torch.cat([b[:c] for b, c in zip(buf, counts)], dim=0))
    return outs[0], outs[1], outs[2], counts


def gather_accepted_padded(idx, params, rho, n_dev, group=None):
    """Asynchronous form: fixed-capacity buffers (rows [0, n_dev) valid) and the
    device-resident count are all-gathered as they are -- no host round trip, so
    steps queue back to back on every rank.  Returns tensors shaped
    [world, cap, ...] plus the [world] count tensor; ``compact_gathered`` turns
    them into the ascending concatenation once the host needs it."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    outs = []
    for t in (idx, params, rho, n_dev):
        buf = torch.empty((world,) + tuple(t.shape), dtype=t.dtype, device=t.device)
        # per-rank views of one buffer: works on gloo (tests) and NCCL alike
        dist.all_gather([buf[r] for r in range(world)], t.contiguous(), group=group)
        outs.append(buf)
    return outs[0], outs[1], outs[2], outs[3].reshape(world)


def compact_gathered(idx, params, rho, counts):
    """Concatenate the valid rows of a padded gather in rank order (synchronises)."""
    import torch
    c = [int(v) for v in counts.tolist()]
    cap = idx.shape[1]
    keep = [min(k, cap) for k in c]
    return (torch.cat([idx[r, :k] for r, k in enumerate(keep)]),
            torch.cat([params[r, :k] for r, k in enumerate(keep)]),
            torch.cat([rho[r, :k] for r, k in enumerate(keep)]), c)


def allreduce_sum(t, group=None):
    import torch.distributed as dist
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return t


def sharded_reject(ctx, model, key, n_total, observed, eps, cap_fraction=0.01, group=None):
    """Config 1 on this rank's shard + the gather of accepted samples.

    Device-resident: outputs are torch CUDA tensors filled by the fused kernel
    path; only the accepted rows travel."""
    import torch
    import torch.distributed as dist
    from . import _abi as A
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    begin, end = shard_range(n_total, world, rank)
    count = end - begin
    cap = max(1024, int(count * cap_fraction))
    dev = torch.device("cuda", ctx.device_info()["device"])
    real = torch.float32 if model.precision == A.VXB_F32 else torch.float64
    # allocate on the library's stream so that the caching allocator's reuse of
    # these buffers is ordered with the kernels that fill them
    with torch.cuda.stream(torch.cuda.ExternalStream(ctx.stream(), device=dev)):
        idx = torch.empty(cap, dtype=torch.int64, device=dev)
        params = torch.empty((cap, model.dim), dtype=real, device=dev)
        rho = torch.empty(cap, dtype=real, device=dev)
        n_dev = torch.empty(1, dtype=torch.int64, device=dev)
    # fully asynchronous: the accepted count stays on the device, the host only
    # enqueues (rows [0, count) of the buffers are valid once the stream drains)
    ctx.abc_reject(model, key, n_total, begin, count, observed, eps, cap, idx=idx,
                   params=params, rho=rho, n_accepted=n_dev)
    if world == 1:
        return idx, params, rho, n_dev
    # the gather of accepted samples over NVLink, on the library's stream, padded to
    # the fixed capacity so that no rank has to read a count back first
    with torch.cuda.stream(torch.cuda.ExternalStream(ctx.stream(), device=dev)):
        return gather_accepted_padded(idx, params, rho, n_dev, group)
