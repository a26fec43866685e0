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


def packed_views(buf, layout, precision, dim, blocks=1):
    """Typed views of `blocks` consecutive packed accepted sets (vxb_accept_layout) held
    in the uint8 tensor `buf`: idx [blocks, cap] int64, params [blocks, cap, dim],
    rho [blocks, cap], count [blocks] int64.  No copy."""
    import torch
    from . import _abi as A
    real, rb = (torch.float32, 4) if precision == A.VXB_F32 else (torch.float64, 8)
    cap, stride = int(layout.cap), int(layout.stride)
    as64, asr = buf.view(torch.int64), buf.view(real)
    idx = torch.as_strided(as64, (blocks, cap), (stride // 8, 1), int(layout.off_idx) // 8)
    count = torch.as_strided(as64, (blocks,), (stride // 8,), int(layout.off_count) // 8)
    params = torch.as_strided(asr, (blocks, cap, dim), (stride // rb, dim, 1), int(layout.off_params) // rb)
    rho = torch.as_strided(asr, (blocks, cap), (stride // rb, 1), int(layout.off_rho) // rb)
    return idx, params, rho, count


def gather_packed(packed_local, world, out=None, group=None):
    """THE exchange of config 1: one all_gather_into_tensor of the fixed-capacity
    (count | idx | theta | rho) block of every rank -- no host round trip, so steps
    queue back to back on every rank.  Works on NCCL (CUDA) and gloo (CPU) alike."""
    import torch
    import torch.distributed as dist
    if out is None:
        out = torch.empty(world * packed_local.numel(), dtype=torch.uint8, device=packed_local.device)
    dist.all_gather_into_tensor(out, packed_local, group=group)
    return out


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


def _force_gather():
    """Diagnostics: VXB_FORCE_GATHER=1 runs the collective even with one rank, so that a
    one-GPU box executes exactly the code path of N > 1 (NCCL init, packed all-gather)."""
    import os
    return bool(os.environ.get("VXB_FORCE_GATHER"))


class RejectBuffers:
    """Output buffers of sharded_reject for this rank: its packed accepted set and
    (several ranks) the gathered blocks of all ranks, allocated on the library's
    stream so that the caching allocator's reuse is ordered with the kernels that
    fill them.  Reusable across steps."""

    def __init__(self, ctx, model, n_total, cap_fraction=0.01, group=None, world=None, rank=None):
        import torch
        from . import lib
        if world is None:
            rank, world = _world(group)
        self.world, self.rank = world, rank
        begin, end = shard_range(n_total, world, rank)
        # every rank uses the capacity of the largest shard: equal block sizes
        largest = shard_range(n_total, world, 0)
        cap = max(1024, int((largest[1] - largest[0]) * cap_fraction))
        self.layout = lib.accept_layout(model.precision, model.dim, cap)
        self.precision, self.dim = model.precision, model.dim
        dev = torch.device("cuda", ctx.device_info()["device"])
        with torch.cuda.stream(torch.cuda.ExternalStream(ctx.stream(), device=dev)):
            self.local = torch.empty(int(self.layout.stride), dtype=torch.uint8, device=dev)
            self.all = (torch.empty(world * int(self.layout.stride), dtype=torch.uint8, device=dev)
                        if world > 1 or _force_gather() else None)

    def local_views(self):
        idx, params, rho, count = packed_views(self.local, self.layout, self.precision, self.dim)
        return idx[0], params[0], rho[0], count

    def gathered_views(self):
        return packed_views(self.all, self.layout, self.precision, self.dim, self.world)


def reject_buffers(ctx, model, n_total, cap_fraction=0.01, group=None):
    return RejectBuffers(ctx, model, n_total, cap_fraction, group)


def sharded_reject(ctx, model, key, n_total, observed, eps, cap_fraction=0.01, group=None,
                   buffers=None, comm=None):
    """Config 1 on this rank's shard + the gather of accepted samples.

    Device-resident and fully asynchronous: the fused kernel path writes the accepted
    rows (and their count) into this rank's packed block; with several ranks ONE
    collective gathers the blocks over NVLink -- torch.distributed's NCCL
    (all_gather_into_tensor) or, with ``comm`` (lib.Comm), the library's own
    communicator through vxb_sharded_abc_reject.  Returns views (idx, theta, rho,
    count): of this rank's block for one rank, of all blocks ([world, ...]) otherwise.
    `buffers` (reject_buffers) lets a caller that steps repeatedly reuse the memory."""
    import torch
    rank, world = (comm.rank, comm.size) if comm is not None else _world(group)
    b = buffers if buffers is not None else RejectBuffers(ctx, model, n_total, cap_fraction, group,
                                                          world, rank)
    if comm is not None:
        ctx.sharded_abc_reject(comm, model, key, n_total, observed, eps, b.layout, b.local, b.all)
        return b.local_views() if b.all is None else b.gathered_views()
    begin, end = shard_range(n_total, world, rank)
    idx, params, rho, n_dev = b.local_views()
    ctx.abc_reject(model, key, n_total, begin, end - begin, observed, eps, int(b.layout.cap),
                   idx=idx, params=params, rho=rho, n_accepted=n_dev)
    if b.all is None:
        return idx, params, rho, n_dev
    with torch.cuda.stream(torch.cuda.ExternalStream(ctx.stream(), device=b.local.device)):
        gather_packed(b.local, world, out=b.all, group=group)
    return b.gathered_views()


# --------------------------------------------------------------------------
# ABC-SMC (config 3) over several GPUs
# --------------------------------------------------------------------------
CHUNK = 256  # the canonical reduction chunk (csrc/vxb_smc.cu: kChunk)


def _world(group):
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(group), dist.get_world_size(group)
    return 0, 1


def allgather_rows(tensors, group=None):
    """All-gather row blocks of different length: one all_gather of the counts,
    then one padded all_gather per tensor; returns the rank-order concatenations
    and the per-rank counts.  With one rank it is the identity.  Synchronises (the
    counts travel through the host): used by the one-shot paths (config 0, the
    weak-informativity test), not inside the ABC-SMC rounds."""
    import torch
    import torch.distributed as dist
    rank, world = _world(group)
    k = int(tensors[0].shape[0])
    if world == 1:
        return list(tensors), [k]
    n_local = torch.tensor([k], dtype=torch.int64, device=tensors[0].device)
    counts = torch.empty(world, dtype=torch.int64, device=n_local.device)
    dist.all_gather([counts[r:r + 1] for r in range(world)], n_local, group=group)
    counts = [int(c) for c in counts.tolist()]
    cap = max(max(counts), 1)
    outs = []
    for t in tensors:
        pad = torch.zeros((cap,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
        pad[:k] = t
        buf = torch.empty((world,) + tuple(pad.shape), dtype=t.dtype, device=t.device)
        dist.all_gather([buf[r] for r in range(world)], pad, group=group)
        outs.append(torch.cat([buf[r, :c] for r, c in enumerate(counts)], dim=0))
    return outs, counts


class DeviceStages:
    """The per-rank stage operations of an ABC-SMC generation on this rank's GPU,
    each one call into the C ABI (include/vexbayes_cuda.h).  Tensors are torch
    CUDA tensors that live on the library's stream; torch only allocates, slices
    and carries them into the collectives.  Every round operation is asynchronous:
    counts and fill levels stay in device memory (the `state` vector)."""

    def __init__(self, ctx):
        import torch
        self.ctx = ctx
        self.device = torch.device("cuda", ctx.device_info()["device"])
        self._stream = torch.cuda.ExternalStream(ctx.stream(), device=self.device)
        self._scratch = {}

    def scope(self):
        import torch
        return torch.cuda.stream(self._stream)

    def _buffers(self, count, dim):
        """Per-round evaluation scratch (theta*, rho, flag), reused across rounds."""
        import torch
        key = (count, dim)
        if key not in self._scratch:
            self._scratch = {key: (
                torch.empty((max(count, 1), dim), dtype=torch.float64, device=self.device),
                torch.empty(max(count, 1), dtype=torch.float64, device=self.device),
                torch.empty(max(count, 1), dtype=torch.uint8, device=self.device))}
        return self._scratch[key]

    def _pack(self, dim, theta, rho, failed, count, eps, layout, block, state, n):
        import ctypes as C
        from .lib import _ptr, u32, u64, f64
        c = self.ctx
        c._check(c.lib.vxb_abcsmc_pack_round(c.handle, u32(dim), _ptr(theta), _ptr(rho), _ptr(failed),
                                             u64(count), f64(eps), C.byref(layout), _ptr(block),
                                             _ptr(state), u64(n)))

    def prior_round(self, model, seed0, n_total, first, count, observed, layout, block, state, n):
        """Generation 0: rows [first, first+count) of the prior predictive job, the
        non-failed ones packed into `block`."""
        from . import models as M
        theta, rho, failed = self._buffers(count, model.dim)
        if count:
            self.ctx.abc_prior_predictive(model, M.keying(seed0), n_total, first, count, observed,
                                          params=theta, rho=rho, failed=failed)
        self._pack(model.dim, theta, rho, failed, count, float("inf"), layout, block, state, n)

    def propose_round(self, model, seed, gen, first, count, theta_prev, cum_prev, chol, observed,
                      eps, layout, block, state, n):
        """Generation >= 1: proposals [first, first+count), the accepted ones packed into
        `block`; skipped on the device once the population is full."""
        import ctypes as C
        from .lib import _ptr, u32, u64, f64
        theta, rho, flag = self._buffers(count, model.dim)
        ch = np.ascontiguousarray(chol, dtype=np.float64)
        obs = np.ascontiguousarray(observed, dtype=np.float64)
        c = self.ctx
        c._check(c.lib.vxb_abcsmc_propose(c.handle, C.byref(model), u64(seed), u32(gen), u64(first),
                                          u64(count), u64(int(theta_prev.shape[0])),
                                          _ptr(theta_prev), _ptr(cum_prev), _ptr(ch), _ptr(obs),
                                          f64(eps), _ptr(theta), _ptr(rho), _ptr(flag),
                                          _ptr(state), u64(n)))
        self._pack(model.dim, theta, rho, None, count, eps, layout, block, state, n)

    def append_round(self, blocks, world, layout, pop_theta, pop_rho, n, state):
        import ctypes as C
        from .lib import _ptr, u32, u64
        c = self.ctx
        c._check(c.lib.vxb_abcsmc_append_round(c.handle, u32(int(pop_theta.shape[1])), _ptr(blocks),
                                               u32(world), C.byref(layout), _ptr(pop_theta),
                                               _ptr(pop_rho), u64(n), _ptr(state)))

    def weights(self, theta_new, theta_prev, w_prev, chol, rng=0):
        """rng: the model's generator -- VXB_RNG_FAST selects the throughput form of the
        weights that the one-GPU driver uses for such a model."""
        import torch
        from .lib import _ptr, i32, u32, u64
        out = torch.empty(int(theta_new.shape[0]), dtype=torch.float64, device=self.device)
        if out.numel() == 0:
            return out
        ch = torch.from_numpy(np.ascontiguousarray(chol, dtype=np.float64)).to(self.device)
        c = self.ctx
        c._check(c.lib.vxb_abcsmc_weights(c.handle, i32(rng), u32(int(theta_new.shape[1])),
                                          u64(int(theta_new.shape[0])), _ptr(theta_new.contiguous()),
                                          u64(int(theta_prev.shape[0])), _ptr(theta_prev),
                                          _ptr(w_prev), _ptr(ch), _ptr(out)))
        return out

    def quantile(self, values, level):
        return self.ctx.quantile(values, level)

    def moments(self, theta, w):
        return self.ctx.weighted_moments(theta, w)

    def cumsum(self, w):
        import torch
        return self.ctx.canon_cumsum(w, torch.empty_like(w))

    def chunk_sums(self, v):
        import torch
        n = int(v.shape[0])
        return self.ctx.canon_chunk_sums(
            v, torch.empty((n + CHUNK - 1) // CHUNK, dtype=torch.float64, device=self.device))

    def normalise_by_totals(self, w_raw, totals):
        """In place: w_raw /= (chunk totals added left to right), all on the device."""
        from .lib import _ptr, u64
        c = self.ctx
        c._check(c.lib.vxb_normalise_by_chunk_totals(c.handle, _ptr(w_raw), u64(int(w_raw.shape[0])),
                                                     _ptr(totals), u64(int(totals.shape[0])), None))
        return w_raw

    def make_kernel(self, cov, scale, jitter):
        from . import lib
        return lib.make_kernel(cov, scale, jitter)


def sharded_abcsmc(stages, model, cfg, observed, group=None):
    """ABC-SMC (BASELINE config 3; scheme of DESIGN.md section 3.3) with the
    proposals of every round and the new particles of every generation sharded
    over the ranks by global index.  Exchanges:

    * per round ONE all_gather_into_tensor of each rank's packed block of accepted
      proposals (count | theta* | rho at a fixed capacity); the blocks are appended in
      rank order = ascending proposal index, so "the first N accepted by proposal
      index" is the same set on every rank and for every world size;
    * per generation one all-gather of the unnormalised importance weights (shards
      aligned to the 256-row canonical chunks, fixed size) and one all-reduce(SUM) of
      the vector of chunk totals -- every entry has exactly one non-zero contributor,
      so the reduction is exact and the weight sum (chunk totals added left to right,
      on the device) is bit-identical to the one-GPU run.

    No per-round host round trip: accepted counts, the fill level of the new
    population and the number of rounds used live in device memory (`state`); rounds
    are issued AHEAD of the host's knowledge from the previous acceptance rate, and a
    round that arrives after the population is full is skipped on the device.  The
    host reads the 4-word state once per batch of rounds (normally once per
    generation, together with the population statistics it needs anyway).

    The previous population (theta, w, rho) is replicated; its statistics (epsilon,
    weighted covariance, cumulative weights) are recomputed on every rank.  `stages`
    supplies the per-rank compute (DeviceStages on a GPU).  Returns the dictionary of
    Context.abcsmc_run."""
    import math
    import torch
    import torch.distributed as dist
    from . import _abi as A, lib
    from .lib import derive_seed
    rank, world = _world(group)
    n, gens, d = int(cfg.particles), int(cfg.generations), int(model.dim)
    round_size = int(cfg.round_size) or n
    max_rounds = int(cfg.max_rounds) or 1000
    if n < 2:
        raise ValueError("insufficient-data: need at least two particles")
    res = dict(epsilon=np.zeros(gens), ess=np.zeros(gens), accept_rate=np.zeros(gens),
               proposals=np.zeros(gens, dtype=np.uint64), mean=np.zeros((gens, d)),
               cov=np.zeros((gens, d, d)))
    n_chunks = (n + CHUNK - 1) // CHUNK
    c_begin, c_end = shard_range(n_chunks, world, rank)
    w_begin, w_end = min(n, c_begin * CHUNK), min(n, c_end * CHUNK)
    w_pad = (shard_range(n_chunks, world, 0)[1]) * CHUNK          # largest weight shard
    w_spans = [(min(n, shard_range(n_chunks, world, r)[0] * CHUNK),
                min(n, shard_range(n_chunks, world, r)[1] * CHUNK)) for r in range(world)]
    seed0 = derive_seed(cfg.seed, [0])
    b, e = shard_range(round_size, world, rank)
    cap = max(1, shard_range(round_size, world, 0)[1])            # largest slice of a round
    layout = lib.accept_layout(A.VXB_F64, d, cap)
    dev = stages.device
    with stages.scope():
        block = torch.zeros(int(layout.stride), dtype=torch.uint8, device=dev)
        blocks = torch.zeros(world * int(layout.stride), dtype=torch.uint8, device=dev) if world > 1 else block
        state = torch.zeros(4, dtype=torch.int64, device=dev)
        pops = [(torch.zeros((n, d), dtype=torch.float64, device=dev),
                 torch.zeros(n, dtype=torch.float64, device=dev)) for _ in range(2)]
        theta = w = rho = None
        rate = 1.0
        for g in range(gens):
            eps, chol, cum = float("inf"), None, None
            if g >= 1:
                eps = stages.quantile(rho, cfg.quantile)
                _, cov, _ = stages.moments(theta, w)
                chol = stages.make_kernel(cov, cfg.kernel_scale, cfg.jitter)
                cum = stages.cumsum(w)
            theta_new, rho_new = pops[g & 1]
            state.zero_()
            issued, got, accepted_total, used = 0, 0, 0, 0
            while got < n and issued < max_rounds:
                # generation 0 accepts every non-failed row: no slack; later generations:
                # the rounds the estimated rate asks for, plus half as many again
                need = (n - got) / (round_size * rate)
                ahead = int(math.ceil(need)) if g == 0 else int(math.ceil(1.5 * need)) + 1
                ahead = max(1, min(ahead, max_rounds - issued))
                for t in range(issued, issued + ahead):
                    first, count = t * round_size + b, e - b
                    if g == 0:
                        stages.prior_round(model, seed0, (t + 1) * round_size, first, count, observed,
                                           layout, block, state, n)
                    else:
                        stages.propose_round(model, cfg.seed, g, first, count, theta, cum, chol,
                                             observed, eps, layout, block, state, n)
                    if world > 1:
                        gather_packed(block, world, out=blocks, group=group)
                    stages.append_round(blocks, world, layout, theta_new, rho_new, n, state)
                issued += ahead
                got, accepted_total, used, _ = (int(v) for v in state.cpu().numpy())  # one read per batch
                if used:
                    rate = max(accepted_total / (used * round_size), 1e-9)
            if got != n:
                raise RuntimeError("empty-set: generation did not fill within max_rounds")
            evaluated = used * round_size
            rate *= 0.8   # the acceptance rate falls from one generation to the next
            if g == 0:
                w_new = torch.full((n,), 1.0 / n, dtype=torch.float64, device=dev)
            else:
                w_local = stages.weights(theta_new[w_begin:w_end], theta, w, chol, rng=int(model.rng))
                totals = torch.zeros(n_chunks, dtype=torch.float64, device=dev)
                if w_end > w_begin:
                    totals[c_begin:c_end] = stages.chunk_sums(w_local)
                if world > 1:
                    padded = torch.zeros(w_pad, dtype=torch.float64, device=dev)
                    padded[:w_end - w_begin] = w_local
                    gathered = torch.empty(world * w_pad, dtype=torch.float64, device=dev)
                    dist.all_gather_into_tensor(gathered, padded, group=group)
                    w_new = torch.cat([gathered[r * w_pad:r * w_pad + (hi - lo)]
                                       for r, (lo, hi) in enumerate(w_spans)])
                    allreduce_sum(totals, group)
                else:
                    w_new = w_local
                w_new = stages.normalise_by_totals(w_new.contiguous(), totals)
            theta, w, rho = theta_new, w_new, rho_new
            mean, cov, s2 = stages.moments(theta, w)
            if not (np.isfinite(s2) and s2 > 0.0):
                raise RuntimeError("degenerate-ensemble: weight sum is not finite")
            res["epsilon"][g], res["ess"][g] = eps, 1.0 / s2
            res["accept_rate"][g] = accepted_total / evaluated
            res["proposals"][g] = evaluated
            res["mean"][g], res["cov"][g] = mean, cov
        res["theta"] = theta.cpu().numpy()
        res["weight"] = w.cpu().numpy()
        res["rho"] = rho.cpu().numpy()
    return res


# --------------------------------------------------------------------------
# configs 0, 2 and 4 over several GPUs
# --------------------------------------------------------------------------
def sharded_select(ctx, model, key, n_total, observed, accept_fraction, group=None):
    """Config 0: every rank simulates its rows, the discrepancies (8 B/row, 8 MB
    at N = 1e6) are all-gathered, and every rank runs the same select_epsilon
    (abc.cpp:75-97) over the full vector -- epsilon and the ascending accepted
    indices are identical on every rank and for every world size.  Returns
    (epsilon, idx tensor, theta tensor of the accepted rows, rho tensor)."""
    import torch
    import torch.distributed as dist
    from . import _abi as A
    rank, world = _world(group)
    begin, end = shard_range(n_total, world, rank)
    count = end - begin
    dev = torch.device("cuda", ctx.device_info()["device"])
    real = torch.float32 if model.precision == A.VXB_F32 else torch.float64
    with torch.cuda.stream(torch.cuda.ExternalStream(ctx.stream(), device=dev)):
        theta = torch.empty((count, model.dim), dtype=real, device=dev)
        rho = torch.empty(count, dtype=real, device=dev)
        failed = torch.empty(count, dtype=torch.uint8, device=dev)
        ctx.abc_prior_predictive(model, key, n_total, begin, count, observed, params=theta,
                                 rho=rho, failed=failed)
        if world > 1:
            (rho_all, failed_all), counts = allgather_rows([rho, failed], group)
        else:
            rho_all, failed_all = rho, failed
        cap = max(1024, int(4 * accept_fraction * n_total) + 64)
        idx = torch.empty(cap, dtype=torch.int64, device=dev)
        eps, _, n_acc = ctx.select_epsilon(rho_all.contiguous(), failed_all.contiguous(),
                                           accept_fraction, cap, model.precision, n_total, idx)
        idx = idx[:min(n_acc, cap)]
        # accepted theta live on the rank that simulated them: gather in rank order
        mine = idx[(idx >= begin) & (idx < end)] - begin
        th_acc = theta.index_select(0, mine)
        if world > 1:
            (th_acc,), _ = allgather_rows([th_acc], group)
        return eps, idx, th_acc, rho_all.index_select(0, idx)


def sharded_counts(local_counts, group=None):
    """Configs 2 and 4: integer counters of disjoint dataset / path ranges add up
    with one all-reduce(SUM); integer sums are exact in any order."""
    rank, world = _world(group)
    if world > 1:
        allreduce_sum(local_counts, group)
    return local_counts


def sharded_weak_info(ctx, cfg, group=None, evidence_fn=None):
    """The weak-informativity test with the hyperparameter rows sharded over the
    ranks (the reference's own task parallelism, weak_info.cpp:248-262): rank r
    estimates the evidences of rows partition(K+1, world, 1)[r]; one all-gather of
    the (rows x N x 2) evidence blocks (2.6 MB at the paper's size); every rank then
    computes the same p-values and cut-offs.  Sampler seeds are keyed by (row,
    dataset), so the table is identical for every world size.  `evidence_fn(first,
    count)` replaces the device stage in the CPU tests."""
    import torch
    from . import lib
    rank, world = _world(group)
    rows = int(cfg.hyper_count) + 1
    begin, end = shard_range(rows, world, rank)
    lam = ctx.weak_info_lambdas(cfg) if ctx is not None else None
    if evidence_fn is None:
        mine = ctx.weak_info_evidence(cfg, lam, begin, end - begin)
        dev = torch.device("cuda", ctx.device_info()["device"])
    else:
        mine = evidence_fn(begin, end - begin)
        dev = torch.device("cpu")
    block = torch.from_numpy(np.ascontiguousarray(mine)).to(dev)
    (ev,), _ = allgather_rows([block], group)
    ev = ev.cpu().numpy()
    gamma, weakly, completed = lib.weak_info_cutoffs(cfg, ev)
    return dict(lambda_=lam, gamma=gamma, weakly=weakly, completed=completed, evidence=ev)
