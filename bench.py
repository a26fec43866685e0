#!/usr/bin/env python
"""bench.py -- headline benchmark of the hot path (BASELINE.json config 1).

Workload: ABC rejection on the stochastic logistic-growth SDE, N = 1e8 prior
samples per step (2000 Euler-Maruyama steps each), acceptance threshold fixed at
the 0.1% quantile taken from config 0 (N = 1e6, seed 1337), particles sharded
evenly over the GPUs (strong scaling, as config 1 states), accepted samples
gathered over NCCL.  One "step" = one full pass over the N particles.

    python bench.py --gpus 1 --steps 5 --warmup 3
    python bench.py --gpus N ...              # starts N ranks itself (torch.distributed.run)
    python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N ...
    python bench.py --impl reference ...      # the reference's CPU path, host cores

Prints ONE JSON line (rank 0).  Inputs are synthetic (seeded); see DESIGN.md.
At N = 1 the line also carries `configs`: every other BASELINE config (0, 2, 3, 4) and
the reference's own workloads (toggle switch, weak-informativity test, TB Gillespie,
resample_multinomial) at full size, each timed with CUDA events under the same NVML
clock sampler as the headline.
"""
import argparse
import json
import math
import os
import socket
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

FLOPS_PER_STEP = 55                     # 47 per N(0,1) + 8 for the update
STEPS_PER_SIM = 2000
FLOPS_PER_SIM = STEPS_PER_SIM * FLOPS_PER_STEP + 3 * 3 + 20 * 3 + 1   # prior + distance
NOMINAL_PEAK = {"f64": 148 * 64 * 2 * 1.965e9 / 1e12, "f32": 148 * 128 * 2 * 1.965e9 / 1e12}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--particles", type=float, default=1e8)
    ap.add_argument("--variant", default="f64_fast",
                    choices=["f64_fast", "f64_ref", "f32_fast", "f32_ref"])
    ap.add_argument("--no-extras", action="store_true", help="skip variants and cpu baseline")
    ap.add_argument("--cpu-sample", type=float, default=4e5)
    ap.add_argument("--comm", default="torch", choices=["torch", "native"],
                    help="N > 1: gather over torch.distributed's NCCL or the library's own "
                         "communicator (vxb_comm_*, bootstrapped through torch.distributed)")
    ap.add_argument("--selftest-dist", action="store_true",
                    help="CPU check of the launch path: gloo ranks, one packed gather, no GPU work")
    return ap.parse_args()


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def spawn_ranks(args):
    """`python bench.py --gpus N` without a launcher: start the N ranks ourselves, the
    way the driver does (torch.distributed.run, one process per GPU, rendezvous on
    127.0.0.1).  NCCL's communicator lines go to stderr (NCCL_DEBUG=INFO, INIT only)."""
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    env.setdefault("OMP_NUM_THREADS", "1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           "--master-port", str(free_port()), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd, env=env)


def selftest_dist(args, rank, world):
    """The launch + exchange path on CPU (gloo): every rank builds a packed accepted
    block (include/vexbayes_cuda.h: vxb_accept_layout) with known contents, ONE
    all_gather_into_tensor moves them, rank 0 checks the rank-order concatenation."""
    import torch
    import torch.distributed as dist
    from paper_1902_09046_b200 import _abi as A, dist as D, lib
    if world > 1:
        dist.init_process_group("gloo")
    lay = lib.accept_layout(A.VXB_F64, 3, 64)
    block = torch.zeros(int(lay.stride), dtype=torch.uint8)
    idx, params, rho, count = D.packed_views(block, lay, A.VXB_F64, 3)
    k = 5 + rank
    begin, _ = D.shard_range(1000, world, rank)
    idx[0, :k] = torch.arange(begin, begin + k)
    rho[0, :k] = 0.5 + rank
    count[0] = k
    allb = D.gather_packed(block, world) if world > 1 else block
    n_acc, g_idx, _, g_rho, over = lib.accept_unpack(lay, A.VXB_F64, 3, world, allb.numpy())
    ok = (n_acc == sum(5 + r for r in range(world)) and not over and bool((np.diff(g_idx.astype(np.int64)) > 0).all()))
    if rank == 0:
        print(json.dumps({"selftest": "dist", "ok": bool(ok), "n_gpus": world, "backend": "gloo",
                          "accepted": int(n_acc), "pid": os.getpid(),
                          "launched_by": "torch.distributed.run" if "TORCHELASTIC_RUN_ID" in os.environ
                          else "direct"}), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0 if ok else 1


class ClockSampler:
    """SM clock, power and throttle reasons DURING the timed region, read through
    NVML in a background thread (polling the nvidia-smi CLI instead stalls the
    launching thread by ~10% on this driver)."""
    REASONS = {"hw_slowdown": 0x8, "sw_power_cap": 0x4, "hw_thermal_slowdown": 0x40,
               "sw_thermal_slowdown": 0x20}

    def __init__(self, device, period=0.25):
        self.device, self.period = device, period
        self.sm, self.pw, self.mask, self.max_sm = [], [], 0, None
        self.stop = threading.Event()
        self.thread = None

    def _handle(self):
        import pynvml
        pynvml.nvmlInit()
        try:
            import torch
            uuid = str(torch.cuda.get_device_properties(self.device).uuid)
            if not uuid.startswith("GPU-"):
                uuid = "GPU-" + uuid
            return pynvml, pynvml.nvmlDeviceGetHandleByUUID(uuid)
        except Exception:
            return pynvml, pynvml.nvmlDeviceGetHandleByIndex(self.device)

    def _run(self):
        try:
            nv, h = self._handle()
            self.max_sm = float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM))
            while not self.stop.is_set():
                self.sm.append(float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)))
                self.pw.append(nv.nvmlDeviceGetPowerUsage(h) / 1000.0)
                self.mask |= int(nv.nvmlDeviceGetCurrentClocksEventReasons(h))
                self.stop.wait(self.period)
        except Exception as e:  # NVML missing: report no samples rather than fail the bench
            self.error = repr(e)

    def __enter__(self):
        if os.environ.get("VXB_BENCH_NO_CLOCKS"):   # diagnostics: is the sampler itself a cost?
            return self
        self.thread = threading.Thread(target=self._run, daemon=True)
        self.thread.start()
        return self

    def __exit__(self, *exc):
        self.stop.set()
        if self.thread is not None:
            self.thread.join(timeout=2)

    def summary(self):
        if not self.sm:
            return {"sm_mhz": None, "sm_max_mhz": self.max_sm, "reasons": [], "samples": 0,
                    "error": getattr(self, "error", None)}
        reasons = sorted(n for n, bit in self.REASONS.items() if self.mask & bit)
        return {"sm_mhz": float(np.median(self.sm)), "sm_min_mhz": min(self.sm),
                "sm_max_mhz": self.max_sm, "power_w_max": max(self.pw), "reasons": reasons,
                "samples": len(self.sm)}


def ncu_traffic(variant):
    """DRAM bytes per launch and the pipe utilisations of the dominant kernel from the
    committed ncu capture (profiles/r2_traffic.json; taken at 2e6 rows per launch).  The
    flop-convention `frac` prices a normal at the reference's 47 flop; the pipe numbers
    say how busy the hardware actually was."""
    try:
        t = json.load(open(os.path.join(ROOT, "profiles", "r2_traffic.json")))
        k = t["kernels"][variant]
        out = {"traffic": k["dram_bytes"],
               "traffic_note": f"ncu dram bytes per launch at {t['rows_per_profiled_launch']} rows "
                               f"(algorithmic: {k['algorithmic_bytes']} B of rho, L2 resident)"}
        for key in ("fp64_pipe_active_pct", "xu_pipe_pct", "issue_active_pct", "alu_pipe_pct",
                    "fma_pipe_pct", "warps_active_pct"):
            if key in k:
                out[key.replace("_pct", "_ncu")] = k[key]
        return out
    except (OSError, KeyError, ValueError):
        return {"traffic": None}


def logistic_variant(name):
    from paper_1902_09046_b200 import _abi as A, models as M
    prec = A.VXB_F32 if name.startswith("f32") else A.VXB_F64
    rng = A.VXB_RNG_FAST if name.endswith("fast") else A.VXB_RNG_REF
    return M.logistic_model(precision=prec, rng=rng)


def run_reference(args, rank, world):
    """The reference's own CPU implementation of the path on the host cores:
    abc::run_prior_predictive (unmodified reference, oracle/_ref) on the logistic
    hooks + the fixed-epsilon accept scan; bounded sample per step."""
    if rank != 0:
        return
    from oracle.pyoracle import Oracle, Ref
    from paper_1902_09046_b200 import _abi as A, models as M
    cores = os.cpu_count() or 1
    m = M.logistic_model()
    sample = int(args.cpu_sample)
    use_ref = Ref.available()
    o = Ref() if use_ref else Oracle(threads=cores)
    theta = [0.5, 100.0, 0.05]
    seed_obs = o.derive_seed(1, [90])
    obs = o.logistic_simulate(m, theta, seed_obs, 0, 0) if use_ref else o.simulate_at(m, theta, seed_obs, 0, 0)
    # config 1 fixes epsilon at config 0's 0.1% quantile (seed 1337, reference-exact
    # RNG, particle keying); its value is a pure function of the seeds, so the arm
    # uses the constant the GPU arm recomputes every run (profiles/r1_bench_1gpu.json)
    eps = 19.712058377057488

    def step(s):
        if use_ref:
            p, summ, rho, f = o.logistic_abc(m, sample, cores, 1, 1337 + s, obs)
        else:
            p, summ, rho, f = o.abc_prior_predictive(m, M.keying(1337 + s), sample, 0, sample, obs)
        return int(((rho <= eps) & (f == 0)).sum())

    for s in range(args.warmup):
        step(s)
    t0 = time.perf_counter()
    for s in range(args.steps):
        step(args.warmup + s)
    dt = time.perf_counter() - t0
    sims = args.steps * sample / dt
    line = {
        "impl": "reference", "metric": "prior-predictive sims/sec (logistic SDE ABC rejection)",
        "value": sims, "unit": "sims/s", "sde_steps_per_s": sims * STEPS_PER_SIM,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * dt / args.steps, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "config1: logistic-SDE ABC rejection, fixed epsilon, fp64",
                   "particles_per_step": sample, "sde_steps_per_particle": STEPS_PER_SIM},
        "cpu_baseline": {"value": sims, "unit": "sims/s", "cores": cores,
                         "kind": "reference" if use_ref else "port",
                         "sample": f"{sample} particles per step (of the 1e8-particle job), "
                                   f"{cores} std::thread workers, reference keying"},
        "e2e": {"value": sims, "unit": "sims/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl != "reference":
        sys.exit(spawn_ranks(args))
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}: launch one rank per GPU "
                 "(python bench.py --gpus N starts them itself)")
    if args.selftest_dist:
        sys.exit(selftest_dist(args, rank, world))

    import torch
    import torch.distributed as dist
    from paper_1902_09046_b200 import _abi as A, dist as D, lib, models as M

    torch.cuda.set_device(local)
    comm, comm_note = None, "single GPU: no collective"
    # VXB_FORCE_GATHER=1 (diagnostics, under a launcher): one rank walks the N > 1 path
    dist_on = world > 1 or (bool(os.environ.get("VXB_FORCE_GATHER")) and "RANK" in os.environ)
    if dist_on:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    ctx = lib.Context(local)
    if dist_on:
        comm_note = "torch.distributed NCCL all_gather_into_tensor of the packed accepted block"
        if args.comm == "native":
            # the library's own NCCL communicator; its unique id travels through
            # torch.distributed.  Every rank must agree on the outcome.
            ok = torch.ones(1, dtype=torch.int32, device=f"cuda:{local}")
            uid = [None]
            if rank == 0:
                try:
                    uid = [lib.comm_unique_id().tobytes()]
                except Exception as e:     # NCCL not loadable: every rank falls back together
                    print(f"bench.py: native communicator unavailable: {e!r}", file=sys.stderr)
            dist.broadcast_object_list(uid, src=0)
            try:
                if uid[0] is None:
                    raise RuntimeError("no unique id")
                comm = lib.Comm(ctx, np.frombuffer(uid[0], dtype=np.uint8), rank, world)
            except Exception as e:  # fall back to torch.distributed rather than lose the run
                ok.zero_()
                print(f"bench.py: rank {rank}: native communicator failed: {e!r}", file=sys.stderr)
            dist.all_reduce(ok, op=dist.ReduceOp.MIN)
            if int(ok.item()) == 1:
                comm_note = f"library NCCL (vxb_sharded_abc_reject, NCCL {lib.comm_version()})"
            else:
                if comm is not None:
                    comm.close()
                comm = None
                comm_note += " (native communicator failed on some rank: fell back)"
    info = ctx.device_info()
    ext = torch.cuda.ExternalStream(ctx.stream(), device=torch.device("cuda", local))
    n_total = int(args.particles)

    # ---- synthetic data: config 0 observation and its 0.1% epsilon
    m_ref = M.logistic_model()
    obs = ctx.simulate_at(m_ref, [0.5, 100.0, 0.05], lib.derive_seed(1, [90]), 0, 0)
    n0 = 1_000_000
    rho0 = torch.empty(n0, dtype=torch.float64, device=f"cuda:{local}")
    ctx.abc_prior_predictive(m_ref, M.keying(1337), n0, 0, n0, obs, rho=rho0)
    eps, _, nacc0 = ctx.select_epsilon(rho0, None, 1e-3, cap=0, precision=A.VXB_F64, n=n0,
                                       idx=np.zeros(1, dtype=np.uint64))
    del rho0

    def barrier():
        if dist_on:
            dist.barrier()
        torch.cuda.synchronize()

    def timed(fn, warmup, steps):
        """W untimed + exactly K timed steps, events on the launching stream, max over ranks."""
        with torch.cuda.stream(ext):
            for s in range(warmup):
                fn(s)
            barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(ext)
            out = None
            for s in range(steps):
                out = fn(warmup + s)
            e1.record(ext)
            barrier()
        ms = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=f"cuda:{local}")
        if dist_on:
            dist.all_reduce(ms, op=dist.ReduceOp.MAX)
        return float(ms.item()), out

    def device_step(model):
        buffers = D.reject_buffers(ctx, model, n_total)   # reused by every step

        def fn(s):
            return D.sharded_reject(ctx, model, M.keying(1337 + s), n_total, obs, eps,
                                    buffers=buffers, comm=comm)
        return fn

    def host_step(model):
        begin, end = D.shard_range(n_total, world, rank)
        cap = max(1024, int((end - begin) * 0.01))
        # the caller's HOST buffers, pinned and reused by every step (a pageable,
        # freshly zeroed 40 MB set per step costs 2 ms of host time against 354 ms)
        real = torch.float32 if model.precision == A.VXB_F32 else torch.float64
        h_idx = torch.empty(cap, dtype=torch.int64, pin_memory=True).numpy().view(np.uint64)
        h_par = torch.empty((cap, model.dim), dtype=real, pin_memory=True).numpy()
        h_rho = torch.empty(cap, dtype=real, pin_memory=True).numpy()

        def fn(s):  # public host-buffer call: H2D of the observation, D2H of the accepted rows
            k, _, _, _ = ctx.abc_reject(model, M.keying(1337 + s), n_total, begin, end - begin, obs,
                                        eps, cap, idx=h_idx, params=h_par, rho=h_rho)
            k = min(k, cap)
            return k, h_idx[:k], h_par[:k], h_rho[:k]
        return fn

    # ---- headline: device-resident
    model = logistic_variant(args.variant)
    ctx.profile_reset()
    with ClockSampler(local) as clocks:
        ms, out = timed(device_step(model), args.warmup, args.steps)
    total_launches = sum(v["launches"] for v in ctx.profile_read().values())
    timed_fraction = args.steps / (args.warmup + args.steps)
    # the dominant kernel's own duration: a separate short pass with the library's
    # per-launch CUDA events switched on (kept out of the headline loop above)
    ctx.profile_enable(True)
    ctx.profile_reset()
    timed(device_step(model), 1, min(args.steps, 3))
    prof = ctx.profile_read()
    ctx.profile_enable(False)
    sims_per_s = args.steps * n_total / (ms * 1e-3)
    n_acc = int(out[3].sum().item())  # device-resident count(s), read once after the timed region
    sim = prof["simulate"]
    kernel_ms = sim["total_ms"] / max(sim["launches"], 1)   # per launch, this rank's shard
    begin, end = D.shard_range(n_total, world, rank)
    kernel_flops = (end - begin) * FLOPS_PER_SIM
    dt_name = "f32" if args.variant.startswith("f32") else "f64"
    peak_meas, _ = ctx.fma_peak(A.VXB_F32 if dt_name == "f32" else A.VXB_F64)
    achieved = kernel_flops / (kernel_ms * 1e-3) / 1e12

    # ---- e2e: host buffers through the public call
    ms_e2e, out_h = timed(host_step(model), args.warmup, args.steps)
    e2e_sims = args.steps * n_total / (ms_e2e * 1e-3)
    real = 4 if dt_name == "f32" else 8
    k_local = len(out_h[1])
    d2h = k_local * (8 + 3 * real + real) + 8
    h2d = obs.nbytes + 256

    line = {
        "metric": "prior-predictive sims/sec (logistic SDE ABC rejection)",
        "value": sims_per_s, "unit": "sims/s", "sde_steps_per_s": sims_per_s * STEPS_PER_SIM,
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": dt_name, "data": "synthetic",
        "config": {"workload": f"config1: logistic-SDE ABC rejection, N={n_total:.0e} particles/step, "
                               f"fixed epsilon from config0, {args.variant}",
                   "particles_per_step": n_total, "sde_steps_per_particle": STEPS_PER_SIM,
                   "epsilon": eps, "accepted_per_step": n_acc, "variant": args.variant,
                   "sharding": f"particles/{world}", "exchange": comm_note,
                   "philox4x32_rounds": int(lib.load().vxb_fast_generator_rounds()),
                   "l2": "no reusable input (compute-bound); per-step rho scratch "
                         f"{(end - begin) * real / 1e6:.0f} MB exceeds L2"},
        "e2e": {"value": e2e_sims, "unit": "sims/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "ms_per_step": ms_e2e / args.steps},
        "gpu_launches": int(round(total_launches * timed_fraction)),
        "roofline": {"bound": f"{dt_name}-pipe", "achieved": achieved, "peak": peak_meas,
                     "unit": "TFLOP/s", "frac": achieved / peak_meas,
                     "peak_nominal": NOMINAL_PEAK[dt_name],
                     "frac_of_nominal": achieved / NOMINAL_PEAK[dt_name],
                     "peak_source": "measured FMA-chain probe (vxb_fma_peak) on this GPU; "
                                    "MEASURED_PEAKS.json has no fp64/fp32 entry",
                     "kernel": "logistic_abc_kernel", "kernel_ms": kernel_ms,
                     "flops_per_sim": FLOPS_PER_SIM, **ncu_traffic(args.variant)},
        "clocks": clocks.summary(),
        "device": info["name"],
    }

    if not args.no_extras:
        variants = {}
        for name in ("f64_fast", "f64_ref", "f32_fast"):
            if name == args.variant:
                variants[name] = {"sims_per_s": sims_per_s, "ms_per_step": ms / args.steps}
                continue
            w, k = min(args.warmup, 2), min(args.steps, 3)
            ms_v, _ = timed(device_step(logistic_variant(name)), w, k)
            pk = NOMINAL_PEAK["f32" if name.startswith("f32") else "f64"]
            sv = k * n_total / (ms_v * 1e-3)
            variants[name] = {"sims_per_s": sv, "ms_per_step": ms_v / k, "steps": k, "warmup": w,
                              "frac_of_nominal_peak": sv * FLOPS_PER_SIM / 1e12 / pk}
        for name, v in variants.items():
            # the hardware's own view next to the flop-convention fraction (ncu capture)
            v.update({k: x for k, x in ncu_traffic(name).items() if k.endswith("_ncu")})
            v["frac_note"] = ("algorithmic flops at the reference's price of 47 per N(0,1) "
                              "(SURVEY.md 8d) over the nominal pipe peak; *_ncu = measured pipe "
                              "utilisation of the same kernel")
        line["variants"] = variants
        if rank == 0 and world == 1:
            # the contract's CPU figure first; everything after it is additional evidence and
            # must never cost the line
            line["cpu_baseline"] = cpu_baseline(args, obs, eps)
            try:
                line["configs"] = all_configs(ctx, timed, obs, local)
                cpu_configs(line["configs"], obs)
            except Exception as e:
                line["configs_error"] = f"{type(e).__name__}: {e}"
            line["opt_in_philox7"] = philox7_arm(args)
            # ---- opt-in early rejection (VXB_OPT_EARLY_REJECT): same job, same accepted set;
            # rows stop once they can no longer be accepted.  NOT the headline: `value`, `e2e`
            # and `roofline` above simulate every row to the end
            def early_arm(name):
                step = device_step(logistic_variant(name))
                with torch.cuda.stream(ext):
                    full = [t.clone() for t in step(99)]
                ctx.set_early_reject(True)
                try:
                    ms_e, _ = timed(step, 1, 3)
                    with torch.cuda.stream(ext):
                        got = step(99)
                    ctx.synchronize()
                finally:
                    ctx.set_early_reject(False)
                k = int(full[3].sum().item())
                same = k == int(got[3].sum().item()) and all(torch.equal(a[:k], b[:k])
                                                             for a, b in zip(full[:3], got[:3]))
                return {"sims_per_s": 3 * n_total / (ms_e * 1e-3), "ms_per_step": ms_e / 3,
                        "speedup_vs_full": variants[name]["ms_per_step"] / (ms_e / 3),
                        "accepted": k, "identical_accepted_set": bool(same)}

            early = {}
            for name in ("f64_fast", "f64_ref", "f32_fast"):
                try:
                    early[name] = early_arm(name)
                except Exception as e:
                    early[name] = {"error": f"{type(e).__name__}: {e}"}
            early["note"] = ("vxb_set_option(VXB_OPT_EARLY_REJECT): a row stops when its partial squared distance "
                             "exceeds epsilon^2; survivors are re-packed between up to six segment launches; "
                             "accepted indices, parameters and distances bit-identical to the full simulation")
            line["opt_in_early_reject"] = early
    if rank == 0:
        print(json.dumps(line), flush=True)
    if comm is not None:
        comm.close()
    ctx.close()
    if dist_on:
        dist.destroy_process_group()


def all_configs(ctx, timed, obs, device):
    """Every other workload at full size, one JSON object each: CUDA-event time per
    pass (W >= 1 warm-up, K >= 3 timed passes, enough of them to give the clock sampler a
    window), units/s, the algorithmic flop rate under SURVEY.md 8(d)'s prices against
    the nominal FP64 peak, and the NVML clock summary of that timed region."""
    import torch
    from paper_1902_09046_b200 import _abi as A, bench_harness as B, lib, models as M
    peak = NOMINAL_PEAK["f64"] * 1e12
    res = {}

    def run(name, fn, units, unit, flops_per_unit=None, target_s=0.6, extra=None, pipe="f64"):
        # calibrate the repetition count on one untimed pass (which is also a warm-up)
        ms1, _ = timed(lambda s: fn(), 1, 1)
        k = max(3, min(200, int(math.ceil(target_s * 1e3 / max(ms1, 1e-3)))))
        with ClockSampler(device, period=0.05) as clocks:
            ms, out = timed(lambda s: fn(), 1, k)
        per = ms / k
        e = {"ms": per, "passes": k, "units": units, "unit": unit,
             "units_per_s": units / (per * 1e-3), "clocks": clocks.summary()}
        if flops_per_unit:
            e["flops_per_unit"] = flops_per_unit
            e["tflops_algorithmic"] = units * flops_per_unit / (per * 1e-3) / 1e12
            e[f"frac_of_nominal_fp{pipe[1:]}"] = (units * flops_per_unit / (per * 1e-3) /
                                                  (NOMINAL_PEAK[pipe] * 1e12))
        if extra:
            e.update(extra(out))
        res[name] = e
        return out

    m = M.logistic_model()
    # ---- config 0: N = 1e6, reference-exact streams, accept the 0.1% nearest
    n0 = 1_000_000
    rho = torch.empty(n0, dtype=torch.float64, device=f"cuda:{device}")
    failed = torch.empty(n0, dtype=torch.uint8, device=f"cuda:{device}")

    def c0(model):
        def fn():
            ctx.abc_prior_predictive(model, M.keying(1337), n0, 0, n0, obs, rho=rho, failed=failed)
            return ctx.select_epsilon(rho, failed, 1e-3, cap=2000, precision=A.VXB_F64, n=n0)
        return fn
    run("config0_exact", c0(m), n0, "sims", FLOPS_PER_SIM,
        extra=lambda o: {"epsilon": o[0], "accepted": o[2]})
    run("config0_fast", c0(M.logistic_model(rng=A.VXB_RNG_FAST)), n0, "sims", FLOPS_PER_SIM,
        extra=lambda o: {"epsilon": o[0], "accepted": o[2]})

    # ---- config 2: 64 lambdas x 1e6 datasets x n = 100
    nl, mt, nd = 64, 1_000_000, 100
    lam = np.array(M.lambda_grid(nl))
    ln = np.array([-0.5 * math.log(2.0 * math.pi * (l * l + 1.0 / nd)) for l in lam])
    ybar = float((3.0 + ctx.rng_fill_gaussian(lib.derive_seed(2, [90]), 0, 0, nd)).mean())
    exact_p = np.array([math.erfc(abs(ybar) / math.sqrt(2.0 * (l * l + 1.0 / nd))) for l in lam])
    for name, rng in (("config2_exact", A.VXB_RNG_REF), ("config2_fast", A.VXB_RNG_FAST)):
        mdl = M.normal_mean_model(nd, rng=rng)
        run(name, lambda mdl=mdl: ctx.ppp_pvalues(mdl, lam, ln, mt, 0, mt, 1337, ybar), nl * mt,
            "datasets", 4960,
            extra=lambda o: {"max_abs_err_vs_closed_form": float(np.abs(o[1] - exact_p).max()),
                             "mc_standard_error_bound": 5e-4})

    # ---- config 3: ABC-SMC, N = 1e5 x 10 generations
    cfg = A.vxb_abcsmc_cfg()
    cfg.particles, cfg.generations = 100_000, 10
    cfg.quantile, cfg.kernel_scale, cfg.jitter, cfg.round_size, cfg.max_rounds, cfg.seed = 0.5, 2.0, 1e-10, 0, 0, 1337
    for name, mdl in (("config3_exact", m), ("config3_fast", M.logistic_model(rng=A.VXB_RNG_FAST))):
        run(name, lambda mdl=mdl: ctx.abcsmc_run(mdl, cfg, obs), cfg.particles * cfg.generations,
            "particle-generations", target_s=1.0,
            extra=lambda o: {"proposals_simulated_upper_bound": int(o["proposals"].sum()),
                             "epsilon_last": float(o["epsilon"][-1]), "ess_last": float(o["ess"][-1]),
                             "weight_pairs": int(cfg.particles) ** 2 * (cfg.generations - 1)})
    # the SPMD multi-GPU driver (vxb_sharded_abcsmc_run) as ONE rank: same bits, rounds
    # issued ahead of the host with the state on the device
    run("config3_fast_spmd_driver_1rank",
        lambda: ctx.sharded_abcsmc_run(None, M.logistic_model(rng=A.VXB_RNG_FAST), cfg, obs),
        cfg.particles * cfg.generations, "particle-generations", target_s=0.6,
        extra=lambda o: {"epsilon_last": float(o["epsilon"][-1]), "rounds_total": int(o["proposals"].sum() // cfg.particles)})
    for name in ("config3_exact", "config3_fast"):
        # flop rate: every proposal priced as a simulation (an upper bound: proposals
        # outside the prior box are not simulated) + 50 flop per importance-weight pair
        e = res[name]
        fl = e["proposals_simulated_upper_bound"] * FLOPS_PER_SIM + e["weight_pairs"] * 50
        e["tflops_algorithmic_upper_bound"] = fl / (e["ms"] * 1e-3) / 1e12
        e["frac_of_nominal_fp64_upper_bound"] = fl / (e["ms"] * 1e-3) / peak

    # ---- config 4: MLMC tau-leap, 6 levels x 1e6 paths
    mc = A.vxb_mlmc_cfg()
    mc.levels, mc.refine, mc.tau0, mc.t_end, mc.paths, mc.seed = 6, 4, 1.0, 30.0, 1_000_000, 1337
    fine = [30 * 4 ** l for l in range(6)]
    steps = mc.paths * sum(f if l == 0 else f + f // 4 for l, f in enumerate(fine))
    flops = mc.paths * (fine[0] * 130 + sum(f * 370 for f in fine[1:]))
    for name, rng, prec in (("config4_exact", A.VXB_RNG_REF, A.VXB_F64), ("config4_fast", A.VXB_RNG_FAST, A.VXB_F64),
                            ("config4_fast_f32", A.VXB_RNG_FAST, A.VXB_F32)):
        mm = M.mm_tauleap_model(rng=rng, precision=prec)
        run(name, lambda mm=mm: ctx.mlmc_tauleap(mm, mc), steps, "path-steps", flops / steps,
            target_s=1.5, extra=lambda o: {"estimate": o["estimate"], "std_error": o["std_error"]},
            pipe="f32" if prec == A.VXB_F32 else "f64")
        # SURVEY 8(d) prices an exp per Poisson draw (370 flop per coupled fine step); the
        # kernels decide a draw of zero from 1 - lam on the raw bits, so the flop rate under
        # that convention is a work-equivalent, not a pipe utilisation (it can exceed 1):
        # path-steps/s is the number for this config
        e = res[name]
        for k in ("frac_of_nominal_fp64", "frac_of_nominal_fp32"):
            if k in e:
                e[k + "_survey_convention"] = e.pop(k)
        e["tflops_survey_convention"] = e.pop("tflops_algorithmic")

    # ---- the paper's toggle-switch ABC: N = 8064, C = 8000, T = 600
    n_t, c_t, t_t = 8064, 8000, 600
    tm = M.toggle_model(t_t, c_t)
    tobs = ctx.simulate_at(tm, M.TOGGLE_MIDPOINT, lib.derive_seed(1337, [90]), 0, 0)
    trho = torch.empty(n_t, dtype=torch.float64, device=f"cuda:{device}")
    cell_steps = n_t * c_t * (t_t - 1)
    run("toggle_exact", lambda: ctx.abc_prior_predictive(tm, M.keying(1337, A.VXB_KEY_WORKER, 16, 4),
                                                         n_t, 0, n_t, tobs, rho=trho),
        cell_steps, "cell-steps", 228, target_s=2.0, extra=lambda o: {"published_best_s": 69.0})
    tmf = M.toggle_model(t_t, c_t, rng=A.VXB_RNG_FAST)
    run("toggle_fast", lambda: ctx.abc_prior_predictive(tmf, M.keying(1337), n_t, 0, n_t, tobs, rho=trho),
        cell_steps, "cell-steps", 228, target_s=1.0, extra=lambda o: {"published_best_s": 69.0})

    # ---- the paper's weak-informativity test: K = N = 400, N_p = 500
    for name, kw in (("weakinfo_exact", {}), ("weakinfo_fast", {"rng": A.VXB_RNG_FAST})):
        wcfg = M.weakinfo_config(hyper_count=400, datasets=400, particles=500, seed=1337, **kw)
        run(name, lambda wcfg=wcfg: ctx.weak_info_test(wcfg), 2 * 401 * 400, "sampler-runs",
            target_s=1.0, extra=lambda o: {"weakly_informative": int(o["weakly"].sum()),
                                           "published_best_s": 90.0})

    # ---- TB Gillespie ABC at the reference's bench sizes (bench.hpp:39-42), 1e6 rows
    n_tb = 1_000_000
    tbm = M.tb_model(10, 10.0, 10000.0)
    tb_obs = B.tb_observed_summaries(ctx, 10, 10.0, 10000.0, 1337, 4)
    tb_rho = torch.empty(n_tb, dtype=torch.float64, device=f"cuda:{device}")
    tb_failed = torch.empty(n_tb, dtype=torch.uint8, device=f"cuda:{device}")
    run("tb_gillespie", lambda: ctx.abc_prior_predictive(tbm, M.keying(1337), n_tb, 0, n_tb, tb_obs,
                                                        rho=tb_rho, failed=tb_failed),
        n_tb, "rows", target_s=3.0)

    # ---- smc::resample_multinomial at N = 1e5, d = 3 (reference: 17.8 ms, smc.cpp:268-300)
    rs = np.random.RandomState(9)
    n_r = 100_000
    lw = torch.from_numpy(rs.normal(size=n_r) * 3).to(f"cuda:{device}")
    parts = torch.from_numpy(rs.normal(size=(n_r, 3))).to(f"cuda:{device}")
    r_out = torch.empty_like(parts)
    r_anc = torch.empty(n_r, dtype=torch.int64, device=f"cuda:{device}")

    def resample():
        ctx._check(ctx.lib.vxb_resample_multinomial(
            ctx.handle, lib.u64(n_r), lib.u32(3), lib._ptr(lw), lib._ptr(parts), lib.u64(77),
            lib.u32(9), lib._ptr(r_out), lib._ptr(r_anc)))
    run("resample_multinomial_1e5", resample, n_r, "particles", target_s=0.3,
        extra=lambda o: {"reference_cpu_ms": 17.8,
                         "note": "bit-exact: host-libm exp + strictly sequential running sum "
                                 "(one dependent DADD per particle)"})
    return res


def cpu_configs(configs, obs):
    """The CPU path of every workload on this box's host cores, on a BOUNDED sample each
    (2-5 s of CPU work; the sample is stated), attached to the matching `configs` entries:
    the unmodified reference (oracle/_ref) where it has the code -- the ABC sampler on
    the logistic hooks + select_epsilon, toggle ABC, the weak-informativity test, TB ABC,
    resample_multinomial -- and this repository's CPU restatement (oracle port) for the
    workloads the reference lacks (configs 2, 3, 4).  Reported baselines, not targets."""
    from oracle.pyoracle import Oracle, Ref
    from paper_1902_09046_b200 import _abi as A, models as M
    cores = os.cpu_count() or 1
    o = Oracle(threads=cores)
    r = Ref() if Ref.available() else None

    def attach(names, kind, sample, units, seconds, unit):
        for name in names:
            if name in configs:
                cpu_rate = units / seconds
                configs[name]["cpu"] = {"kind": kind, "cores": cores, "sample": sample,
                                        "seconds": seconds, "units_per_s": cpu_rate, "unit": unit,
                                        "gpu_over_cpu": configs[name]["units_per_s"] / cpu_rate}

    def clock(fn):
        t0 = time.perf_counter()
        out = fn()
        return out, time.perf_counter() - t0

    m = M.logistic_model()
    try:
        # config 0 on 3e5 of its 1e6 rows: prior-predictive set + select_epsilon
        n0 = 300_000
        if r is not None:
            (_, dt) = clock(lambda: r.select_epsilon(*r.logistic_abc(m, n0, cores, 1, 1337, obs)[2:4], 1e-3))
            kind = "reference"
        else:
            (_, dt) = clock(lambda: o.select_epsilon(*o.abc_prior_predictive(m, M.keying(1337), n0, 0, n0, obs)[2:4], 1e-3))
            kind = "port"
        attach(("config0_exact", "config0_fast"), kind, "3e5 of 1e6 sims + select_epsilon over them", n0, dt, "sims")
        # config 2: 64 lambdas x 1e5 of the 1e6 datasets
        nl, mt, nd = 64, 100_000, 100
        lam = np.array(M.lambda_grid(nl))
        ln = np.array([-0.5 * math.log(2.0 * math.pi * (l * l + 1.0 / nd)) for l in lam])
        (_, dt) = clock(lambda: o.ppp_pvalues(M.normal_mean_model(nd), lam, ln, mt, 0, mt, 1337, 2.9))
        attach(("config2_exact", "config2_fast"), "port", "64 lambdas x 1e5 of 1e6 datasets", nl * mt, dt, "datasets")
        # config 3: N = 5e3 x 10 generations (the weights are O(N^2): not a linear sample)
        cfg = A.vxb_abcsmc_cfg()
        cfg.particles, cfg.generations = 5_000, 10
        cfg.quantile, cfg.kernel_scale, cfg.jitter, cfg.round_size, cfg.max_rounds, cfg.seed = 0.5, 2.0, 1e-10, 0, 0, 1337
        (_, dt) = clock(lambda: o.abcsmc_run(m, cfg, obs))
        for name in ("config3_exact", "config3_fast"):
            if name in configs:
                configs[name]["cpu"] = {"kind": "port", "cores": cores, "seconds": dt,
                                        "sample": "N = 5e3 x 10 generations (1/20 of the particles, 1/400 "
                                                  "of the weight pairs): not comparable unit for unit"}
        # config 4: 6 levels x 2e3 of the 1e6 paths
        mc = A.vxb_mlmc_cfg()
        mc.levels, mc.refine, mc.tau0, mc.t_end, mc.paths, mc.seed = 6, 4, 1.0, 30.0, 2_000, 1337
        fine = [30 * 4 ** l for l in range(6)]
        steps = mc.paths * sum(f if l == 0 else f + f // 4 for l, f in enumerate(fine))
        (_, dt) = clock(lambda: o.mlmc_tauleap(M.mm_tauleap_model(), mc))
        attach(("config4_exact", "config4_fast", "config4_fast_f32"), "port", "6 levels x 2e3 of 1e6 paths", steps, dt,
               "path-steps")
        if r is not None:
            # toggle ABC: 32 of the 8064 samples at the paper's C = 8000, T = 600
            n_t = 32
            (_, dt) = clock(lambda: r.toggle_abc(600, 8000, n_t, cores, 4, 1337))
            attach(("toggle_exact", "toggle_fast"), "reference", "32 of 8064 samples (C = 8000, T = 600)",
                   n_t * 8000 * 599, dt, "cell-steps")
            # weak-informativity test: K = 10, N = 40 (880 of the 320 800 sampler runs)
            (_, dt) = clock(lambda: r.weak_info_test(10, 40, 500, workers=cores, seed=1337))
            attach(("weakinfo_exact", "weakinfo_fast"), "reference", "K = 10, N = 40: 880 of 320 800 sampler runs",
                   2 * 11 * 40, dt, "sampler-runs")
            # TB Gillespie ABC: 4096 of the 1e6 rows
            tb_obs = r.tb_observed(10, 10.0, 10000.0, 1337)
            (_, dt) = clock(lambda: r.tb_abc_particle(10, 10.0, 10000.0, 0, 4096, 1337, tb_obs))
            attach(("tb_gillespie",), "reference", "4096 of 1e6 rows", 4096, dt, "rows")
            # resample_multinomial, full size, single thread (as the reference runs it)
            rs = np.random.RandomState(9)
            lw, parts = rs.normal(size=100_000) * 3, rs.normal(size=(100_000, 3))
            r.resample_multinomial(lw, parts, 77, 9)
            (_, dt) = clock(lambda: [r.resample_multinomial(lw, parts, 77, 9) for _ in range(5)])
            attach(("resample_multinomial_1e5",), "reference", "full size, one thread, mean of 5 calls", 100_000, dt / 5, "particles")
            configs["resample_multinomial_1e5"]["cpu"]["cores"] = 1
    except Exception as e:   # a CPU figure must never cost the line
        configs["cpu_error"] = repr(e)


def philox7_arm(args):
    """The documented opt-in build (Philox4x32-7 throughput generator, build.py --rounds7)
    through this same script in a subprocess, so that its number sits under the same
    clock sampler: headline value, kernel fraction, clocks.  Not the product default."""
    from paper_1902_09046_b200 import build
    if not os.path.exists(build.LIB_ROUNDS7) or os.environ.get("VXB_LIBRARY"):
        return None
    try:
        run = subprocess.run([sys.executable, os.path.abspath(__file__), "--gpus", "1", "--steps", "3",
                              "--warmup", "3", "--no-extras", "--particles", str(args.particles)],
                             capture_output=True, text=True, timeout=300,
                             env=dict(os.environ, VXB_LIBRARY=build.LIB_ROUNDS7))
        b = json.loads([l for l in run.stdout.splitlines() if l.startswith("{")][-1])
        return {"philox4x32_rounds": b["config"]["philox4x32_rounds"], "value": b["value"], "unit": b["unit"],
                "ms_per_step": b["ms_per_step"], "e2e": b["e2e"]["value"],
                "frac_of_nominal": b["roofline"]["frac_of_nominal"], "clocks": b["clocks"],
                "accepted_per_step": b["config"]["accepted_per_step"],
                "note": "opt-in build, statistics in profiles/r2_philox7.json; the product library runs 10 rounds"}
    except Exception as e:  # the opt-in arm must never cost the main line
        return {"error": repr(e)}


def cpu_baseline(args, obs, eps):
    """The reference CPU path on this box's host cores, bounded sample (rank 0, N=1)."""
    from oracle.pyoracle import Oracle, Ref
    from paper_1902_09046_b200 import models as M
    cores = os.cpu_count() or 1
    m = M.logistic_model()
    sample = int(args.cpu_sample)
    use_ref = Ref.available()
    o = Ref() if use_ref else Oracle(threads=cores)

    def step(s):
        if use_ref:
            return o.logistic_abc(m, sample, cores, 1, 1337 + s, obs)
        return o.abc_prior_predictive(m, M.keying(1337 + s), sample, 0, sample, obs)

    step(0)  # one discarded warm-up, then 3 replicates (bench.cpp:140-172 protocol)
    t0 = time.perf_counter()
    for s in range(3):
        p, summ, rho, f = step(1 + s)
        int(((rho <= eps) & (f == 0)).sum())
    dt = (time.perf_counter() - t0) / 3
    return {"value": sample / dt, "unit": "sims/s", "cores": cores,
            "kind": "reference" if use_ref else "port",
            "sample": f"{sample} particles (of the 1e8-particle job; scales linearly), "
                      f"{cores} std::thread workers"}


if __name__ == "__main__":
    main()
