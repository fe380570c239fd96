#!/usr/bin/env python
"""Benchmark: grid-node updates/s (forward sweep + adjoint) on the 4096^2
Randers fp64 workload (BASELINE.json configs[2], the metric's own config).

One step = one forward solve + loss gradient + backward (identify stencils,
adjoint, parameter gradients) of one 4096^2 grid, inputs resident in HBM.
Work unit: W = 4 K (N^2 - |S|) + n_records node-updates,
K = the solve's iteration count (identical to the reference's by parity).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N > 1 is launched by torchrun: every rank solves its own grid (independent
scenes, "weak" scaling, no data-path collective); time = max over ranks.
--impl reference times the reference's own CPU implementation (oracle/_ref,
compiled from /root/reference's sources) on all host cores, on the same C3
fields: one strip of rows per thread, two iterations of the reference solve
per step (reference_arm).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "grid-node updates/s (fwd sweep + adjoint) at 4096² Randers fp64; % HBM roofline"
UNIT = "node-updates/s"
BYTES_FWD = 56.0   # G 24 + b 16 + T read 8 + T write 8 per forward node-update
BYTES_BWD = 96.0   # per adjoint node: T, G, b, dL/dT read + 5 gradients written


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=3)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--n", "--grid", dest="n", type=int, default=4096,
                   help="grid size (default: the metric's 4096); spell it --grid under torchrun, whose parser "
                        "takes --n as an abbreviation of its own options")
    p.add_argument("--drift", type=float, default=0.2)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--cpu-n", type=int, default=1024, help="grid of the bounded CPU sample")
    p.add_argument("--workload", default="c3", choices=["c3", "c4", "c5"],
                   help="c3: the metric's single 4096^2 grid (default); c4: the batched inverse "
                        "config, 64 scenes of 2048^2 sharded over the ranks; c5: the training config, "
                        "256 samples of 1024^2 through encoder -> projection -> solve, DDP over the "
                        "ranks (c4/c5 print informational lines)")
    p.add_argument("--scenes", type=int, default=None, help="c4/c5: scenes (samples) in the whole job "
                                                              "(default 64 / 256)")
    p.add_argument("--encoder", default="bf16", choices=["fp32", "bf16"],
                   help="c5: encoder arithmetic (bf16 autocast + channels-last, or fp32); the solver is fp64")
    p.add_argument("--chunk", type=int, default=8, help="c4/c5: scenes per batched call (micro-batch)")
    p.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                   help="process-group backend for N>1 (gloo: CPU-side collectives, lets several ranks share one "
                        "GPU in tests; ranks then map to GPUs round-robin)")
    return p.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.device), "--query-gpu=" + self.Q,
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.rows.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 3 + i and "Active" in r[3 + i]
                          and r[3 + i].strip().lower() not in ("not active",)})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def load_fp64_peak():
    """Measured FP64 pipe peak on this pool's B200 (scripts/ubench/fp64_peak.cu,
    profiles/r02_fp64_peak.json): DADD/DMUL thread-ops per second."""
    try:
        with open(os.path.join(ROOT, "profiles", "r02_fp64_peak.json")) as f:
            d = json.load(f)
        return max(float(d["dadd_tops"]), float(d["dmul_tops"])) * 1e12, "measured (scripts/ubench/fp64_peak.cu)"
    except Exception:
        return 148 * 64 * 1.965e9, "nominal 148 SMs x 64 lanes x 1.965 GHz"


def load_traffic():
    """dram bytes per sweep launch from the committed ncu capture, if any."""
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return d.get("sweep_dram_bytes_per_launch"), d.get("sweep_launch_n"), d.get("sweep_algorithmic_bytes")
    except Exception:
        return None, None, None


def load_fp64_inst():
    """FP64 work per sweep launch at C3 from the committed ncu counts
    (profiles/ncu_summary.json "sweep_fp64_counts", captured with --metrics
    on scripts/prof_solve.py 4096): executed DADD + DMUL + DFMA thread
    instructions (predicated-on lanes only), and the FP64-pipe warp
    instructions."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
            d = json.load(f)
        c = d["sweep_fp64_counts"]
        thread = sum(float(c[f"sm__sass_thread_inst_executed_op_{op}_pred_on.sum"]) for op in ("dadd", "dmul", "dfma"))
        return thread, float(c["smsp__inst_executed_pipe_fp64.sum"])
    except Exception:
        return None, None


def load_c3_reference():
    """The reference library's own C3 forward + adjoint at the stated config
    (4096^2, the bench's inputs), timed once on a GPU box's host
    (scripts/cpu_c3_reference.py -> profiles/r02_cpu_c3_reference.json)."""
    try:
        with open(os.path.join(ROOT, "profiles", "r02_cpu_c3_reference.json")) as f:
            return json.load(f)
    except Exception:
        return None


# ---------------------------------------------------------------------------
def cpu_baseline(cpu_n: int, drift: float):
    """Bounded sample of the same workload on 1 host core through the
    reference library itself (oracle/_ref), else the C port (oracle/)."""
    import numpy as np

    from paper_2603_00035_b200 import workload as wl
    F = wl.host_fields(cpu_n, 1, drift)
    src = wl.host_point_source(cpu_n, cpu_n)
    obs = wl.host_observation_mask(src)
    vals = np.zeros((cpu_n, cpu_n))
    h = 1.0 / cpu_n
    try:
        from oracle.pyoracle import RefLib
        R = RefLib()
        wall, times, K, nrec, conv = R.pipeline(*F, src, obs, vals, h, 1e-6, 50, 1, 1)
        kind = "reference"
    except Exception:
        from oracle.pyoracle import Oracle
        O = Oracle()
        t0 = time.time()
        times, K, nrec = O.pipeline(*F, src, obs, vals, h, 1e-6, 50)
        wall = time.time() - t0
        kind = "port"
    W = wl.node_updates(K, cpu_n * cpu_n, 1, nrec)
    return {"value": W / wall, "unit": UNIT, "cores": 1, "kind": kind, "host": host_cpu(),
            "sample": f"{cpu_n}x{cpu_n} Randers (same recipe), one forward+adjoint solve, K={K}, "
                      f"{W} node-updates in {wall:.1f} s on 1 core (reference is single-threaded)"}


def cpu_batch_baseline(n: int, drift: float, tag: str):
    """SURVEY §8d for the batched configs: `nproc` independent problems run
    concurrently through the reference library (one std::thread each), on a
    bounded sample (n x n problems); aggregate node-updates/s."""
    import numpy as np

    from oracle.pyoracle import RefLib
    from paper_2603_00035_b200 import workload as wl
    R = RefLib()
    F = R.random_feasible_fields(n, 1, drift)
    src = np.zeros((n, n), np.uint8)
    src[n // 2, n // 2] = 1
    obs = R.observation_mask(src, 2024, 0.3)
    threads = os.cpu_count() or 1
    wall, times, K, nrec, conv = R.pipeline(*F, src, obs, np.zeros((n, n)), 1.0 / n, 1e-6, 50, threads, threads)
    W = wl.node_updates(K, n * n, 1, nrec) * threads
    return {"value": W / wall, "unit": UNIT, "cores": threads, "kind": "reference", "host": host_cpu(),
            "sample": f"{tag}: {threads} concurrent {n}x{n} Randers forward+adjoint problems (one per thread, "
                      f"K={K}) through the reference library, {wall:.1f} s"}


def host_cpu():
    """nproc and the CPU model of the host the CPU numbers ran on."""
    model = "unknown"
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"nproc": os.cpu_count(), "model": model}


def reference_arm(args, rank, world):
    """--impl reference: the reference's own CPU path on all host threads, on
    this arm's config (C3: the 4096^2 fields of workload.host_fields(n, 1,
    drift), the bench's own inputs), each step a bounded sample of it.

    One reference solve of the whole C3 grid takes ~330 s on one core, so a
    step cannot be a solve.  The sample: the C3 fields cut into one strip of
    rows per host thread (the strips tile the grid), a point source at each
    strip's centre, and per step every thread runs the reference `solve` on
    its strip for two iterations (max_iters = 2, the C3 tol) -- all threads
    concurrently.  The strips keep the C3 row width, so row and column passes
    walk memory with the C3 grid's strides.  Forward node updates only (the
    adjoint is ~3% of the reference's C3 time, profiles/r02_cpu_c3_reference
    .json); W = 4 * iterations * strip nodes, summed over the strips."""
    if rank != 0:
        return
    import numpy as np

    from paper_2603_00035_b200 import workload as wl
    try:
        from oracle.pyoracle import RefLib
        R = RefLib()
    except Exception as exc:
        print(json.dumps({"impl": "reference", "unavailable": f"oracle/_ref not built ({exc})"}), flush=True)
        return
    n = args.n
    nthreads = max(1, min(os.cpu_count() or 1, n // 8))
    F = wl.host_fields(n, 1, args.drift)
    bounds = [(n * i) // nthreads for i in range(nthreads + 1)]
    rows = max(bounds[i + 1] - bounds[i] for i in range(nthreads))
    # equal strip heights (the last strips repeat rows when n % threads != 0)
    starts = [min(bounds[i], n - rows) for i in range(nthreads)]
    planes = [np.stack([f[r0:r0 + rows] for r0 in starts]) for f in F]
    src = np.zeros((nthreads, rows, n), np.uint8)
    src[:, rows // 2, n // 2] = 1
    h = 1.0 / n
    its_per_step = 2
    rates = []
    K = None
    for step in range(args.warmup + args.steps):
        wall, its = R.solve_batch(*planes, src, h, 1e-6, its_per_step)
        K = its
        W = 4 * int(np.sum(its)) * rows * n
        if step >= args.warmup:
            rates.append((W, wall))
    Wt = sum(w for w, _ in rates)
    Tt = sum(t for _, t in rates)
    value = Wt / Tt
    sample = (f"each step: the C3 fields (workload.host_fields({n}, 1, {args.drift})) cut into {nthreads} strips of "
              f"{rows}x{n} (one per host thread, tiling the grid), a point source at each strip's centre, the "
              f"reference library's solve run {its_per_step} iterations on every strip concurrently "
              f"(iterations {sorted(set(int(k) for k in K))}); forward node-updates only")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * Tt / max(1, len(rates)),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (deterministic host-generated correlated-noise Randers fields, projected)",
        "config": {"workload": f"C3: full Randers metric with drift, {n}x{n}, forward + adjoint, fp64",
                   "grid": f"{n}x{n}", "sample": f"{nthreads} strips of {rows}x{n}, {its_per_step} iterations "
                                                 f"each per step", "threads": nthreads},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": nthreads, "kind": "reference", "host": host_cpu(),
                         "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    c3 = load_c3_reference()
    if c3:
        line["c3_full"] = {k: c3[k] for k in ("grid", "K", "seconds", "node_updates_per_s", "cores", "how")
                           if k in c3}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
def c4_main(args, rank, world, local):
    """BASELINE.json configs[3]: `scenes` independent 2048^2
    Randers scenes (own metric per scene, seed = scene index), sharded by
    scene over the ranks (sharding.shard_range; no data-path collective).
    One step = every scene of the rank once through the data term of
    objective_and_grad: batched solve (concurrent grid slots) -> loss
    gradient -> fused backward, `chunk` scenes per call, inputs resident."""
    import numpy as np
    import torch

    local = local % torch.cuda.device_count()  # gloo tests: several ranks on one GPU
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group("gloo")
    import paper_2603_00035_b200 as rfk
    from paper_2603_00035_b200 import workload as wl
    from paper_2603_00035_b200.sharding import shard_range

    n = 2048 if args.n == 4096 else args.n
    h = 1.0 / n
    scenes = args.scenes or 64
    lo, hi = shard_range(scenes, rank, world)
    ctx = rfk.Context(local)
    stream = torch.cuda.current_stream(dev)
    ctx.set_stream(stream.cuda_stream)
    # per scene s a truth field (seed s) observed through
    # generate_observations(density 0.07, noise 0, seed s) (inversion.cpp:
    # 387-437), and the current estimate (another field, seed 1000 + s) at
    # which one objective_and_grad data term is evaluated per step
    chunks = []
    for c0 in range(lo, hi, args.chunk):
        ids = list(range(c0, min(hi, c0 + args.chunk)))
        src1 = wl.point_source(n, n, device=dev)
        obs_l, val_l = [], []
        for s_id in ids:
            truth = wl.randers_fields(n, s_id, args.drift, device=dev)
            o, v = rfk.generate_observations(*truth, src1, h, 0.07, 0.0, s_id, ctx=ctx)
            obs_l.append(o[0])
            val_l.append(v[0])
        per = [wl.randers_fields(n, 1000 + s_id, args.drift, device=dev) for s_id in ids]
        F = [torch.stack([p[i] for p in per]) for i in range(5)]
        src = src1.expand(len(ids), n, n).contiguous()
        obs = torch.stack(obs_l)
        vals = torch.stack(val_l)
        chunks.append((F, src, obs, vals))
    torch.cuda.synchronize()
    out = {}

    def step():
        for i, (F, src, obs, vals) in enumerate(chunks):
            t, rep = rfk.solve(*F, src, h, ctx=ctx)
            g, loss, unr = rfk.loss_grad_mse(t, obs, vals, exact=False, ctx=ctx)
            lam, grads, cl = rfk.backward(t, *F, src, h, g, want_lambda=False, ctx=ctx)
            out[i] = (t, rep)

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    W_rank = 0
    for i, (F, src, obs, vals) in enumerate(chunks):
        t, rep = out[i]
        its = np.atleast_1d(np.asarray(rep.iterations))
        nrec = ((t < 1e9) & (src == 0)).flatten(1).sum(1).cpu().numpy()
        W_rank += sum(wl.node_updates(int(k), n * n, 1, int(r)) for k, r in zip(its, nrec))
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    launches0 = ctx.launches
    with ClockSampler(local) as clk:
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
    t_ms = e0.elapsed_time(e1)
    launches = ctx.launches - launches0
    W_job = W_rank
    if world > 1:
        from paper_2603_00035_b200.sharding import reduce_step_stats
        t_ms, W_job = reduce_step_stats(t_ms, float(W_rank))
    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        try:
            cpu = cpu_batch_baseline(512, args.drift, "C4")
        except Exception as exc:
            cpu = {"value": None, "sample": f"failed: {exc}"}
    if rank == 0:
        line = {
            "metric": "grid-node updates/s (fwd sweep + adjoint), C4 batch of 2048² Randers fp64 scenes",
            "value": W_job * args.steps / (t_ms / 1e3), "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (device-generated correlated-noise Randers fields per scene, projected); "
                    "observations from generate_observations(density 0.07, noise 0) of a truth field",
            "cpu_baseline": cpu,
            "config": {"workload": f"C4: {scenes} scenes of {n}x{n}, one objective_and_grad data term per scene "
                                   f"(solve + loss + identify/adjoint/gradients), sharded by scene over {world} "
                                   f"rank(s)",
                       "grid": f"{n}x{n}", "scenes": scenes, "scenes_per_call": args.chunk,
                       "node_updates_per_step": int(W_job), "tol": 1e-6, "max_iters": 50,
                       "l2": "inputs larger than L2", "parallelism": f"batch-sharded x{world}"},
            "clocks": clk.summary(), "gpu_launches": int(launches),
            "note": "informational: the headline is the default (C3) line",
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def c5_main(args, rank, world, local):
    """BASELINE.json configs[4]: `scenes` samples of 1024^2
    (3 correlated-noise covariate channels each) through the encoder ->
    feasibility projection -> eikonal solve -> masked MSE, backward through
    the adjoint and the projection VJP into the encoder, one Adam step per
    step.  Samples are sharded over the ranks; the encoder is wrapped in DDP
    (NCCL all-reduce of its gradients, the only collective); each rank
    accumulates over micro-batches of `chunk` samples.  Targets come from a
    fixed random "truth" encoder (setup, untimed)."""
    import numpy as np
    import torch

    local = local % torch.cuda.device_count()  # gloo tests: several ranks on one GPU
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group("gloo")
    import paper_2603_00035_b200 as rfk
    from paper_2603_00035_b200 import torch_ops, training
    from paper_2603_00035_b200 import workload as wl
    from paper_2603_00035_b200.sharding import reduce_step_stats, shard_range

    n = 1024 if args.n == 4096 else args.n
    h = 1.0 / n
    scenes = args.scenes or 256
    lo, hi = shard_range(scenes, rank, world)
    torch.manual_seed(1234)
    truth = training.RandersEncoder().to(dev)
    torch.manual_seed(7)
    model = training.prepare_encoder(training.RandersEncoder().to(dev), args.encoder)
    if world > 1:
        model = torch.nn.parallel.DistributedDataParallel(model, device_ids=[local])
    opt = torch.optim.Adam(model.parameters(), lr=1e-3)
    src1 = wl.point_source(n, n, device=dev)
    obs1 = wl.observation_mask(src1)
    micro = []
    with torch.no_grad():
        for c0 in range(lo, hi, args.chunk):
            ids = list(range(c0, min(hi, c0 + args.chunk)))
            cov = torch.stack([torch.stack([wl.correlated_noise(n, n, 3, 3 * s + k, device=dev) for k in range(3)])
                               for s in ids]).float()
            src = src1.expand(len(ids), n, n).contiguous()
            obs = obs1.expand(len(ids), n, n).contiguous()
            tgt, _ = rfk.solve(*training.raw_to_fields(truth(cov)), src, h)
            micro.append((training.encoder_input(cov, args.encoder), src, obs, tgt))
    torch.cuda.synchronize()
    nm = len(micro)

    def step():
        opt.zero_grad(set_to_none=True)
        for i, batch in enumerate(micro):
            last = i == nm - 1
            if world > 1 and not last:
                with model.no_sync():
                    (training.c5_loss(model, *batch, h, precision=args.encoder) / nm).backward()
            else:
                (training.c5_loss(model, *batch, h, precision=args.encoder) / nm).backward()
        opt.step()

    for _ in range(max(3, args.warmup)):
        step()
    stats = []
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    torch_ops.collect_solve_stats(stats)
    launches0 = rfk.context().launches
    stream = torch.cuda.current_stream(dev)
    with ClockSampler(local) as clk:
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
    torch_ops.collect_solve_stats(None)
    launches = rfk.context().launches - launches0
    t_ms = e0.elapsed_time(e1)
    # work the timed steps did: every solve's own iteration count and records
    W_rank = 0
    for its, t, src in stats:
        its = np.atleast_1d(np.asarray(its))
        nrec = ((t < 1e9) & (src == 0)).flatten(1).sum(1).cpu().numpy()
        W_rank += sum(wl.node_updates(int(k), n * n, 1, int(r)) for k, r in zip(its, nrec))
    del stats
    W_job = W_rank
    if world > 1:
        t_ms, W_job = reduce_step_stats(t_ms, float(W_rank))
    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        try:
            cpu = cpu_batch_baseline(256, args.drift, "C5 solver part")
        except Exception as exc:
            cpu = {"value": None, "sample": f"failed: {exc}"}
    if rank == 0:
        ms = t_ms / args.steps
        line = {
            "metric": "grid-node updates/s (fwd sweep + adjoint), C5 encoder training on 1024² Randers fp64 samples",
            "cpu_baseline": cpu,
            "value": W_job / (t_ms / 1e3), "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": f"f64 solver, {args.encoder} encoder",
            "data": "synthetic (correlated-noise covariates, targets from a fixed random encoder)",
            "config": {"workload": f"C5: {scenes} samples of {n}x{n}, encoder (5x3x3 conv, 64 ch) -> "
                                   f"projection -> solve -> masked MSE -> adjoint -> projection VJP -> "
                                   f"encoder backward, Adam; DDP x{world}",
                       "grid": f"{n}x{n}", "samples": scenes, "micro_batch": args.chunk,
                       "samples_per_s": scenes / (ms / 1e3), "node_updates_per_step": int(W_job / args.steps),
                       "parallelism": f"data-parallel x{world} (NCCL all-reduce of encoder gradients)"},
            "clocks": clk.summary(), "gpu_launches": int(launches),
            "note": "informational: the headline is the default (C3) line",
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def main():
    args = parse()
    rank, world, local = dist_env()
    if args.impl == "reference":
        return reference_arm(args, rank, world)
    if args.workload == "c4":
        return c4_main(args, rank, world, local)
    if args.workload == "c5":
        return c5_main(args, rank, world, local)

    import numpy as np
    import torch

    local = local % torch.cuda.device_count()  # gloo tests: several ranks on one GPU
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group("gloo")

    import paper_2603_00035_b200 as rfk
    from paper_2603_00035_b200 import workload as wl

    ctx = rfk.Context(local)
    stream = torch.cuda.current_stream(dev)
    ctx.set_stream(stream.cuda_stream)
    n = args.n
    h = 1.0 / n
    # the deterministic host generator: rank 0's inputs are exactly those of
    # the full-size parity golden (tests/golden/large_hashes.json "c3")
    Fh = wl.host_fields(n, 1 + rank, args.drift)
    srch = wl.host_point_source(n, n)
    obsh = wl.host_observation_mask(srch)
    input_digest = wl.fields_digest(*Fh, srch, obsh)
    F = [torch.as_tensor(x).to(dev) for x in Fh]
    src = torch.as_tensor(srch).to(dev)
    obs = torch.as_tensor(obsh).to(dev)
    vals = torch.zeros((n, n), dtype=torch.float64, device=dev)
    del Fh
    torch.cuda.synchronize()

    state = {}

    def step():
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        t, rep = rfk.solve(*F, src, h, ctx=ctx)
        e1.record(stream)
        g, loss, unr = rfk.loss_grad_mse(t, obs, vals, exact=False, ctx=ctx)
        lam, grads, cl = rfk.backward(t, *F, src, h, g, want_lambda=False, ctx=ctx)
        state.update(t=t, rep=rep, grads=grads, e0=e0, e1=e1, loss=loss)
        return rep

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    nrec = int(((state["t"] < 1e9) & (src == 0)).sum())
    K = state["rep"].iterations
    W_step = wl.node_updates(K, n * n, 1, nrec)
    W_fwd = 4 * K * (n * n - 1)

    # ---- timed region (device-resident inputs) ----
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    launches0 = ctx.launches
    sweep_events = []
    with ClockSampler(local) as clk:
        start = torch.cuda.Event(enable_timing=True)
        end = torch.cuda.Event(enable_timing=True)
        start.record(stream)
        for _ in range(args.steps):
            step()
            sweep_events.append((state["e0"], state["e1"]))
        end.record(stream)
        torch.cuda.synchronize()
    launches = ctx.launches - launches0
    t_ms = start.elapsed_time(end)
    sweep_times = [a.elapsed_time(b) for a, b in sweep_events]
    if world > 1:
        tt = torch.tensor([t_ms], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        t_ms = float(tt.item())
    ms_per_step = t_ms / args.steps
    # each rank solves its own scene (seed 1 + rank), so K and the record
    # count differ per rank: the job's work is the sum over ranks
    W_job = W_step
    if world > 1:
        wt = torch.tensor([W_step], dtype=torch.int64, device=dev)
        torch.distributed.all_reduce(wt, op=torch.distributed.ReduceOp.SUM)
        W_job = int(wt.item())
    value = W_job * args.steps / (t_ms / 1e3)

    # ---- roofline of the dominant kernel (the sweep) ----
    peak, peak_kind = load_peaks()
    sweep_s = statistics.mean(sweep_times) / 1e3
    alg_bytes = W_fwd * BYTES_FWD
    achieved = alg_bytes / sweep_s / 1e9
    traffic, _, _ = load_traffic()
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": traffic, "peak_source": f"{peak_kind} hbm_gbs",
                "kernel": "sweep_kernel<16>", "kernel_ms": sweep_s * 1e3,
                "kernel_share": sweep_s * 1e3 / ms_per_step,
                "algorithmic_bytes": alg_bytes}
    # the FP64 pipe, side by side: measured pipe
    # peak vs the sweep's FP64 instructions per launch (committed ncu capture)
    fp64_peak, fp64_src = load_fp64_peak()
    fp64_thread, fp64_warp = load_fp64_inst()
    if fp64_thread and n == 4096:
        fp64_rate = fp64_thread / sweep_s
        roofline["fp64"] = {"achieved": fp64_rate / 1e12, "peak": fp64_peak / 1e12, "unit": "T thread-ops/s",
                            "frac": fp64_rate / fp64_peak, "peak_source": fp64_src,
                            "thread_ops_per_launch": fp64_thread, "fp64_pipe_warp_inst_per_launch": fp64_warp,
                            "inst_source": "profiles/ncu_summary.json sweep_fp64_counts (DADD+DMUL+DFMA, "
                                           "predicated-on lanes, one C3 solve)"}
    # the latency bound that actually binds: the exact
    # Gauss-Seidel order's dependency DAG has a longest path of ~2 NL + NW node
    # updates per pass; with overlapped passes an iteration costs ~4 * 2 NL
    # (scripts/sim/critpath.c) -> K * 8 N + N node-update latencies per solve
    crit = K * 8 * n + n
    # the latency roof: the dependent chain of one dirty node update read off
    # the sweep's SASS: donor load -> 23 dependent FP64 ops
    # at 23 cycles (disc 8, sqrt 7 + MUFU, Markstein 4, validity 2) + compare
    # / select hops + the fold's shared-memory round trip + relax store,
    # step barrier and the next donor load: ~715 cycles at 1965 MHz
    chain_min = 715.0
    cyc = sweep_s * 1.965e9 / crit
    roofline["critical_path"] = {"node_updates_on_path": crit, "us_per_node_update_on_path": sweep_s * 1e6 / crit,
                                 "cycles_per_node_update_at_max_clock": cyc,
                                 "chain_cycles_min_estimate": chain_min,
                                 "latency_frac": chain_min / cyc,
                                 "note": "latency roof = critical path x the dependent chain of one dirty node "
                                         "update (SASS estimate); every unit of the path counted as dirty"}

    # ---- e2e: the same step through the C ABI with host buffers ----
    e2e = None
    if rank == 0 or world > 1:
        pin = lambda x: x.cpu().pin_memory().numpy()
        Fh = [pin(x) for x in F]
        srch, obsh, valsh = pin(src), pin(obs), pin(vals)
        gout = torch.empty((5, n, n), dtype=torch.float64).pin_memory().numpy()
        ctx_h = rfk.Context(local)

        def host_step():
            # objective_and_grad (inversion.cpp:25-73) through the C ABI with
            # host buffers: parameters + observation set in, 5 gradient
            # planes + the loss out, once per step
            return rfk.objective_and_grad(*Fh, srch, obsh, valsh, h, exact=False, out=gout, ctx=ctx_h)
        host_step()
        nbytes = lambda *xs: int(sum(x.nbytes for x in xs))
        h2d = nbytes(*Fh, srch, obsh, valsh)
        d2h = nbytes(gout) + 8 + 4
        t0 = time.perf_counter()
        e2e_steps = max(1, min(args.steps, 2))
        for _ in range(e2e_steps):
            host_step()
        te = (time.perf_counter() - t0) / e2e_steps
        if world > 1:  # the slowest rank's wall time
            tt = torch.tensor([te], dtype=torch.float64, device=dev)
            torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
            te = float(tt.item())
        e2e = {"value": W_job / te, "unit": UNIT, "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h,
               "api": "rfk_objective_and_grad (RFK_MEM_HOST, pinned buffers): solve + loss + identify/adjoint/gradients"}

    # informational, outside the timed regions: the fp32 mode's forward on the
    # same fields, against the fp64 forward of the timed steps
    fp32 = None
    if rank == 0 and world == 1:
        try:
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            rfk.solve_f32(*F, src, h, ctx=ctx)  # warm-up (workspace)
            e0.record(stream)
            t32, rep32 = rfk.solve_f32(*F, src, h, ctx=ctx)
            e1.record(stream)
            torch.cuda.synchronize()
            t64 = state["t"]
            m = t64 < 1e9
            rel = ((t32.double() - t64).abs()[m] / t64[m].abs().clamp_min(1e-3)).max().item()
            fp32 = {"forward_ms": e0.elapsed_time(e1), "fp64_forward_ms": statistics.mean(sweep_times),
                    "K": int(rep32.iterations), "max_rel_err_vs_fp64": rel,
                    "api": "rfk_solve_f32 (not the headline: the metric is fp64)"}
        except Exception as exc:
            fp32 = {"failed": str(exc)}

    # informational: batched forward (C4-like, 4 grids of (n/2)^2 on one metric,
    # 4 sources) -- grids run concurrently in slots
    batch = None
    if rank == 0 and world == 1:
        try:
            nb, B = n // 2, 4
            Fb = wl.randers_fields(nb, 7, args.drift, device=dev)
            sb = torch.zeros((B, nb, nb), dtype=torch.uint8, device=dev)
            for b in range(B):
                sb[b, (nb // 2 + 97 * b) % nb, (nb // 3 + 61 * b) % nb] = 1
            rfk.solve(*Fb, sb, 1.0 / nb, ctx=ctx)  # warm-up (workspace)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            tb, rb = rfk.solve(*Fb, sb, 1.0 / nb, ctx=ctx)
            e1.record(stream)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1)
            wf = sum(4 * int(k) * (nb * nb - 1) for k in np.asarray(rb.iterations))
            batch = {"grids": B, "grid": f"{nb}x{nb}", "forward_ms": ms,
                     "forward_node_updates_per_s": wf / (ms / 1e3),
                     "single_grid_forward_node_updates_per_s": W_fwd / statistics.mean(sweep_times) * 1e3,
                     "note": "informational; the headline is the single C3 grid"}
        except Exception as exc:
            batch = {"failed": str(exc)}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_baseline(args.cpu_n, args.drift)
        except Exception as exc:  # the baseline must not sink the bench line
            cpu = {"value": None, "unit": UNIT, "cores": 1, "kind": "reference", "sample": f"failed: {exc}"}

    c3ref = load_c3_reference() if (rank == 0 and n == 4096) else None
    if cpu is not None and c3ref:
        cpu["c3_full"] = c3ref
        if c3ref.get("node_updates_per_s"):
            cpu["c3_full_ratio_e2e"] = (e2e["value"] / c3ref["node_updates_per_s"]) if e2e else None
            cpu["c3_full_ratio_value"] = value / c3ref["node_updates_per_s"]
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (deterministic host-generated correlated-noise Randers fields, projected)",
            "config": {"workload": f"C3: full Randers metric with drift, {n}x{n}, forward + adjoint, fp64",
                       "input_digest": input_digest,
                       "parity": "rank 0's inputs are tests/golden/large_hashes.json c3; T, K, records, lambda and "
                                 "gradients bit-identical to the reference library (tests/test_fullsize_parity_gpu.py)",
                       "grid": f"{n}x{n}", "sources": 1, "tol": 1e-6, "max_iters": 50, "K": K,
                       "node_updates_per_step": W_job, "n_records": nrec,
                       "l2": "inputs larger than L2 (5 x 128 MiB fp64 parameter planes)",
                       "parallelism": f"replicas x{world} (one grid per GPU)"},
            "roofline": roofline,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "clocks": clk.summary(),
            "gpu_launches": int(launches),
            "fp32_mode": fp32,
            "batch_mode": batch,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
