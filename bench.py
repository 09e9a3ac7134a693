"""Benchmark: pipelined diffusion training step (BASELINE.json metric
"train samples/sec at 1/2/4/8 B200; bubble ratio; speedup vs unfilled 1F1B").

    python bench.py --gpus N --steps K --warmup W [--impl ours|reference] [--config c2]
    (N > 1: torchrun --nproc-per-node N ... bench.py --gpus N ...)

Workload (configs[1] of BASELINE.json): SD v2.1 U-Net (865M, trainable) + frozen
OpenCLIP ViT-H text encoder (23 layers) + frozen SD VAE encoder, 256 px, bf16
compute with fp32 master weights / AdamW, synthetic data and random init.
Per GPU 32 samples per iteration (weak scaling): world batch 32 N; N = 1 -> S = D = 1;
N = 2 -> S = D = 2, M = 4; N = 4 -> S = D = 4, M = 4; N = 8 -> S = D = 4, M = 4, 2 groups (c2/c4);
c3: S = N/2 stages x 2 replicas over D = N; c5: S = D = N, M = 2N (see `layout`). N > 1 plans from
a profile measured on the box and NCCL-measured CommCosts (profiling_run).

value  : world samples/s, inputs resident in HBM, device-timed (CUDA events) over exactly K
         iterations after W warm-ups, max over ranks.
e2e    : same metric through the public Trainer API with inputs in pinned host memory:
         every step copies its batch slices H2D and reads the loss D2H (.item()).
Every iteration also runs the frozen encoders for the next batch (cross-iteration fill /
tail) and the AdamW step: nothing is skipped inside the timed region.
"""

from __future__ import annotations

import argparse
import datetime
import gc
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

METRIC = "train samples/sec"
WORKLOADS = {
    "c2": ("c2: SD v2.1 U-Net (trainable, 865M) + OpenCLIP ViT-H text (23 layers, frozen) + "
           "SD VAE encoder (frozen), 256px, 32 samples/GPU/iteration"),
    "c3": ("c3: ControlNet v1.0 branch (trainable, 364M) -> locked SD v2.1 decoder; frozen VAE, "
           "OpenCLIP-H, hint, locked U-Net encoder; 512px, 32 samples/GPU/iteration"),
    "c4": ("c4: cascaded base 64px U-Net (316M) + SR 256px U-Net (133M), bidirectional pipelines, "
           "frozen T5-large-shaped encoder (128 tokens) + image pyramid, self-cond p=0.5, 32 samples/GPU"),
    "c5": ("c5: SD U-Net at model channels 512 (trainable, 2.19B) + OpenCLIP-H + SD VAE, 256px, "
           "32 samples/GPU/iteration"),
}
WORKLOAD = WORKLOADS["c2"]


def layout(n, config="c2"):
    """Pipeline layout per GPU count and configuration: c2 / c4 follow
    "4-stage pipeline x 2 DP" at N=8 (S = D = 4, two groups); c3 runs S = 4 stages over D = 8
    devices (every stage replicated twice, reference partitioner.py:69-84); c5 is the "8-stage
    pipeline on 8xB200" with M = 16 (BASELINE.json configs[4]). Fewer GPUs shrink the pipeline."""
    if n == 1:
        return dict(S=1, D=1, M=1)
    if config == "c5":
        return dict(S=n, D=n, M=2 * n)
    if config == "c3" and n >= 4:
        return dict(S=n // 2, D=n, M=4)
    S = min(n, 4)
    return dict(S=S, D=S, M=4)


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


class Clocks:
    """nvidia-smi sampler running during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.out = ""
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        return False

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in (self.out or "").splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        load = [s for s in sm if s > 0.5 * max(sm)] or sm
        return {"sm_mhz": statistics.median(load), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


def dist_setup(n, share_gpu=False):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != n:
        raise SystemExit(f"--gpus {n} but WORLD_SIZE={world}")
    if share_gpu:
        # TEST ONLY: all ranks on cuda:0, gloo with host-staged P2P (exercises the N > 1 code
        # path on a single-GPU box; the numbers are meaningless)
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        # a hung peer fails the job after DP_NCCL_TIMEOUT_S instead of blocking forever (the
        # NCCL watchdog aborts the communicators; every sub-group inherits the timeout)
        to = datetime.timedelta(seconds=int(os.environ.get("DP_NCCL_TIMEOUT_S", "600")))
        if share_gpu:
            dist.init_process_group("gloo", timeout=to)
        else:
            # device_id binds the default group to this GPU: its communicator and every
            # sub-group's (split from it) are created eagerly at setup, not on the first send
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"), timeout=to)
    return rank, world, local


def max_over_ranks(x, world):
    if world == 1:
        return x
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([x], device=dev, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.item()


def clock_hz():
    """Cycles per second for the lead spin: the B200's max SM clock, so a spin lasts >= lead_ms at any clock."""
    return 1.965e9


def barrier(world):
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()


def timed_steps(trainer, K, world, *, read_loss=False, kernel_timer=False, lead_ms=0.0):
    """K steps between CUDA events (max over ranks). lead_ms > 0 (the per-launch event pass only): every
    step starts with a spin kernel of that length on the executor's streams, so the host enqueues the step's
    ~2000 launches and ~4000 timing events while the GPU is busy and each bracketed interval holds the
    kernel's device time rather than the host's launch latency (the event pass is host-bound otherwise);
    the spins are timed by their own events and subtracted."""
    from paper_2405_01248_b200 import telemetry

    barrier(world)
    telemetry.reset()
    # automatic garbage collection off inside the timed loop (collected just before, as training
    # loops with manual GC do): a collection pause stalls the host thread that feeds ~2000 launches
    # per step and showed up as sporadic 10% dips of the e2e pass
    gc.collect()
    gc.disable()
    if kernel_timer:
        telemetry.timer.start(reserve=2 * 2500 * K)
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    losses = []
    host_loss = torch.empty(K, dtype=torch.float32, pin_memory=True) if read_loss else None
    spins = []
    lead_streams = []
    if lead_ms > 0 and trainer.ex.streams.cuda:
        lead_streams = [trainer.ex.streams.compute, trainer.ex.streams.fill]
        if trainer.ex.opt_stream is not None:
            lead_streams.append(trainer.ex.opt_stream)
    for i in range(K):
        if lead_streams:
            cyc = int(lead_ms * 1e-3 * clock_hz())
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(lead_streams[0]):
                e0.record()
                torch.cuda._sleep(cyc)
                e1.record()
            spins.append((e0, e1))
            for st in lead_streams[1:]:
                st.wait_stream(lead_streams[0])
        loss = trainer.step()
        if read_loss:
            # the step's loss crosses to pinned host memory every step (async D2H: the host does not
            # drain the GPU between steps, as in a training loop with asynchronous logging)
            host_loss[i:i + 1].copy_(trainer.ex.total_loss(), non_blocking=True)
    b.record()
    torch.cuda.synchronize()
    gc.enable()
    if read_loss:
        losses = host_loss.tolist()
        if not all(v == v for v in losses):
            raise SystemExit(f"non-finite loss in the e2e run: {losses}")
    ms = a.elapsed_time(b) - sum(e0.elapsed_time(e1) for e0, e1 in spins)
    kstats = telemetry.timer.stop() if kernel_timer else None
    launches = telemetry.total_launches()
    barrier(world)
    return max_over_ranks(ms, world), kstats, launches, losses


def cpu_reference(steps, warmup, sample=1):
    """The reference's CPU path for this workload: the sequential fp32 oracle training step
    (oracle/train_step.py) on host cores, `sample` samples per step."""
    from oracle import train_step
    from paper_2405_01248_b200 import diffusion, networks, nn

    torch.set_num_threads(os.cpu_count() or 1)
    params = {}
    for C in (networks.SDUNet, networks.SDVAEEncoder, networks.CLIPTextEncoder):
        c = C()
        params[c.name] = nn.init_state(c.store.param_specs(), 0)
    ds = diffusion.DataSpec(2, sample, 256, 32, 4, 77, 49408, 1000, 0.0)
    sab, s1m = diffusion.noise_schedule()
    times = []
    for i in range(warmup + steps):
        batch = diffusion.make_batch(ds, i)
        t0 = time.perf_counter()
        train_step.train("c2", params, [batch], sab, s1m)
        dt = time.perf_counter() - t0
        if i >= warmup:
            times.append(dt)
    return sample * len(times) / sum(times), torch.get_num_threads()


def planner_cpu_baseline(reps=10):
    """BASELINE.md §4 CPU baseline #1: the REFERENCE planner's evaluate_point (baseline/_ref, the
    unmodified pipefill package) on the measured c2 B200 profile at the N=8 layout (S = D = 4, M = 4,
    world 8, world batch 256), single-threaded Python, best of `reps` (perf_counter)."""
    ref = os.path.join(ROOT, "baseline", "_ref")
    prof_path = os.path.join(ROOT, "profiles", "r01_c2_measured_profile_D4_M4.json")
    if not os.path.isdir(os.path.join(ref, "pipefill")) or not os.path.exists(prof_path):
        return None
    if ref not in sys.path:
        sys.path.append(ref)
    import importlib

    Rpl = importlib.import_module("pipefill.planner")
    Rpr = importlib.import_module("pipefill.profile")
    prof = Rpr.load_profile(prof_path)
    cl = Rpr.ClusterConfig(8, Rpr.CommCosts(2.0e11, 2e-5, 3.0e11, 1e-5))
    best = float("inf")
    for _ in range(reps):
        t0 = time.perf_counter()
        Rpl.evaluate_point(prof, cl, 4, 4, 4, 256, bubble_min_len=0.002)
        best = min(best, time.perf_counter() - t0)
    return {"value": best * 1e3, "unit": "ms per evaluate_point", "cores": 1, "kind": "reference",
            "sample": "reference pipefill evaluate_point(S=4, M=4, D=4, world 8, batch 256) on the measured "
                      "c2 profile, best of 10"}


def reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    # bounded: each step is one sample (~20 s on 8 cores); cap the run at ~4 minutes
    steps = max(1, min(args.steps, 8))
    warm = 1 if args.warmup > 0 else 0
    v, cores = cpu_reference(steps, warm)
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "samples/s", "n_gpus": args.gpus,
            "steps": steps, "warmup": warm, "ms_per_step": 1000.0 / v, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": WORKLOAD, "cpu_sample": "1 sample per step"},
            "cpu_baseline": {"value": v, "unit": "samples/s", "cores": cores, "kind": "port",
                             "sample": f"{steps} steps x 1 sample of the c2 step (oracle/train_step.py, fp32)"},
            "e2e": {"value": v, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--per-gpu-batch", type=int, default=32)
    ap.add_argument("--debug-share-gpu", action="store_true",
                    help="TEST ONLY: run all ranks on cuda:0 over gloo (validates the N>1 path)")
    ap.add_argument("--trace-out", default=None, help="write the measured schedule as a trace-event JSON")
    ap.add_argument("--config", default="c2", choices=sorted(WORKLOADS) + ["c3-small", "c4-small", "c5-small"],
                    help="the headline (BASELINE.json metric) workload is c2; c3..c5 for reference")
    ap.add_argument("--graph", action="store_true",
                    help="N=1: replay the captured iteration as a CUDA graph (measured: no gain, GPU-bound)")
    args = ap.parse_args()
    if args.impl == "reference":
        return reference_arm(args)
    args.warmup = max(args.warmup, 3)

    rank, world, local = dist_setup(args.gpus, args.debug_share_gpu)
    from paper_2405_01248_b200 import engine

    lay = layout(world, args.config.split("-")[0])
    wb = args.per_gpu_batch * world
    profile = comm = None
    if lay["S"] > 1:
        # measured per-layer costs (rank 0) and NCCL p2p / allreduce costs (all ranks), shared so
        # every rank plans from identical inputs
        from paper_2405_01248_b200 import profiling_run
        profile, comm = profiling_run.shared_profile(args.config, world, rank, wb, with_comm=True, **lay)
    trainer = engine.Trainer.create(args.config, world=world, rank=rank, world_batch=wb, profile=profile,
                                    device=f"cuda:{local}", comm=comm, **lay)
    W, K = args.warmup, args.steps
    trainer.prefetch(2 * W + 2 * K + 2, mode="device")
    for _ in range(W):
        trainer.step()
    use_graph = world == 1 and args.graph
    if use_graph:
        # N = 1: the whole iteration (U-Net fwd/bwd, AdamW, next batch's VAE + CLIP) is
        # captured once and replayed as one CUDA graph (no per-kernel host dispatch)
        trainer.enable_cuda_graph()
        for _ in range(W):
            trainer.step()
    torch.cuda.reset_peak_memory_stats()  # the memory line reflects training steps only
    with Clocks(local) as clk:
        ms, _, launches, _ = timed_steps(trainer, K, world)
    value = wb * K / (ms / 1000.0)
    if use_graph:
        trainer._graph = None

    # e2e pass right after the value pass (same machine state, before the long instrumented passes):
    # pinned-host inputs copied H2D inside every step and the loss read back
    e2e = None
    if not args.no_e2e:
        trainer.feed_mode = "host"
        trainer.prefetch(K + W + 3, mode="host")
        # warm-up without a host sync per step: the host runs ahead of the GPU as in the timed loop,
        # so the copy-stream allocator pools reach their steady state before timing
        for _ in range(max(2, W)):
            trainer.step()
        trainer.ex.total_loss().item()
        ms_e, _, _, _ = timed_steps(trainer, K, world, read_loss=True)
        h2d = _h2d_bytes_per_step(trainer)
        e2e = {"value": wb * K / (ms_e / 1000.0), "unit": "samples/s", "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": 4}
        trainer.feed_mode = "device"
        trainer.prefetch(K + 3, mode="device")

    # roofline pass (eager, after the timed ones): every libdpipe launch bracketed by CUDA events on
    # its stream (the events break programmatic dependent launch, so this pass runs slower), each step
    # behind a 60 ms lead spin so the GPU does not wait on the host inside a bracket
    # The optimizer's overlap with the final backward is switched off for this pass only: the AdamW slices
    # otherwise run concurrently on the optimizer stream and every bracketed GEMM of the last backward
    # shares the SMs with them, so its interval is not that kernel's duration.
    ovl = trainer.ex.overlap_sync
    trainer.ex.overlap_sync = False
    try:
        ms_k, kstats, _, _ = timed_steps(trainer, K, world, kernel_timer=True, lead_ms=60.0)
    finally:
        trainer.ex.overlap_sync = ovl

    # measured bubble ratio: one traced iteration after the timed region, task intervals from
    # CUDA events on their streams, bubbles / ratio by the planner's own definitions
    barrier(world)
    trainer.step(trace=True)
    sched_meas, _, br_meas = trainer.measured()
    br_meas_unf = None
    if args.trace_out and rank == 0:
        # measured schedule in the reference's trace-event format (scheduler.py:483-519)
        from paper_2405_01248_b200.pipefill import scheduler as psched
        psched.export_trace(sched_meas, args.trace_out)

    # speedup vs the same executor's unfilled pipeline (frozen part data-parallel, un-overlapped)
    speedup = 1.0
    if lay["S"] > 1:
        unf = engine.Trainer.create(args.config, world=world, rank=rank, world_batch=wb, profile=profile,
                                    device=f"cuda:{local}", filled=False, comm=comm, **lay)
        unf.prefetch(W + K + 1, mode="device")
        for _ in range(W):
            unf.step()
        ms_u, _, _, _ = timed_steps(unf, K, world)
        speedup = ms_u / ms
        barrier(world)
        unf.step(trace=True)
        _, _, br_meas_unf = unf.measured()
        del unf

    # memory-feasibility model vs the measured peak of this run (memory.py)
    mem = {"measured_peak_gb": round(torch.cuda.max_memory_allocated() / 1e9, 2)}
    try:
        mem["predicted_gb"] = round(trainer.memory_report()[trainer.ex.dev] / 1e9, 2)
    except Exception as e:  # the report is informative; never fail the bench line on it
        mem["predicted_error"] = str(e)[:120]

    pk, pk_kind = peaks()
    roof = None
    if kstats:
        # the dominant kernel: tc_gemm_kernel (every linear / conv / attention contraction)
        gem = [v for f, v in kstats.items() if f.startswith("tcgen05_gemm")]
        st = {"ms": sum(v["ms"] for v in gem), "flops": sum(v["flops"] for v in gem),
              "launches": sum(v["launches"] for v in gem)}
        ach = st["flops"] / (st["ms"] / 1000.0) / 1e12
        peak = pk.get("bf16_tflops_sustained", pk.get("bf16_tflops"))
        breakdown = {f: {"ms_per_step": round(v["ms"] / K, 3), "launches_per_step": v["launches"] / K,
                         **({"tflops": round(v["flops"] / max(v["ms"], 1e-9) / 1e9, 1)} if v["flops"] else {})}
                     for f, v in sorted(kstats.items(), key=lambda kv: -kv[1]["ms"])}
        roof = {"bound": "tensor", "kernel": "tc_gemm_kernel (tcgen05_gemm.*)", "achieved": ach,
                "peak": peak, "unit": "TFLOP/s", "frac": ach / peak,
                "peak_kind": f"{pk_kind} bf16_tflops_sustained", "traffic": _ncu_traffic("tcgen05_gemm"),
                "share_of_step": st["ms"] / ms_k, "launches_per_step": st["launches"] / K,
                "flops_per_launch": st["flops"] / max(1, st["launches"]),
                "timed_step_ms_with_events": ms_k / K, "breakdown": breakdown}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and args.config == "c2":
        v, cores = cpu_reference(2, 1)
        cpu = {"value": v, "unit": "samples/s", "cores": cores, "kind": "port",
               "sample": "2 timed steps x 1 sample of the c2 training step after 1 warm-up step, CPU oracle "
                         "(oracle/train_step.py, fp32)",
               "planner": planner_cpu_baseline()}

    if rank == 0:
        res = trainer.ex.plan_result
        line = {
            "metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": world, "steps": K,
            "warmup": W, "ms_per_step": ms / K, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic (seeded), random init",
            "config": {"workload": WORKLOADS.get(args.config, args.config + " (reduced test variant)"), "world_batch": wb, "group_batch": wb * lay["D"] // world,
                       "S": lay["S"], "M": lay["M"], "D": lay["D"], "groups": world // lay["D"],
                       "parallelism": f"pp{lay['S']}xdp{world // lay['S']}",
                       "l2": "working set (weights 1.7 GB bf16 + activations) >> 126 MB L2",
                       "dispatch": "cuda_graph" if use_graph else "eager"},
            "bubble_ratio_predicted_before": res["bubble_ratio_before"],
            "bubble_ratio_predicted_after": res["bubble_ratio_after"],
            "bubble_ratio_measured": br_meas,
            "bubble_ratio_measured_unfilled": br_meas_unf,
            "speedup_vs_unfilled": speedup,
            "e2e": e2e, "gpu_launches": launches, "roofline": roof, "cpu_baseline": cpu, "memory": mem,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def _h2d_bytes_per_step(trainer):
    """Bytes this rank copies host->device in one steady-state step (counted from the copies)."""
    from paper_2405_01248_b200.engine import InputFeed

    trainer.prefetch(2, mode="host")
    before = InputFeed.h2d_total
    trainer.step()
    torch.cuda.synchronize()
    return int(InputFeed.h2d_total - before)


def _ncu_traffic(fam):
    """DRAM bytes per launch of the family's representative kernel from one committed ncu --set full
    capture (profiles/ncu_traffic.json), or None."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as fh:
            v = json.load(fh).get(fam)
        return v if isinstance(v, (int, float)) else None
    except (OSError, ValueError):
        return None


if __name__ == "__main__":
    main()
