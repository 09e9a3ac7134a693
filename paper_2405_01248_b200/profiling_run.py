"""Measured `model-profile/v1` and `CommCosts` for a configuration (the paper's "Fig. 6 step 1",
PAPER.md:260,728-729), produced on rank 0 and shared with every rank so that all ranks plan from
the identical inputs (the planner is deterministic given its inputs, reference planner.py:190-240).

* `measure`: per-layer costs of every backbone and every frozen component of the configuration
  (profiler.measure_profile), layer-0 inputs built from the configuration's own batch fields
  (DataSpec with its latent channels and extra fields: ControlNet hint, cascaded SR noise) plus the
  producers' final outputs for dependent frozen components (model.frozen_deps, e.g. vae/text ->
  locked U-Net encoder in c3); the dependencies are carried into the profile.
* `measure_comm`: NCCL micro-benchmark filling the planner's analytic comm model (reference
  profile.py:39-61, used at partitioner.py:186-197): point-to-point send/recv between ranks 0 and 1
  and allreduce over every rank, each at a small and a large message; latency and bandwidth are
  the intercept and slope of the two-point fit (device-timed, max over ranks).
"""

from __future__ import annotations

from dataclasses import replace

import torch
import torch.distributed as dist

from . import engine
from .diffusion import DataSpec, make_batch
from .pipefill.filler import VALID_LOCAL_SIZES
from .pipefill.profile import CommCosts
from .profiler import measure_profile, probe_specs

# Used only when there is no peer to measure against (world 1: the plan has no communication).
DEFAULT_COMM = CommCosts(2.0e11, 2e-5, 3.0e11, 1e-5)


def _rand_state(spec, k, device, grad_ok=True, gen=None):
    st = {}
    for name, v in spec.items():
        shape, dt = v[0], v[1]
        grad = v[2] if len(v) > 2 else False
        if dt in (torch.int64, torch.int32):
            t = torch.randint(0, 1000, (k,) + tuple(shape), device=device, dtype=dt)
        else:
            t = torch.randn((k,) + tuple(shape), device=device).to(dt)
            if grad and grad_ok:
                t.requires_grad_(True)
        st[name] = t
    return st


def measure(cfg, group_batch, D, M, device, reps=3):
    model = engine.build_model(cfg, device)
    c = engine.CONFIGS[cfg]
    ds = DataSpec(c.config_id, 1, c.image, c.latent, c.zc, c.text_len, c.vocab, 1000, c.selfcond_p,
                  extra=c.extra)
    feed = engine.InputFeed(make_batch(ds, 10 ** 6), device, c.dtype)
    live_all, fspecs = probe_specs(model, lambda k: feed.get(k, 0, 1), device)
    mb = group_batch // M
    bb_keys = sorted({1} | {max(1, mb // r) for r in range(1, D + 1)} | {-(-mb // r) for r in range(1, D + 1)})
    fr_keys = sorted({1, 2} | set(VALID_LOCAL_SIZES) | {max(1, group_batch // d) for d in range(1, D + 1)}
                     | {-(-group_batch // d) for d in range(1, D + 1)})
    fr_keys = [k for k in fr_keys if k <= group_batch]
    # layer-0 inputs of the frozen components: the configuration's own batch fields (one synthetic
    # batch of the largest key, sliced), plus the producers' final outputs for dependent components
    big = engine.InputFeed(make_batch(replace(ds, world_batch=max(fr_keys)), 10 ** 6 + 2), device, c.dtype)
    deps = tuple(getattr(model, "frozen_deps", ()))

    def make_state(which, layer, k):
        if isinstance(which, tuple):  # ("backbone", pipe)
            return _rand_state(live_all[which[1]][layer], k, device)
        if layer == 0:
            st = {f: big.get(f, 0, k) for f in model.frozen[which].inputs}
            for prod, cons in deps:
                if cons == which:
                    st.update(_rand_state(fspecs[prod][-1], k, device))
            return st
        return _rand_state(fspecs[which][layer - 1], k, device)

    prof = measure_profile(model, live_all, fspecs, make_state, group_batch=group_batch, D=D, M=M, reps=reps,
                           device=device, bb_keys=bb_keys, frozen_keys=fr_keys)
    del model, big
    torch.cuda.empty_cache()
    return prof


def _timed_ms(fn, reps, device):
    fn()
    torch.cuda.synchronize(device)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize(device)
    return a.elapsed_time(b) / reps


def _max_over_ranks(x, device):
    t = torch.tensor([x], device=device, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.item()


def _fit(sizes, secs):
    (n0, n1), (t0, t1) = sizes, secs
    bw = (n1 - n0) / max(t1 - t0, 1e-9)
    lat = max(0.0, t0 - n0 / bw)
    return bw, lat


def measure_comm(world, rank, device, small=1 << 16, large=64 << 20, reps=10):
    """CommCosts measured over NCCL on this job's ranks (collective: every rank calls it).
    p2p: rank 0 -> rank 1 send/recv (one NVSwitch hop, uniform to every peer); ar: allreduce of
    fp32 buffers over all ranks (bytes = buffer size, the planner's grad_bytes convention)."""
    if world == 1 or not dist.is_initialized() or dist.get_backend() != "nccl":
        return DEFAULT_COMM  # nothing to measure (gloo: the host-staged test transport)
    dev = torch.device(device)
    p2p_t, ar_t = [], []
    for n in (small, large):
        buf = torch.zeros(n // 4, device=dev, dtype=torch.float32)

        def p2p():
            if rank == 0:
                dist.send(buf, dst=1)
            elif rank == 1:
                dist.recv(buf, src=0)

        dist.barrier()
        p2p_t.append(_max_over_ranks(_timed_ms(p2p, reps, dev), dev) * 1e-3)
        dist.barrier()
        ar_t.append(_max_over_ranks(_timed_ms(lambda: dist.all_reduce(buf), reps, dev), dev) * 1e-3)
        del buf
    bw_p, lat_p = _fit((small, large), p2p_t)
    bw_a, lat_a = _fit((small, large), ar_t)
    return CommCosts(bw_a, lat_a, bw_p, lat_p)


def shared_profile(cfg, world, rank, world_batch, S, D, M, with_comm=False):
    """The measured profile (rank 0) broadcast to every rank; with_comm=True also returns the
    measured CommCosts (every rank takes part in the NCCL micro-benchmark)."""
    group_batch = world_batch * D // world
    obj = [None]
    if rank == 0:
        obj[0] = measure(cfg, group_batch, D, M, f"cuda:{torch.cuda.current_device()}")
    if world > 1:
        dist.broadcast_object_list(obj, src=0)
    if not with_comm:
        return obj[0]
    comm = measure_comm(world, rank, f"cuda:{torch.cuda.current_device()}")
    if world > 1:
        box = [comm]
        dist.broadcast_object_list(box, src=0)
        comm = box[0]
    return obj[0], comm
