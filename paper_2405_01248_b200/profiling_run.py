"""Measured `model-profile/v1` for a configuration, produced on rank 0 and shared with
every rank so that all ranks plan from the identical profile (the planner is
deterministic given its inputs, reference planner.py:190-240)."""

from __future__ import annotations

import torch
import torch.distributed as dist

from . import engine
from .diffusion import make_batch
from .pipefill.filler import VALID_LOCAL_SIZES
from .profiler import measure_profile, probe_specs


def _rand_state(spec, k, device, grad_ok=True):
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
    from dataclasses import replace
    from .diffusion import DataSpec
    ds = DataSpec(c.config_id, 1, c.image, c.latent, 4, c.text_len, c.vocab, 1000, c.selfcond_p)
    feed = engine.InputFeed(make_batch(ds, 10 ** 6), device, c.dtype)
    live_all, fspecs = probe_specs(model, lambda k: feed.get(k, 0, 1), device)
    live = live_all[0]
    mb = group_batch // M
    bb_keys = sorted({1} | {max(1, mb // r) for r in range(1, D + 1)} | {-(-mb // r) for r in range(1, D + 1)})
    fr_keys = sorted({1, 2} | set(VALID_LOCAL_SIZES) | {max(1, group_batch // d) for d in range(1, D + 1)}
                     | {-(-group_batch // d) for d in range(1, D + 1)})
    fr_keys = [k for k in fr_keys if k <= group_batch]
    frozen_inputs = {0: {"images": ((c.image, c.image, 3), torch.float32)},
                     1: {"ids": ((c.text_len,), torch.int64)}}

    def make_state(which, layer, k):
        if which == "backbone":
            return _rand_state(live[layer], k, device)
        if layer == 0:
            st = _rand_state(frozen_inputs[which], k, device)
            if "ids" in st:
                st["ids"] = st["ids"] % c.vocab
            return st
        return _rand_state(fspecs[which][layer - 1], k, device)

    prof = measure_profile(model, live, fspecs, make_state, group_batch=group_batch, D=D, M=M, reps=reps,
                           device=device, bb_keys=bb_keys, frozen_keys=fr_keys)
    del model
    torch.cuda.empty_cache()
    return prof


def shared_profile(cfg, world, rank, world_batch, S, D, M):
    group_batch = world_batch * D // world
    obj = [None]
    if rank == 0:
        obj[0] = measure(cfg, group_batch, D, M, f"cuda:{torch.cuda.current_device()}")
    if world > 1:
        dist.broadcast_object_list(obj, src=0)
    return obj[0]
