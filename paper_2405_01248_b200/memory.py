"""Memory-feasibility model of a pipelined training plan (the reference planner has no
memory model, while the paper hits memory limits).

Per device of a GroupProgram the model adds
  * trainable parameters of the stage(s) it hosts: fp32 master + compute copy (bf16) + fp32 grad + AdamW m, v
    + the cached flip-transposed bf16 copy the dgrads read (nn.FLIP_CACHE; upper bound: every weight)
    (20 B/parameter in bf16 configurations, 16 B in fp32 ones where the master is the compute copy);
  * frozen components, replicated on every device (fp32 master + compute copy);
  * activations autograd keeps for the backward: per backbone layer, bytes per sample measured on the device
    (`measure_layer_activation_bytes`) x the stage's per-replica micro-batch x the micro-batches in flight at
    the stage. The planner's simulator dispatches forwards eagerly (reference scheduler.py:1-10,165-179: a
    ready forward runs whenever no backward is ready), not warm-up-capped 1F1B, so the in-flight depth is
    counted from the device's replayed instruction order (`inflight_depth`: max over the program of
    forwards minus backwards of that stage), e.g. 8 at S=4, M=8 on stage 0 where 1F1B would hold 4;
  * frozen outputs held for the next iteration (latents / context of the group batch, twice: being produced
    and being consumed), plus the largest frozen layer's input + output over the group batch (transient).
`check_plan` raises MemoryError when a device exceeds the budget; the planner API itself is unchanged.
"""

from __future__ import annotations

import math

import torch

B200_HBM_BYTES = 183_359 * 2**20   # nvidia-smi total of one B200


def _store_bytes(store, trainable):
    n = store.numel()
    if not trainable:
        return n * (4 + (2 if store.dtype != torch.float32 else 0))
    return n * _param_bytes(store)


def measure_layer_activation_bytes(model, batch_fn, device, batch=2):
    """Per backbone, per layer: bytes per sample allocated (and kept alive for the backward) by the
    layer's forward with autograd recording, measured with torch.cuda.memory_allocated on `device`."""
    from .adapter import topo_order

    dev = torch.device(device)
    fro = {}
    deps = getattr(model, "frozen_deps", ())
    finals = {}
    with torch.no_grad():
        for c in topo_order(len(model.frozen), deps):
            f = model.frozen[c]
            st = {k: batch_fn(k, batch) for k in f.inputs}
            for s_, d in deps:
                if d == c:
                    st.update(finals[s_])
            for layer in f.component.layers:
                st = layer(st)
            finals[c] = st
            fro.update(st)
    t = batch_fn("t", batch)
    out = []
    for pipe, bb in enumerate(model.backbones):
        nf = model.noise_field(pipe)
        st, _ = model.stage0_inputs(fro, t, batch_fn(nf, batch), pipe=pipe)
        per_layer = []
        ctx = bb.grad_context() if hasattr(bb, "grad_context") else torch.enable_grad()
        keep = []
        with ctx:
            for k, v in list(st.items()):
                if v.is_floating_point() and k not in ("noise",):
                    st[k] = v.detach().requires_grad_(True)
            torch.cuda.synchronize(dev)
            base = torch.cuda.memory_allocated(dev)
            for layer in bb.layers:
                st = layer(st)
                keep.append(st)
                torch.cuda.synchronize(dev)
                now = torch.cuda.memory_allocated(dev)
                per_layer.append(max(0, now - base) / batch)
                base = now
        del keep, st
        torch.cuda.synchronize(dev)
        out.append(per_layer)
    return out


def inflight_depth(prog, dev, pipe=0):
    """Peak number of micro-batches whose forward has run and whose backward has not, over the
    instruction order of `dev` in GroupProgram `prog` (the order the executor replays), for `pipe`."""
    live = peak = 0
    for ins in prog.device_program(dev).instrs:
        if ins[0] in ("fwd", "bwd") and ins[3] == pipe:
            live += 1 if ins[0] == "fwd" else -1
            peak = max(peak, live)
    return peak


def _param_bytes(store):
    """Trainable bytes per parameter: fp32 master + grad + AdamW m, v (16) + bf16 compute copy (2)
    + the cached flip-transposed bf16 copy the dgrads read (2, nn.FLIP_CACHE; upper bound: every weight)."""
    from . import nn
    bf16 = store.dtype != torch.float32
    return 16 + (2 if bf16 else 0) + (2 if bf16 and nn.FLIP_CACHE else 0)


def predict_device_bytes(prog, model, act_bytes, frozen_specs=None):
    """{device: bytes} for one GroupProgram (adapter.build_group_program) of `model`."""
    frozen = sum(_store_bytes(f.component.store, False) for f in model.frozen
                 if getattr(f.component, "store", None) is not None
                 and f.component.store is not getattr(model.backbone, "store", None))
    held = 0
    transient = 0
    if frozen_specs:
        def nbytes(spec):
            return sum(math.prod(shape) * torch.tensor([], dtype=dt).element_size() for shape, dt in spec.values())
        for c, specs in enumerate(frozen_specs):
            held += 2 * nbytes(specs[-1]) * prog.group_batch
            # a frozen layer's input + output for the largest piece a device runs (<= the group batch)
            for j in range(1, len(specs)):
                transient = max(transient, (nbytes(specs[j - 1]) + nbytes(specs[j])) * prog.group_batch)
    held += transient
    out = {}
    for dev in range(prog.D):
        dp = prog.device_program(dev)
        stages = list(dp.stages) if dp.stages else [dp.stage]
        total = frozen + held
        for pi, st in enumerate(stages):
            if st is None:
                continue
            pl = prog.pipes[pi]
            bb = model.backbones[pl.backbone]
            lo, hi = pl.stage_ranges[st]
            a, b = bb.stage_slice(lo, hi)
            total += (b - a) * _param_bytes(bb.store)
            r = pl.stage_devices[st][1] - pl.stage_devices[st][0]
            micro = -(-prog.micro_batch // r)
            inflight = inflight_depth(prog, dev, pi)
            total += sum(act_bytes[pl.backbone][lo:hi]) * micro * inflight
        out[dev] = int(total)
    return out


def check_plan(prog, model, act_bytes, frozen_specs=None, budget=B200_HBM_BYTES, headroom=0.9):
    """Raise MemoryError when a device of the plan is predicted above `headroom` x `budget`."""
    pred = predict_device_bytes(prog, model, act_bytes, frozen_specs)
    worst = max(pred.values())
    if worst > headroom * budget:
        dev = max(pred, key=pred.get)
        raise MemoryError(f"plan needs {worst / 2**30:.1f} GiB on device {dev} "
                          f"(budget {headroom * budget / 2**30:.1f} GiB)")
    return pred
