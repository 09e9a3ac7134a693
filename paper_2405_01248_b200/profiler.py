"""B200 profiler: emits the reference's `model-profile/v1` document (reference
profile.py:36,76-130,346-363) for a TrainModel, replacing the paper's
"Fig. 6 step 1" on-hardware profiling that the reference swaps
for file ingestion.

* `live_specs` / `frozen_specs`: shape probes (batch 1) of the live set at every
  backbone layer boundary and of every frozen layer's output — the executor
  allocates its P2P buffers from them, and the comm-byte fields come from them
  (the WHOLE live set, not just the hidden state: SURVEY.md §7 "U-Net skip
  connections crossing stage cuts").
* `measure_profile`: per-layer forward / backward times measured with CUDA events
  at every batch key the planner will query (B/r for each replication, the fill
  partial sizes 4..96, remaining/d, up to the group batch).
* `synthetic_profile`: analytic costs (linear in batch) for CPU tests and dry runs.
"""

from __future__ import annotations

import math

import torch

from .pipefill.profile import ComponentProfile, LayerCost, ModelProfile
from .pipefill.filler import VALID_LOCAL_SIZES


def _spec_of(state):
    return {k: (tuple(v.shape[1:]), v.dtype, bool(v.requires_grad)) for k, v in state.items()}


def _bytes_per_sample(spec, grad_only=False):
    tot = 0
    for shape, dt, g in spec.values():
        if grad_only and not g:
            continue
        tot += math.prod(shape) * torch.tensor([], dtype=dt).element_size()
    return tot


def probe_specs(model, batch_fn, device):
    """Run one sample through every layer; returns (live_specs, frozen_specs). Frozen components
    run in dependency order; a dependent component's first layer also sees its producers'
    final outputs (model.frozen_deps: (producer, consumer) index pairs)."""
    from .adapter import topo_order

    deps = getattr(model, "frozen_deps", ())
    frozen_specs = [None] * len(model.frozen)
    finals = {}
    fro = {}
    for c in topo_order(len(model.frozen), deps):
        f = model.frozen[c]
        st = {k: batch_fn(k) for k in f.inputs}
        for s_, d in deps:
            if d == c:
                st.update(finals[s_])
        specs = []
        with torch.no_grad():
            for layer in f.component.layers:
                st = layer(st)
                specs.append({k: (tuple(v.shape[1:]), v.dtype) for k, v in st.items()})
        frozen_specs[c] = specs
        finals[c] = st
        fro.update(st)
    t = batch_fn("t")
    live_all = []
    for pipe, bb in enumerate(getattr(model, "backbones", None) or [model.backbone]):
        nf = model.noise_field(pipe) if hasattr(model, "noise_field") else "noise"
        st, _ = model.stage0_inputs(fro, t, batch_fn(nf), pipe=pipe)
        live = [_spec_of(st)]
        ctx = bb.grad_context() if hasattr(bb, "grad_context") else torch.enable_grad()
        with ctx:
            for layer in bb.layers:
                st = layer(st)
                live.append(_spec_of(st))
        live_all.append(live)
    return live_all, frozen_specs


def _keys(group_batch, D, M, extra=()):
    ks = {1, 2, 3, 4}
    mb = group_batch // M
    for r in range(1, D + 1):
        ks.add(max(1, mb // r))
        ks.add(max(1, -(-mb // r)))
    for d in range(1, D + 1):
        ks.add(max(1, group_batch // d))
        ks.add(max(1, -(-group_batch // d)))
    ks.update(VALID_LOCAL_SIZES)
    ks.update(extra)
    return sorted(k for k in ks if k >= 1)


def synthetic_profile(model, live_specs, frozen_specs, *, group_batch, D, M, fwd_per_sample=1e-3,
                      bwd_factor=2.0, frozen_per_sample=5e-4, backbone_weights=None,
                      frozen_weights=None, names=None):
    """Costs linear in batch: layer j fwd = w_j * fwd_per_sample * b (bwd = bwd_factor x).
    live_specs: per backbone, the probed live sets (a single backbone's list is accepted)."""
    keys = _keys(group_batch, D, M)
    if live_specs and isinstance(live_specs[0], dict):
        live_specs = [live_specs]
    backbones = []
    for bi, bb in enumerate(getattr(model, "backbones", None) or [model.backbone]):
        live = live_specs[bi]
        L = len(bb.layers)
        bw = backbone_weights or [1.0] * L
        layers = []
        for j in range(L):
            out_spec = live[j + 1]
            fb = _bytes_per_sample(out_spec)
            gb = _bytes_per_sample(out_spec, grad_only=True)
            layers.append(LayerCost(
                fwd_time={k: bw[j] * fwd_per_sample * k for k in keys},
                bwd_time={k: bw[j] * bwd_factor * fwd_per_sample * k for k in keys},
                fwd_comm_bytes={k: fb * k for k in keys},
                bwd_comm_bytes={k: gb * k for k in keys},
                grad_bytes={k: 0 for k in keys},
                out_bytes={k: _bytes_per_sample({"out": live[-1]["out"]}) * k for k in keys},
            ))
        backbones.append(ComponentProfile(name=f"{getattr(bb, 'name', 'backbone')}{bi if bi else ''}",
                                          layers=layers, trainable=True))
    frozen = []
    for c, f in enumerate(model.frozen):
        fw = (frozen_weights or {}).get(c) or [1.0] * len(f.component.layers)
        fl = []
        for j, spec in enumerate(frozen_specs[c]):
            ob = sum(math.prod(s) * torch.tensor([], dtype=dt).element_size() for s, dt in spec.values())
            fl.append(LayerCost(
                fwd_time={k: fw[j] * frozen_per_sample * k for k in keys},
                bwd_time={k: 0.0 for k in keys},
                fwd_comm_bytes={k: ob * k for k in keys},
                bwd_comm_bytes={k: 0 for k in keys},
                grad_bytes={k: 0 for k in keys},
                out_bytes={k: ob * k for k in keys},
            ))
        nm = (names or {}).get(c, getattr(f.component, "name", f"frozen{c}"))
        frozen.append(ComponentProfile(name=nm, layers=fl, trainable=False))
    names_ = [c.name for c in frozen]
    deps = tuple((names_[a], names_[b]) for a, b in getattr(model, "frozen_deps", ()))
    return ModelProfile(backbones=tuple(backbones), frozen=tuple(frozen), frozen_deps=deps,
                        selfcond_prob=getattr(model, "selfcond_p", 0.0))


def _param_bytes(component, layer_idx):
    tot = 0
    for p in component.store.params.values():
        if component.layer_of_param(p.name) == layer_idx:
            tot += p.numel * 4
    return tot


def measure_profile(model, live_specs, frozen_specs, make_state, *, group_batch, D, M, reps=3,
                    device="cuda", bb_keys=None, frozen_keys=None):
    """Measured per-layer costs on this GPU (CUDA events, median of `reps` after a warm-up).

    make_state(component_index or ("backbone", pipe), layer, batch) -> input state dict for that
    layer (random tensors of the probed shapes). Every backbone of a two-backbone model is profiled
    and the model's frozen dependencies (producer, consumer) are carried into the profile by name. Backward time of a backbone layer = time of
    torch.autograd.backward over its grad-carrying outputs with unit-random gradients.
    """
    keys = bb_keys or _keys(group_batch, D, M)
    fkeys = frozen_keys or _keys(group_batch, D, M)

    def timed(fn):
        fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b) * 1e-3)
        ts.sort()
        return ts[len(ts) // 2]

    if live_specs and isinstance(live_specs[0], dict):
        live_specs = [live_specs]  # single-backbone form
    backbones = []
    for pipe, bb in enumerate(getattr(model, "backbones", None) or [model.backbone]):
        live = live_specs[pipe]
        layers = []
        for j, fn in enumerate(bb.layers):
            fwd, bwd = {}, {}
            for k in keys:
                st = make_state(("backbone", pipe), j, k)

                def run_f():
                    with bb.grad_context():
                        return fn(dict(st))

                fwd[k] = timed(lambda: run_f())
                spec = live[j + 1]
                names = [n for n in sorted(spec) if spec[n][2]]

                def run_b():
                    out = run_f()
                    ts = [out[n] for n in names if out[n].requires_grad]
                    if ts:
                        torch.autograd.backward(ts, [torch.randn_like(t) for t in ts])

                tb = timed(run_b)
                bwd[k] = max(tb - fwd[k], 1e-7)
                bb.store.zero_grad()
            out_spec = live[j + 1]
            fb = _bytes_per_sample(out_spec)
            gb = _bytes_per_sample(out_spec, grad_only=True)
            pb = _param_bytes(bb, j)
            layers.append(LayerCost(fwd_time=fwd, bwd_time=bwd,
                                    fwd_comm_bytes={k: fb * k for k in keys},
                                    bwd_comm_bytes={k: gb * k for k in keys},
                                    grad_bytes={k: pb for k in keys},
                                    out_bytes={k: _bytes_per_sample({"out": live[-1]["out"]}) * k
                                               for k in keys}))
        backbones.append(ComponentProfile(name=f"{getattr(bb, 'name', 'backbone')}{pipe if pipe else ''}",
                                          layers=layers, trainable=True))
    frozen = []
    for c, f in enumerate(model.frozen):
        fl = []
        for j, fn in enumerate(f.component.layers):
            fwd = {}
            for k in fkeys:
                st = make_state(c, j, k)
                with torch.no_grad():
                    fwd[k] = timed(lambda: fn(dict(st)))
            spec = frozen_specs[c][j]
            ob = sum(math.prod(s) * torch.tensor([], dtype=dt).element_size() for s, dt in spec.values())
            fl.append(LayerCost(fwd_time=fwd, bwd_time={k: 0.0 for k in fkeys},
                                fwd_comm_bytes={k: ob * k for k in fkeys},
                                bwd_comm_bytes={k: 0 for k in fkeys}, grad_bytes={k: 0 for k in fkeys},
                                out_bytes={k: ob * k for k in fkeys}))
        frozen.append(ComponentProfile(name=getattr(f.component, "name", f"frozen{c}"), layers=fl,
                                       trainable=False))
    names_ = [c.name for c in frozen]
    deps = tuple((names_[a], names_[b]) for a, b in getattr(model, "frozen_deps", ()))
    return ModelProfile(backbones=tuple(backbones), frozen=tuple(frozen), frozen_deps=deps,
                        selfcond_prob=getattr(model, "selfcond_p", 0.0))
