"""Public API of the executor: build a configuration's TrainModel, plan it with
the reference planner API (pipefill.planner.evaluate_point, unchanged), adapt
the plan into per-rank programs and run training iterations.

    trainer = engine.Trainer.create("c1", world=1, rank=0, S=1, M=1, D=1)
    loss = trainer.step()          # one pipelined training iteration (host batch -> loss)

Configurations (BASELINE.json configs):
  c1  tiny DiT (4 blocks, d=256) + tiny VAE encoder + tiny text encoder, 128 px, fp32,
      self-conditioning p=0.5
  c2  SD v2.1 U-Net + OpenCLIP ViT-H text (23 layers) + SD VAE encoder, 256 px, bf16
  c3  ControlNet v1.0: trainable ControlNet branch -> locked SD v2.1 decoder (one backbone
      chain); frozen VAE, OpenCLIP-H text, hint map and the LOCKED U-Net encoder (frozen
      dependencies vae->enc, text->enc), 512 px, bf16
  c4  cascaded two-backbone model (CDM): 64 px base U-Net + 256 px super-resolution U-Net
      (bidirectional pipelines), frozen T5-large-shaped encoder (128 tokens) and image pyramid,
      self-conditioning p=0.5 on both pipes, pixel space, bf16
  c5  scaled-up SD U-Net (model channels 512 -> 2.2B parameters) + OpenCLIP-H + SD VAE, 256 px
  *-small  reduced resolution / encoder depth variants of c3..c5 for the parity tests
"""

from __future__ import annotations

import os
from dataclasses import dataclass, replace

import torch

from . import ops as kops
from .adapter import build_group_program
from .diffusion import DataSpec, make_batch, noise_schedule
from .networks import (CLIPTextEncoder, ControlNet, HintImage, ImagePyramid, LockedUNetEncoder, SDUNet,
                       SDVAEEncoder, T5Encoder, TinyDiT, TinyTextEncoder, TinyVAEEncoder)
from .nn import grad_anchor
from .pipefill import filler, planner, profile as pprof, scheduler
from .profiler import probe_specs, synthetic_profile
from .runtime import FrozenSpec, PipelineExecutor, TrainModel


@dataclass(frozen=True)
class ConfigSpec:
    name: str
    dtype: torch.dtype
    image: int
    latent: int
    text_len: int
    vocab: int
    selfcond_p: float
    config_id: int
    zc: int = 4
    extra: tuple = ()   # extra batch fields (diffusion.DataSpec.extra)
    family: str = ""    # model family (defaults to name)
    depth: int = 0      # text-encoder depth override (small variants)


# Bubbles shorter than this are not filled. The reference default (scheduler.py MIN_BUBBLE_LEN,
# 10 ms) was tuned for A100 layer times; on B200 a U-Net stage of one micro-batch
# runs in a few ms and kernel launches cost microseconds, so the executor passes 2 ms through the
# planner's own `bubble_min_len` argument (measured c2 profile, S=D=4, M=4: predicted speedup over
# the unfilled pipeline 1.12x at 10 ms, 1.18x at 2 ms; tests/test_c5_plan.py).
B200_BUBBLE_MIN_LEN = 0.002

_C = torch.bfloat16
CONFIGS = {
    "c1": ConfigSpec("c1", torch.float32, 128, 32, 16, 1000, 0.5, 1),
    "c2": ConfigSpec("c2", _C, 256, 32, 77, 49408, 0.0, 2),
    "c3": ConfigSpec("c3", _C, 512, 64, 77, 49408, 0.0, 3, extra=(("hint", "bernoulli", 512, 3),)),
    "c4": ConfigSpec("c4", _C, 256, 64, 128, 32128, 0.5, 4, zc=3, extra=(("noise_sr", "noise", 256, 3),)),
    "c5": ConfigSpec("c5", _C, 256, 32, 77, 49408, 0.0, 5),
    "c3-small": ConfigSpec("c3-small", _C, 128, 16, 77, 49408, 0.0, 3, extra=(("hint", "bernoulli", 128, 3),),
                           family="c3", depth=2),
    "c4-small": ConfigSpec("c4-small", _C, 64, 16, 16, 32128, 0.5, 4, zc=3,
                           extra=(("noise_sr", "noise", 64, 3),), family="c4", depth=2),
    "c5-small": ConfigSpec("c5-small", _C, 128, 16, 77, 49408, 0.0, 5, family="c5", depth=2),
}

# model-size parameters of the cascaded configuration (c4): pixel-space U-Nets
CDM_BASE = dict(mc=192, mult=(1, 2, 3, 4), attn_levels=(1, 2, 3))
CDM_SR = dict(mc=128, mult=(1, 2, 4, 4), attn_levels=(3,))
C5_MC = 512


def _attach_grad_context(comp, device):
    comp.grad_context = lambda: grad_anchor(True, device)
    return comp


def build_model(cfg: str | ConfigSpec, device="cuda", seed=0, states=None, small=False):
    """Materialise the components of a configuration on `device` (deterministic init).
    `states` optionally maps component name -> parameter dict (e.g. for parity tests)."""
    c = CONFIGS[cfg] if isinstance(cfg, str) else cfg
    states = states or {}
    fam = c.family or c.name
    if fam in ("c3", "c4", "c5"):
        return _build_ext(c, fam, device, seed, states)
    if c.name == "c1":
        bb = TinyDiT(c.dtype, img=c.latent, cin=8, cout=4)
        vae = TinyVAEEncoder(c.dtype)
        txt = TinyTextEncoder(c.dtype)
        sc_ch = 4
    elif c.name == "c2":
        bb = SDUNet(c.dtype)
        vae = SDVAEEncoder(c.dtype)
        txt = CLIPTextEncoder(c.dtype, layers=2 if small else 23)
        sc_ch = 0
    else:
        raise KeyError(c.name)
    for comp in (bb, vae, txt):
        comp.materialize(device, seed, states.get(comp.name))
    _attach_grad_context(bb, device)
    sab, s1m = noise_schedule()
    model = TrainModel(bb, [FrozenSpec(vae, ("images",)), FrozenSpec(txt, ("ids",))], kops,
                       sab.to(device), s1m.to(device), selfcond_channels=sc_ch,
                       adamw=dict(lr=1e-4, betas=(0.9, 0.999), eps=1e-8, weight_decay=0.01))
    model.selfcond_p = c.selfcond_p
    model.cfg = c
    return model


def _finish(model, c, device, comps, seed, states):
    for comp in comps:
        comp.materialize(device, seed, states.get(comp.name))
    for bb in model.backbones:
        _attach_grad_context(bb, device)
    model.cfg = c
    model.selfcond_p = c.selfcond_p
    return model


def _build_ext(c, fam, device, seed, states):
    """c3 (ControlNet), c4 (cascaded two-backbone), c5 (2.2B U-Net)."""
    sab, s1m = noise_schedule()
    sab, s1m = sab.to(device), s1m.to(device)
    adam = dict(lr=1e-4, betas=(0.9, 0.999), eps=1e-8, weight_decay=0.01)
    depth = c.depth or 23
    if fam == "c5":
        bb = SDUNet(c.dtype, mc=C5_MC)
        vae, txt = SDVAEEncoder(c.dtype), CLIPTextEncoder(c.dtype, layers=depth)
        model = TrainModel(bb, [FrozenSpec(vae, ("images",)), FrozenSpec(txt, ("ids",))], kops, sab, s1m,
                           adamw=adam)
        return _finish(model, c, device, (bb, vae, txt), seed, states)
    if fam == "c3":
        locked = SDUNet(c.dtype, trainable=False, name="unet_locked")
        enc = LockedUNetEncoder(locked)
        enc.sqrt_ab, enc.sqrt_1mab = sab, s1m
        bb = ControlNet(locked, c.dtype)
        vae, txt, hint = SDVAEEncoder(c.dtype), CLIPTextEncoder(c.dtype, layers=depth), HintImage(c.dtype)
        frozen = [FrozenSpec(vae, ("images",)), FrozenSpec(txt, ("ids",)), FrozenSpec(hint, ("hint",)),
                  FrozenSpec(enc, ("t", "noise"))]
        model = TrainModel(bb, frozen, kops, sab, s1m, adamw=adam)
        model.frozen_deps = ((0, 3), (1, 3))
        return _finish(model, c, device, (bb, vae, txt, hint, enc), seed, states)
    # c4: cascaded diffusion, two backbones sharing the frozen outputs
    sc = 3 if c.selfcond_p > 0 else 0
    base = SDUNet(c.dtype, cin=3 + sc, cout=3, name="unet_base", **CDM_BASE)
    sr = SDUNet(c.dtype, cin=6 + sc, cout=3, name="unet_sr", **CDM_SR)
    t5 = T5Encoder(c.dtype, vocab=c.vocab, L=c.text_len, layers=c.depth or 24)
    pyr = ImagePyramid(c.dtype, factor=c.image // c.latent)
    io = [dict(latent="latent", noise="noise", cond=None, drop=("img_sr", "lowres")),
          dict(latent="img_sr", noise="noise_sr", cond="lowres", drop=("latent",))]
    model = TrainModel(base, [FrozenSpec(pyr, ("images",)), FrozenSpec(t5, ("ids",))], kops, sab, s1m,
                       selfcond_channels=sc, adamw=adam, backbones=[base, sr], pipe_io=io)
    return _finish(model, c, device, (base, sr, pyr, t5), seed, states)


class InputFeed:
    """Batch fields for one iteration. mode 'device': the whole world batch is resident on
    the device (bench `value`); mode 'host': slices are copied from pinned host memory
    when used (bench `e2e`), and the copied bytes are counted (per feed and globally in
    InputFeed.h2d_total)."""

    h2d_total = 0

    def __init__(self, batch, device, dtype, mode="device"):
        self.device = torch.device(device)
        self.dtype = dtype
        self.mode = mode
        self.h2d_bytes = 0
        fields = batch.fields()
        if mode == "device":
            self.f = {k: self._cast(k, v.to(self.device, non_blocking=True)) for k, v in fields.items()}
        else:
            self.f = {k: (v.pin_memory() if self.device.type == "cuda" else v) for k, v in fields.items()}
        self.selfcond = batch.selfcond

    def _cast(self, k, v):
        if v.is_floating_point() and k != "t" and v.dtype != self.dtype:
            return v.to(self.dtype)
        return v

    def stage(self, fields, stream):
        """Host mode: start the H2D copies of whole `fields` on `stream` now (pinned memory ->
        device); later `get`s of those fields wait on the copy event instead of copying inline, so
        the transfer overlaps compute (the bytes still count as this step's H2D traffic)."""
        if self.mode != "host" or self.device.type != "cuda":
            return
        self.staged = getattr(self, "staged", {})
        with torch.cuda.stream(stream):
            for k in fields:
                if k in self.f and k not in self.staged:
                    v = self.f[k].to(self.device, non_blocking=True)
                    n = v.numel() * v.element_size()
                    self.h2d_bytes += n
                    InputFeed.h2d_total += n
                    self.staged[k] = v
            self.staged_ev = torch.cuda.Event()
            self.staged_ev.record(stream)

    def get(self, k, lo, hi):
        st = getattr(self, "staged", None)
        if st and k in st:
            cur = torch.cuda.current_stream(self.device)
            cur.wait_event(self.staged_ev)
            v = st[k]
            v.record_stream(cur)
            return self._cast(k, v[lo:hi])
        v = self.f[k][lo:hi]
        if self.mode == "host":
            v = v.to(self.device, non_blocking=True)
            self.h2d_bytes += v.numel() * v.element_size()
            InputFeed.h2d_total += v.numel() * v.element_size()
            v = self._cast(k, v)
        return v

    def t(self, lo, hi):
        return self.get("t", lo, hi)

    def noise(self, lo, hi):
        return self.get("noise", lo, hi)


def plan_programs(prof, world, S, M, D, world_batch, frozen_counts, bubble_min_len=B200_BUBBLE_MIN_LEN,
                  cluster_comm=None):
    """Reference planner calls -> {selfcond: GroupProgram} plus the warm-up program."""
    comm = cluster_comm or pprof.CommCosts(2.0e11, 2e-5, 3.0e11, 1e-5)
    cluster = pprof.ClusterConfig(world, comm)
    res = planner.evaluate_point(prof, cluster, S, M, D, world_batch, bubble_min_len=bubble_min_len)
    plan = res["plan"]
    group_batch = plan.config.global_batch
    deps = tuple(prof.frozen_dep_indices())
    programs = {}
    if res["mode"] == planner.MODE_BIDIRECTIONAL and prof.selfcond_prob > 0:
        # two backbones with self-conditioning: the reference's bidirectional schedule has no
        # fwd_sc tasks (planner.py:115-118). Default: the opt-in planner extension simulates both
        # pipes WITH the pass (planning_ext) so that fills are placed against the
        # schedule the executor runs; DP_SC_OUTSIDE_PLAN=1 keeps the reference schedule and runs
        # the pass ahead of the planned tasks instead
        if os.environ.get("DP_SC_OUTSIDE_PLAN", "0") == "1":
            programs[True] = build_group_program(res, frozen_counts, selfcond=True, frozen_deps=deps)
        else:
            from .planning_ext import evaluate_point_selfcond

            res_sc = evaluate_point_selfcond(prof, cluster, S, M, D, world_batch, bubble_min_len=bubble_min_len)
            programs[True] = build_group_program(res_sc, frozen_counts, selfcond=True, frozen_deps=deps)
            programs[True].plan_result = res_sc
        programs[False] = build_group_program(res, frozen_counts, selfcond=False, frozen_deps=deps)
    elif res["mode"] == planner.MODE_SELFCOND:
        programs[True] = build_group_program(res, frozen_counts, selfcond=True, frozen_deps=deps)
        pre = scheduler.build_schedule(plan, prof, cluster, selfcond=False)
        fill = filler.fill_all(scheduler.extract_bubbles(pre, bubble_min_len), prof, group_batch, pre)
        programs[False] = build_group_program(dict(plan=plan, pre_fill_schedule=pre, fill=fill),
                                              frozen_counts, selfcond=False, frozen_deps=deps)
    else:
        programs[False] = build_group_program(res, frozen_counts, selfcond=False, frozen_deps=deps)
        programs[True] = programs[False]
    pre = res["pre_fill_schedule"]
    warm = filler.fill_all([], prof, group_batch, pre)
    warm_prog = build_group_program(dict(plan=plan, pre_fill_schedule=pre, fill=warm), frozen_counts,
                                    selfcond=False, frozen_deps=deps)
    unfilled = build_group_program(dict(plan=plan, pre_fill_schedule=pre, fill=warm), frozen_counts,
                                   selfcond=False, frozen_deps=deps)
    return res, programs, warm_prog, unfilled


class Trainer:
    """One rank of a pipelined training job."""

    def __init__(self, model, cfg, executor, data_spec, device, feed_mode="device"):
        self.model, self.cfg, self.ex, self.data_spec = model, cfg, executor, data_spec
        self.device = device
        self.it = 0
        self.feed_mode = feed_mode
        self._next = None

    @classmethod
    def create(cls, cfg="c1", *, world=1, rank=0, S=1, M=1, D=1, world_batch=None, device=None,
               seed=0, states=None, profile=None, filled=True, feed_mode="device", small=False,
               bubble_min_len=B200_BUBBLE_MIN_LEN, comm=None, program_file=None):
        c = CONFIGS[cfg] if isinstance(cfg, str) else cfg
        device = device or (f"cuda:{torch.cuda.current_device()}" if torch.cuda.is_available() else "cpu")
        model = build_model(c, device, seed, states, small=small)
        world_batch = world_batch or 8 * world
        ds = DataSpec(c.config_id, world_batch, c.image, c.latent, c.zc, c.text_len, c.vocab, 1000,
                      c.selfcond_p, extra=c.extra)
        return cls.from_model(model, c, ds, world=world, rank=rank, S=S, M=M, D=D, device=device,
                              profile=profile, filled=filled, feed_mode=feed_mode,
                              bubble_min_len=bubble_min_len, comm=comm, program_file=program_file)

    @classmethod
    def from_model(cls, model, cfg, ds, *, world=1, rank=0, S=1, M=1, D=1, device="cuda", profile=None,
                   filled=True, feed_mode="device", bubble_min_len=B200_BUBBLE_MIN_LEN, comm=None,
                   check_memory=None, program_file=None):
        """Plan and wire an already-built TrainModel (any component implementation).
        check_memory (default: on CUDA devices): gate the plan with the memory-feasibility model
        (memory.check_plan raises MemoryError before the first step when a device would overflow)."""
        world_batch = ds.world_batch
        probe = make_batch(replace(ds, world_batch=1), 10 ** 6)
        pfeed = InputFeed(probe, device, cfg.dtype)
        live, fspecs = probe_specs(model, lambda k: pfeed.get(k, 0, 1), device)  # per backbone
        counts = [len(f.component.layers) for f in model.frozen]
        if profile is None:
            profile = synthetic_profile(model, live, fspecs, group_batch=world_batch * D // world, D=D, M=M)
        if program_file is not None:
            # a shipped per-rank program (adapter.save_rank_programs): no planning on this rank
            from .adapter import load_rank_program

            prank, docs = load_rank_program(program_file)
            if prank != rank:
                raise ValueError(f"{program_file} holds the program of rank {prank}, not {rank}")
            res, warm = None, docs["warmup"]
            programs = {False: docs["plain"], True: docs["selfcond"]}
        else:
            res, programs, warm, unfilled = plan_programs(profile, world, S, M, D, world_batch, counts,
                                                          bubble_min_len, comm)
            if not filled:
                programs = {False: unfilled, True: unfilled}
        # per pipe: mean squared error over that pipe's noise tensor (two-backbone models sum them)
        scales = [1.0 / (world_batch * pfeed.get(model.noise_field(p), 0, 1).numel())
                  for p in range(len(model.backbones))]
        ex = PipelineExecutor(model, programs, rank=rank, world=world, device=device, live_specs=live,
                              frozen_specs=fspecs, loss_scale=scales if len(scales) > 1 else scales[0],
                              warm_program=warm)
        ex.plan_result = res
        t = cls(model, cfg, ex, ds, device, feed_mode)
        t.profile = profile
        if check_memory is None:
            check_memory = torch.device(device).type == "cuda"
        if check_memory:
            t.memory_report(check=True)
        return t

    def save_programs(self, directory):
        """Ship this job's plan as one program file per rank (adapter.PROGRAM_FORMAT: per-device
        instruction order, frozen pieces with sample ranges, transfers; the plain, self-conditioned
        and warm-up programs); Trainer.create(..., program_file=<dir>/rank<r>.json) runs it."""
        from .adapter import save_rank_programs

        ex = self.ex
        progs = {"plain": ex.programs[False], "selfcond": ex.programs[True], "warmup": ex.warm_program}
        return save_rank_programs(ex.prog0, directory, groups=ex.world // ex.D, programs=progs)

    def prefetch(self, n, mode=None):
        """Pre-build the feeds of iterations [it, it + n] (device-resident or pinned host)
        so that no batch synthesis happens inside a timed region."""
        mode = mode or self.feed_mode
        self._prefetched = {i: InputFeed(make_batch(self.data_spec, i), self.device, self.cfg.dtype, mode)
                            for i in range(self.it, self.it + n + 1)}

    def _feed(self, i):
        pre = getattr(self, "_prefetched", None)
        if pre and i in pre:
            return pre.pop(i)
        return InputFeed(make_batch(self.data_spec, i), self.device, self.cfg.dtype, self.feed_mode)

    # ------------------------------------------------------------------ CUDA graphs (world 1)
    def enable_cuda_graph(self):
        """Capture one steady-state iteration (U-Net fwd/bwd, AdamW, next batch's frozen
        encoders) into a CUDA graph and replay it from then on. Single GPU only (the pipeline
        programs of N > 1 interleave NCCL P2P); needs a fixed self-conditioning branch."""
        from .runtime import _Streams
        from . import telemetry

        if self.ex.world != 1 or self.cfg.selfcond_p not in (0.0, 1.0):
            raise ValueError("CUDA-graph replay needs world == 1 and a fixed self-conditioning branch")
        if self.it == 0 and not self.ex.frozen_ready:
            self.warmup_frozen()
        # multi-stream capture: the executor's compute stream forks from the capturing stream and the
        # optimizer stream from compute events, so the AdamW slices stay overlapped with the backward
        # inside the graph (DP_GRAPH_SINGLE_STREAM=1: everything on the capture stream)
        if os.environ.get("DP_GRAPH_SINGLE_STREAM", "0") != "0":
            self.ex.streams = _Streams(self.ex.device, single=True)
        torch.cuda.synchronize()
        self._g_cur = InputFeed(make_batch(self.data_spec, self.it), self.device, self.cfg.dtype, "device")
        self._g_nxt = InputFeed(make_batch(self.data_spec, self.it + 1), self.device, self.cfg.dtype, "device")
        # refresh the eager state so that frozen_ready holds batch `it` (capture executes nothing)
        g_in = self.ex.frozen_ready
        cur, nxt = self._g_cur, self._g_nxt
        gb = self.ex.gb_of()
        graph = torch.cuda.CUDAGraph()
        side = torch.cuda.Stream(device=self.device)
        side.wait_stream(torch.cuda.current_stream(self.device))
        n0 = telemetry.total_launches()
        with torch.cuda.stream(side):
            self.ex.inputs = cur
            with torch.cuda.graph(graph, stream=side):
                loss = self.ex.run_iteration(lambda f, lo, hi: nxt.get(f, gb + lo, gb + hi),
                                             cur.selfcond, has_next=True)
        torch.cuda.current_stream(self.device).wait_stream(side)
        self._graph_launches = telemetry.total_launches() - n0
        self._graph = graph
        self._graph_loss = loss
        self._graph_in = g_in
        self._graph_out = self.ex.frozen_ready
        self.ex.frozen_ready = g_in

    def _graph_step(self):
        from . import telemetry

        cur_b = self._feed(self.it)
        nxt_b = self._feed(self.it + 1)
        # every field the captured iteration reads: the current batch's fields (t, noise, extra
        # fields such as a second pipe's noise) and every frozen component's inputs of the next batch
        # (images, ids, ControlNet hint, the locked encoder's t / noise)
        for k in self._g_cur.f:
            self._g_cur.f[k].copy_(cur_b.get(k, 0, cur_b.f[k].shape[0]), non_blocking=True)
        for k in sorted({f for spec in self.model.frozen for f in spec.inputs}):
            self._g_nxt.f[k].copy_(nxt_b.get(k, 0, nxt_b.f[k].shape[0]), non_blocking=True)
        self._graph.replay()
        # frozen outputs of batch it+1 (graph outputs) -> the buffers the next replay reads
        for c, pieces in self._graph_out.items():
            for (a, b, st), (a2, b2, st2) in zip(pieces, self._graph_in[c]):
                for k in st:
                    st2[k].copy_(st[k], non_blocking=True)
        telemetry.count("cuda_graph_replay", self._graph_launches)
        self.it += 1
        return self._graph_loss

    def warmup_frozen(self):
        self._cur = self._feed(self.it)
        self.ex.warmup(lambda f, lo, hi: self._cur.get(f, self.ex.gb_of() + lo, self.ex.gb_of() + hi))

    def step(self, has_next=True, trace=False):
        """One iteration: train on batch `it` (frozen outputs ready), fill batch it+1.
        trace=True records measured task intervals (see `measured`)."""
        if getattr(self, "_graph", None) is not None and has_next and not trace:
            return self._graph_step()
        if self.it == 0 and not self.ex.frozen_ready:
            self.warmup_frozen()
        cur = self._cur
        nxt = self._feed(self.it + 1) if has_next else None
        if nxt is not None and nxt.mode == "host" and self.ex.world == 1 and self.ex.streams.cuda:
            # the next batch's encoder inputs are consumed by this iteration's fills / tail
            if getattr(self, "_copy_stream", None) is None:
                self._copy_stream = torch.cuda.Stream(device=self.ex.device)
            nxt.stage([f for spec in self.model.frozen for f in spec.inputs], self._copy_stream)
        self.ex.inputs = cur
        gb = self.ex.gb_of()
        raw = (lambda f, lo, hi: nxt.get(f, gb + lo, gb + hi)) if nxt is not None else None
        loss = self.ex.run_iteration(raw, cur.selfcond, has_next=has_next, trace=trace)
        self._cur = nxt
        self.it += 1
        return loss

    def memory_report(self, batch=2, check=False):
        """Predicted bytes per device of this rank's pipeline group (memory.py: parameters, frozen
        weights, activations kept for the backward x micro-batches in flight, held frozen outputs):
        the maximum over the iteration programs the executor may run. check=True raises MemoryError
        when a device exceeds the B200 budget (memory.check_plan)."""
        from . import memory

        act = getattr(self, "_act_bytes", None)
        if act is None:
            probe = make_batch(replace(self.data_spec, world_batch=batch), 10 ** 6 + 1)
            feed = InputFeed(probe, self.device, self.cfg.dtype)
            act = memory.measure_layer_activation_bytes(self.model, lambda k, b: feed.get(k, 0, b), self.device,
                                                        batch)
            self._act_bytes = act
        out = {}
        for prog in {id(p): p for p in self.ex.programs.values()}.values():
            fn = memory.check_plan if check else memory.predict_device_bytes
            for d, v in fn(prog, self.model, act, self.ex.frozen_specs).items():
                out[d] = max(out.get(d, 0), v)
        return out

    def measured(self, min_len=0.0):
        """Measured schedule of the last traced step (collective over the job): returns
        (Schedule, bubbles, bubble_ratio) computed with the planner's own extract_bubbles /
        bubble_ratio (reference scheduler.py:395,434) on barrier-aligned task times; the tail
        counts as busy (planner.py:172-175)."""
        sched = self.ex.measured_schedule()
        bubbles = scheduler.extract_bubbles(sched, min_len)
        return sched, bubbles, scheduler.bubble_ratio(sched, bubbles)
