"""Pipelined training executor: replays the planner's schedule on real devices.

One process per GPU (torch.distributed; NCCL on B200, gloo for CPU tests).
Rank r = group * D + local device; group g is one pipeline replica of the
planner's D-device group (reference planner.py:10-15,151-158).

Per iteration i (cross-iteration filling):
  * the backbone trains on batch i, whose frozen outputs (latents, context) were
    computed during iteration i-1 (iteration 0 is preceded by a warm-up frozen pass);
  * every rank executes its DeviceProgram (adapter.py) in order:
      fwd / fwd_sc / bwd  on the high-priority compute stream, live sets moving by P2P
      fill                on the low-priority fill stream, gated on the event of the
                          compute task that precedes the bubble; frozen work for batch i+1
      sync                per-stage flat-gradient allreduce + flat AdamW
      tail, deliver       leftover frozen work, then frozen outputs -> stage-0 owners.

P2P uses one 2-rank process group per (kind, src, dst) so that every link is a FIFO
whose send and receive orders agree by construction: forward activations, backward
gradients, self-conditioning feedback and frozen transfers never share a queue.

Compute is abstracted by `TrainModel` (backbone + frozen components with layer lists);
the executor itself never touches kernels, so the same control plane runs on CPU/gloo in
tests with torch-op layers and on B200 with the libdpipe components.
"""

from __future__ import annotations

import contextlib
import time
from dataclasses import dataclass

import torch
import torch.distributed as dist

from .adapter import GroupProgram, backbone_transfers, input_layers, split_range

# ============================================================================ model bundle


@dataclass
class FrozenSpec:
    component: object            # networks.Component (or a test double): .layers, .run
    inputs: tuple                # raw batch fields consumed by layer 0 ("images" / "ids")


class TrainModel:
    """Backbone + frozen components + diffusion glue, independent of placement.

    `ops` provides the few fused kernels the glue needs (q_sample, pred_x0, mse,
    concat); on B200 it is paper_2405_01248_b200.ops, in CPU tests a torch stand-in.
    """

    def __init__(self, backbone, frozen, ops, sqrt_ab, sqrt_1mab, selfcond_channels=0,
                 grad_scale=1.0, adamw=None, backbones=None, pipe_io=None):
        self.backbone = backbone
        self.backbones = list(backbones) if backbones else [backbone]
        # per backbone: which frozen output is x0, which batch field is its noise and which
        # frozen output (if any) is concatenated as conditioning (cascaded super-resolution)
        self.pipe_io = pipe_io or [dict(latent="latent", noise="noise", cond=None)] * len(self.backbones)
        self.frozen = frozen
        self.ops = ops
        self.sqrt_ab = sqrt_ab
        self.sqrt_1mab = sqrt_1mab
        self.sc_ch = selfcond_channels
        self.adamw = adamw or {}

    # -- stage 0 input construction ------------------------------------------------------
    def stage0_inputs(self, frozen_out, t, noise, x0_sc=None, pipe=0):
        """frozen_out: merged dict of frozen outputs (latent, ctx, pooled) for these samples.
        `pipe` selects the backbone of a two-backbone (bidirectional) model; both backbones of
        a cascaded model share the frozen outputs and the noise draw."""
        o = self.ops
        io = self.pipe_io[pipe]
        x0 = frozen_out[io["latent"]]
        xt = o.q_sample(x0, noise, t, self.sqrt_ab, self.sqrt_1mab)
        x = xt
        if io.get("cond"):
            x = o.concat_last(x, frozen_out[io["cond"]])
        if self.sc_ch:
            sc = x0_sc if x0_sc is not None else torch.zeros_like(xt)
            x = o.concat_last(x, sc)
        st = {"x": x, "t": t, "noise": noise}
        skip = {io["latent"], io.get("cond")} | set(io.get("drop", ()))
        for k, v in frozen_out.items():
            if k not in skip:
                st[k] = v
        return st, xt

    def noise_field(self, pipe=0):
        return self.pipe_io[pipe]["noise"]


# ============================================================================ helpers


def _cat(parts):
    parts = [p for p in parts if p is not None]
    if len(parts) == 1:
        return parts[0]
    return torch.cat(parts, 0)


_ALIGN = 16


def _seg_bytes(shape, dtype, n):
    """Bytes of n samples of a per-sample `shape` tensor, padded to the packing alignment."""
    nb = n * int(torch.Size(shape).numel()) * torch.empty((), dtype=dtype).element_size()
    return -(-nb // _ALIGN) * _ALIGN


def pack(tensors):
    """One flat byte buffer holding `tensors` back to back (16-byte aligned segments): a live set
    or a frozen activation crosses a link as ONE message instead of one per tensor."""
    parts = []
    for t in tensors:
        b = t.detach().contiguous().reshape(-1).view(torch.uint8)
        parts.append(b)
        pad = -b.numel() % _ALIGN
        if pad:
            parts.append(torch.zeros(pad, dtype=torch.uint8, device=t.device))
    return parts[0] if len(parts) == 1 else torch.cat(parts)


def unpack(flat, layout, n):
    """Views into a received flat buffer: layout = [(name, per-sample shape, dtype)] in packing
    order, n samples each (no copies)."""
    out, off = {}, 0
    for name, shape, dt in layout:
        nb = _seg_bytes(shape, dt, n)
        numel = n * int(torch.Size(shape).numel())
        esz = torch.empty((), dtype=dt).element_size()
        out[name] = flat[off:off + numel * esz].view(dt).view((n,) + tuple(shape))
        off += nb
    return out


def packed_bytes(layout, n):
    return sum(_seg_bytes(shape, dt, n) for _, shape, dt in layout)


class _Streams:
    def __init__(self, device, single=False):
        self.cuda = device.type == "cuda" and not single
        if self.cuda:
            self.compute = torch.cuda.Stream(device=device, priority=-1)
            self.fill = torch.cuda.Stream(device=device, priority=0)
        else:
            self.compute = self.fill = None

    def on(self, which):
        if not self.cuda:
            return contextlib.nullcontext()
        return torch.cuda.stream(self.compute if which == "compute" else self.fill)

    def event(self, which):
        if not self.cuda:
            return None
        ev = torch.cuda.Event()
        ev.record(self.compute if which == "compute" else self.fill)
        return ev

    def wait(self, which, ev):
        if ev is None or not self.cuda:
            return
        (self.compute if which == "compute" else self.fill).wait_event(ev)

    def join(self):
        if self.cuda:
            self.compute.wait_stream(self.fill)

    def record(self, t, which):
        if self.cuda and t is not None and t.is_cuda:
            t.record_stream(self.compute if which == "compute" else self.fill)


class _StagedRecv:
    """Work handle of a host-staged receive: completes the gloo receive, then copies to the device."""

    def __init__(self, work, host, dst):
        self.work, self.host, self.dst = work, host, dst

    def wait(self):
        self.work.wait()
        self.dst.copy_(self.host)


def staged():
    """TEST transport: gloo cannot move CUDA tensors point-to-point, so the multi-process GPU
    tests (several ranks sharing one GPU) stage P2P and allreduce through host memory. The
    product transport is NCCL (device buffers, NVLink)."""
    return dist.is_initialized() and dist.get_backend() == "gloo" and torch.cuda.is_available()


class Links:
    """2-rank process groups per (kind, src, dst); kinds: fwd, bwd, fb (self-cond feedback), frz."""

    def __init__(self, rank, world, needed):
        self.rank = rank
        self.pg = {}
        self.staged = world > 1 and staged()
        if world == 1:
            return
        for key in sorted(needed):
            kind, a, b = key
            g = dist.new_group(ranks=sorted({a, b}))
            self.pg[key] = g

    def isend(self, kind, t, dst):
        if _DEBUG:
            print(f"[r{self.rank}] send {kind} -> {dst} {tuple(t.shape)}", flush=True)
        if self.staged and t.is_cuda:
            t = t.detach().to("cpu")
        return dist.isend(t.contiguous(), dst=dst, group=self.pg[(kind, self.rank, dst)])

    def irecv(self, kind, t, src):
        if _DEBUG:
            print(f"[r{self.rank}] recv {kind} <- {src} {tuple(t.shape)}", flush=True)
        if self.staged and t.is_cuda:
            host = torch.empty(t.shape, dtype=t.dtype)
            return _StagedRecv(dist.irecv(host, src=src, group=self.pg[(kind, src, self.rank)]), host, t)
        return dist.irecv(t, src=src, group=self.pg[(kind, src, self.rank)])


_DEBUG = bool(int(__import__("os").environ.get("DP_DEBUG_P2P", "0")))
_OVL_SIDE = __import__("os").environ.get("DP_OVL_STREAM", "opt") == "opt"  # experiments: "compute"
_EARLY_TAIL = bool(int(__import__("os").environ.get("DP_EARLY_TAIL", "0")))  # experiments
# single-device frozen tail (no transfers) replayed as one CUDA graph per (program, tail): the ~350 launches of
# the next batch's VAE + text-encoder forwards leave the host's critical path (DP_TAIL_GRAPH=0: eager)
_TAIL_GRAPH = bool(int(__import__("os").environ.get("DP_TAIL_GRAPH", "1")))
# DP_LATE_OPT_JOIN=1: the compute stream joins the optimizer stream at the end of the iteration instead of
# at the sync task. Off by default: measured neutral at N=1, and with per-slice gradient snapshots on (the
# parity tests) c2 iterations hung in the device synchronize with it on (tools/hang_probe.py: 2 of 3 snapshot
# runs, and the c2 parity / optimizer-overlap test files; the run with it off completed;
# profiles/r02_hang_probe.txt)
_LATE_OPT_JOIN = bool(int(__import__("os").environ.get("DP_LATE_OPT_JOIN", "0")))


class _Tracer:
    """Measured per-task times of one iteration on this rank (SURVEY §8d "measured bubble
    ratio"): CUDA events on the stream each task runs on (host clock on CPU), relative to an
    origin recorded on the compute stream when the iteration starts. `tasks()` returns
    pipefill `Task`s in seconds so the planner's own `extract_bubbles` / `bubble_ratio`
    (scheduler.py:395,434 of the reference) can be applied to the measured schedule."""

    def __init__(self, streams, dev):
        self.streams, self.dev = streams, dev
        self.recs = []
        self.cuda = streams.cuda
        if self.cuda:
            self.t0 = torch.cuda.Event(enable_timing=True)
            self.t0.record(streams.compute)
        else:
            self.t0 = time.perf_counter()

    def _mark(self, which):
        if not self.cuda:
            return time.perf_counter()
        ev = torch.cuda.Event(enable_timing=True)
        ev.record(self.streams.compute if which == "compute" else self.streams.fill)
        return ev

    @contextlib.contextmanager
    def task(self, which, kind, m=None, s=None, direction="down", tag=""):
        a = self._mark(which)
        yield
        self.recs.append((kind, m, s, direction, tag, a, self._mark(which)))

    def tasks(self):
        from .pipefill.scheduler import Task

        out = []
        if self.cuda:
            self.streams.compute.synchronize()
            self.streams.fill.synchronize()
        for kind, m, s, d, tag, a, b in self.recs:
            if self.cuda:
                ta, tb = self.t0.elapsed_time(a) * 1e-3, self.t0.elapsed_time(b) * 1e-3
            else:
                ta, tb = a - self.t0, b - self.t0
            out.append(Task(self.dev, kind, m, s, d, max(0.0, ta), max(0.0, tb), tag))
        return out


# ============================================================================ executor


class PipelineExecutor:
    OVERLAP_CTAS = int(__import__("os").environ.get("DP_OVL_CTAS", "296"))  # grid cap of AdamW chunks next to the backward
    def __init__(self, model: TrainModel, programs: dict, *, rank=0, world=1, device="cuda",
                 live_specs=None, frozen_specs=None, loss_scale=1.0, inputs=None, warm_program=None):
        """programs: {False: GroupProgram, True: GroupProgram (self-cond activated)} built from
        the same partition; `inputs` provides host/device batch slices (InputFeed).
        live_specs: per pipe (backbone) a list over layer boundaries of {name: (shape, dtype, grad)}."""
        self.model = model
        self.programs = programs
        self.prog0 = programs[False]
        self.warm_program = warm_program  # iteration-0 frozen pass (its links are created up front)
        self.rank, self.world = rank, world
        self.D = self.prog0.D
        self.group, self.dev = divmod(rank, self.D)
        self.device = torch.device(device)
        self.streams = _Streams(self.device)
        self.npipes = len(self.prog0.pipes)
        if live_specs is not None and live_specs and isinstance(live_specs[0], dict):
            live_specs = [live_specs]  # single-backbone form
        self.live_specs = live_specs
        self.frozen_specs = frozen_specs  # [comp][layer] -> {name: (shape, dtype)}
        self.loss_scale = loss_scale
        self.inputs = inputs
        p = self.prog0.device_program(self.dev)
        self.stages = list(p.stages) if p.stages else [p.stage]
        self.stage, self.replica = self.stages[0], p.replica
        self.param_ranges = []
        for pi, st in enumerate(self.stages):
            if st is None:
                self.param_ranges.append(None)
                continue
            lo, hi = self.prog0.pipes[pi].stage_ranges[st]
            self.param_ranges.append(self._backbone(pi).stage_slice(lo, hi))
        self.param_range = self.param_ranges[0]
        self.links = Links(rank, world, self._needed_links())
        self._stage_pgs = self._make_stage_groups()
        self.frozen_ready = {}   # for the NEXT iteration: comp -> list[(lo, hi, state)] on stage-0 owners
        self.loss_buf = torch.zeros(1, device=self.device, dtype=torch.float32)
        # optimizer overlapped with the stage's final backward (the planner's sync task starts
        # with the final backward, scheduler.py:202-207): layer-group allreduce + AdamW chunks on a
        # side stream as soon as autograd has finished their gradients (CUDA, NCCL or world 1)
        self.overlap_sync = self.streams.cuda and not (world > 1 and staged())
        self.opt_stream = torch.cuda.Stream(device=self.device, priority=0) if self.streams.cuda else None
        self.grad_snapshots = None  # list -> reduced flat grad slices (lo, hi, grad) captured before each AdamW
        self.grad_snapshot_pipes = []  # backbone index of each snapshot
        self._frz_sends = []        # in-flight frozen-activation sends (kept alive until deliver)

    # ---------------------------------------------------------------- setup
    def _backbone(self, pipe):
        bbs = getattr(self.model, "backbones", None) or [self.model.backbone]
        return bbs[self.prog0.pipes[pipe].backbone]

    def gb_of(self):
        """Offset of this rank's pipeline group in the world batch."""
        return self.group * self.prog0.group_batch

    def _grank(self, dev):
        return self.group * self.D + dev

    def _needed_links(self):
        need = set()
        progs = list(self.programs.values()) + ([self.warm_program] if self.warm_program else [])
        for g in range(self.world // self.D):
            base = g * self.D
            for prog in progs:
                for pi, pl in enumerate(prog.pipes):
                    for s in range(prog.S - 1):
                        for m in range(prog.M):
                            for i, j, a, b in backbone_transfers(prog, s, m, pi):
                                src = base + pl.stage_devices[s][0] + i
                                dst = base + pl.stage_devices[s + 1][0] + j
                                need.add((f"fwd{pi}", src, dst))
                                need.add((f"bwd{pi}", dst, src))
                if prog.selfcond and prog.S > 1:
                    for pi, pl in enumerate(prog.pipes):
                        for m in range(prog.M):
                            for i, j, a, b in self._feedback_pieces(prog, m, pi):
                                need.add((f"fb{pi}", base + pl.stage_devices[-1][0] + i,
                                          base + pl.stage_devices[0][0] + j))
                for t in list(prog.transfers) + list(prog.deliveries):
                    if t.src != t.dst:
                        need.add(("frz", base + t.src, base + t.dst))
        return need

    def _make_stage_groups(self):
        """Per pipe: the process group over every replica of this device's stage (all groups)."""
        mine = [None] * self.npipes
        if self.world == 1:
            return mine
        for pi, pl in enumerate(self.prog0.pipes):
            for s in range(self.prog0.S):
                a, b = pl.stage_devices[s]
                ranks = [g * self.D + d for g in range(self.world // self.D) for d in range(a, b)]
                pg = dist.new_group(ranks=ranks) if len(ranks) > 1 else None
                if s == self.stages[pi]:
                    mine[pi] = pg
        return mine

    @staticmethod
    def _feedback_pieces(prog, m, pi=0):
        lo, hi = prog.micro_range(m)
        a0, a1 = prog.pipes[pi].stage_devices[-1]
        b0, b1 = prog.pipes[pi].stage_devices[0]
        out = []
        for i, (sa, sb) in enumerate(split_range(lo, hi, a1 - a0)):
            for j, (da, db) in enumerate(split_range(lo, hi, b1 - b0)):
                a, b = max(sa, da), min(sb, db)
                if b > a:
                    out.append((i, j, a, b))
        return out

    # ---------------------------------------------------------------- frozen work
    def _run_frozen_piece(self, piece, store, raw):
        comp = self.model.frozen[piece.comp]
        if piece.layer == 0:
            st = {f: raw(f, piece.lo, piece.hi) for f in comp.inputs}
            for ic, il in input_layers(piece.comp, 0, self.prog.frozen_layers, self.prog.frozen_deps):
                st.update(self._gather_frozen(store, ic, il, piece.lo, piece.hi))
        else:
            st = self._gather_frozen(store, piece.comp, piece.layer - 1, piece.lo, piece.hi)
        with torch.no_grad():
            out = comp.component.layers[piece.layer](st)
        store.setdefault((piece.comp, piece.layer), []).append((piece.lo, piece.hi, out))
        return out

    def _gather_frozen(self, store, comp, layer, lo, hi):
        parts = []
        for a, b, st in store.get((comp, layer), []):
            x, y = max(a, lo), min(b, hi)
            if y > x:
                parts.append((x, {k: v[x - a:y - a] for k, v in st.items()}))
        parts.sort(key=lambda q: q[0])
        cov = sum(next(iter(p[1].values())).shape[0] for p in parts)
        if cov != hi - lo:
            raise RuntimeError(f"frozen comp {comp} layer {layer} [{lo},{hi}) missing on device "
                               f"{self.dev} (have {cov})")
        keys = parts[0][1].keys()
        return {k: _cat([p[1][k] for p in parts]) for k in keys}

    def _post_frozen_sends(self, prog, piece, out, sent):
        """Send every transfer this piece's output feeds (production order)."""
        for t in prog.transfers:
            if (t.src == self.dev and t.comp == piece.comp and t.layer == piece.layer
                    and piece.lo <= t.lo and t.hi <= piece.hi and t.dst != self.dev):
                flat = pack([out[k][t.lo - piece.lo:t.hi - piece.lo] for k in sorted(out)])
                self._frz_sends.append(self.links.isend("frz", flat, self._grank(t.dst)))
                sent.add(t.seq)

    def _recv_frozen_upto(self, prog, store, need_seq, posted):
        """Post receives (in production order) for every transfer to this device up to
        `need_seq`, wait for them, and add them to `store`."""
        for t in prog.transfers:
            if t.seq > need_seq:
                break
            if t.dst != self.dev or t.src == self.dev or t.seq in posted:
                continue
            layout = self._frozen_layout(t.comp, t.layer)
            flat = torch.empty(packed_bytes(layout, t.hi - t.lo), device=self.device, dtype=torch.uint8)
            posted[t.seq] = (t, flat, self.links.irecv("frz", flat, self._grank(t.src)))
        for seq, (t, flat, work) in list(posted.items()):
            if work is not None and seq <= need_seq:
                work.wait()
                bufs = unpack(flat, self._frozen_layout(t.comp, t.layer), t.hi - t.lo)
                store.setdefault((t.comp, t.layer), []).append((t.lo, t.hi, bufs))
                posted[seq] = (t, flat, None)

    def _frozen_layout(self, comp, layer):
        spec = self.frozen_specs[comp][layer]
        return [(k, spec[k][0], spec[k][1]) for k in sorted(spec)]

    def _run_pieces(self, prog, pieces, store, raw, posted, sent):
        for piece in pieces:
            if piece.device != self.dev:
                continue
            inputs = set(input_layers(piece.comp, piece.layer, prog.frozen_layers, prog.frozen_deps))
            need = [t.seq for t in prog.transfers
                    if t.dst == self.dev and (t.comp, t.layer) in inputs
                    and t.lo < piece.hi and piece.lo < t.hi]
            if need:
                self._recv_frozen_upto(prog, store, max(need), posted)
            out = self._run_frozen_piece(piece, store, raw)
            self._post_frozen_sends(prog, piece, out, sent)

    def _tail_graphable(self, prog):
        from . import telemetry

        # not inside another capture (whole-iteration graphs), not while the bench brackets every launch
        return (_TAIL_GRAPH and self.world == 1 and self.streams.cuda and not prog.transfers
                and all(piece.device == self.dev for piece in prog.tail)
                and not telemetry.timer.active and not torch.cuda.is_current_stream_capturing())

    def _run_tail_graphed(self, prog, store, raw):
        """The frozen tail of a single-device program as one CUDA graph: the next batch's raw fields are
        copied into static buffers, the graph replays every piece, and the outputs the delivery reads
        (the last layer of each component) are cloned out of the graph's memory pool (the next replay
        overwrites it while this iteration's successor still consumes them)."""
        key = id(prog)
        ent = self._tail_graphs.get(key) if hasattr(self, "_tail_graphs") else None
        if ent is None:
            if not hasattr(self, "_tail_graphs"):
                self._tail_graphs = {}
            fields = sorted({f for piece in prog.tail if piece.layer == 0
                             for f in self.model.frozen[piece.comp].inputs})
            lo0 = min(piece.lo for piece in prog.tail)
            hi0 = max(piece.hi for piece in prog.tail)
            static = {f: raw(f, lo0, hi0).clone() for f in fields}
            sraw = lambda f, lo, hi: static[f][lo - lo0:hi - lo0]  # noqa: E731
            finals = {(t.comp, t.layer) for t in prog.deliveries}
            cap_store = {}
            g = torch.cuda.CUDAGraph()
            cur = torch.cuda.current_stream(self.device)
            with torch.cuda.graph(g, stream=cur):
                self._run_pieces(prog, prog.tail, cap_store, sraw, {}, set())
            ent = dict(graph=g, static=static, lo0=lo0, hi0=hi0, fields=fields,
                       outs={k: v for k, v in cap_store.items() if k in finals})
            self._tail_graphs[key] = ent
        for f in ent["fields"]:
            ent["static"][f].copy_(raw(f, ent["lo0"], ent["hi0"]), non_blocking=True)
        ent["graph"].replay()
        for k, parts in ent["outs"].items():
            store.setdefault(k, []).extend((a, b, {n: v.clone() for n, v in st.items()}) for a, b, st in parts)

    def _deliver(self, prog, store, posted):
        """Final frozen outputs -> first-stage owners of every pipe (used next iteration)."""
        if prog.transfers:
            self._recv_frozen_upto(prog, store, prog.transfers[-1].seq, posted)
        ready = {}
        sends = []
        recvs = []
        for t in prog.deliveries:
            if t.src == self.dev:
                comp_out = self._gather_frozen(store, t.comp, t.layer, t.lo, t.hi)
                if t.dst == self.dev:
                    ready.setdefault(t.comp, []).append((t.lo, t.hi, comp_out))
                else:
                    flat = pack([comp_out[k] for k in sorted(comp_out)])
                    sends.append(self.links.isend("frz", flat, self._grank(t.dst)))
            elif t.dst == self.dev:
                layout = self._frozen_layout(t.comp, t.layer)
                flat = torch.empty(packed_bytes(layout, t.hi - t.lo), device=self.device, dtype=torch.uint8)
                recvs.append((t, flat, self.links.irecv("frz", flat, self._grank(t.src))))
        for t, flat, w in recvs:
            w.wait()
            ready.setdefault(t.comp, []).append(
                (t.lo, t.hi, unpack(flat, self._frozen_layout(t.comp, t.layer), t.hi - t.lo)))
        for w in sends + self._frz_sends:
            w.wait()
        self._frz_sends = []
        return ready

    def frozen_for(self, frozen_ready, lo, hi):
        """Merged frozen outputs of samples [lo, hi) (group-local) on this stage-0 device."""
        merged = {}
        for c, pieces in frozen_ready.items():
            parts = []
            for a, b, st in pieces:
                x, y = max(a, lo), min(b, hi)
                if y > x:
                    parts.append((x, {k: v[x - a:y - a] for k, v in st.items()}))
            if not parts:
                continue
            parts.sort(key=lambda q: q[0])
            for k in parts[0][1]:
                merged[k] = _cat([p[1][k] for p in parts])
        return merged

    # ---------------------------------------------------------------- backbone
    def _stage_forward(self, pi, st_in, grad, hooks=False):
        lo, hi = self.prog.pipes[pi].stage_ranges[self.stages[pi]]
        bb = self._backbone(pi)
        if grad:
            anchor_ctx = getattr(bb, "grad_context", None)
            ctx = anchor_ctx() if anchor_ctx else contextlib.nullcontext()
            with ctx:
                if hooks:
                    return self._run_hooked(pi, bb, st_in, lo, hi)
                return bb.run(st_in, lo, hi)
        with torch.no_grad():
            return bb.run(st_in, lo, hi)

    # ---------------------------------------------------------------- optimizer overlap
    def _run_hooked(self, pi, bb, st, lo, hi):
        """Forward of the stage's LAST micro-batch layer by layer, with a gradient hook on every
        layer's input hidden state: when autograd completes grad(h_j), layers > j have finished
        their backward (one layer of lag covers side branches such as the time embedding), so
        their parameter slice can be reduced and updated while layers <= j still run backward."""
        self._ovl_top[pi] = hi
        for j in range(lo, hi):
            h = st.get("h") if isinstance(st, dict) else None
            if j > lo and torch.is_tensor(h) and h.requires_grad:
                h.register_hook(self._layer_hook(pi, j + 1))
            st = bb.layers[j](st)
        return st

    def _layer_hook(self, pi, new_top):
        def hook(_g):
            self._update_layers(pi, new_top)
        return hook

    def _update_layers(self, pi, new_top, final=False):
        """Allreduce + AdamW of the parameter slice of layers [new_top, top) on the optimizer
        stream, ordered after everything the compute stream has enqueued so far."""
        top = self._ovl_top.get(pi)
        if top is None or new_top >= top:
            return
        bb = self._backbone(pi)
        store = bb.store
        a, b = bb.stage_slice(new_top, top)
        lo, hi = self.param_ranges[pi]
        a, b = max(a, lo), min(b, hi)
        self._ovl_top[pi] = new_top
        if b <= a and not final:
            return
        st = self.opt_stream if _OVL_SIDE else self.streams.compute
        if st is not self.streams.compute:
            ev = torch.cuda.Event()
            ev.record(self.streams.compute)
            st.wait_event(ev)
        with torch.cuda.stream(st):
            if not self._ovl_begun.get(pi):
                store.adamw_begin(**self.model.adamw)
                self._ovl_begun[pi] = True
            if b > a:
                pg = self._stage_pgs[pi]
                if pg is not None:
                    dist.all_reduce(store.grad[a:b], group=pg)
                if self.grad_snapshots is not None:
                    # parity tests: the reduced gradient slice exactly as this AdamW chunk reads it
                    self._snapshot(store, a, b, self.prog.pipes[pi].backbone)
                # background chunks: one CTA per SM at most (see dp_adamw_apply); the final chunk
                # at the sync point has the machine to itself
                store.adamw_apply((a, b), max_ctas=0 if (final and not _LATE_OPT_JOIN) else self.OVERLAP_CTAS,
                                  zero_grad=True,
                                  **self.model.adamw)

    def _sync_overlapped(self, pi):
        lo_l, _ = self.prog.pipes[pi].stage_ranges[self.stages[pi]]
        self._update_layers(pi, lo_l, final=True)
        if not _LATE_OPT_JOIN:
            self.streams.compute.wait_stream(self.opt_stream)
        # else: the compute stream joins the optimizer stream at the END of the iteration, so the last AdamW
        # slices (HBM-bound) run under the frozen tail / fills that follow the sync (tensor-bound VAE convs,
        # text-encoder GEMMs), which never read the backbone's parameters; the next iteration's forward
        # is ordered after every update by that join

    def _spec(self, pi, boundary):
        return self.live_specs[pi][boundary]

    def _fwd(self, pi, m, sc_pass):
        prog = self.prog
        pl = prog.pipes[pi]
        S = prog.S
        s = self.stages[pi]
        lo_r, hi_r = prog.replica_range(s, m, self.replica, pi)
        n = hi_r - lo_r
        key = (pi, m, sc_pass)
        if s == 0:
            fro = self.frozen_for(self.frozen_cur, lo_r, hi_r)
            t = self.inputs.t(self.gb + lo_r, self.gb + hi_r)
            noise = self.inputs.get(self.model.noise_field(pl.backbone), self.gb + lo_r, self.gb + hi_r)
            x0_sc = None
            if not sc_pass and prog.selfcond:
                eps_sc = self._feedback_in.pop((pi, m))
                x0_sc = self.model.ops.pred_x0(self._xt[(pi, m)], eps_sc, t, self.model.sqrt_ab,
                                               self.model.sqrt_1mab)
            st_in, xt = self.model.stage0_inputs(fro, t, noise, x0_sc, pipe=pl.backbone)
            if sc_pass:
                self._xt[(pi, m)] = xt
        else:
            st_in = self._recv_live(pi, s, m, n, lo_r)
        if not sc_pass:
            spec0 = self._spec(pi, pl.stage_ranges[s][0])
            for k, v in st_in.items():
                if v.is_floating_point() and spec0.get(k, (0, 0, False))[2]:
                    v.requires_grad_(True)
        hooks = (not sc_pass and self._ovl_on and self._last_m.get(pi) == m)
        out = self._stage_forward(pi, st_in, grad=not sc_pass, hooks=hooks)
        if s == S - 1:
            if sc_pass:
                self._send_feedback(pi, m, out["out"].detach(), lo_r)
            else:
                pred = out["out"]
                dpred = torch.empty_like(pred)
                ls = self.loss_scale[pl.backbone] if isinstance(self.loss_scale, (list, tuple)) else self.loss_scale
                self.model.ops.mse(pred.detach(), out["noise"], self.loss_buf, ls, dpred)
                self._saved[key] = (st_in, [pred], [dpred])
        else:
            if not sc_pass:
                self._saved[key] = (st_in, out, None)
            self._send_live(pi, s, m, out, lo_r)

    def _bwd(self, pi, m):
        prog = self.prog
        pl = prog.pipes[pi]
        s = self.stages[pi]
        st_in, outs, grads = self._saved.pop((pi, m, False))
        if s == prog.S - 1:
            torch.autograd.backward(outs, grads)
        else:
            lo_r, hi_r = prog.replica_range(s, m, self.replica, pi)
            spec = self._spec(pi, pl.stage_ranges[s][1])
            names = [k for k in sorted(spec) if spec[k][2]]
            gin = self._recv_grads(pi, s, m, hi_r - lo_r, lo_r, names)
            ts = [outs[k] for k in names if outs[k].requires_grad]
            gs = [gin[k] for k in names if outs[k].requires_grad]
            if ts:
                torch.autograd.backward(ts, gs)
        if s > 0:
            spec = self._spec(pi, pl.stage_ranges[s][0])
            names = [k for k in sorted(spec) if spec[k][2]]
            grads_in = {k: (st_in[k].grad if st_in[k].grad is not None else torch.zeros_like(st_in[k]))
                        for k in names}
            lo_r, _ = prog.replica_range(s, m, self.replica, pi)
            self._send_grads(pi, s, m, grads_in, lo_r)

    # live-set P2P -------------------------------------------------------------------------
    def _pieces(self, pi, s, m, as_src):
        """(peer_replica, lo, hi) pieces of micro m crossing cut s -> s+1 of pipe pi for this device."""
        out = []
        for i, j, a, b in backbone_transfers(self.prog, s, m, pi):
            if as_src and i == self.replica:
                out.append((j, a, b))
            if not as_src and j == self.replica:
                out.append((i, a, b))
        return out

    def _send_live(self, pi, s, m, out, lo_r):
        pl = self.prog.pipes[pi]
        spec = self._spec(pi, pl.stage_ranges[s][1])
        dst0 = pl.stage_devices[s + 1][0]
        for j, a, b in self._pieces(pi, s, m, True):
            flat = pack([out[k][a - lo_r:b - lo_r] for k in sorted(spec)])
            self._pending.append(self.links.isend(f"fwd{pi}", flat, self._grank(dst0 + j)))

    def _recv_packed(self, kind, layout, n, pieces, src0, lo_r):
        """Receive one packed message per piece (peer replica, lo, hi) and return the per-name
        tensors of all n samples: views of the message when one piece covers them, else
        assembled from the pieces."""
        msgs = []
        for i, a, b in pieces:
            flat = torch.empty(packed_bytes(layout, b - a), device=self.device, dtype=torch.uint8)
            msgs.append((a, b, flat, self.links.irecv(kind, flat, self._grank(src0 + i))))
        for *_, w in msgs:
            w.wait()
        if len(msgs) == 1 and msgs[0][1] - msgs[0][0] == n:
            return unpack(msgs[0][2], layout, n)
        bufs = {k: torch.empty((n,) + tuple(shape), device=self.device, dtype=dt) for k, shape, dt in layout}
        for a, b, flat, _ in msgs:
            for k, v in unpack(flat, layout, b - a).items():
                bufs[k][a - lo_r:b - lo_r].copy_(v)
        return bufs

    def _recv_live(self, pi, s, m, n, lo_r):
        pl = self.prog.pipes[pi]
        spec = self._spec(pi, pl.stage_ranges[s][0])
        layout = [(k, spec[k][0], spec[k][1]) for k in sorted(spec)]
        return self._recv_packed(f"fwd{pi}", layout, n, self._pieces(pi, s - 1, m, False),
                                 pl.stage_devices[s - 1][0], lo_r)

    def _send_grads(self, pi, s, m, grads, lo_r):
        src0 = self.prog.pipes[pi].stage_devices[s - 1][0]
        for i, a, b in self._pieces(pi, s - 1, m, False):
            flat = pack([grads[k][a - lo_r:b - lo_r] for k in sorted(grads)])
            self._pending.append(self.links.isend(f"bwd{pi}", flat, self._grank(src0 + i)))

    def _recv_grads(self, pi, s, m, n, lo_r, names):
        pl = self.prog.pipes[pi]
        spec = self._spec(pi, pl.stage_ranges[s][1])
        layout = [(k, spec[k][0], spec[k][1]) for k in sorted(names)]
        return self._recv_packed(f"bwd{pi}", layout, n, self._pieces(pi, s, m, True),
                                 pl.stage_devices[s + 1][0], lo_r)

    def _send_feedback(self, pi, m, eps, lo_r):
        prog = self.prog
        if prog.S == 1:
            self._feedback_in[(pi, m)] = eps
            return
        b0 = prog.pipes[pi].stage_devices[0][0]
        for i, j, a, b in self._feedback_pieces(prog, m, pi):
            if i == self.replica:
                self._pending.append(self.links.isend(f"fb{pi}", eps[a - lo_r:b - lo_r], self._grank(b0 + j)))

    def _recv_feedback(self, pi, m):
        prog = self.prog
        lo_r, hi_r = prog.replica_range(0, m, self.replica, pi)
        spec = self._spec(pi, -1)["out"]
        buf = torch.empty((hi_r - lo_r,) + tuple(spec[0]), device=self.device, dtype=spec[1])
        a0 = prog.pipes[pi].stage_devices[-1][0]
        works = [self.links.irecv(f"fb{pi}", buf[a - lo_r:b - lo_r], self._grank(a0 + i))
                 for i, j, a, b in self._feedback_pieces(prog, m, pi) if j == self.replica]
        for w in works:
            w.wait()
        self._feedback_in[(pi, m)] = buf

    # ---------------------------------------------------------------- sync
    def _sync(self, pi):
        if self._ovl_on and pi in self._ovl_top:
            return self._sync_overlapped(pi)
        store = self._backbone(pi).store
        lo, hi = self.param_ranges[pi]
        if hasattr(store, "pre_allreduce"):
            store.pre_allreduce()
        pg = self._stage_pgs[pi]
        if pg is not None and hi > lo:
            if self.links.staged and store.grad.is_cuda:
                host = store.grad[lo:hi].cpu()
                dist.all_reduce(host, group=pg)
                store.grad[lo:hi].copy_(host)
            else:
                dist.all_reduce(store.grad[lo:hi], group=pg)
        if self.grad_snapshots is not None:
            self._snapshot(store, lo, hi, self.prog.pipes[pi].backbone)
        store.adamw_step(rng=(lo, hi), **self.model.adamw)
        store.zero_grad((lo, hi))

    # ---------------------------------------------------------------- iteration
    def warmup(self, raw_next):
        """Iteration-0 warm-up: the frozen part of batch 0 alone, run as a
        data-parallel tail over the group's D devices."""
        self.prog = prog = self.warm_program
        store, posted, sent = {}, {}, set()
        with self.streams.on("fill"):
            self._run_pieces(prog, prog.tail, store, raw_next, posted, sent)
        self.streams.join()
        with self.streams.on("compute"):
            self.frozen_ready = self._deliver(prog, store, posted)

    def run_iteration(self, raw_next, selfcond, has_next=True, trace=False):
        """One training iteration on the current batch; fills compute batch i+1 (`raw_next`).
        trace=True records every task's measured interval (see `measured_tasks`)."""
        self.prog = prog = self.programs[bool(selfcond)]
        self.frozen_cur = self.frozen_ready
        self.frozen_ready = {}
        self.gb = self.group * prog.group_batch
        self._saved, self._xt, self._feedback_in, self._pending = {}, {}, {}, []
        store, posted, sent = {}, {}, set()
        self.loss_buf.zero_()
        if self.grad_snapshots is not None:
            self._alloc_snapshot_bufs()
        tr = self.tracer = _Tracer(self.streams, self.dev) if trace else None
        # optimizer overlap: the micro-batch of each pipe's final backward on this device
        self._ovl_on = self.overlap_sync and self.streams.cuda
        self._ovl_top, self._ovl_begun, self._last_m = {}, {}, {}
        for ins in prog.device_program(self.dev).instrs:
            if ins[0] == "bwd":
                self._last_m[ins[3]] = ins[1]
        task = tr.task if tr else (lambda *a, **k: contextlib.nullcontext())
        last_compute_ev = None
        if self.streams.cuda:
            # every stream of the iteration is forked from the caller's stream: ordered after its work, and
            # part of a CUDA-graph capture that runs on it (a join with a never-forked stream would make the
            # capture depend on uncaptured work)
            cur = torch.cuda.current_stream(self.device)
            for st in (self.streams.compute, self.streams.fill, self.opt_stream):
                if st is not None:
                    st.wait_stream(cur)
        instrs = prog.device_program(self.dev).instrs
        early_tail = _EARLY_TAIL and self.world == 1 and self.streams.cuda and has_next and bool(prog.tail)
        if early_tail:
            # experiment: the single-device tail (no bubbles) issued on the low-priority fill stream at
            # the start of the iteration, concurrent with the backbone
            with self.streams.on("fill"), task("fill", "fill", tag="tail"):
                self._run_pieces(prog, prog.tail, store, raw_next, posted, sent)
        for ins in instrs:
            kind = ins[0]
            if kind in ("fwd", "fwd_sc", "bwd"):
                _, m, s, pi = ins
                with self.streams.on("compute"), task("compute", kind, m, s, prog.pipes[pi].direction):
                    if kind == "fwd" and s == 0 and prog.selfcond and prog.S > 1:
                        self._recv_feedback(pi, m)
                    if kind == "bwd":
                        self._bwd(pi, m)
                    else:
                        self._fwd(pi, m, kind == "fwd_sc")
                    last_compute_ev = self.streams.event("compute")
            elif kind == "fill":
                if not has_next:
                    continue
                self.streams.wait("fill", last_compute_ev)
                with self.streams.on("fill"), task("fill", "fill", tag=f"bubble{ins[1]}"):
                    self._run_pieces(prog, prog.fills[ins[1]], store, raw_next, posted, sent)
            elif kind == "sync":
                with self.streams.on("compute"), task("compute", "sync", s=self.stages[ins[2]],
                                                      direction=prog.pipes[ins[2]].direction):
                    self._sync(ins[2])
            elif kind == "tail":
                if not has_next or early_tail:
                    continue
                self.streams.join()
                # leftover frozen work: busy time (planner.py:172-175), recorded as a fill task
                with self.streams.on("compute"), task("compute", "fill", tag="tail"):
                    if self._tail_graphable(prog) and not trace:
                        self._run_tail_graphed(prog, store, raw_next)
                    else:
                        self._run_pieces(prog, prog.tail, store, raw_next, posted, sent)
            elif kind == "deliver":
                self.streams.join()
                with self.streams.on("compute"), task("compute", "p2p_comm", tag="deliver"):
                    if has_next:
                        self.frozen_ready = self._deliver(prog, store, posted)
                    for w in self._pending:
                        w.wait()
        if self.streams.cuda:
            if self.opt_stream is not None:
                self.streams.compute.wait_stream(self.opt_stream)
            torch.cuda.current_stream(self.device).wait_stream(self.streams.compute)
        return self.loss_buf

    def _snapshot(self, store, a, b, backbone):
        """Copy grad[a:b] into the store's preallocated snapshot buffer on the current stream (no
        allocation inside the backward: a cudaMalloc / cudaFree there synchronises the device from
        the autograd thread)."""
        buf = self._snap_bufs[id(store)]
        buf[a:b].copy_(store.grad[a:b])
        self.grad_snapshots.append((a, b, buf[a:b]))
        self.grad_snapshot_pipes.append(backbone)

    def _alloc_snapshot_bufs(self):
        if not hasattr(self, "_snap_bufs"):
            self._snap_bufs = {}
        for pi in range(len(self.prog0.pipes)):
            st = self._backbone(pi).store
            if id(st) not in self._snap_bufs and getattr(st, "grad", None) is not None:
                self._snap_bufs[id(st)] = torch.empty_like(st.grad)

    def take_grad_snapshots(self):
        """Parity tests: the reduced gradients captured since the last call (grad_snapshots = []
        enables capture), assembled per backbone index into full flat fp32 host tensors (zeros
        outside the stages this rank hosts); clears the capture list."""
        torch.cuda.synchronize(self.device) if self.device.type == "cuda" else None
        out = {}
        for (lo, hi, g), bi in zip(self.grad_snapshots or [], self.grad_snapshot_pipes):
            bbs = getattr(self.model, "backbones", None) or [self.model.backbone]
            flat = out.setdefault(bi, torch.zeros(bbs[bi].store.grad.numel(), dtype=torch.float32))
            flat[lo:hi] = g.float().cpu()
        if self.grad_snapshots is not None:
            self.grad_snapshots.clear()
            self.grad_snapshot_pipes.clear()
        return out

    def measured_tasks(self):
        """Measured tasks of the last traced iteration on this rank (device = local index)."""
        return self.tracer.tasks() if getattr(self, "tracer", None) else []

    def measured_schedule(self):
        """Gather every rank's measured tasks of the last traced iteration; returns the
        measured pipefill `Schedule` of this rank's pipeline group (collective call)."""
        from .pipefill.scheduler import Schedule

        mine = self.measured_tasks()
        if self.world > 1:
            allt = [None] * self.world
            dist.all_gather_object(allt, mine)
            allt = allt[self.group * self.D:(self.group + 1) * self.D]
        else:
            allt = [mine]
        tasks = [t for ts in allt for t in ts]
        makespan = max((t.end for t in tasks), default=0.0)
        return Schedule(tasks, makespan, self.D)

    def total_loss(self):
        """Sum of the loss over all ranks (only last-stage ranks contribute)."""
        if self.world > 1:
            if self.links.staged and self.loss_buf.is_cuda:
                host = self.loss_buf.cpu()
                dist.all_reduce(host)
                self.loss_buf.copy_(host)
            else:
                dist.all_reduce(self.loss_buf)
        return self.loss_buf
