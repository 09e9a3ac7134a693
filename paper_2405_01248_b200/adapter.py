"""Plan adapter: the planner's outputs -> per-rank instruction programs.

This is the executor-side half of the paper's "instruction generation" step
(Fig. 6 step 6), which the reference leaves out.
Input is exactly what the reference API returns (planner.evaluate_point,
reference planner.py:141-187): the PartitionPlan, the simulated Schedule
(scheduler.py:320-332) and the FillPlan (filler.py:245-276). Output, per
group-local device:

  ("fwd" | "fwd_sc" | "bwd", micro, stage, pipe)  compute tasks in simulated start order
                                             (pipe 0 = "down" backbone, 1 = "up" backbone of a
                                             bidirectional plan, partitioner.py:402-501)
  ("fill", bubble_idx)                       frozen work of one bubble, placed after the
                                             device's last compute task ending <= bubble.start
  ("sync", stage, pipe)                      per-stage gradient allreduce + AdamW, right after
                                             the stage's final backward (scheduler.py:202-207)
  ("tail",)                                  leftover frozen work over all D devices
  ("deliver",)                               frozen outputs -> stage-0 consumers (next iteration)

plus the sample-range bookkeeping the reference only tracks as counts
(filler.py:89,240): every frozen (component, layer) piece gets
a concrete [lo, hi) range of the group batch on a concrete device, processed in
ascending sample order, split contiguously and near-evenly over the bubble's
sorted idle devices. From the pieces the adapter
derives every frozen-activation transfer (src, dst, component, layer, range)
in global production order, which both endpoints enumerate identically.
"""

from __future__ import annotations

from dataclasses import dataclass, field

from .pipefill.scheduler import group_device_ranges

EPS = 1e-12


def split_range(lo, hi, parts):
    """Contiguous near-even split of [lo, hi) into `parts` ranges (possibly empty)."""
    n = hi - lo
    return [(lo + (k * n) // parts, lo + ((k + 1) * n) // parts) for k in range(parts)]


@dataclass(frozen=True)
class Piece:
    """Frozen work item: layer `layer` of frozen component `comp` over samples [lo, hi) on `device`."""

    comp: int
    layer: int
    lo: int
    hi: int
    device: int
    phase: int          # production order: index of the fill (bubble) or len(fills) for the tail


@dataclass(frozen=True)
class Transfer:
    src: int
    dst: int
    comp: int
    layer: int          # producer layer (its outputs move)
    lo: int
    hi: int
    seq: int            # global production order


@dataclass
class DeviceProgram:
    device: int
    stage: int | None              # stage of pipe 0 hosted here
    replica: int | None
    instrs: list = field(default_factory=list)
    stages: tuple = ()             # per pipe: flow stage hosted on this device (or None)


@dataclass(frozen=True)
class PipeLayout:
    """One backbone pipeline: flow stage s holds layers stage_ranges[s] on the group-local
    devices stage_devices[s]. The up pipe of a bidirectional plan runs flow stage j on device
    group S-1-j (scheduler.py:273-276)."""

    direction: str
    backbone: int
    stage_ranges: tuple
    stage_devices: tuple


@dataclass
class GroupProgram:
    """Everything one pipeline group (D devices) executes in one iteration."""

    D: int
    S: int
    M: int
    group_batch: int
    micro_batch: int
    stage_ranges: list          # stage -> (lo, hi) backbone layers
    stage_devices: list         # stage -> (first, last+1) group-local devices
    devices: list               # DeviceProgram per group-local device
    fills: list                 # per bubble: list[Piece] in execution order
    tail: list                  # list[Piece]
    transfers: list             # list[Transfer] in production order
    deliveries: list            # list[Transfer] (layer = last layer) final outputs -> stage 0
    frozen_layers: list         # per frozen component: number of layers
    selfcond: bool
    frozen_deps: tuple = ()     # (producer, consumer) frozen component indices
    pipes: tuple = ()           # PipeLayout per backbone pipeline (1, or 2 when bidirectional)

    def device_program(self, dev):
        return self.devices[dev]

    def micro_range(self, m):
        return m * self.micro_batch, (m + 1) * self.micro_batch

    def replica_range(self, stage, m, replica, pipe=0):
        first, last = self.pipes[pipe].stage_devices[stage]
        lo, hi = self.micro_range(m)
        return split_range(lo, hi, last - first)[replica]

    def stage_of(self, dev):
        for s, (a, b) in enumerate(self.stage_devices):
            if a <= dev < b:
                return s, dev - a
        raise ValueError(dev)

    # ---- standalone program documents (Fig. 6 step 6: "instruction generation").
    # The reference's plan document carries task counts only (planner.py:312-317); these carry the
    # per-device instruction order, the frozen pieces with their sample ranges and every transfer,
    # so a launcher can ship one file per rank and the executor runs it without re-planning.

    def to_dict(self):
        return {"format": PROGRAM_FORMAT, "D": self.D, "S": self.S, "M": self.M,
                "group_batch": self.group_batch, "micro_batch": self.micro_batch,
                "stage_ranges": [list(r) for r in self.stage_ranges],
                "stage_devices": [list(r) for r in self.stage_devices],
                "devices": [{"device": d.device, "stage": d.stage, "replica": d.replica,
                             "stages": list(d.stages), "instrs": [list(i) for i in d.instrs]}
                            for d in self.devices],
                "fills": [[_piece_row(p) for p in ps] for ps in self.fills],
                "tail": [_piece_row(p) for p in self.tail],
                "transfers": [_transfer_row(t) for t in self.transfers],
                "deliveries": [_transfer_row(t) for t in self.deliveries],
                "frozen_layers": list(self.frozen_layers), "selfcond": bool(self.selfcond),
                "frozen_deps": [list(d) for d in self.frozen_deps],
                "pipes": [{"direction": pl.direction, "backbone": pl.backbone,
                           "stage_ranges": [list(r) for r in pl.stage_ranges],
                           "stage_devices": [list(r) for r in pl.stage_devices]} for pl in self.pipes]}

    @classmethod
    def from_dict(cls, d):
        if d.get("format") != PROGRAM_FORMAT:
            raise ValueError(f"not a {PROGRAM_FORMAT} document: format={d.get('format')!r}")
        devices = [DeviceProgram(x["device"], x["stage"], x["replica"], [tuple(i) for i in x["instrs"]],
                                 tuple(x["stages"])) for x in d["devices"]]
        return cls(D=d["D"], S=d["S"], M=d["M"], group_batch=d["group_batch"], micro_batch=d["micro_batch"],
                   stage_ranges=[tuple(r) for r in d["stage_ranges"]],
                   stage_devices=[tuple(r) for r in d["stage_devices"]], devices=devices,
                   fills=[[Piece(*r) for r in ps] for ps in d["fills"]], tail=[Piece(*r) for r in d["tail"]],
                   transfers=[Transfer(*r) for r in d["transfers"]],
                   deliveries=[Transfer(*r) for r in d["deliveries"]],
                   frozen_layers=list(d["frozen_layers"]), selfcond=d["selfcond"],
                   frozen_deps=tuple(tuple(x) for x in d["frozen_deps"]),
                   pipes=tuple(PipeLayout(p["direction"], p["backbone"], tuple(tuple(r) for r in p["stage_ranges"]),
                                          tuple(tuple(r) for r in p["stage_devices"])) for p in d["pipes"]))

    def rank_document(self, dev, group=0, rank=None):
        """The program of group-local device `dev` as a standalone document: the group-level
        layout (stage ranges / devices, pieces, transfers — every rank of the group needs them to
        address its peers) plus `device` = the instruction list this rank executes."""
        doc = self.to_dict()
        doc["rank"] = {"device": dev, "group": group, "rank": group * self.D + dev if rank is None else rank}
        return doc


PROGRAM_FORMAT = "dpipe-program/v1"


def _piece_row(p):
    return [p.comp, p.layer, p.lo, p.hi, p.device, p.phase]


def _transfer_row(t):
    return [t.src, t.dst, t.comp, t.layer, t.lo, t.hi, t.seq]


def save_rank_programs(prog, directory, groups=1, programs=None):
    """Write one `rank<r>.json` per rank of a `groups`-group job (PROGRAM_FORMAT). `programs` maps
    an iteration kind ("plain" / "selfcond") to a GroupProgram when self-conditioning makes the
    executor pick one of two programs per iteration; each rank file then holds both."""
    import json
    import os

    os.makedirs(directory, exist_ok=True)
    progs = programs or {"plain": prog}
    paths = []
    for g in range(groups):
        for dev in range(prog.D):
            r = g * prog.D + dev
            doc = {"format": PROGRAM_FORMAT + "+rank", "rank": r, "group": g, "device": dev,
                   "programs": {k: p.rank_document(dev, g, r) for k, p in progs.items()}}
            path = os.path.join(directory, f"rank{r}.json")
            with open(path, "w") as f:
                json.dump(doc, f, sort_keys=True, separators=(",", ":"))
            paths.append(path)
    return paths


def load_rank_program(path):
    """-> (rank, {kind: GroupProgram}) from a file written by save_rank_programs."""
    import json

    with open(path) as f:
        doc = json.load(f)
    if doc.get("format") != PROGRAM_FORMAT + "+rank":
        raise ValueError(f"{path}: not a {PROGRAM_FORMAT} rank document")
    return doc["rank"], {k: GroupProgram.from_dict(v) for k, v in doc["programs"].items()}


def _pipes(plan):
    groups = group_device_ranges(plan)
    down = plan.stages_down
    pipes = [PipeLayout("down", down[0].backbone, tuple(tuple(st.layer_range) for st in down),
                        tuple(groups))]
    up = plan.stages_up
    if up:
        n = len(up)
        pipes.append(PipeLayout("up", up[0].backbone, tuple(tuple(st.layer_range) for st in up),
                                tuple(groups[n - 1 - j] for j in range(n))))
    return tuple(pipes)


def build_group_program(result, frozen_layer_counts, selfcond=None, frozen_deps=()):
    """Adapt one `evaluate_point` result (or an equivalent dict with plan/schedule/fill
    built for the non-activated self-conditioning iterations) into a GroupProgram."""
    plan = result["plan"]
    schedule = result["pre_fill_schedule"]
    fill = result["fill"]
    cfg = plan.config
    D, S, M, B = cfg.group_size, cfg.num_stages, cfg.num_microbatches, cfg.global_batch
    pipes = _pipes(plan)
    stage_ranges, stage_devices = list(pipes[0].stage_ranges), list(pipes[0].stage_devices)
    sc = cfg.selfcond if selfcond is None else selfcond
    pipe_of = {p.direction: i for i, p in enumerate(pipes)}

    devices = []
    for dev in range(D):
        stages = []
        rep = None
        for pl in pipes:
            st = None
            for s_, (a, b) in enumerate(pl.stage_devices):
                if a <= dev < b:
                    st, rep = s_, dev - a
            stages.append(st)
        devices.append(DeviceProgram(dev, stages[0], rep, stages=tuple(stages)))

    # ---- compute tasks per device, in the simulator's per-device order
    compute = {dev: [] for dev in range(D)}
    for t in schedule.tasks:  # sorted by (device, start, end, kind, micro)
        if t.kind in ("fwd", "bwd", "fwd_sc"):
            compute[t.device].append(t)
    for dev in range(D):
        compute[dev].sort(key=lambda t: (t.start, t.end, t.kind, t.micro_batch))

    # ---- frozen pieces with concrete sample ranges (ascending per (comp, layer))
    done = [[0] * n for n in frozen_layer_counts]
    fills = []
    for bi, f in enumerate(fill.fills):
        pieces = []
        if f.fill_time > 0:
            idle = sorted(f.bubble.idle_devices)
            work = []
            for c in sorted(f.full_layers):
                for layer in f.full_layers[c]:
                    n = f.full_samples[(c, layer)]
                    work.append((c, layer, n))
            if f.partial is not None:
                work.append((f.partial.component, f.partial.layer, f.partial.samples))
            for c, layer, n in work:
                lo = done[c][layer]
                hi = lo + n
                done[c][layer] = hi
                for dev, (a, b) in zip(idle, split_range(lo, hi, len(idle))):
                    if b > a:
                        pieces.append(Piece(c, layer, a, b, dev, bi))
        fills.append(pieces)
    tail = []
    tail_phase = len(fill.fills)
    for tw in _topo_tail(fill.tail, frozen_layer_counts, frozen_deps):
        lo = done[tw.component][tw.layer]
        hi = lo + tw.samples
        done[tw.component][tw.layer] = hi
        for dev, (a, b) in enumerate(split_range(lo, hi, D)):
            if b > a:
                tail.append(Piece(tw.component, tw.layer, a, b, dev, tail_phase))
    for c, n in enumerate(frozen_layer_counts):
        for layer in range(n):
            if done[c][layer] != B:
                raise RuntimeError(f"frozen component {c} layer {layer}: {done[c][layer]} of {B} samples "
                                   "covered by the fill plan")

    # ---- instruction placement
    for dev in range(D):
        prog = devices[dev]
        items = []  # (sort_time, tiebreak, instr)
        for t in compute[dev]:
            items.append((t.start, 1, (t.kind, t.micro_batch, t.stage, pipe_of[t.direction])))
        for bi, f in enumerate(fill.fills):
            if any(p.device == dev for p in fills[bi]):
                # after every compute task ending <= bubble.start; before those starting >= it
                items.append((f.bubble.start, 0, ("fill", bi)))
        items.sort(key=lambda x: (x[0], x[1]))
        instrs = [it[2] for it in items]
        if sc and len(pipes) > 1 and not any(t.kind == "fwd_sc" for t in compute[dev]):
            # The reference's bidirectional simulator has no self-conditioning pass
            # (planner.py:115-118, scheduler.py:346-347). Run it outside the plan (SURVEY
            # Appendix B.1): every pipe's no-grad forward of all micro-batches, pipe by pipe in
            # flow order, before the planned tasks; feedback reaches stage 0 before its fwd.
            pre = []
            for pi, st in enumerate(prog.stages):
                if st is not None:
                    pre += [("fwd_sc", m, st, pi) for m in range(M)]
            instrs = pre + instrs
        for pi, st in enumerate(prog.stages):
            if st is not None:
                last_bwd = max(i for i, ins in enumerate(instrs)
                               if ins[0] == "bwd" and ins[2] == st and ins[3] == pi)
                instrs.insert(last_bwd + 1, ("sync", st, pi))
        if any(p.device == dev for p in tail):
            instrs.append(("tail",))
        instrs.append(("deliver",))
        prog.instrs = instrs

    transfers, deliveries = _data_plan(fills, tail, frozen_layer_counts, B, M,
                                       [pl.stage_devices[0] for pl in pipes], frozen_deps)
    return GroupProgram(D=D, S=S, M=M, group_batch=B, micro_batch=B // M, stage_ranges=stage_ranges,
                        stage_devices=stage_devices, devices=devices, fills=fills, tail=tail,
                        transfers=transfers, deliveries=deliveries,
                        frozen_layers=list(frozen_layer_counts), selfcond=sc,
                        frozen_deps=tuple(tuple(d) for d in frozen_deps), pipes=pipes)


def topo_order(n, deps):
    """Frozen components in a dependency-respecting order (Kahn, lowest index first): the
    reference validates the dependency graph as a DAG (profile.py:184-210) but emits the tail
    in component-index order (filler.py:256-262), which is only safe for sorted DAGs."""
    preds = {c: {s for s, d in deps if d == c} for c in range(n)}
    done, order = set(), []
    while len(order) < n:
        nxt = min(c for c in range(n) if c not in done and preds[c] <= done)
        order.append(nxt)
        done.add(nxt)
    return order


def _topo_tail(tail, counts, deps=()):
    rank = {c: i for i, c in enumerate(topo_order(len(counts), deps))}
    return sorted(tail, key=lambda t: (rank[t.component], t.layer))


def _overlaps(pieces, lo, hi):
    for p in pieces:
        a, b = max(lo, p.lo), min(hi, p.hi)
        if b > a:
            yield p, a, b


def input_layers(comp, layer, counts, deps):
    """(component, layer) outputs a piece of `layer` of `comp` consumes: the previous layer, or
    for layer 0 the final layers of the components it depends on (e.g. ControlNet's frozen
    U-Net encoder on the VAE latents and the text context)."""
    if layer > 0:
        return [(comp, layer - 1)]
    return [(s, counts[s] - 1) for s, d in deps if d == comp]


def _data_plan(fills, tail, counts, B, M, first_groups, deps=()):
    """Frozen-activation transfers in production order, and final-output deliveries."""
    produced = {}  # (comp, layer) -> list[Piece]
    order = [p for ps in fills for p in ps] + list(tail)
    transfers = []
    seq = 0
    for p in order:
        for ic, il in input_layers(p.comp, p.layer, counts, deps):
            got = list(_overlaps(produced.get((ic, il), ()), p.lo, p.hi))
            if sum(b - a for _, a, b in got) != p.hi - p.lo:
                raise RuntimeError(f"frozen ({p.comp},{p.layer}) [{p.lo},{p.hi}) runs before its input "
                                   f"({ic},{il}) is produced")
            for src, a, b in got:
                if src.device != p.device:
                    transfers.append(Transfer(src.device, p.device, ic, il, a, b, seq))
                    seq += 1
        produced.setdefault((p.comp, p.layer), []).append(p)
    # transfers are discovered in consumption order; re-sort by producer order so that both
    # ends post them in the order the producer can send them
    pos = {(p.comp, p.layer, p.lo, p.hi, p.device): i for i, p in enumerate(order)}

    def prod_index(t):
        for src, a, b in _overlaps(produced[(t.comp, t.layer)], t.lo, t.hi):
            if src.device == t.src and a == t.lo and b == t.hi:
                return pos[(src.comp, src.layer, src.lo, src.hi, src.device)]
        raise AssertionError(t)

    transfers.sort(key=lambda t: (prod_index(t), t.seq))
    transfers = [Transfer(t.src, t.dst, t.comp, t.layer, t.lo, t.hi, i) for i, t in enumerate(transfers)]
    # final frozen outputs -> the first-stage owners of every pipe (each sample to the replica
    # that runs it; a device owning the first stage of both pipes receives it once)
    deliveries = []
    seen = set()
    mb = B // M
    k = 0
    for first, last in first_groups:
        r0 = last - first
        for c, n in enumerate(counts):
            final = produced.get((c, n - 1), [])
            for m in range(M):
                for rep, (lo, hi) in enumerate(split_range(m * mb, (m + 1) * mb, r0)):
                    for src, a, b in _overlaps(final, lo, hi):
                        key = (src.device, first + rep, c, a, b)
                        if key in seen:
                            continue
                        seen.add(key)
                        deliveries.append(Transfer(src.device, first + rep, c, n - 1, a, b, k))
                        k += 1
    return transfers, deliveries


def backbone_transfers(prog: GroupProgram, stage, m, pipe=0):
    """Live-set pieces crossing the cut stage -> stage+1 of a pipe for micro-batch m:
    [(src_replica, dst_replica, lo, hi)] (the reverse for gradients)."""
    out = []
    a0, a1 = prog.pipes[pipe].stage_devices[stage]
    b0, b1 = prog.pipes[pipe].stage_devices[stage + 1]
    lo, hi = prog.micro_range(m)
    src = split_range(lo, hi, a1 - a0)
    dst = split_range(lo, hi, b1 - b0)
    for i, (sa, sb) in enumerate(src):
        for j, (da, db) in enumerate(dst):
            a, b = max(sa, da), min(sb, db)
            if b > a:
                out.append((i, j, a, b))
    return out
