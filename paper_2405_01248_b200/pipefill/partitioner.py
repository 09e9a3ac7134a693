"""Stage partitioning of the trainable backbone(s) (paper §4, Eqs. 1-15).

Restates reference partitioner.py:34-674 with identical arithmetic and
tie-breaking so plans match the reference bit-for-bit:

* stage values at local batch B/r (``StageEvaluator``, reference :130-211);
* a memoised DP over (layer prefix, stages, devices) whose sub-results are
  Pareto sets of (w, w_sc, y) so the max/max objective stays exact
  (reference :267-340);
* bidirectional pairing of two backbones on shared device groups
  (reference :402-501);
* the exhaustive oracle used by the tests (reference :520-644).

The executor instantiates ``StageAssignment.layer_range`` / ``replicas`` of the
returned ``PartitionPlan`` as its pipeline stages.
"""

from __future__ import annotations

import itertools
from dataclasses import dataclass

from .errors import ExtrapolationError, InfeasibleError, OracleTooLargeError, ValidationError
from .profile import ClusterConfig, ComponentProfile, ModelProfile, cost_at

DOWN = "down"
UP = "up"

_LOOKUP_FIELDS = ("fwd_time", "bwd_time", "grad_bytes", "fwd_comm_bytes", "bwd_comm_bytes",
                  "out_bytes")


@dataclass(frozen=True)
class PlanConfig:
    num_stages: int
    num_microbatches: int
    group_size: int
    global_batch: int
    micro_batch: int = 0
    selfcond: bool = False

    def __post_init__(self):
        for attr in ("num_stages", "num_microbatches", "group_size", "global_batch"):
            val = getattr(self, attr)
            if not isinstance(val, int) or val < 1:
                raise ValidationError(f"PlanConfig.{attr} must be a positive integer, got {val!r}")
        if self.num_stages > self.group_size:
            raise ValidationError(
                f"num_stages ({self.num_stages}) cannot exceed group_size ({self.group_size})")
        if self.global_batch % self.num_microbatches:
            raise ValidationError(
                f"global_batch ({self.global_batch}) not divisible by "
                f"num_microbatches ({self.num_microbatches})")
        mb = self.global_batch // self.num_microbatches
        if self.micro_batch == 0:
            object.__setattr__(self, "micro_batch", mb)
        elif self.micro_batch != mb:
            raise ValidationError(
                f"micro_batch ({self.micro_batch}) != global_batch / num_microbatches ({mb})")


@dataclass(frozen=True)
class StageAssignment:
    backbone: int
    layer_range: tuple
    replicas: int
    direction: str = DOWN

    def __post_init__(self):
        lo, hi = self.layer_range
        if hi <= lo:
            raise ValidationError(f"stage layer_range {self.layer_range} must be non-empty")
        if self.replicas < 1:
            raise ValidationError(f"stage replicas must be >= 1, got {self.replicas}")


@dataclass(frozen=True)
class StageCosts:
    t0: float
    t_sync: float
    t_comp: float
    gap: float


@dataclass
class PartitionPlan:
    config: PlanConfig
    stages: list
    objective: float
    per_stage: list
    t_max: float
    t_max_sc: float | None = None
    feedback_time: float = 0.0
    m_cdm: int | None = None
    selfcond_prob: float = 0.0

    @property
    def stages_down(self):
        return [s for s in self.stages if s.direction == DOWN]

    @property
    def stages_up(self):
        return [s for s in self.stages if s.direction == UP]


@dataclass(frozen=True)
class StageValue:
    """Costs of one candidate stage (layers [lo, hi) on r replicas)."""

    fwd: float
    bwd: float
    fwd_comm: float
    bwd_comm: float
    t_sync: float
    t_comp: float
    gap: float
    t0: float
    t0_sc: float
    compute: float


class StageEvaluator:
    """Memoised stage costing for one backbone at micro-batch B (local B/r).

    ``p2p_factor`` multiplies the bandwidth term of boundary transfers
    (2 when two pipeline directions share the links).
    """

    def __init__(self, component: ComponentProfile, cluster: ClusterConfig, micro_batch: int,
                 p2p_factor: float = 1.0):
        self.layers = component.layers
        self.num_layers = len(self.layers)
        self.comm = cluster.comm
        self.micro_batch = micro_batch
        self.p2p_factor = p2p_factor
        self._per_layer = {}
        self._per_stage = {}

    def layer_costs(self, idx: int, r: int):
        key = (idx, r)
        try:
            return self._per_layer[key]
        except KeyError:
            pass
        local = self.micro_batch // r
        try:
            val = tuple(cost_at(self.layers[idx], f, local) for f in _LOOKUP_FIELDS)
        except ExtrapolationError:
            val = None
        self._per_layer[key] = val
        return val

    def stage(self, lo: int, hi: int, r: int):
        key = (lo, hi, r)
        if key not in self._per_stage:
            self._per_stage[key] = self._compute(lo, hi, r)
        return self._per_stage[key]

    def _compute(self, lo, hi, r):
        if r < 1 or self.micro_batch % r:
            return None
        f_sum = b_sum = g_sum = 0.0
        for i in range(lo, hi):
            c = self.layer_costs(i, r)
            if c is None:
                return None
            f_sum += c[0]
            b_sum += c[1]
            g_sum += c[2]
        cm = self.comm
        if hi < self.num_layers:
            edge = self.layer_costs(hi - 1, r)
            if edge is None:
                return None
            f_comm = self.p2p_factor * edge[3] / cm.bandwidth_p2p + cm.latency_p2p
            b_comm = self.p2p_factor * edge[4] / cm.bandwidth_p2p + cm.latency_p2p
        else:
            f_comm = b_comm = 0.0
        sync = g_sum / cm.bandwidth_ar + cm.latency_ar
        return StageValue(
            fwd=f_sum, bwd=b_sum, fwd_comm=f_comm, bwd_comm=b_comm, t_sync=sync, t_comp=b_sum,
            gap=sync - b_sum, t0=max(f_sum + b_sum, f_comm + b_comm),
            t0_sc=max(2.0 * f_sum + b_sum, 2.0 * f_comm + b_comm), compute=f_sum + b_sum,
        )

    def feedback_time(self, r: int):
        """Self-conditioning feedback: last layer's output back to stage 0."""
        last = self.layer_costs(self.num_layers - 1, r)
        if last is None:
            return None
        return last[5] / self.comm.bandwidth_p2p + self.comm.latency_p2p


# reference-compatible private name (scheduler and tests import it)
_BackboneCosts = StageEvaluator


def stage_cost_single(profile: ModelProfile, cluster: ClusterConfig, layer_range, r: int,
                      micro_batch: int, selfcond: bool = False, backbone: int = 0) -> StageCosts:
    ev_all = StageEvaluator(profile.backbones[backbone], cluster, micro_batch)
    lo, hi = layer_range
    ev = ev_all.stage(lo, hi, r)
    if ev is None:
        if micro_batch % r:
            raise InfeasibleError(f"micro_batch {micro_batch} not divisible by replicas {r}")
        local = micro_batch // r
        layers = profile.backbones[backbone].layers
        for i in range(lo, hi):  # surface the ExtrapolationError that made it infeasible
            for f in _LOOKUP_FIELDS:
                cost_at(layers[i], f, local)
        raise InfeasibleError(f"stage {layer_range} at r={r} cannot be costed")
    return StageCosts(t0=ev.t0_sc if selfcond else ev.t0, t_sync=ev.t_sync, t_comp=ev.t_comp,
                      gap=ev.gap)


def selfcond_objective(t_max: float, t_max_sc: float, p: float) -> float:
    """E[bound] when the extra forward activates with probability p (paper Eq. 8)."""
    if not 0.0 <= p <= 1.0:
        raise ValidationError(f"activation probability must be in [0, 1], got {p!r}")
    return p * t_max_sc + (1.0 - p) * t_max


def _pos(x: float) -> float:
    return x if x > 0.0 else 0.0


def _pareto(cands):
    """Pareto frontier over the first three coordinates; after sorting, the
    lexicographically smallest of exact ties survives."""
    cands.sort()
    front = []
    for c in cands:
        dominated = False
        for f in front:
            if f[0] <= c[0] and f[1] <= c[1] and f[2] <= c[2]:
                dominated = True
                break
        if dominated:
            continue
        front = [f for f in front if not (c[0] <= f[0] and c[1] <= f[1] and c[2] <= f[2])]
        front.append(c)
    return front


def _rep_options(devices: int, stages_left: int, equal_r):
    if equal_r is None:
        return list(range(1, devices - stages_left + 2))
    return [equal_r] if devices - equal_r >= (stages_left - 1) * equal_r else []


class _ChainDP:
    """DP over prefixes of one backbone: solve(l, s, d) = Pareto set of
    (w, w_sc, y, max_compute, ranges, reps) for layers [0, l) in s stages on d devices."""

    def __init__(self, ev: StageEvaluator, equal_r):
        self.ev = ev
        self.equal_r = equal_r
        self.memo = {}

    def extend(self, acc, l, s, d, out):
        ev = self.ev
        for r in _rep_options(d, s, self.equal_r):
            for cut in range(s - 1, l):
                sv = ev.stage(cut, l, r)
                if sv is None:
                    continue
                for w, wsc, y, mc, rngs, reps in self.solve(cut, s - 1, d - r):
                    out.append((max(w, sv.t0), max(wsc, sv.t0_sc), max(y, sv.gap),
                                max(mc, sv.compute), rngs + ((cut, l),), reps + (r,)))
        return out

    def solve(self, l, s, d):
        key = (l, s, d)
        hit = self.memo.get(key)
        if hit is not None:
            return hit
        if s == 1:
            sv = self.ev.stage(0, l, d)
            res = [] if sv is None else [(sv.t0, sv.t0_sc, sv.gap, sv.compute, ((0, l),), (d,))]
        else:
            res = _pareto(self.extend(None, l, s, d, []))
        self.memo[key] = res
        return res


def _single_candidates(ev: StageEvaluator, cfg: PlanConfig, equal_r):
    L, S, D = ev.num_layers, cfg.num_stages, cfg.group_size
    if S == 1:
        sv = ev.stage(0, L, D)
        return [] if sv is None else [(sv.t0, sv.t0_sc, sv.gap, sv.compute, ((0, L),), (D,))]
    # the last stage stays outside the memo: its replication sets the feedback time
    return _ChainDP(ev, equal_r).extend(None, L, S, D, [])


def _select_single(ev: StageEvaluator, cfg: PlanConfig, p: float, candidates):
    slots = cfg.num_microbatches + 2 * cfg.num_stages - 2
    winner = None
    for w, wsc, y, mc, rngs, reps in candidates:
        bound = slots * w + _pos(y)
        fb = ev.feedback_time(reps[-1])
        if p > 0.0:
            if fb is None:
                continue
        elif fb is None:
            fb = 0.0
        bound_sc = slots * wsc + _pos(y) + fb
        key = (selfcond_objective(bound, bound_sc, p), mc, rngs, reps)
        if winner is None or key < winner[0]:
            winner = (key, bound, bound_sc, fb, rngs, reps)
    return winner


def _stage_costs_for(ev: StageEvaluator, rngs, reps, selfcond: bool):
    out = []
    for (lo, hi), r in zip(rngs, reps):
        sv = ev.stage(lo, hi, r)
        out.append(StageCosts(t0=sv.t0_sc if selfcond else sv.t0, t_sync=sv.t_sync,
                              t_comp=sv.t_comp, gap=sv.gap))
    return out


def _single_plan(ev, cfg, p, winner):
    key, bound, bound_sc, fb, rngs, reps = winner
    return PartitionPlan(
        config=cfg,
        stages=[StageAssignment(backbone=0, layer_range=rg, replicas=r) for rg, r in zip(rngs, reps)],
        objective=key[0],
        per_stage=_stage_costs_for(ev, rngs, reps, cfg.selfcond),
        t_max=bound, t_max_sc=bound_sc, feedback_time=fb, selfcond_prob=p,
    )


def partition_single(profile: ModelProfile, cluster: ClusterConfig, cfg: PlanConfig, *,
                     equal_replication: bool = True) -> PartitionPlan:
    """Optimal single-backbone partition (reference partitioner.py:364-399)."""
    if len(profile.backbones) != 1:
        raise ValueError("partition_single requires a profile with exactly one backbone")
    comp = profile.backbones[0]
    L, S, D = len(comp.layers), cfg.num_stages, cfg.group_size
    _check_common(cluster, cfg)
    if L < S:
        raise InfeasibleError(f"backbone has {L} layers, cannot form {S} stages")
    equal_r = _equal_replication(cfg) if equal_replication else None
    ev = StageEvaluator(comp, cluster, cfg.micro_batch)
    p = profile.selfcond_prob if cfg.selfcond else 0.0
    winner = _select_single(ev, cfg, p, _single_candidates(ev, cfg, equal_r))
    if winner is None:
        raise InfeasibleError(
            f"no feasible partition for S={S}, D={D}: every replication split "
            "violates batch divisibility or the profiled batch range")
    return _single_plan(ev, cfg, p, winner)


def _bidirectional_candidates(down: StageEvaluator, up: StageEvaluator, cfg: PlanConfig, equal_r):
    """(w, y, max_compute, ranges_down, ranges_up, reps) in device-group order:
    group g hosts a down range and an up range (reference :402-447)."""
    Ld, Lu = down.num_layers, up.num_layers
    memo = {}

    def solve(ld, lu, s, d):
        key = (ld, lu, s, d)
        if key in memo:
            return memo[key]
        if s == 1:
            a = down.stage(0, ld, d)
            b = up.stage(Lu - lu, Lu, d)
            res = [] if a is None or b is None else [(
                max(a.t0, b.t0), max(a.gap, b.gap), max(a.compute, b.compute),
                ((0, ld),), ((Lu - lu, Lu),), (d,))]
        else:
            res = []
            for r in _rep_options(d, s, equal_r):
                for cut in range(s - 1, ld):
                    a = down.stage(cut, ld, r)
                    if a is None:
                        continue
                    for take in range(1, lu - s + 2):
                        b = up.stage(Lu - lu, Lu - lu + take, r)
                        if b is None:
                            continue
                        for w, y, mc, rd, ru, reps in solve(cut, lu - take, s - 1, d - r):
                            res.append((max(w, a.t0, b.t0), max(y, a.gap, b.gap),
                                        max(mc, a.compute, b.compute), rd + ((cut, ld),),
                                        ru + ((Lu - lu, Lu - lu + take),), reps + (r,)))
            res = _pareto(res)
        memo[key] = res
        return res

    return solve(Ld, Lu, cfg.num_stages, cfg.group_size)


def _bidirectional_plan(cfg, down, up, slots, key, rd, ru, reps):
    stages = [StageAssignment(backbone=0, layer_range=rg, replicas=r, direction=DOWN)
              for rg, r in zip(rd, reps)]
    # up stages in flow order: the up pipeline enters on the last device group
    stages += [StageAssignment(backbone=1, layer_range=rg, replicas=r, direction=UP)
               for rg, r in zip(reversed(ru), reversed(reps))]
    per_stage = []
    for st in stages:
        sv = (down if st.backbone == 0 else up).stage(st.layer_range[0], st.layer_range[1],
                                                       st.replicas)
        per_stage.append(StageCosts(t0=sv.t0, t_sync=sv.t_sync, t_comp=sv.t_comp, gap=sv.gap))
    return PartitionPlan(config=cfg, stages=stages, objective=key[0], per_stage=per_stage,
                         t_max=key[0], m_cdm=slots)


def partition_bidirectional(profile: ModelProfile, cluster: ClusterConfig, cfg: PlanConfig, *,
                            equal_replication: bool = True, m_cdm_fn=None) -> PartitionPlan:
    """Paired partition of two backbones pipelined in opposite directions
    (reference partitioner.py:450-501; paper Eqs. 9-15)."""
    if len(profile.backbones) != 2:
        raise ValueError("partition_bidirectional requires a profile with exactly two backbones")
    _check_common(cluster, cfg)
    S, D, M = cfg.num_stages, cfg.group_size, cfg.num_microbatches
    Ld, Lu = (len(b.layers) for b in profile.backbones)
    if min(Ld, Lu) < S:
        raise InfeasibleError(f"backbones have {Ld} and {Lu} layers, cannot both form {S} stages")
    equal_r = _equal_replication(cfg) if equal_replication else None
    down = StageEvaluator(profile.backbones[0], cluster, cfg.micro_batch, p2p_factor=2.0)
    up = StageEvaluator(profile.backbones[1], cluster, cfg.micro_batch, p2p_factor=2.0)
    if m_cdm_fn is None:
        from .scheduler import m_cdm as m_cdm_fn
    slots = m_cdm_fn(S, M)
    mult = slots + 2 * S - 2
    winner = None
    for w, y, mc, rd, ru, reps in _bidirectional_candidates(down, up, cfg, equal_r):
        key = (mult * w + _pos(y), mc, rd, ru, reps)
        if winner is None or key < winner[0]:
            winner = (key, rd, ru, reps)
    if winner is None:
        raise InfeasibleError(f"no feasible bidirectional partition for S={S}, D={D}")
    key, rd, ru, reps = winner
    return _bidirectional_plan(cfg, down, up, slots, key, rd, ru, reps)


def _check_common(cluster: ClusterConfig, cfg: PlanConfig) -> None:
    if cluster.world_size % cfg.group_size:
        raise InfeasibleError(
            f"group_size {cfg.group_size} does not divide world_size {cluster.world_size}")


def _equal_replication(cfg: PlanConfig) -> int:
    if cfg.group_size % cfg.num_stages:
        raise InfeasibleError(
            f"equal replication needs num_stages ({cfg.num_stages}) to divide "
            f"group_size ({cfg.group_size})")
    return cfg.group_size // cfg.num_stages


# ------------------------------------------------------------------ exhaustive oracle

ORACLE_MAX_LAYERS = 10
ORACLE_MAX_STAGES = 4
ORACLE_MAX_DEVICES = 6


def _compositions(total: int, parts: int):
    if parts == 1:
        yield (total,)
        return
    for head in range(1, total - parts + 2):
        for tail in _compositions(total - head, parts - 1):
            yield (head,) + tail


def _cuts_to_ranges(cuts, L):
    edges = (0, *cuts, L)
    return tuple(zip(edges[:-1], edges[1:]))


def brute_force_partition(profile: ModelProfile, cluster: ClusterConfig, cfg: PlanConfig, *,
                          equal_replication: bool = True, m_cdm_fn=None) -> PartitionPlan:
    """Enumerate every contiguous partition and replication split (test oracle)."""
    S, D = cfg.num_stages, cfg.group_size
    if (S > ORACLE_MAX_STAGES or D > ORACLE_MAX_DEVICES
            or any(len(b.layers) > ORACLE_MAX_LAYERS for b in profile.backbones)):
        raise OracleTooLargeError(
            f"oracle guards exceeded (L<={ORACLE_MAX_LAYERS}, S<={ORACLE_MAX_STAGES}, "
            f"D<={ORACLE_MAX_DEVICES})")
    _check_common(cluster, cfg)
    if equal_replication:
        rep_sets = [(_equal_replication(cfg),) * S]
    else:
        rep_sets = list(_compositions(D, S))
    if len(profile.backbones) == 1:
        return _brute_single(profile, cluster, cfg, rep_sets)
    return _brute_bidirectional(profile, cluster, cfg, rep_sets, m_cdm_fn)


def _brute_single(profile, cluster, cfg, rep_sets):
    comp = profile.backbones[0]
    L, S = len(comp.layers), cfg.num_stages
    if L < S:
        raise InfeasibleError(f"backbone has {L} layers, cannot form {S} stages")
    ev = StageEvaluator(comp, cluster, cfg.micro_batch)
    p = profile.selfcond_prob if cfg.selfcond else 0.0
    cands = []
    for cuts in itertools.combinations(range(1, L), S - 1):
        rngs = _cuts_to_ranges(cuts, L)
        for reps in rep_sets:
            svs = [ev.stage(lo, hi, r) for (lo, hi), r in zip(rngs, reps)]
            if None in svs:
                continue
            cands.append((max(s.t0 for s in svs), max(s.t0_sc for s in svs),
                          max(s.gap for s in svs), max(s.compute for s in svs), rngs, reps))
    winner = _select_single(ev, cfg, p, cands)
    if winner is None:
        raise InfeasibleError("oracle found no feasible partition")
    return _single_plan(ev, cfg, p, winner)


def _brute_bidirectional(profile, cluster, cfg, rep_sets, m_cdm_fn):
    S, M = cfg.num_stages, cfg.num_microbatches
    Ld, Lu = (len(b.layers) for b in profile.backbones)
    if min(Ld, Lu) < S:
        raise InfeasibleError(f"backbones have {Ld} and {Lu} layers, cannot both form {S} stages")
    down = StageEvaluator(profile.backbones[0], cluster, cfg.micro_batch, p2p_factor=2.0)
    up = StageEvaluator(profile.backbones[1], cluster, cfg.micro_batch, p2p_factor=2.0)
    if m_cdm_fn is None:
        from .scheduler import m_cdm as m_cdm_fn
    slots = m_cdm_fn(S, M)
    mult = slots + 2 * S - 2
    winner = None
    for cuts_d in itertools.combinations(range(1, Ld), S - 1):
        rd = _cuts_to_ranges(cuts_d, Ld)
        for cuts_u in itertools.combinations(range(1, Lu), S - 1):
            ru = tuple(reversed(_cuts_to_ranges(cuts_u, Lu)))  # group order
            for reps in rep_sets:
                evs = [down.stage(lo, hi, r) for (lo, hi), r in zip(rd, reps)]
                evs += [up.stage(lo, hi, r) for (lo, hi), r in zip(ru, reps)]
                if None in evs:
                    continue
                key = (mult * max(e.t0 for e in evs) + _pos(max(e.gap for e in evs)),
                       max(e.compute for e in evs), rd, ru, reps)
                if winner is None or key < winner[0]:
                    winner = (key, rd, ru, reps)
    if winner is None:
        raise InfeasibleError("oracle found no feasible bidirectional partition")
    key, rd, ru, reps = winner
    return _bidirectional_plan(cfg, down, up, slots, key, rd, ru, reps)


def validate_plan(plan: PartitionPlan, profile: ModelProfile, *,
                  equal_replication: bool = True) -> None:
    D = plan.config.group_size
    down_reps = [s.replicas for s in plan.stages_down]
    if sum(down_reps) != D:
        raise ValidationError("down-stage replicas do not sum to the group size")
    ups = plan.stages_up
    if ups:
        if sum(s.replicas for s in ups) != D:
            raise ValidationError("up-stage replicas do not sum to the group size")
        if [s.replicas for s in reversed(ups)] != down_reps:
            raise ValidationError("up stages must share the down stages' device groups")
    if equal_replication and len({s.replicas for s in plan.stages}) > 1:
        raise ValidationError(f"equal replication violated: {sorted({s.replicas for s in plan.stages})}")
    for b, comp in enumerate(profile.backbones):
        rngs = sorted(s.layer_range for s in plan.stages if s.backbone == b)
        if not rngs:
            continue
        if rngs[0][0] != 0 or rngs[-1][1] != len(comp.layers):
            raise ValidationError(f"backbone {b} ranges do not cover all layers")
        for (_, end), (start, _) in zip(rngs, rngs[1:]):
            if end != start:
                raise ValidationError(f"backbone {b} ranges not contiguous at {end} vs {start}")
