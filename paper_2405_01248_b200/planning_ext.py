"""Opt-in planner extension: self-conditioning in bidirectional (two-backbone) plans.

NOT part of the reference API (which stays byte-compatible in `pipefill/`). The reference drops
self-conditioning whenever a profile has two backbones: `_planning_mode` returns bidirectional
(reference planner.py:115-118) and `build_bidirectional_schedule` simulates both pipes without
the extra forward (scheduler.py:346-347), although the paper says the bidirectional schedule "can
readily extend" to it. Config c4 (cascaded base + super-resolution U-Nets, each
self-conditioned) needs exactly that, so this module reuses the reference simulator's own
self-conditioning rules per pipe (fwd_sc tasks of every micro-batch flow down the pipe, the
last stage's output returns to stage 0 as feedback, and `fwd` of stage 0 waits for it;
scheduler.py:129-141,219-237) in the two-pipe simulation:

  * partition: the reference's `partition_bidirectional` (unchanged objective);
  * schedule: both pipes with `selfcond=True`, p2p time doubled as in the bidirectional
    schedule, and each pipe's feedback costed on ITS backbone's last layer at the last stage's
    replication (StageEvaluator.feedback_time; the reference's plan carries the down pipe's only);
  * fill / metrics: the reference's extract_bubbles / fill_all / apply_fill_plan / bubble_ratio.

`evaluate_point_selfcond` returns the same dict as the reference `evaluate_point`, so the adapter
builds the self-conditioned program from it like any other plan; the predicted c4 schedule then
contains the pass the executor runs (the measured-vs-predicted gap of the "outside the plan"
fallback, disappears).
"""

from __future__ import annotations

from dataclasses import replace

from .pipefill import filler, scheduler
from .pipefill.errors import InfeasibleError, ValidationError
from .pipefill.partitioner import PlanConfig, StageEvaluator, partition_bidirectional
from .pipefill.scheduler import DOWN, UP, PipelineSimulator, _expand, _pipe_timings, bubble_ratio, extract_bubbles


def _pipe_feedback(plan, profile, cluster, direction):
    stages = plan.stages_down if direction == DOWN else plan.stages_up
    ev = StageEvaluator(profile.backbones[stages[0].backbone], cluster, plan.config.micro_batch, p2p_factor=2.0)
    fb = ev.feedback_time(stages[-1].replicas)
    if fb is None:
        raise ValidationError(f"{direction} pipe: self-conditioning feedback cannot be costed")
    return 2.0 * (fb - cluster.comm.latency_p2p) + cluster.comm.latency_p2p


def build_bidirectional_schedule_selfcond(plan, profile, cluster):
    """Both pipes of a bidirectional plan with the self-conditioning forward."""
    if not plan.stages_up:
        return scheduler.build_schedule(plan, profile, cluster, selfcond=True)
    pipes = []
    for d in (DOWN, UP):
        pt = _pipe_timings(plan, profile, cluster, d, True, 2.0)
        pipes.append(replace(pt, feedback=_pipe_feedback(plan, profile, cluster, d)))
    comp, comm = PipelineSimulator(len(pipes[0].groups), pipes).run()
    return _expand(plan, pipes, comp, comm)


def evaluate_point_selfcond(profile, cluster, S, M, D, world_batch, *,
                            bubble_min_len=scheduler.MIN_BUBBLE_LEN, equal_replication=True):
    """`evaluate_point` (reference planner.py:141-187) for a two-backbone profile with the
    self-conditioning forward in both pipes; same result keys, mode "bidirectional+selfcond"."""
    if len(profile.backbones) != 2:
        raise ValidationError("evaluate_point_selfcond plans two-backbone (bidirectional) profiles")
    if cluster.world_size % D:
        raise InfeasibleError(f"group size {D} does not divide world size {cluster.world_size}")
    copies = cluster.world_size // D
    if world_batch % copies:
        raise InfeasibleError(f"global batch {world_batch} not divisible by {copies} group replicas")
    group_batch = world_batch // copies
    cfg = PlanConfig(num_stages=S, num_microbatches=M, group_size=D, global_batch=group_batch, selfcond=False)
    plan = partition_bidirectional(profile, cluster, cfg, equal_replication=equal_replication)
    pre = build_bidirectional_schedule_selfcond(plan, profile, cluster)
    fill = filler.fill_all(extract_bubbles(pre, bubble_min_len), profile, group_batch, pre)
    post = filler.apply_fill_plan(pre, fill)
    before = bubble_ratio(pre, extract_bubbles(pre, 0.0))
    idle_left = sum(b.duration * len(b.idle_devices) for b in extract_bubbles(post, 0.0))
    iter_time = post.makespan + fill.tail_time
    return {"plan": plan, "schedule": post, "pre_fill_schedule": pre, "fill": fill,
            "predicted_iter_time": iter_time, "bubble_ratio_before": before,
            "bubble_ratio_after": idle_left / (iter_time * D) if iter_time > 0 else 0.0,
            "throughput": copies * group_batch / iter_time if iter_time > 0 else 0.0,
            "mode": "bidirectional+selfcond"}


__all__ = ["build_bidirectional_schedule_selfcond", "evaluate_point_selfcond", "UP", "DOWN"]
