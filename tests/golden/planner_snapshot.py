"""Duck-typed JSON snapshot of planner outputs, shared by the golden-vector
generator (run against the reference `pipefill`) and the parity tests (run
against paper_2405_01248_b200.pipefill). Floats survive JSON exactly (repr
round trip), so snapshot equality is bit-exact equality."""

import random


def task_row(t):
    return [t.device, t.kind, t.micro_batch, t.stage, t.direction, t.start, t.end, t.tag]


def bubble_row(b):
    return [b.start, b.end, sorted(b.idle_devices)]


def fill_row(f):
    return {
        "bubble": bubble_row(f.bubble),
        "full_layers": {str(c): list(v) for c, v in sorted(f.full_layers.items())},
        "full_samples": [[c, l, n] for (c, l), n in sorted(f.full_samples.items())],
        "partial": None if f.partial is None else [f.partial.component, f.partial.layer,
                                                   f.partial.samples],
        "fill_time": f.fill_time,
    }


def plan_row(plan):
    return {
        "stages": [[s.backbone, list(s.layer_range), s.replicas, s.direction] for s in plan.stages],
        "per_stage": [[c.t0, c.t_sync, c.t_comp, c.gap] for c in plan.per_stage],
        "objective": plan.objective, "t_max": plan.t_max, "t_max_sc": plan.t_max_sc,
        "feedback_time": plan.feedback_time, "m_cdm": plan.m_cdm,
        "selfcond_prob": plan.selfcond_prob,
        "micro_batch": plan.config.micro_batch,
    }


def point_snapshot(res, extract_bubbles):
    pre = res["pre_fill_schedule"]
    return {
        "plan": plan_row(res["plan"]),
        "pre_tasks": [task_row(t) for t in pre.tasks],
        "pre_makespan": pre.makespan,
        "post_tasks": [task_row(t) for t in res["schedule"].tasks],
        "post_makespan": res["schedule"].makespan,
        "bubbles": [bubble_row(b) for b in extract_bubbles(pre, 0.0)],
        "fills": [fill_row(f) for f in res["fill"].fills],
        "tail": [[t.component, t.layer, t.samples, t.time] for t in res["fill"].tail],
        "residual": res["fill"].residual_bubble_time,
        "tail_time": res["fill"].tail_time,
        "iter": res["predicted_iter_time"],
        "before": res["bubble_ratio_before"],
        "after": res["bubble_ratio_after"],
        "throughput": res["throughput"],
        "mode": res["mode"],
    }


KEYS = (1, 2, 4, 8, 12, 16, 24, 32, 48, 64, 96, 128, 256)


def synthetic_profile_doc(seed, n_backbones=1, n_frozen=2, selfcond_prob=0.0, layers=(6, 14),
                          frozen_layers=(2, 10), frozen_scale=1.0, deps=True):
    """Deterministic synthetic model-profile/v1 document (pure Python RNG)."""
    rng = random.Random(seed)

    def layer(trainable, scale):
        base = rng.uniform(2e-4, 4e-3) * scale
        expo = rng.uniform(0.75, 1.0)
        fwd = {k: base * k ** expo for k in KEYS}
        act = rng.randint(2 ** 14, 2 ** 20)
        return {
            "fwd_time": {str(k): v for k, v in fwd.items()},
            "bwd_time": {str(k): (2.0 * v if trainable else 0.0) for k, v in fwd.items()},
            "fwd_comm_bytes": {str(k): k * act for k in KEYS},
            "bwd_comm_bytes": {str(k): k * act for k in KEYS},
            "grad_bytes": {str(k): (rng.randint(10 ** 6, 10 ** 8) if trainable else 0) for k in KEYS},
            "out_bytes": {str(k): k * rng.randint(2 ** 12, 2 ** 16) for k in KEYS},
        }

    doc = {
        "format": "model-profile/v1",
        "selfcond_prob": selfcond_prob,
        "backbones": [{"name": f"unet{i}", "trainable": True,
                       "layers": [layer(True, 1.0) for _ in range(rng.randint(*layers))]}
                      for i in range(n_backbones)],
        "frozen": [{"name": f"enc{i}", "trainable": False,
                    "layers": [layer(False, frozen_scale) for _ in range(rng.randint(*frozen_layers))]}
                   for i in range(n_frozen)],
        "frozen_deps": [["enc0", "enc1"]] if deps and n_frozen >= 2 and rng.random() < 0.5 else [],
    }
    return doc
