"""Config c5 plan (CPU): the 2.2B U-Net on an 8-stage pipeline over 8 devices, M = 16, world batch
256, with per-layer costs from the measured c2 profile on B200
(profiles/r01_c2_measured_profile_D4_M4.json; backbone scaled by the measured c5/c2 step-time
ratio, VAE/CLIP as measured, all linear in batch). The reference planner must split long VAE
layers into partial batches (filler.py:75-242), and the executor's program for every device must
cover each frozen (component, layer) exactly once over the group batch."""

import json
import os

from paper_2405_01248_b200.adapter import build_group_program
from paper_2405_01248_b200.pipefill import planner, profile

HERE = os.path.dirname(os.path.abspath(__file__))
PROF = os.path.join(HERE, "..", "profiles", "r01_c2_measured_profile_D4_M4.json")
KEYS = sorted({1, 2, 3, 4, 6, 8, 10, 12, 16, 20, 24, 32, 40, 48, 64, 80, 96, 128, 192, 256})


def _linear(cost, scale):
    ks = sorted(cost, key=int)
    k = ks[-1]
    per = cost[k] / int(k) * scale
    return {b: per * b for b in KEYS}


def _layer(d, scale, frozen):
    return profile.LayerCost(
        fwd_time=_linear(d["fwd_time"], scale),
        bwd_time={b: 0.0 for b in KEYS} if frozen else _linear(d["bwd_time"], scale),
        fwd_comm_bytes={b: int(v) for b, v in _linear(d["fwd_comm_bytes"], 1.0).items()},
        bwd_comm_bytes={b: 0 for b in KEYS} if frozen else
        {b: int(v) for b, v in _linear(d["bwd_comm_bytes"], 1.0).items()},
        grad_bytes={b: int(list(d["grad_bytes"].values())[0] * (1 if frozen else 2.53)) for b in KEYS},
        out_bytes={b: int(v) for b, v in _linear(d["out_bytes"], 1.0).items()})


def c5_profile():
    d = json.load(open(PROF))
    bb = d["backbones"][0]
    # measured on B200 (profiles/r01_bench_n1_c5.jsonl vs r01_bench_n1_latest.jsonl): the c5 step
    # is ~1.4x the c2 step while the frozen encoders are unchanged -> backbone x ~2.0
    backbone = profile.ComponentProfile("unet_c5", tuple(_layer(l, 2.0, False) for l in bb["layers"]), True)
    frozen = tuple(profile.ComponentProfile(f["name"], tuple(_layer(l, 1.0, True) for l in f["layers"]), False)
                   for f in d["frozen"])
    return profile.ModelProfile((backbone,), frozen, (), 0.0)


def test_c5_eight_stage_plan_uses_partial_batches():
    prof = c5_profile()
    cluster = profile.ClusterConfig(8, profile.CommCosts(7.7e11, 1e-5, 7.25e11, 2e-5))
    from paper_2405_01248_b200.engine import B200_BUBBLE_MIN_LEN
    res = planner.evaluate_point(prof, cluster, 8, 16, 8, 256, bubble_min_len=B200_BUBBLE_MIN_LEN)
    fill = res["fill"]
    assert res["bubble_ratio_after"] < res["bubble_ratio_before"]
    assert fill.tail_time == 0.0  # every frozen layer fits in the bubbles
    partials = [f.partial for f in fill.fills if f.partial is not None]
    assert partials, "no partial-batch splitting in the c5 fill plan"
    vae = [c.name for c in prof.frozen].index("vae")
    assert any(p.component == vae for p in partials)
    counts = [len(c.layers) for c in prof.frozen]
    prog = build_group_program(res, counts)
    B = prog.group_batch
    cov = {}
    for pieces in prog.fills + [prog.tail]:
        for p in pieces:
            cov.setdefault((p.comp, p.layer), []).append((p.lo, p.hi))
    for c, n in enumerate(counts):
        for layer in range(n):
            iv = sorted(cov[(c, layer)])
            assert iv[0][0] == 0 and iv[-1][1] == B
            assert all(a[1] == b[0] for a, b in zip(iv, iv[1:]))
    # every device runs its stage's 2 x M compute tasks plus one sync
    for dev in range(8):
        ins = prog.device_program(dev).instrs
        assert sum(1 for i in ins if i[0] in ("fwd", "bwd")) == 32
        assert sum(1 for i in ins if i[0] == "sync") == 1
