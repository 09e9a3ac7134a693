"""Plan adapter (CPU): the per-device programs replay the reference planner's Schedule and
FillPlan exactly — every simulated compute task once, in simulated order; every frozen
(component, layer) covered over the whole group batch exactly once; fills placed in their
bubbles; transfers and deliveries consistent with the pieces."""

import random

import pytest

from paper_2405_01248_b200.adapter import build_group_program, split_range
from paper_2405_01248_b200.pipefill import filler, planner, profile, scheduler


def _profile(seed, L=8, frozen=(5, 3), p=0.0, keys=(1, 2, 3, 4, 6, 8, 12, 16, 24, 32, 48, 64, 96, 128),
             backbones=1):
    rnd = random.Random(seed)

    def layer(f, b, frozen_layer=False):
        return profile.LayerCost(
            fwd_time={k: f * k for k in keys}, bwd_time={k: (0.0 if frozen_layer else b * k) for k in keys},
            fwd_comm_bytes={k: 1000 * k for k in keys}, bwd_comm_bytes={k: (0 if frozen_layer else 1000 * k) for k in keys},
            grad_bytes={k: 0 if frozen_layer else 4000 for k in keys}, out_bytes={k: 100 * k for k in keys})

    bbs = tuple(profile.ComponentProfile(f"bb{k}", [layer(rnd.uniform(0.5, 2) * 1e-3, rnd.uniform(1, 4) * 1e-3)
                                                    for _ in range(L)], True) for k in range(backbones))
    fr = [profile.ComponentProfile(f"f{i}", [layer(rnd.uniform(0.2, 1.5) * 1e-3, 0, True) for _ in range(n)],
                                   False) for i, n in enumerate(frozen)]
    return profile.ModelProfile(bbs, tuple(fr), (), p)


@pytest.mark.parametrize("seed,S,M,D,p,nb", [(0, 2, 4, 2, 0.0, 1), (1, 4, 4, 4, 0.0, 1), (2, 4, 8, 4, 0.0, 1),
                                             (3, 2, 4, 4, 0.0, 1), (4, 4, 4, 4, 0.5, 1), (5, 3, 6, 3, 0.0, 1),
                                             (6, 2, 4, 2, 0.0, 2), (7, 4, 4, 4, 0.0, 2)])
def test_programs_replay_schedule_and_fill(seed, S, M, D, p, nb):
    prof = _profile(seed, p=p, backbones=nb)
    cluster = profile.ClusterConfig(D, profile.CommCosts(2e11, 1e-5, 3e11, 1e-5))
    res = planner.evaluate_point(prof, cluster, S, M, D, 64 * M // 4)
    counts = [len(c.layers) for c in prof.frozen]
    prog = build_group_program(res, counts)
    B = prog.group_batch
    # 1. compute tasks: exactly the schedule's, per device, in start order
    sched = res["pre_fill_schedule"]
    for dev in range(D):
        want = [(t.kind, t.micro_batch, t.stage, 0 if t.direction == "down" else 1) for t in sorted(
            (t for t in sched.tasks if t.device == dev and t.kind in ("fwd", "bwd", "fwd_sc")),
            key=lambda t: (t.start, t.end))]
        got = [i for i in prog.devices[dev].instrs if i[0] in ("fwd", "bwd", "fwd_sc")]
        assert got == want
        kinds = [i[0] for i in prog.devices[dev].instrs]
        assert kinds[-1] == "deliver" and kinds.count("sync") == len(prog.pipes)
        for pi in range(len(prog.pipes)):
            last_bwd = max(k for k, i in enumerate(prog.devices[dev].instrs) if i[0] == "bwd" and i[3] == pi)
            assert prog.devices[dev].instrs[last_bwd + 1][:1] == ("sync",)
    # 2. frozen coverage: each (comp, layer) sample range covered exactly once
    for c, n in enumerate(counts):
        for layer in range(n):
            cov = [0] * B
            for ps in prog.fills + [prog.tail]:
                for pc in ps:
                    if pc.comp == c and pc.layer == layer:
                        for s in range(pc.lo, pc.hi):
                            cov[s] += 1
            assert cov == [1] * B, (c, layer)
    # 3. fill pieces run on the bubble's idle devices, sample counts match the FillPlan
    for f, pieces in zip(res["fill"].fills, prog.fills):
        assert {pc.device for pc in pieces} <= set(f.bubble.idle_devices)
        per = {}
        for pc in pieces:
            per[(pc.comp, pc.layer)] = per.get((pc.comp, pc.layer), 0) + pc.hi - pc.lo
        want = dict(f.full_samples)
        if f.partial is not None:
            key = (f.partial.component, f.partial.layer)
            want[key] = want.get(key, 0) + f.partial.samples
        assert per == {k: v for k, v in want.items() if v}
    # 4. every fill instruction sits before compute tasks starting after its bubble
    for dev in range(D):
        tasks = sorted((t for t in sched.tasks if t.device == dev and t.kind in ("fwd", "bwd", "fwd_sc")),
                       key=lambda t: (t.start, t.end))
        k = 0
        for ins in prog.devices[dev].instrs:
            if ins[0] in ("fwd", "bwd", "fwd_sc"):
                k += 1
            if ins[0] == "fill":
                b = res["fill"].fills[ins[1]].bubble
                assert all(t.end <= b.start + 1e-12 for t in tasks[:k])
                assert all(t.start >= b.end - 1e-12 for t in tasks[k:])
    # 5. transfers move data between different devices, ordered by production
    assert [t.seq for t in prog.transfers] == list(range(len(prog.transfers)))
    assert all(t.src != t.dst for t in prog.transfers)


def test_split_range():
    assert split_range(0, 10, 3) == [(0, 3), (3, 6), (6, 10)]
    assert split_range(5, 7, 4) == [(5, 5), (5, 6), (6, 6), (6, 7)]


@pytest.mark.parametrize("seed,S,M,D,p,nb", [(0, 2, 4, 2, 0.0, 1), (4, 4, 4, 4, 0.5, 1), (7, 4, 4, 4, 0.0, 2)])
def test_program_documents_round_trip(tmp_path, seed, S, M, D, p, nb):
    """The standalone per-rank program format: to_dict/from_dict and the rank
    files reproduce the in-memory programs exactly, and reject foreign documents."""
    import dataclasses
    import json

    from paper_2405_01248_b200.adapter import GroupProgram, load_rank_program, save_rank_programs

    prof = _profile(seed, p=p, backbones=nb)
    cluster = profile.ClusterConfig(2 * D, profile.CommCosts(2e11, 1e-5, 3e11, 1e-5))
    res = planner.evaluate_point(prof, cluster, S, M, D, 64 * M // 4)
    counts = [len(c.layers) for c in prof.frozen]
    prog = build_group_program(res, counts, selfcond=bool(p) or None)
    doc = json.loads(json.dumps(prog.to_dict()))
    assert dataclasses.asdict(GroupProgram.from_dict(doc)) == dataclasses.asdict(prog)
    paths = save_rank_programs(prog, str(tmp_path), groups=2, programs={"plain": prog, "selfcond": prog})
    assert len(paths) == 2 * D
    for r, path in enumerate(paths):
        rank, progs = load_rank_program(path)
        assert rank == r and set(progs) == {"plain", "selfcond"}
        assert dataclasses.asdict(progs["plain"]) == dataclasses.asdict(prog)
    with pytest.raises(ValueError):
        GroupProgram.from_dict({"format": "pipeline-plan/v1"})


def test_bidirectional_selfcond_extension():
    """Opt-in planner extension (planning_ext): both pipes of a two-backbone plan
    carry the self-conditioning forward with the reference simulator's own rules; the
    programs built from it contain the planned fwd_sc tasks instead of an out-of-plan pass."""
    from paper_2405_01248_b200.planning_ext import evaluate_point_selfcond

    prof = _profile(11, backbones=2, p=0.5)
    cluster = profile.ClusterConfig(4, profile.CommCosts(2e11, 1e-5, 3e11, 1e-5))
    ref = planner.evaluate_point(prof, cluster, 4, 4, 4, 64)
    ext = evaluate_point_selfcond(prof, cluster, 4, 4, 4, 64)
    assert ref["mode"] == planner.MODE_BIDIRECTIONAL
    assert ext["plan"].stages_down == ref["plan"].stages_down and ext["plan"].stages_up == ref["plan"].stages_up
    sc = [t for t in ext["pre_fill_schedule"].tasks if t.kind == "fwd_sc"]
    assert not any(t.kind == "fwd_sc" for t in ref["pre_fill_schedule"].tasks)
    assert len(sc) == 2 * 4 * 4  # both pipes, every stage, every micro-batch
    assert ext["pre_fill_schedule"].makespan > ref["pre_fill_schedule"].makespan
    # stage 0 of each pipe runs fwd(m) only after the pass of m left the pipe's last stage
    for d in ("down", "up"):
        tasks = [t for t in ext["pre_fill_schedule"].tasks if t.direction == d]
        for m in range(4):
            last_sc = max(t.end for t in tasks if t.kind == "fwd_sc" and t.micro_batch == m and t.stage == 3)
            first = min(t.start for t in tasks if t.kind == "fwd" and t.micro_batch == m and t.stage == 0)
            assert first >= last_sc - 1e-12
    counts = [len(c.layers) for c in prof.frozen]
    prog = build_group_program(ext, counts, selfcond=True)
    for dp in prog.devices:
        n_sc = sum(1 for i in dp.instrs if i[0] == "fwd_sc")
        assert n_sc == 2 * 4 and dp.instrs.index(next(i for i in dp.instrs if i[0] == "fwd_sc")) >= 0
    # the planned order interleaves the pass with the other pipe's tasks (not a prefix block)
    assert any(dp.instrs[0][0] != "fwd_sc" or dp.instrs[2 * 4 - 1][0] != "fwd_sc" for dp in prog.devices)
