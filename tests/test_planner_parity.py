"""Planner parity: paper_2405_01248_b200.pipefill vs the reference `pipefill`.

* golden fixtures (tests/golden/planner_cases.json, generated from the
  reference by tests/golden/make_planner_golden.py) — always run;
* live randomized comparison against the reference when it is importable
  (this container: /root/reference; elsewhere baseline/_ref);
* SPEC.md known-answer examples and the acceptance properties
  (DP == brute force, 1F1B identities, fill coverage/capacity, determinism).
"""

import json
import math
import os
import random
import sys

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "golden"))

from planner_snapshot import point_snapshot, synthetic_profile_doc  # noqa: E402

from paper_2405_01248_b200.pipefill import (  # noqa: E402
    errors, filler, partitioner, planner, profile, scheduler)

GOLDEN = os.path.join(HERE, "golden", "planner_cases.json")


def _load_cases():
    with open(GOLDEN) as fh:
        return json.load(fh)["cases"]


def _norm(x):
    """JSON round trip (tuples -> lists) so snapshots compare like the fixture."""
    return json.loads(json.dumps(x, sort_keys=True))


@pytest.mark.parametrize("case", _load_cases(), ids=lambda c: c["name"])
def test_golden_planner_case(case):
    prof = profile.profile_from_dict(case["profile"])
    cl = profile.ClusterConfig(case["world"], profile.CommCosts(*case["comm"]))
    for pt in case["points"]:
        S, M, D = pt["point"]
        if "error" in pt:
            with pytest.raises(errors.PipefillError) as exc:
                planner.evaluate_point(prof, cl, S, M, D, case["world_batch"],
                                       bubble_min_len=case["bubble_min_len"],
                                       equal_replication=case["equal_replication"])
            assert type(exc.value).__name__ == pt["error"]
            assert str(exc.value) == pt["message"]
            continue
        res = planner.evaluate_point(prof, cl, S, M, D, case["world_batch"],
                                     bubble_min_len=case["bubble_min_len"],
                                     equal_replication=case["equal_replication"])
        got = _norm(point_snapshot(res, scheduler.extract_bubbles))
        want = pt["result"]
        for key in want:
            assert got[key] == want[key], f"{case['name']} {pt['point']} field {key}"
    if "error" in case["search"]:
        with pytest.raises(errors.NoFeasiblePlanError):
            planner.search(prof, cl, planner.default_search_space(prof, cl, case["world_batch"]),
                           bubble_min_len=case["bubble_min_len"],
                           equal_replication=case["equal_replication"])
    else:
        rep = planner.search(prof, cl, planner.default_search_space(prof, cl, case["world_batch"]),
                             bubble_min_len=case["bubble_min_len"],
                             equal_replication=case["equal_replication"])
        assert _norm(planner.plan_document(rep)) == case["search"]


def _reference():
    for cand in ("/root/reference/pkg/src",
                 os.path.join(os.path.dirname(HERE), "baseline", "_ref")):
        if os.path.isdir(os.path.join(cand, "pipefill")):
            if cand not in sys.path:
                sys.path.append(cand)
            import importlib

            return importlib.import_module("pipefill")
    return None


@pytest.mark.skipif(_reference() is None, reason="reference pipefill not importable here")
def test_live_random_parity_with_reference():
    import importlib

    ref = _reference()
    Rpl = importlib.import_module("pipefill.planner")
    Rpr = importlib.import_module("pipefill.profile")
    Rsc = importlib.import_module("pipefill.scheduler")
    rng = random.Random(1234)
    compared = 0
    for it in range(60):
        nb = 2 if rng.random() < 0.25 else 1
        doc = synthetic_profile_doc(seed=1000 + it, n_backbones=nb, n_frozen=rng.randint(0, 3),
                                    selfcond_prob=rng.choice([0.0, 0.5, 1.0]) if nb == 1 else 0.0,
                                    layers=(3, 10), frozen_layers=(1, 8),
                                    frozen_scale=rng.choice([0.5, 1.0, 3.0]))
        world = rng.choice([2, 4, 8])
        comm = (rng.uniform(1e10, 3e11), rng.uniform(0, 1e-4), rng.uniform(1e10, 3e11),
                rng.uniform(0, 1e-4))
        wb = rng.choice([32, 64, 128, 256])
        eq = rng.random() < 0.7
        mlen = rng.choice([0.0, 0.005, 0.010])
        rp, mp = Rpr.profile_from_dict(doc), profile.profile_from_dict(doc)
        rc = Rpr.ClusterConfig(world, Rpr.CommCosts(*comm))
        mc = profile.ClusterConfig(world, profile.CommCosts(*comm))
        for S, M, D in Rpl.default_search_space(rp, rc, wb).points()[:12]:
            try:
                r = _norm(point_snapshot(Rpl.evaluate_point(rp, rc, S, M, D, wb, bubble_min_len=mlen,
                                                            equal_replication=eq),
                                         Rsc.extract_bubbles))
            except ref.PipefillError as exc:
                r = ("err", type(exc).__name__, str(exc))
            try:
                m = _norm(point_snapshot(planner.evaluate_point(mp, mc, S, M, D, wb,
                                                                bubble_min_len=mlen,
                                                                equal_replication=eq),
                                         scheduler.extract_bubbles))
            except errors.PipefillError as exc:
                m = ("err", type(exc).__name__, str(exc))
            assert r == m, (it, S, M, D)
            compared += 1
    assert compared > 300


# ------------------------------------------------------------------ SPEC.md known answers

def _const_layer(fwd, bwd, keys=(1, 2, 4, 8, 16, 32, 64)):
    return profile.LayerCost(
        fwd_time={k: fwd for k in keys}, bwd_time={k: bwd for k in keys},
        fwd_comm_bytes={k: 0 for k in keys}, bwd_comm_bytes={k: 0 for k in keys},
        grad_bytes={k: 0 for k in keys}, out_bytes={k: 0 for k in keys})


ZERO_COMM = profile.ClusterConfig(8, profile.CommCosts(1e30, 0.0, 1e30, 0.0))


def test_cost_at_known_answers():
    lc = profile.LayerCost(fwd_time={8: 0.010, 16: 0.020}, bwd_time={8: 0.0, 16: 0.0},
                           fwd_comm_bytes={8: 0, 16: 0}, bwd_comm_bytes={8: 0, 16: 0},
                           grad_bytes={8: 0, 16: 0}, out_bytes={8: 0, 16: 0})
    assert profile.cost_at(lc, "fwd_time", 8) == 0.010
    assert profile.cost_at(lc, "fwd_time", 12) == pytest.approx(0.015, abs=1e-15)
    with pytest.raises(errors.ExtrapolationError):
        profile.cost_at(lc, "fwd_time", 4)


def test_stage_cost_known_answers():
    prof = profile.ModelProfile(backbones=(profile.ComponentProfile("b", (_const_layer(2.0, 4.0),), True),))
    sc = partitioner.stage_cost_single(prof, ZERO_COMM, (0, 1), 1, 4)
    assert (sc.t0, sc.t_comp, sc.gap) == (6.0, 4.0, -4.0)
    assert sc.t_sync == pytest.approx(0.0, abs=1e-20)
    assert partitioner.stage_cost_single(prof, ZERO_COMM, (0, 1), 1, 4, selfcond=True).t0 == 8.0


def test_partition_known_answers():
    one = profile.ModelProfile(backbones=(profile.ComponentProfile("b", (_const_layer(2.0, 4.0),), True),))
    cl1 = profile.ClusterConfig(1, profile.CommCosts(1e30, 0.0, 1e30, 0.0))
    plan = partitioner.partition_single(one, cl1, partitioner.PlanConfig(1, 4, 1, 4))
    assert plan.objective == 24.0
    four = profile.ModelProfile(backbones=(profile.ComponentProfile(
        "b", tuple(_const_layer(1.0, 2.0) for _ in range(4)), True),))
    cl2 = profile.ClusterConfig(2, profile.CommCosts(1e30, 0.0, 1e30, 0.0))
    plan = partitioner.partition_single(four, cl2, partitioner.PlanConfig(2, 4, 2, 8))
    assert plan.objective == 36.0
    assert [s.layer_range for s in plan.stages] == [(0, 2), (2, 4)]


def test_selfcond_objective_known_answers():
    assert partitioner.selfcond_objective(24.0, 32.0, 0.0) == 24.0
    assert partitioner.selfcond_objective(24.0, 32.0, 1.0) == 32.0
    assert partitioner.selfcond_objective(24.0, 32.0, 0.5) == 28.0


def _uniform_plan(S, M, tf=1.0, tb=1.0):
    prof = profile.ModelProfile(backbones=(profile.ComponentProfile(
        "b", tuple(_const_layer(tf, tb) for _ in range(S)), True),))
    cl = profile.ClusterConfig(S, profile.CommCosts(1e30, 0.0, 1e30, 0.0))
    cfg = partitioner.PlanConfig(S, M, S, M)
    return prof, cl, partitioner.partition_single(prof, cl, cfg)


@pytest.mark.parametrize("S", [2, 3, 4, 8])
@pytest.mark.parametrize("M", [2, 4, 8, 16])
def test_1f1b_identities(S, M):  # SPEC.md acceptance 3
    prof, cl, plan = _uniform_plan(S, M, 0.25, 0.25)
    sched = scheduler.build_schedule(plan, prof, cl)
    assert abs(sched.makespan - (M + S - 1) * 0.5) < 1e-12
    ratio = scheduler.bubble_ratio(sched, scheduler.extract_bubbles(sched, 0.0))
    assert abs(ratio - (S - 1) / (M + S - 1)) < 1e-12
    assert scheduler.critical_path(sched)[1] == 2 * (M + S - 1)


def test_fig2_first_bubble_and_s1():
    prof, cl, plan = _uniform_plan(4, 4, 0.25, 0.25)
    b0 = scheduler.extract_bubbles(scheduler.build_schedule(plan, prof, cl), 0.0)[0]
    assert (b0.start, b0.end, set(b0.idle_devices)) == (0.0, 0.25, {1, 2, 3})
    one = profile.ModelProfile(backbones=(profile.ComponentProfile("b", (_const_layer(2.0, 4.0),), True),))
    cl1 = profile.ClusterConfig(1, profile.CommCosts(1e30, 0.0, 1e30, 0.0))
    plan = partitioner.partition_single(one, cl1, partitioner.PlanConfig(1, 2, 1, 2))
    s = scheduler.build_schedule(plan, one, cl1)
    assert s.makespan == 12.0 and scheduler.extract_bubbles(s, 0.0) == []


def _frozen_profile(costs_by_comp):
    keys = (1, 2, 4, 8, 16, 32, 64, 128)
    comps = []
    for i, costs in enumerate(costs_by_comp):
        layers = tuple(profile.LayerCost(
            fwd_time={k: c * k for k in keys}, bwd_time={k: 0.0 for k in keys},
            fwd_comm_bytes={k: 0 for k in keys}, bwd_comm_bytes={k: 0 for k in keys},
            grad_bytes={k: 0 for k in keys}, out_bytes={k: 0 for k in keys}) for c in costs)
        comps.append(profile.ComponentProfile(f"f{i}", layers, False))
    bb = profile.ComponentProfile("b", (_const_layer(1.0, 1.0),), True)
    return profile.ModelProfile(backbones=(bb,), frozen=tuple(comps))


def test_ffc_known_answers():  # SPEC.md:282-284 (B/d = 1 so costs are per layer)
    st = filler.FillState(_frozen_profile([[3, 3, 3]]), 1)
    assert [v for v, _ in filler.ffc(st, 7.0, 1)] == [(2,)]
    st = filler.FillState(_frozen_profile([[4], [3, 3]]), 1)
    assert sorted(v for v, _ in filler.ffc(st, 7.0, 1)) == [(0, 2), (1, 1)]
    st = filler.FillState(_frozen_profile([[4], [3, 3]]), 1)
    assert [v for v, _ in filler.ffc(st, 0.0, 1)] == [(0, 0)]


def test_partial_continuation():  # 64 remaining, fits 16 -> 48 left
    prof = _frozen_profile([[1.0]])
    st = filler.FillState(prof, 64)
    bub = scheduler.Bubble(0.0, 16.5, frozenset({0}))
    f = filler.fill_bubble(st, 64, bub)
    assert f.partial.samples == 16 and st.remaining[0][0] == 48


def test_dp_equals_brute_force():  # SPEC.md acceptance 1
    rng = random.Random(7)
    for it in range(120):
        nb = 2 if it % 4 == 3 else 1
        doc = synthetic_profile_doc(seed=50 + it, n_backbones=nb, n_frozen=0, layers=(2, 7),
                                    selfcond_prob=rng.choice([0.0, 0.5]) if nb == 1 else 0.0)
        prof = profile.profile_from_dict(doc)
        D = rng.choice([1, 2, 3, 4])
        S = rng.randint(1, min(D, 3))
        M = rng.choice([1, 2, 4])
        cl = profile.ClusterConfig(D, profile.CommCosts(rng.uniform(1e9, 1e11), 1e-5,
                                                        rng.uniform(1e9, 1e11), 1e-5))
        eq = D % S == 0 and rng.random() < 0.5
        cfg = partitioner.PlanConfig(S, M, D, 8 * M, selfcond=prof.selfcond_prob > 0)
        try:
            fn = partitioner.partition_bidirectional if nb == 2 else partitioner.partition_single
            dp = fn(prof, cl, cfg, equal_replication=eq)
        except errors.InfeasibleError:
            with pytest.raises(errors.InfeasibleError):
                partitioner.brute_force_partition(prof, cl, cfg, equal_replication=eq)
            continue
        bf = partitioner.brute_force_partition(prof, cl, cfg, equal_replication=eq)
        assert math.isclose(dp.objective, bf.objective, rel_tol=1e-12)
        partitioner.validate_plan(dp, prof, equal_replication=eq)


def test_fill_coverage_and_capacity():  # SPEC.md acceptance 5
    for it in range(40):
        nb = 2 if it % 5 == 4 else 1
        doc = synthetic_profile_doc(seed=300 + it, n_backbones=nb, n_frozen=3,
                                    selfcond_prob=0.5 if (it % 3 == 0 and nb == 1) else 0.0,
                                    frozen_scale=2.0)
        prof = profile.profile_from_dict(doc)
        cl = profile.ClusterConfig(4, profile.CommCosts(1e11, 1e-5, 1e11, 1e-5))
        res = planner.evaluate_point(prof, cl, 4 if nb == 1 else 2, 4, 4, 128)
        gb = res["plan"].config.global_batch
        seen = {}
        for f in res["fill"].fills:
            assert f.fill_time <= f.bubble.duration + 1e-15
            for (c, l), n in f.full_samples.items():
                seen[(c, l)] = seen.get((c, l), 0) + n
            if f.partial is not None:
                k = (f.partial.component, f.partial.layer)
                seen[k] = seen.get(k, 0) + f.partial.samples
        for t in res["fill"].tail:
            seen[(t.component, t.layer)] = seen.get((t.component, t.layer), 0) + t.samples
        for c, comp in enumerate(prof.frozen):
            for l in range(len(comp.layers)):
                assert seen.get((c, l), 0) == gb


def test_plan_document_determinism_and_roundtrip(tmp_path):  # SPEC.md acceptance 8
    prof = profile.profile_from_dict(synthetic_profile_doc(seed=11, n_frozen=2))
    cl = profile.ClusterConfig(4, profile.CommCosts(1e11, 1e-5, 1e11, 1e-5))
    space = planner.default_search_space(prof, cl, 64)
    a = planner.emit_plan(planner.search(prof, cl, space), tmp_path / "a.json")
    planner.emit_plan(planner.search(prof, cl, space), tmp_path / "b.json")
    assert (tmp_path / "a.json").read_bytes() == (tmp_path / "b.json").read_bytes()
    assert planner.load_plan(tmp_path / "a.json") == _norm(a)


def test_profile_roundtrip_and_validation(tmp_path):
    doc = synthetic_profile_doc(seed=21, n_frozen=2)
    prof = profile.profile_from_dict(doc)
    profile.save_profile(prof, tmp_path / "p.json")
    assert profile.load_profile(tmp_path / "p.json") == prof
    bad = json.loads(json.dumps(doc))
    bad["frozen_deps"] = [["enc0", "enc1"], ["enc1", "enc0"]]
    with pytest.raises(errors.ValidationError, match="acyclic"):
        profile.profile_from_dict(bad)
    bad = json.loads(json.dumps(doc))
    bad["frozen"][0]["layers"][0]["bwd_time"]["1"] = 1.0
    with pytest.raises(errors.ValidationError, match="zero bwd_time"):
        profile.profile_from_dict(bad)
    bad = json.loads(json.dumps(doc))
    bad["format"] = "nope"
    with pytest.raises(errors.ParseError):
        profile.profile_from_dict(bad)


@pytest.mark.skipif(_reference() is None, reason="reference pipefill not importable here")
def test_reference_plans_drive_the_adapter_identically():
    """The drop-in boundary: the REFERENCE planner's own evaluate_point output (reference
    planner.py:141-187), fed to the executor's adapter (adapter.build_group_program), yields
    per-device programs identical to those from the restated planner — the executor runs the
    reference's plans unchanged."""
    import dataclasses
    import importlib

    from paper_2405_01248_b200.adapter import build_group_program

    _reference()
    Rpl = importlib.import_module("pipefill.planner")
    Rpr = importlib.import_module("pipefill.profile")
    rng = random.Random(4321)
    compared = 0
    for it in range(40):
        nb = 2 if rng.random() < 0.25 else 1
        doc = synthetic_profile_doc(seed=2000 + it, n_backbones=nb, n_frozen=rng.randint(1, 3),
                                    selfcond_prob=rng.choice([0.0, 0.5]) if nb == 1 else 0.0,
                                    layers=(3, 10), frozen_layers=(1, 8), frozen_scale=rng.choice([0.5, 1.0, 3.0]))
        world = rng.choice([2, 4, 8])
        comm = (rng.uniform(1e10, 3e11), rng.uniform(0, 1e-4), rng.uniform(1e10, 3e11), rng.uniform(0, 1e-4))
        wb = rng.choice([32, 64, 128])
        rp, mp = Rpr.profile_from_dict(doc), profile.profile_from_dict(doc)
        rc = Rpr.ClusterConfig(world, Rpr.CommCosts(*comm))
        mc = profile.ClusterConfig(world, profile.CommCosts(*comm))
        counts = [len(c["layers"]) for c in doc["frozen"]]
        for S, M, D in Rpl.default_search_space(rp, rc, wb).points()[:6]:
            try:
                r = Rpl.evaluate_point(rp, rc, S, M, D, wb, bubble_min_len=0.005)
                m = planner.evaluate_point(mp, mc, S, M, D, wb, bubble_min_len=0.005)
            except Exception:
                continue
            deps = tuple(mp.frozen_dep_indices())
            for sc in (False, True) if r["mode"] == "selfcond" else (False,):
                pr = build_group_program(r, counts, selfcond=sc or None, frozen_deps=deps)
                pm = build_group_program(m, counts, selfcond=sc or None, frozen_deps=deps)
                assert dataclasses.asdict(pr) == dataclasses.asdict(pm), (it, S, M, D)
                compared += 1
    assert compared > 60
