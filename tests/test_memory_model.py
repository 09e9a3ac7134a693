"""Memory-feasibility model (CPU): in-flight depth under the planner's eager-forward schedule.

The reference simulator dispatches a ready forward whenever no backward is ready
(scheduler.py:1-10,165-179), so stage 0 holds more micro-batches than warm-up-capped 1F1B
(min(M, S - s)). memory.inflight_depth counts them from the program the executor replays."""

import pytest

from paper_2405_01248_b200 import memory
from paper_2405_01248_b200.adapter import build_group_program
from paper_2405_01248_b200.pipefill import planner, profile

KEYS = (1, 2, 4, 8, 16, 32, 64, 128, 256)


def _uniform(L):
    def layer(frozen=False):
        return profile.LayerCost(
            fwd_time={k: 1e-3 * k for k in KEYS}, bwd_time={k: (0.0 if frozen else 2e-3 * k) for k in KEYS},
            fwd_comm_bytes={k: 1000 * k for k in KEYS}, bwd_comm_bytes={k: 0 if frozen else 1000 * k for k in KEYS},
            grad_bytes={k: 0 if frozen else 4000 for k in KEYS}, out_bytes={k: 100 * k for k in KEYS})

    bb = profile.ComponentProfile("unet", [layer() for _ in range(L)], True)
    fr = profile.ComponentProfile("vae", [layer(True) for _ in range(4)], False)
    return profile.ModelProfile((bb,), (fr,), (), 0.0)


@pytest.mark.parametrize("S,M,want", [(4, 8, 8), (8, 16, 16), (4, 16, 13)])
def test_inflight_depth_eager_forward(S, M, want):
    prof = _uniform(16)
    cluster = profile.ClusterConfig(S, profile.CommCosts(2e11, 1e-5, 3e11, 1e-5))
    res = planner.evaluate_point(prof, cluster, S, M, S, 8 * M)
    prog = build_group_program(res, [4])
    got = memory.inflight_depth(prog, 0)
    assert got == want, (S, M, got)
    # independent count on the reference-format simulated Schedule: forwards started minus
    # backwards started on device 0, in simulated start order
    live = peak = 0
    for t in sorted((t for t in res["pre_fill_schedule"].tasks if t.device == 0 and t.kind in ("fwd", "bwd")),
                    key=lambda t: (t.start, t.end)):
        live += 1 if t.kind == "fwd" else -1
        peak = max(peak, live)
    assert peak == got
    assert got > min(M, S)  # warm-up-capped 1F1B would under-count
    # never below warm-up-capped 1F1B, never above M, last stage holds one
    for dev in range(S):
        d = memory.inflight_depth(prog, dev)
        assert min(M, S - dev) <= d <= M
    assert memory.inflight_depth(prog, S - 1) == 1
