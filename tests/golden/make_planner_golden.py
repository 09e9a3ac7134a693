"""Generate tests/golden/planner_cases.json from the REFERENCE planner.

Run in the build container (needs /root/reference or baseline/_ref):
    python tests/golden/make_planner_golden.py
The fixture pins the restated planner (paper_2405_01248_b200.pipefill)
bit-exactly: every case stores the profile document, the cluster, the query
and the reference's full outputs (partition, simulated tasks, bubbles, fills,
tail, metrics, and the plan document of a grid search).
"""

import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
for cand in ("/root/reference/pkg/src", os.path.join(ROOT, "baseline", "_ref")):
    if os.path.isdir(os.path.join(cand, "pipefill")):
        sys.path.insert(0, cand)
        break
sys.path.insert(0, HERE)

import pipefill  # noqa: E402  (the reference)
from pipefill import planner, profile, scheduler  # noqa: E402

from planner_snapshot import point_snapshot, synthetic_profile_doc  # noqa: E402

assert "paper_2405_01248_b200" not in pipefill.__file__

CASES = [
    # (name, profile kwargs, world, comm, world_batch, points, bubble_min_len, equal_replication)
    ("sd21_like_s4m4", dict(seed=1, n_frozen=2, frozen_scale=1.0), 8,
     (2.0e11, 5e-5, 3.0e11, 1e-5), 256, [(4, 4, 4), (4, 8, 4), (2, 4, 2), (1, 1, 1)], 0.010, True),
    ("sd21_like_uneq", dict(seed=2, n_frozen=2), 8, (1.0e11, 1e-4, 1.0e11, 2e-5), 128,
     [(3, 4, 4), (2, 8, 4)], 0.005, False),
    ("selfcond_half", dict(seed=3, n_frozen=1, selfcond_prob=0.5), 4, (5e10, 1e-4, 8e10, 1e-5),
     64, [(2, 4, 2), (4, 4, 4), (2, 2, 4)], 0.010, True),
    ("selfcond_one", dict(seed=4, n_frozen=2, selfcond_prob=1.0), 4, (5e10, 1e-4, 8e10, 1e-5), 64,
     [(2, 4, 2), (4, 8, 4)], 0.0, True),
    ("cdm_bidir", dict(seed=5, n_backbones=2, n_frozen=1, layers=(5, 9)), 4,
     (8e10, 5e-5, 8e10, 1e-5), 64, [(2, 2, 2), (2, 4, 4), (4, 4, 4)], 0.010, True),
    ("many_frozen", dict(seed=6, n_frozen=3, frozen_layers=(4, 12), frozen_scale=2.0), 8,
     (2e11, 5e-5, 3e11, 1e-5), 256, [(4, 4, 4), (8, 16, 8), (2, 8, 8)], 0.010, True),
    ("tiny_c1", dict(seed=7, n_frozen=2, layers=(4, 6), frozen_layers=(2, 4)), 2,
     (5e10, 1e-5, 5e10, 1e-5), 32, [(2, 4, 2), (1, 4, 1)], 0.0, True),
]


def main():
    out = []
    for name, pkw, world, comm, wb, points, mlen, eq in CASES:
        doc = synthetic_profile_doc(**pkw)
        prof = profile.profile_from_dict(doc)
        cl = profile.ClusterConfig(world, profile.CommCosts(*comm))
        pts = []
        for S, M, D in points:
            try:
                res = planner.evaluate_point(prof, cl, S, M, D, wb, bubble_min_len=mlen,
                                             equal_replication=eq)
                pts.append({"point": [S, M, D], "result": point_snapshot(res, scheduler.extract_bubbles)})
            except pipefill.PipefillError as exc:
                pts.append({"point": [S, M, D], "error": type(exc).__name__, "message": str(exc)})
        try:
            rep = planner.search(prof, cl, planner.default_search_space(prof, cl, wb),
                                 bubble_min_len=mlen, equal_replication=eq)
            search_doc = planner.plan_document(rep)
        except pipefill.PipefillError as exc:
            search_doc = {"error": type(exc).__name__, "message": str(exc)}
        out.append({"name": name, "profile": doc, "world": world, "comm": list(comm),
                    "world_batch": wb, "bubble_min_len": mlen, "equal_replication": eq,
                    "points": pts, "search": search_doc})
    path = os.path.join(HERE, "planner_cases.json")
    with open(path, "w") as fh:
        json.dump({"generator": "tests/golden/make_planner_golden.py",
                   "reference": "pipefill 0.1.0 (/root/reference/pkg/src)", "cases": out}, fh,
                  sort_keys=True, separators=(",", ":"))
        fh.write("\n")
    print(path, os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()
