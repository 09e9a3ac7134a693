"""Measure the c2 model-profile/v1 on one B200 (what bench.py does on rank 0 for N > 1) and save it."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2405_01248_b200 import profiling_run  # noqa: E402
from paper_2405_01248_b200.pipefill import profile as pprof  # noqa: E402

D, M, gb = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
t0 = time.time()
prof = profiling_run.measure("c2", gb, D, M, "cuda:0")
print("profiled in", round(time.time() - t0, 1), "s")
os.makedirs("gpurun_out", exist_ok=True)
pprof.save_profile(prof, f"gpurun_out/c2_profile_D{D}_M{M}_gb{gb}.json")
bb = prof.backbones[0]
print("backbone layers", len(bb.layers), "frozen", [len(c.layers) for c in prof.frozen])
