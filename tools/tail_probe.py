"""c2 N=1 step time with the frozen tail at the end (default) vs issued concurrently (DP_EARLY_TAIL)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2405_01248_b200 import engine  # noqa: E402

tr = engine.Trainer.create("c2", world=1, rank=0, S=1, M=1, D=1, world_batch=32)
tr.prefetch(40)
for _ in range(3):
    tr.step()
for _ in range(2):
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10):
        tr.step()
    b.record()
    torch.cuda.synchronize()
    print(os.environ.get("DP_EARLY_TAIL", "0"), "ms/step", round(a.elapsed_time(b) / 10, 2), flush=True)
