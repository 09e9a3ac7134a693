"""Step time with device-resident vs pinned-host feeds (alternating), c2, N=1 (diagnostics)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2405_01248_b200 import engine  # noqa: E402

tr = engine.Trainer.create("c2", world=1, rank=0, S=1, M=1, D=1, world_batch=32)
for _ in range(3):
    tr.step()
for mode in ("device", "host", "device", "host"):
    tr.feed_mode = mode
    tr.prefetch(12, mode=mode)
    for _ in range(2):
        tr.step()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(8):
        tr.step()
    b.record()
    torch.cuda.synchronize()
    print(mode, "ms/step", a.elapsed_time(b) / 8, flush=True)
