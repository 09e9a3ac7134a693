"""Is the N=1 step host-bound? Compare host dispatch time of Trainer.step() with its GPU time."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2405_01248_b200 import engine  # noqa: E402

tr = engine.Trainer.create("c2", world=1, rank=0, S=1, M=1, D=1, world_batch=int(sys.argv[1]) if len(sys.argv) > 1 else 32)
tr.prefetch(12)
for _ in range(3):
    tr.step()
torch.cuda.synchronize()
for _ in range(3):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    a.record()
    tr.step()
    t1 = time.perf_counter()
    b.record()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"host dispatch {1e3 * (t1 - t0):.1f} ms, gpu {a.elapsed_time(b):.1f} ms, wall {1e3 * (t2 - t0):.1f} ms")
