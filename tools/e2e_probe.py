"""Per-step timeline of the e2e (pinned-host feed) loop: GPU time per step from CUDA events recorded
between steps (no host sync inside the loop) and host dispatch time per step, to locate the sporadic
e2e dips (a slow step on the GPU side vs a host stall)."""
import gc
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2405_01248_b200 import engine  # noqa: E402

tr = engine.Trainer.create("c2", world=1, rank=0, S=1, M=1, D=1, world_batch=32)
tr.prefetch(8, mode="device")
for _ in range(3):
    tr.step()
n = 40
tr.feed_mode = "host"
tr.prefetch(n + 8, mode="host")
for _ in range(4):  # warm-up without per-step syncs (host ahead of the GPU, as in the timed loop)
    tr.step()
tr.ex.total_loss().item()
torch.cuda.synchronize()
gc.collect()
gc.disable()
evs = [torch.cuda.Event(enable_timing=True) for _ in range(n + 1)]
host = []
evs[0].record()
for i in range(n):
    t0 = time.perf_counter()
    tr.step()
    host.append(1e3 * (time.perf_counter() - t0))
    evs[i + 1].record()
torch.cuda.synchronize()
gc.enable()
gpu = [evs[i].elapsed_time(evs[i + 1]) for i in range(n)]
for i in range(n):
    print(f"step {i:2d}: gpu {gpu[i]:6.1f} ms  host {host[i]:6.1f} ms")
print(f"mean gpu {sum(gpu) / n:.2f} ms, max {max(gpu):.1f}; mean host {sum(host) / n:.2f}, max {max(host):.1f}")
