"""One steady-state c2 training step bracketed by cudaProfilerStart/Stop, for
`ncu --profile-from-start off` launch lists (per-kernel device time of exactly one step)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2405_01248_b200 import engine  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
tr = engine.Trainer.create(cfg, world=1, rank=0, S=1, M=1, D=1, world_batch=32)
tr.prefetch(8)
for _ in range(3):
    tr.step()
torch.cuda.synchronize()
torch.cuda.profiler.start()
tr.step()
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("done")
