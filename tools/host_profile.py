"""cProfile of the host side of steady-state c2 steps (where the ~50 ms of dispatch per step goes)."""
import cProfile
import os
import pstats
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2405_01248_b200 import engine  # noqa: E402

tr = engine.Trainer.create("c2", world=1, rank=0, S=1, M=1, D=1, world_batch=32)
tr.prefetch(12)
for _ in range(3):
    tr.step()
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(3):
    tr.step()
torch.cuda.synchronize()
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(35)
