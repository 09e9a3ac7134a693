"""Step time of c2 with the optimizer overlap off / on / hooks-only (diagnostics)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2405_01248_b200 import engine  # noqa: E402

tr = engine.Trainer.create("c2", world=1, rank=0, S=1, M=1, D=1, world_batch=32)
tr.prefetch(40)
for mode in ("off", "on", "off", "noop", "on"):
    ex = tr.ex
    ex.overlap_sync = mode == "on" or mode == "noop"
    if mode == "noop":
        ex._update_layers_orig = getattr(ex, "_update_layers_orig", ex._update_layers)
        ex._update_layers = lambda pi, nt, final=False: (ex._update_layers_orig(pi, nt, final) if final else
                                                         ex._ovl_top.__setitem__(pi, ex._ovl_top[pi]))
    elif hasattr(ex, "_update_layers_orig"):
        ex._update_layers = ex._update_layers_orig
    for _ in range(2):
        tr.step()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    a.record()
    for _ in range(5):
        tr.step()
    b.record()
    torch.cuda.synchronize()
    print(mode, "gpu ms/step", a.elapsed_time(b) / 5, "host ms/step", (time.perf_counter() - t0) * 200, flush=True)
