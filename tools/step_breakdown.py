"""Per-launch-site breakdown of one c2 training step (GEMMs labelled by M x N x K)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2405_01248_b200 import engine, telemetry  # noqa: E402

telemetry.SHAPES = True
tr = engine.Trainer.create("c2", world=1, rank=0, S=1, M=1, D=1, world_batch=32)
tr.prefetch(8)
for _ in range(3):
    tr.step()
torch.cuda.synchronize()
telemetry.timer.start(reserve=20000)
tr.step()
st = telemetry.timer.stop()
tot = sum(v["ms"] for v in st.values())
rows = sorted(st.items(), key=lambda kv: -kv[1]["ms"])
print(f"total {tot:.2f} ms over {sum(v['launches'] for v in st.values())} launches")
for k, v in rows[:90]:
    tf = f"{v['flops'] / max(v['ms'], 1e-9) / 1e9:7.1f} TF/s" if v["flops"] else ""
    print(f"{v['ms']:8.3f} ms {v['launches']:4d}x  {tf}  {k}")
