"""Where does the GPU wait for the host? One c2 step with every libdpipe launch bracketed by native CUDA
events (telemetry timer): busy = sum of bracket durations, idle = gaps between consecutive brackets on the
compute stream (launch order), attributed to the family of the launch that ends the gap.
  python tools/gpu_idle.py [--steps 2]
"""
import argparse
import os
import sys
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2405_01248_b200 import engine, telemetry  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--serial-optimizer", action="store_true")
    args = ap.parse_args()
    tr = engine.Trainer.create("c2", world=1, rank=0, S=1, M=1, D=1, world_batch=32)
    tr.prefetch(args.steps + 6)
    for _ in range(3):
        tr.step()
    torch.cuda.synchronize()
    if args.serial_optimizer:
        tr.ex.overlap_sync = False
    for s in range(args.steps):
        telemetry.timer.start(reserve=12000)
        t0 = torch.cuda.Event(enable_timing=True)
        t0.record()
        tr.step()
        t1 = torch.cuda.Event(enable_timing=True)
        t1.record()
        torch.cuda.synchronize()
        recs = list(telemetry.timer.records)
        nat = telemetry.timer.native
        span = t0.elapsed_time(t1)
        ivs = []
        for fam, fl, a, b in recs:
            st = nat.dp_timing_elapsed(0, a) if a else 0.0
            en = nat.dp_timing_elapsed(0, b)
            ivs.append((st, en, fam))
        telemetry.timer.stop()
        ivs.sort()
        busy = 0.0
        gaps = defaultdict(float)
        cur_end = ivs[0][0] if ivs else 0.0
        for st, en, fam in ivs:
            if st > cur_end:
                gaps[fam] += st - cur_end
            busy += max(0.0, en - max(st, cur_end))
            cur_end = max(cur_end, en)
        idle = sum(gaps.values())
        print(f"step {s}: span {span:.2f} ms, bracketed union {busy:.2f} ms, gaps {idle:.2f} ms over {len(ivs)} launches")
        for fam, g in sorted(gaps.items(), key=lambda kv: -kv[1])[:12]:
            print(f"   {g:7.3f} ms idle before {fam}")


if __name__ == "__main__":
    main()
