"""Run one conv pass a few times (for ncu captures): python tools/conv_one.py N H W C K stride fwd|dgrad|wgrad [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2405_01248_b200 import ops  # noqa: E402

N, H, W, C, K, st = (int(v) for v in sys.argv[1:7])
kind = sys.argv[7]
reps = int(sys.argv[8]) if len(sys.argv) > 8 else 3
P, Q = H // st, W // st
x = torch.randn(N, H, W, C, device="cuda").bfloat16()
w = (torch.randn(K, 3, 3, C, device="cuda") * 0.05).bfloat16()
dy = torch.randn(N, P, Q, K, device="cuda").bfloat16()
dw = torch.zeros(K, 3, 3, C, device="cuda")
for _ in range(reps):
    if kind == "fwd":
        ops.conv2d(x, w, stride=st, pad=(1, 1), out_hw=(P, Q))
    elif kind == "dgrad":
        ops.conv2d_dgrad(dy, w, x.shape, stride=st, pad=(1, 1))
    else:
        ops.conv2d_wgrad(dy, x, dw, stride=st, pad=(1, 1))
torch.cuda.synchronize()
print("done")
