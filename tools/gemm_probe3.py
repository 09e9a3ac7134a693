"""Short-K GEGLU projection of the c2 U-Net (32768x2560x320) for ncu source-level stall analysis."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2405_01248_b200 import ops  # noqa: E402

a = torch.randn(32768, 320, device="cuda").bfloat16()
w = torch.randn(2560, 320, device="cuda").bfloat16()
y = torch.empty(32768, 2560, device="cuda").bfloat16()
for _ in range(3):
    ops.linear(a, w, out=y)
torch.cuda.synchronize()
print("done")
