"""Residual-epilogue linears of the c2 step for ncu: CLIP attention out (2464x1024x1024 + residual)
and U-Net level-0 projection (32768x320x320 + residual), plus the same without residual."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2405_01248_b200 import ops  # noqa: E402

torch.manual_seed(0)
a1 = torch.randn(2464, 1024, device="cuda").bfloat16()
w1 = torch.randn(1024, 1024, device="cuda").bfloat16()
r1 = torch.randn(2464, 1024, device="cuda").bfloat16()
a2 = torch.randn(32768, 320, device="cuda").bfloat16()
w2 = torch.randn(320, 320, device="cuda").bfloat16()
r2 = torch.randn(32768, 320, device="cuda").bfloat16()
b2 = torch.randn(320, device="cuda")
for _ in range(2):
    ops.linear(a1, w1, residual=r1)
    ops.linear(a1, w1)
    ops.linear(a2, w2, bias=b2, residual=r2)
    ops.linear(a2, w2, bias=b2)
torch.cuda.synchronize()
print("done")
