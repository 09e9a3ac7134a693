"""A few back-to-back small linear GEMMs (U-Net level-2 / CLIP shapes) for ncu --set full."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2405_01248_b200 import ops  # noqa: E402

for (M, N, K) in [(2048, 1280, 1280), (8192, 640, 640)]:
    x = torch.randn(M, K, device="cuda").bfloat16()
    w = torch.randn(N, K, device="cuda").bfloat16()
    y = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    for _ in range(3):
        ops.linear(x, w, out=y)
torch.cuda.synchronize()
print("done")
