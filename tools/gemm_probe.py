"""Representative tcgen05 GEMM/conv launches of the c2 step (for ncu --set full captures):
level-0 U-Net conv fwd/dgrad/wgrad (32x32x320), VAE level-1 conv fwd (128x128x128),
U-Net level-0 proj linear (32768x320x320 + residual), CLIP fc1 (2464x4096x1024)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2405_01248_b200 import ops  # noqa: E402

torch.manual_seed(0)
x = torch.randn(32, 32, 32, 320, device="cuda").bfloat16()
w = (torch.randn(320, 3, 3, 320, device="cuda") * 0.05).bfloat16()
dy = torch.randn(32, 32, 32, 320, device="cuda").bfloat16()
dw = torch.zeros(320, 3, 3, 320, device="cuda")
xv = torch.randn(8, 128, 128, 128, device="cuda").bfloat16()
wv = (torch.randn(128, 3, 3, 128, device="cuda") * 0.05).bfloat16()
f = torch.randn(32768, 320, device="cuda").bfloat16()
g = torch.randn(320, 320, device="cuda").bfloat16()
r = torch.randn(32768, 320, device="cuda").bfloat16()
c = torch.randn(2464, 1024, device="cuda").bfloat16()
c2 = torch.randn(4096, 1024, device="cuda").bfloat16()
for _ in range(2):   # warm-up (first launch of each shape also sets kernel attributes)
    ops.conv2d(x, w)                       # 1 conv fwd
    ops.conv2d_dgrad(dy, w, x.shape)       # 2 conv dgrad
    ops.conv2d_wgrad(dy, x, dw)            # 3 conv wgrad
    ops.conv2d(xv, wv)                     # 4 VAE conv fwd
    ops.linear(f, g, residual=r)           # 5 short-K linear + residual
    ops.linear(c, c2)                      # 6 CLIP fc1
torch.cuda.synchronize()
print("done")
