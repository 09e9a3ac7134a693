"""Run a few representative tcgen05 GEMM/conv launches (for ncu --set full captures)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2405_01248_b200 import ops  # noqa: E402

torch.manual_seed(0)
x = torch.randn(32, 32, 32, 320, device="cuda").bfloat16()
w = (torch.randn(320, 3, 3, 320, device="cuda") * 0.05).bfloat16()
a = torch.randn(8192, 8192, device="cuda").bfloat16()
b = torch.randn(8192, 8192, device="cuda").bfloat16()
f = torch.randn(32768, 320, device="cuda").bfloat16()
g = torch.randn(2560, 320, device="cuda").bfloat16()
dy = torch.randn(32, 32, 32, 320, device="cuda").bfloat16()
dw = torch.zeros(320, 3, 3, 320, device="cuda")
for _ in range(2):   # warm-up (first launch of each shape also sets kernel attributes)
    ops.conv2d(x, w)                       # 1 conv fwd, level-0 U-Net (M=32768 N=320 K=2880)
    ops.linear(a, b)                       # 2 square 8192^3
    ops.linear(f, g)                       # 3 GEGLU proj (M=32768 N=2560 K=320)
    ops.conv2d_wgrad(dy, x, dw)            # 4 conv wgrad (M=320 N=2880 K=32768)
    ops.conv2d_dgrad(dy, w, x.shape)       # 5 conv dgrad
torch.cuda.synchronize()
print("done")
