"""One GroupNorm(+SiLU) forward and backward per U-Net shape, for ncu (--set full)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2405_01248_b200 import ops  # noqa: E402

for shape in [(32, 32, 32, 640), (32, 32, 32, 320)]:
    x = torch.randn(*shape, device="cuda").bfloat16()
    C = shape[-1]
    g = torch.ones(C, device="cuda")
    b = torch.zeros(C, device="cuda")
    y, m, r = ops.group_norm(x, g, b, 32, 1e-6, True)
    dy = torch.randn_like(x)
    dg = torch.zeros(C, device="cuda")
    db = torch.zeros(C, device="cuda")
    ops.group_norm_bwd(x, dy, g, b, m, r, 32, True, dg, db)
torch.cuda.synchronize()
print("done")
