"""LayerNorm backward (affine, parameter grads, accumulate into the residual branch) device time at
the U-Net transformer shapes; CUDA-graph replay of 10 calls."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2405_01248_b200 import ops  # noqa: E402
from gn_bench import t  # noqa: E402

for rows, C in [(32768, 320), (8192, 640), (2048, 1280), (2464, 1024)]:
    x = torch.randn(rows, C, device="cuda").bfloat16()
    g = torch.randn(C, device="cuda")
    b = torch.randn(C, device="cuda")
    y, m, r = ops.layer_norm(x, g, b, 1e-5)
    dy = torch.randn_like(x)
    acc = torch.randn_like(x)
    dg = torch.zeros(C, device="cuda")
    db = torch.zeros(C, device="cuda")
    ms = t(lambda: ops.layer_norm_bwd(x, dy, g, m, r, dgamma=dg, dbeta=db, accumulate_into=acc))
    nb = x.numel() * 2 * 4
    print(f"({rows}, {C}) bwd+acc {ms * 1e3:7.1f} us {nb / ms / 1e6:6.0f} GB/s")

for rows, C in [(32768, 320), (8192, 640), (2048, 1280), (2464, 1024)]:
    x = torch.randn(rows, C, device="cuda").bfloat16()
    g = torch.randn(C, device="cuda")
    b = torch.randn(C, device="cuda")
    ms = t(lambda: ops.layer_norm(x, g, b, 1e-5))
    print(f"({rows}, {C}) fwd {ms * 1e3:7.1f} us {x.numel() * 4 / ms / 1e6:6.0f} GB/s")
