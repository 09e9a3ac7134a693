"""LayerNorm fwd / bwd (affine, parameter grads, accumulate into the residual branch) device time at the
U-Net / CLIP transformer shapes. CUDA-graph replay of 8 calls rotating over 4 input copies (> L2 for the
large shapes, so the bandwidth figures are HBM, not L2)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2405_01248_b200 import ops  # noqa: E402
from gn_bench import t  # noqa: E402

NC = 4
for rows, C in [(32768, 320), (8192, 640), (2048, 1280), (2464, 1024)]:
    xs = [torch.randn(rows, C, device="cuda").bfloat16() for _ in range(NC)]
    g = torch.randn(C, device="cuda")
    b = torch.randn(C, device="cuda")
    ys = [ops.layer_norm(x, g, b, 1e-5) for x in xs]
    dys = [torch.randn_like(xs[0]) for _ in range(NC)]
    accs = [torch.randn_like(xs[0]) for _ in range(NC)]
    dg = torch.zeros(C, device="cuda")
    db = torch.zeros(C, device="cuda")
    it = [0]

    def bwd():
        i = it[0] % NC
        it[0] += 1
        ops.layer_norm_bwd(xs[i], dys[i], g, ys[i][1], ys[i][2], dgamma=dg, dbeta=db, accumulate_into=accs[i])

    def fwd():
        i = it[0] % NC
        it[0] += 1
        ops.layer_norm(xs[i], g, b, 1e-5)
    msb = t(bwd, reps=8)
    msf = t(fwd, reps=8)
    nb = rows * C * 2
    print(f"({rows}, {C}) bwd+acc+pg {msb * 1e3:7.1f} us {4 * nb / msb / 1e6:6.0f} GB/s (4 passes) | "
          f"fwd {msf * 1e3:6.1f} us {2 * nb / msf / 1e6:6.0f} GB/s")
