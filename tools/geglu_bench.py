"""ff1 + GEGLU at the U-Net shapes: unfused (GEMM, then the GEGLU kernel) vs the GEMM's GEGLU epilogue."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import torch  # noqa: E402

from paper_2405_01248_b200 import ops  # noqa: E402
from gemm_bench import timeit  # noqa: E402

for M, C in [(32768, 320), (8192, 640), (2048, 1280)]:
    x = torch.randn(M, C, device="cuda").bfloat16()
    w = (torch.randn(8 * C, C, device="cuda") / C ** 0.5).bfloat16()
    b = torch.randn(8 * C, device="cuda")
    h = torch.empty(M, 8 * C, device="cuda", dtype=torch.bfloat16)
    y = torch.empty(M, 4 * C, device="cuda", dtype=torch.bfloat16)
    t_un = timeit(lambda: ops.geglu(ops.linear(x, w, bias=b, out=h)))
    t_fu = timeit(lambda: ops.linear_geglu(x, w, b, h_out=h, y_out=y))
    print(f"({M}, {C}): unfused {t_un:7.1f} us  fused {t_fu:7.1f} us")

# backward through ff2: dgrad GEMM + GEGLU backward kernel vs the GEGLU-backward epilogue
for M, C in [(32768, 320), (8192, 640), (2048, 1280)]:
    F_ = 4 * C
    dy = torch.randn(M, C, device="cuda").bfloat16()
    w2 = (torch.randn(C, F_, device="cuda") / F_ ** 0.5).bfloat16()
    h = torch.randn(M, 2 * F_, device="cuda").bfloat16()

    class _S:
        def register_flip(self, p):
            pass

    class _P:
        wt = None
        wt_fn = None
        flip_args = None
    c1, c2 = (_S(), _P()), (_S(), _P())
    t_un = timeit(lambda: ops.geglu_bwd(h, ops.linear_dgrad(dy, w2, cache=c1)))
    t_fu = timeit(lambda: ops.linear_dgrad_geglu(dy, w2, h, cache=c2))
    print(f"bwd ({M}, {C}): unfused {t_un:7.1f} us  fused {t_fu:7.1f} us")
