"""Run one linear GEMM shape/pass a few times (for ncu captures): python tools/gemm_one.py M N K fwd|dgrad|wgrad [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2405_01248_b200 import ops  # noqa: E402

M, N, K = (int(v) for v in sys.argv[1:4])
kind = sys.argv[4]
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 3
x = torch.randn(M, K, device="cuda").bfloat16()
w = torch.randn(N, K, device="cuda").bfloat16()
bias = torch.randn(N, device="cuda")
dy = torch.randn(M, N, device="cuda").bfloat16()
dw = torch.zeros(N, K, device="cuda")
for _ in range(reps):
    if kind == "fwd":
        ops.linear(x, w, bias=bias)
    elif kind == "dgrad":
        ops.gemm(dy, w.t().contiguous(), torch.empty(M, K, device="cuda", dtype=torch.bfloat16), M=M, N=K, K=N,
                 a_ld=N, b_ld=N, d_ld=K)
    else:
        ops.linear_wgrad(dy, x, dw)
torch.cuda.synchronize()
print("done")
