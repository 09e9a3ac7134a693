"""One flash fwd + bwd at the U-Net level-0 self-attention shape (32 x 1024 tokens x 5 heads) for ncu."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2405_01248_b200 import ops  # noqa: E402

B, N, H = 32, 1024, 5
C = H * 64
qkv = torch.randn(B, N, 3 * C, device="cuda").bfloat16()
o = torch.empty(B, N, C, device="cuda").bfloat16()
lse = torch.empty(B, H, N, device="cuda")
kp, vp = qkv.view(-1)[C:], qkv.view(-1)[2 * C:]
do = torch.randn_like(o)
dq = torch.empty_like(qkv)
for _ in range(2):
    ops.flash_attn_fwd(qkv, kp, vp, o, B=B, N=N, Nk=N, heads=H, q_ld=3 * C, kv_ld=3 * C, o_ld=C, scale=0.125,
                       lse=lse)
    ops.flash_attn_bwd(qkv, kp, vp, o, do, dq, dq.view(-1)[C:], dq.view(-1)[2 * C:], lse, B=B, N=N, Nk=N,
                       heads=H, q_ld=3 * C, kv_ld=3 * C, o_ld=C, do_ld=C, dq_ld=3 * C, dkv_ld=3 * C, scale=0.125)
torch.cuda.synchronize()
print("done")
