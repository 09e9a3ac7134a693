"""Fused attention micro-benchmark on one B200: libdpipe flash fwd/bwd (hd 64) vs torch SDPA
(cuDNN / flash backends) on the SD v2.1 U-Net shapes of the c2 step. CUDA events, warm-up."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.nn.functional as F  # noqa: E402

from paper_2405_01248_b200 import ops  # noqa: E402


def timeit(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps * 1e-3


for (B, N, Nk, H) in [(32, 1024, 1024, 5), (32, 256, 256, 10), (32, 64, 64, 20), (32, 1024, 77, 5),
                      (32, 256, 77, 10), (8, 4096, 4096, 5)]:
    C = H * 64
    self_attn = N == Nk
    if self_attn:
        qkv = torch.randn(B, N, 3 * C, device="cuda").bfloat16()
        q, src, q_ld, kv_ld, k_off, v_off = qkv, qkv, 3 * C, 3 * C, C, 2 * C
    else:
        q = torch.randn(B, N, C, device="cuda").bfloat16()
        src = torch.randn(B, Nk, 2 * C, device="cuda").bfloat16()
        q_ld, kv_ld, k_off, v_off = C, 2 * C, 0, C
    o = torch.empty(B, N, C, device="cuda").bfloat16()
    lse = torch.empty(B, H, N, device="cuda")
    kp, vp = src.view(-1)[k_off:], src.view(-1)[v_off:]
    fwd = lambda: ops.flash_attn_fwd(q, kp, vp, o, B=B, N=N, Nk=Nk, heads=H, q_ld=q_ld, kv_ld=kv_ld,  # noqa: E731
                                     o_ld=C, scale=0.125, lse=lse)
    tf = timeit(fwd)
    do = torch.randn_like(o)
    dq = torch.empty_like(q)
    dsrc = dq if self_attn else torch.empty_like(src)
    bwd = lambda: ops.flash_attn_bwd(q, kp, vp, o, do, dq, dsrc.view(-1)[k_off:], dsrc.view(-1)[v_off:],  # noqa: E731
                                     lse, B=B, N=N, Nk=Nk, heads=H, q_ld=q_ld, kv_ld=kv_ld, o_ld=C, do_ld=C,
                                     dq_ld=q_ld, dkv_ld=kv_ld, scale=0.125)
    tb = timeit(bwd)
    qt = torch.randn(B, H, N, 64, device="cuda").bfloat16().requires_grad_()
    kt = torch.randn(B, H, Nk, 64, device="cuda").bfloat16().requires_grad_()
    vt = torch.randn(B, H, Nk, 64, device="cuda").bfloat16().requires_grad_()
    ts = timeit(lambda: F.scaled_dot_product_attention(qt, kt, vt))
    ot = F.scaled_dot_product_attention(qt, kt, vt)
    g = torch.randn_like(ot)
    tsb = timeit(lambda: torch.autograd.grad(ot, (qt, kt, vt), g, retain_graph=True))
    fl = 4.0 * B * H * N * Nk * 64
    print(json.dumps(dict(shape=[B, N, Nk, H], fwd_us=tf * 1e6, fwd_tflops=fl / tf / 1e12,
                          bwd_us=tb * 1e6, bwd_tflops=2.5 * fl / tb / 1e12,
                          sdpa_fwd_tflops=fl / ts / 1e12, sdpa_bwd_tflops=2.5 * fl / tsb / 1e12)), flush=True)
