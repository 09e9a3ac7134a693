"""Kernel micro-benchmarks on one B200: libdpipe GEMM / implicit conv vs torch (cuBLAS/cuDNN).

CUDA-event timing on the launching stream, warm-up first, L2 flushed between reps.
Prints one line per shape with TFLOP/s for ours and torch's.
"""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.nn.functional as F
from paper_2405_01248_b200 import ops

torch.backends.cuda.matmul.allow_tf32 = False
flush = torch.empty(256 * 1024 * 1024, dtype=torch.int8, device="cuda")


def timeit(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        flush.zero_()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); fn(); e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    ts.sort()
    return ts[len(ts) // 2] * 1e-3


rows = []
for (M, N, K) in [(8192, 8192, 8192), (32768, 320, 1280), (32768, 2560, 320), (32768, 320, 2880),
                  (8192, 640, 5760), (2048, 1280, 11520), (4096, 4096, 4096)]:
    a = torch.randn(M, K, device="cuda").bfloat16()
    b = torch.randn(N, K, device="cuda").bfloat16()
    out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    t1 = timeit(lambda: ops.linear(a, b, out=out))
    t2 = timeit(lambda: torch.matmul(a, b.t(), out=out))
    fl = 2 * M * N * K
    rows.append(dict(kind="gemm", shape=[M, N, K], ours_tflops=fl / t1 / 1e12, torch_tflops=fl / t2 / 1e12))
    print(json.dumps(rows[-1]), flush=True)

for (Nb, H, C, K) in [(32, 32, 320, 320), (32, 16, 640, 640), (32, 8, 1280, 1280), (32, 4, 1280, 1280),
                      (32, 32, 640, 320), (8, 128, 128, 128), (8, 64, 256, 256)]:
    x = torch.randn(Nb, H, H, C, device="cuda").bfloat16()
    w = (torch.randn(K, 3, 3, C, device="cuda") * 0.05).bfloat16()
    xc = x.permute(0, 3, 1, 2).contiguous(memory_format=torch.channels_last)
    wc = w.permute(0, 3, 1, 2).contiguous(memory_format=torch.channels_last)
    t1 = timeit(lambda: ops.conv2d(x, w, stride=1, pad=(1, 1)))
    t2 = timeit(lambda: F.conv2d(xc, wc, padding=1))
    dy = torch.randn(Nb, H, H, K, device="cuda").bfloat16()
    dw = torch.zeros(K, 3, 3, C, device="cuda")
    t3 = timeit(lambda: ops.conv2d_wgrad(dy, x, dw, stride=1, pad=(1, 1)))
    t4 = timeit(lambda: ops.conv2d_dgrad(dy, w, x.shape, stride=1, pad=(1, 1)))
    fl = 2 * Nb * H * H * K * 9 * C
    rows.append(dict(kind="conv3x3", shape=[Nb, H, H, C, K], fwd_tflops=fl / t1 / 1e12,
                     torch_fwd_tflops=fl / t2 / 1e12, wgrad_tflops=fl / t3 / 1e12, dgrad_tflops=fl / t4 / 1e12))
    print(json.dumps(rows[-1]), flush=True)
