"""Device time of the c2 step's linear shapes: libdpipe fwd / dgrad / wgrad vs torch.matmul (cuBLAS),
CUDA events around a CUDA graph of 20 back-to-back calls (weights and activations L2-resident across reps is what
the step sees for the small weights; the activations here exceed L2 for M >= 8192)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2405_01248_b200 import ops  # noqa: E402


def timeit(fn, reps=20):
    """Device time per call: `reps` calls captured in one CUDA graph (host launch cost excluded)."""
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        for _ in range(3):
            fn()
    torch.cuda.current_stream().wait_stream(side)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps):
            fn()
    g.replay()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    g.replay()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps * 1e-3


SHAPES = [(32768, 320, 320), (32768, 960, 320), (32768, 2560, 320), (32768, 320, 1280),
          (8192, 640, 640), (8192, 1920, 640), (8192, 5120, 640), (8192, 640, 2560),
          (2048, 1280, 1280), (2048, 3840, 1280), (2048, 10240, 1280), (2048, 1280, 5120),
          (2464, 1024, 1024), (2464, 3072, 1024), (2464, 4096, 1024), (2464, 1024, 4096)]
for (M, N, K) in SHAPES:
    x = torch.randn(M, K, device="cuda").bfloat16()
    w = torch.randn(N, K, device="cuda").bfloat16()
    dy = torch.randn(M, N, device="cuda").bfloat16()
    y = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    dw = torch.zeros(N, K, device="cuda")
    fl = 2.0 * M * N * K
    r = dict(shape=[M, N, K])
    r["fwd_us"] = timeit(lambda: ops.linear(x, w, out=y)) * 1e6
    r["fwd_cublas_us"] = timeit(lambda: torch.matmul(x, w.t(), out=y)) * 1e6
    r["dgrad_us"] = timeit(lambda: ops.linear_dgrad(dy, w)) * 1e6
    r["dgrad_cublas_us"] = timeit(lambda: torch.matmul(dy, w)) * 1e6
    r["wgrad_us"] = timeit(lambda: ops.linear_wgrad(dy, x, dw)) * 1e6
    r["wgrad_cublas_us"] = timeit(lambda: torch.matmul(dy.t(), x)) * 1e6
    r["fwd_tflops"] = fl / r["fwd_us"] / 1e6
    print(json.dumps({k: (round(v, 1) if isinstance(v, float) else v) for k, v in r.items()}), flush=True)
