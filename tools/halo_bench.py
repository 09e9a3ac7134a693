"""VAE-resolution 3x3 convs: halo strips on/off (DP_HALO env) — CUDA-graph-free event timing."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2405_01248_b200 import ops  # noqa: E402


def timeit(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e-3


for (Nb, H, C, K) in [(32, 256, 128, 128), (32, 128, 128, 256), (32, 128, 256, 256), (8, 256, 256, 256),
                      (32, 256, 64, 128)]:
    x = torch.randn(Nb, H, H, C, device="cuda").bfloat16()
    w = (torch.randn(K, 3, 3, C, device="cuda") * 0.05).bfloat16()
    t = timeit(lambda: ops.conv2d(x, w))
    fl = 2 * Nb * H * H * K * 9 * C
    print(json.dumps(dict(halo=os.environ.get("DP_HALO", "1"), shape=[Nb, H, H, C, K], us=t * 1e6,
                          tflops=fl / t / 1e12)), flush=True)
