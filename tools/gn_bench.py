"""GroupNorm fwd/bwd achieved HBM bandwidth at the VAE / U-Net shapes."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2405_01248_b200 import ops  # noqa: E402


def t(fn, reps=10):
    """Device time per call: the calls are captured in a CUDA graph (no host dispatch gaps)."""
    fn()
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            for _ in range(reps):
                fn()
    torch.cuda.current_stream().wait_stream(s)
    g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    g.replay()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


for shape in ([] if __name__ != "__main__" else [(32, 256, 256, 128), (32, 128, 128, 256), (32, 64, 64, 512), (32, 32, 32, 320), (32, 32, 32, 640),
              (32, 16, 16, 1280), (32, 8, 8, 2560), (32, 8, 8, 1280), (32, 4, 4, 1280), (32, 4, 4, 2560)]):
    x = torch.randn(*shape, device="cuda").bfloat16()
    C = shape[-1]
    g = torch.ones(C, device="cuda")
    b = torch.zeros(C, device="cuda")
    y, m, r = ops.group_norm(x, g, b, 32, 1e-6, True)
    ms = t(lambda: ops.group_norm(x, g, b, 32, 1e-6, True))
    nb = x.numel() * 2
    dy = torch.randn_like(x)
    dg = torch.zeros(C, device="cuda")
    db = torch.zeros(C, device="cuda")
    msb = t(lambda: ops.group_norm_bwd(x, dy, g, b, m, r, 32, True, dg, db))
    print(f"{shape}: fwd {ms * 1e3:8.1f} us  {3 * nb / ms / 1e6:7.0f} GB/s (3 passes) | "
          f"bwd {msb * 1e3:8.1f} us {5 * nb / msb / 1e6:7.0f} GB/s (5 passes)")
