"""3x3 conv shapes of the c2 step (U-Net 32x32..4x4 levels, VAE 256..32) as the step runs them, against cuDNN
(torch channels_last bf16) on the same shapes: fwd (+bias), dgrad (cached flip copy where the step uses one),
wgrad (fp32 accumulate; cuDNN: bf16 weight grad). Device time per call from a CUDA graph of `reps` calls.
  python tools/conv_bench.py [--json out.json]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.nn.functional as F  # noqa: E402

from paper_2405_01248_b200 import ops  # noqa: E402
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from gemm_bench import timeit  # noqa: E402

# (N, H, W, C, K, stride, launches per c2 step of each pass)
SHAPES = [(32, 32, 32, 320, 320, 1), (32, 32, 32, 640, 320, 1), (32, 16, 16, 640, 640, 1),
          (32, 16, 16, 1280, 640, 1), (32, 8, 8, 1280, 1280, 1), (32, 8, 8, 2560, 1280, 1),
          (32, 4, 4, 1280, 1280, 1), (32, 4, 4, 2560, 1280, 1), (32, 32, 32, 320, 320, 2),
          (32, 16, 16, 640, 640, 2), (32, 8, 8, 1280, 1280, 2),
          (32, 256, 256, 128, 128, 1), (32, 128, 128, 256, 256, 1), (32, 64, 64, 512, 512, 1),
          (32, 32, 32, 512, 512, 1)]


class _P:
    def __init__(self):
        self.wt = None
        self.wt_fn = None


class _Store:
    def register_flip(self, p):
        pass


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--json", default=None)
    ap.add_argument("--no-cudnn", action="store_true")
    args = ap.parse_args()
    rows = []
    for (N, H, W, C, K, st) in SHAPES:
        P, Q = H // st, W // st
        x = torch.randn(N, H, W, C, device="cuda").bfloat16()
        w = (torch.randn(K, 3, 3, C, device="cuda") * 0.05).bfloat16()
        bias = torch.randn(K, device="cuda")
        dy = torch.randn(N, P, Q, K, device="cuda").bfloat16()
        dw = torch.zeros(K, 3, 3, C, device="cuda")
        fl = 2.0 * N * P * Q * K * 9 * C
        r = dict(shape=[N, H, W, C, K, st])
        if st == 1:
            out = torch.empty(N, P, Q, K, device="cuda", dtype=torch.bfloat16)
            r["fwd_us"] = timeit(lambda: ops.conv2d(x, w, bias=bias, out=out))
        else:
            r["fwd_us"] = timeit(lambda: ops.conv2d(x, w, stride=2, bias=bias, pad=(1, 1), out_hw=(P, Q)))
        cache = (_Store(), _P())
        ops.conv2d_dgrad(dy, w, x.shape, stride=st, pad=(1, 1), cache=cache)
        r["dgrad_us"] = timeit(lambda: ops.conv2d_dgrad(dy, w, x.shape, stride=st, pad=(1, 1), cache=cache))
        r["wgrad_us"] = timeit(lambda: ops.conv2d_wgrad(dy, x, dw, stride=st, pad=(1, 1)))
        if not args.no_cudnn:
            xc = x.permute(0, 3, 1, 2)  # NCHW view of NHWC memory = channels_last
            wc = w.permute(0, 3, 1, 2)
            dyc = dy.permute(0, 3, 1, 2)
            bb = bias.bfloat16()
            r["fwd_cudnn_us"] = timeit(lambda: F.conv2d(xc, wc, bb, stride=st, padding=1))
            r["dgrad_cudnn_us"] = timeit(lambda: torch.ops.aten.convolution_backward(
                dyc, xc, wc, None, [st, st], [1, 1], [1, 1], False, [0, 0], 1, [True, False, False]))
            r["wgrad_cudnn_us"] = timeit(lambda: torch.ops.aten.convolution_backward(
                dyc, xc, wc, None, [st, st], [1, 1], [1, 1], False, [0, 0], 1, [False, True, False]))
        for k in ("fwd", "dgrad", "wgrad"):
            r[f"{k}_tflops"] = fl / r[f"{k}_us"] / 1e6
            if f"{k}_cudnn_us" in r:
                r[f"{k}_vs_cudnn"] = r[f"{k}_us"] / r[f"{k}_cudnn_us"]
        rows.append(r)
        print(json.dumps({k: (round(v, 2) if isinstance(v, float) else v) for k, v in r.items()}), flush=True)
    if args.json:
        with open(args.json, "w") as f:
            json.dump(rows, f)


if __name__ == "__main__":
    main()
