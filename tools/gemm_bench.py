"""Linear GEMM shapes of the c2 step as the step runs them, against cuBLAS (torch.mm) on the same shapes:
  fwd    y[M,N] (bf16) = x[M,K] w[N,K]^T + bias      (ops.linear)
  dgrad  dx[M,K] (bf16) = dy[M,N] w                  (ops.linear_dgrad with the cached flip: B K-major)
  wgrad  dW[N,K] (fp32) += dy^T x                    (ops.linear_wgrad; cuBLAS: torch.mm(..., out_dtype=fp32))
Device time per call from CUDA events around a CUDA graph of `reps` back-to-back calls (no host cost).
  python tools/gemm_bench.py [--json out.json] [--only fwd,dgrad,wgrad]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2405_01248_b200 import ops  # noqa: E402


def timeit(fn, reps=20):
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
    return s.elapsed_time(e) / reps * 1e3  # us


# (M, N, K, launches per c2 step of each pass): U-Net transformer linears (levels 0-2 + mid), CLIP (fwd only)
SHAPES = [(32768, 320, 320, 3), (32768, 960, 320, 1), (32768, 2560, 320, 1), (32768, 320, 1280, 1),
          (8192, 640, 640, 3), (8192, 1920, 640, 1), (8192, 5120, 640, 1), (8192, 640, 2560, 1),
          (2048, 1280, 1280, 3), (2048, 3840, 1280, 1), (2048, 10240, 1280, 1), (2048, 1280, 5120, 1),
          (32768, 640, 1024, 0), (2464, 1024, 1024, 0), (2464, 3072, 1024, 0), (2464, 4096, 1024, 0),
          (2464, 1024, 4096, 0), (32, 1280, 1280, 0), (32, 320, 1280, 0), (32, 640, 1280, 0)]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--json", default=None)
    ap.add_argument("--only", default="fwd,dgrad,wgrad")
    args = ap.parse_args()
    passes = args.only.split(",")
    rows = []
    for (M, N, K, _) in SHAPES:
        x = torch.randn(M, K, device="cuda").bfloat16()
        w = torch.randn(N, K, device="cuda").bfloat16()
        wt = w.t().contiguous()
        bias = torch.randn(N, device="cuda")
        dy = torch.randn(M, N, device="cuda").bfloat16()
        y = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        dx = torch.empty(M, K, device="cuda", dtype=torch.bfloat16)
        dw = torch.zeros(N, K, device="cuda")
        fl = 2.0 * M * N * K
        r = dict(shape=[M, N, K])
        if "fwd" in passes:
            r["fwd_us"] = timeit(lambda: ops.linear(x, w, bias=bias, out=y))
            r["fwd_cublas_us"] = timeit(lambda: torch.addmm(bias.bfloat16(), x, w.t(), out=y))
        if "dgrad" in passes:
            cache = (_Store(), _P(wt))
            r["dgrad_us"] = timeit(lambda: ops.linear_dgrad(dy, w, out=dx, cache=cache))
            r["dgrad_cublas_us"] = timeit(lambda: torch.mm(dy, w, out=dx))
            # the weight read MN-major in place (no flip-transposed copy)
            r["dgrad_mn_us"] = timeit(lambda: ops.gemm(dy, w, dx, M=M, N=K, K=N, a_ld=N, b_ld=K, b_mn=True, d_ld=K))
        if "wgrad" in passes and M >= 1024:
            r["wgrad_us"] = timeit(lambda: ops.linear_wgrad(dy, x, dw))
            r["wgrad_cublas_us"] = timeit(lambda: torch.mm(dy.t(), x, out_dtype=torch.float32))
        for k in ("fwd", "dgrad", "wgrad"):
            if f"{k}_us" in r:
                r[f"{k}_tflops"] = fl / r[f"{k}_us"] / 1e6
                r[f"{k}_vs_cublas"] = r[f"{k}_us"] / r[f"{k}_cublas_us"]
        rows.append(r)
        print(json.dumps({k: (round(v, 2) if isinstance(v, float) else v) for k, v in r.items()}), flush=True)
    if args.json:
        with open(args.json, "w") as f:
            json.dump(rows, f)


class _P:
    """a parameter whose cached dgrad copy (wt) is already present (what the step sees after iteration 0)"""

    def __init__(self, wt):
        self.wt = wt


class _Store:
    def register_flip(self, p):
        pass


if __name__ == "__main__":
    main()
