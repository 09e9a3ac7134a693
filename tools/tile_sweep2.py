"""Device-time tile sweep (CUDA-graph timing, no host gaps) for mid-size linears of the c2 step:
DP_FORCE_BN x DP_FORCE_CG x DP_SPLITK_FRAC, with and without the residual epilogue."""
import json
import os
import subprocess
import sys

SHAPES = [(2048, 1280, 1280), (8192, 640, 640), (32768, 320, 320), (2464, 1024, 1024), (2464, 1024, 4096),
          (32768, 2560, 320), (8192, 5120, 640), (32768, 320, 1280)]

if len(sys.argv) > 1 and sys.argv[1] == "child":
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch
    from paper_2405_01248_b200 import ops

    def t(fn, reps=20):
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
        return a.elapsed_time(b) / reps * 1e-3
    out = {}
    for (M, N, K) in SHAPES:
        x = torch.randn(M, K, device="cuda").bfloat16()
        w = torch.randn(N, K, device="cuda").bfloat16()
        r = torch.randn(M, N, device="cuda").bfloat16()
        y = torch.empty(M, N, device="cuda").bfloat16()
        fl = 2 * M * N * K
        out[f"{M}x{N}x{K}"] = round(fl / t(lambda: ops.linear(x, w, out=y)) / 1e12)
        out[f"{M}x{N}x{K}+r"] = round(fl / t(lambda: ops.linear(x, w, residual=r, out=y)) / 1e12)
    print(json.dumps(out))
else:
    combos = [("0", "0", "50")] + [(bn, cg, "50") for bn in ("128", "160", "192", "256") for cg in ("1", "2")] + \
             [("0", "0", "0"), ("0", "0", "100")]
    for bn, cg, sk in combos:
        env = dict(os.environ, DP_FORCE_BN=bn, DP_FORCE_CG=cg, DP_SPLITK_FRAC=sk)
        r = subprocess.run([sys.executable, __file__, "child"], env=env, capture_output=True, text=True)
        print(f"BN={bn} CG={cg} SK={sk}", r.stdout.strip()[-900:] or r.stderr[-300:], flush=True)
