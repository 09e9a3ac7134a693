"""Device-time (CUDA graph) sweep of weight-gradient GEMMs: stream-K vs split-K targets (DP_SK_TARGET),
tile widths (DP_FORCE_BN / DP_FORCE_CG)."""
import json
import os
import subprocess
import sys

if len(sys.argv) > 1 and sys.argv[1] == "child":
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch
    from paper_2405_01248_b200 import ops

    def t(fn, reps=10):
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
    for (T, N, K) in [(32768, 320, 320), (8192, 640, 640), (2048, 1280, 1280), (32768, 2560, 320)]:
        dy = torch.randn(T, N, device="cuda").bfloat16()
        x = torch.randn(T, K, device="cuda").bfloat16()
        dw = torch.zeros(N, K, device="cuda")
        out[f"lin {N}x{K}x{T}"] = round(2 * T * N * K / t(lambda: ops.linear_wgrad(dy, x, dw)) / 1e12)
    for (Nb, H, C, Ko) in [(32, 32, 320, 320), (32, 16, 640, 640), (32, 8, 1280, 1280), (32, 4, 1280, 1280)]:
        x = torch.randn(Nb, H, H, C, device="cuda").bfloat16()
        dy = torch.randn(Nb, H, H, Ko, device="cuda").bfloat16()
        dw = torch.zeros(Ko, 3, 3, C, device="cuda")
        out[f"conv {H}x{H}x{C}->{Ko}"] = round(2 * Nb * H * H * Ko * 9 * C / t(lambda: ops.conv2d_wgrad(dy, x, dw)) / 1e12)
    print(json.dumps(out))
else:
    for sk in ["0", "37", "74", "148", "296"]:
        env = dict(os.environ, DP_SK_TARGET=sk)
        r = subprocess.run([sys.executable, __file__, "child"], env=env, capture_output=True, text=True)
        print(f"SK_TARGET={sk}", r.stdout.strip()[-600:] or r.stderr[-300:], flush=True)
