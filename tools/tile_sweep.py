"""Tile-shape sweep for representative U-Net GEMM/conv shapes (DP_FORCE_BN / DP_FORCE_CG)."""
import json
import os
import subprocess
import sys

if len(sys.argv) > 1 and sys.argv[1] == "child":
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch
    from paper_2405_01248_b200 import ops
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.int8, device="cuda")

    def t(fn):
        for _ in range(3):
            fn()
        ts = []
        for _ in range(10):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); fn(); b.record(); torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        ts.sort()
        return ts[5] * 1e-3
    out = {}
    x = torch.randn(32, 32, 32, 320, device="cuda").bfloat16()
    w = (torch.randn(320, 3, 3, 320, device="cuda") * 0.05).bfloat16()
    out["conv0_fwd"] = 2 * 32768 * 320 * 2880 / t(lambda: ops.conv2d(x, w)) / 1e12
    a = torch.randn(32768, 320, device="cuda").bfloat16()
    b = torch.randn(320, 320, device="cuda").bfloat16()
    out["lin_32768x320x320"] = 2 * 32768 * 320 * 320 / t(lambda: ops.linear(a, b)) / 1e12
    a2 = torch.randn(32768, 2880, device="cuda").bfloat16()
    b2 = torch.randn(320, 2880, device="cuda").bfloat16()
    out["lin_32768x320x2880"] = 2 * 32768 * 320 * 2880 / t(lambda: ops.linear(a2, b2)) / 1e12
    a3 = torch.randn(32768, 320, device="cuda").bfloat16()
    b3 = torch.randn(2560, 320, device="cuda").bfloat16()
    out["lin_32768x2560x320"] = 2 * 32768 * 2560 * 320 / t(lambda: ops.linear(a3, b3)) / 1e12
    x2 = torch.randn(32, 16, 16, 640, device="cuda").bfloat16()
    w2 = (torch.randn(640, 3, 3, 640, device="cuda") * 0.05).bfloat16()
    out["conv1_fwd"] = 2 * 8192 * 640 * 5760 / t(lambda: ops.conv2d(x2, w2)) / 1e12
    print(json.dumps(out))
else:
    for bn in ["0", "128", "160", "192", "256"]:
        for cg in ["0", "1", "2"]:
            env = dict(os.environ, DP_FORCE_BN=bn, DP_FORCE_CG=cg)
            r = subprocess.run([sys.executable, __file__, "child"], env=env, capture_output=True, text=True)
            print(f"BN={bn} CG={cg}", r.stdout.strip()[-400:] or r.stderr[-300:], flush=True)
