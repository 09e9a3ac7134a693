"""Device time of every libdpipe launch of one training step, without host overhead.

Records every C-ABI call of one step (argument structs copied by value), then replays the
first call of every distinct signature 10x inside a CUDA graph (device time per call, warm L2,
none of the ctypes / Python launch cost) and weights it by the signature's launch count. Pointers stay valid because the caching allocator
keeps its segments mapped (the replay reads stale data; calls that index memory through
data-dependent ids — embeddings, timestep tables — are skipped).

Prints per-signature totals (GEMM shapes, conv geometry, other kernels) sorted by time, and
optionally compares each linear GEMM signature with cuBLAS (torch.matmul) on fresh tensors.

  python tools/kernel_replay.py [--config c2] [--top 60] [--cublas] [--json out.json]
"""
import argparse
import ctypes
import json
import os
import sys
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2405_01248_b200 import _lib, engine  # noqa: E402

SKIP = {"dp_embed", "dp_q_sample", "dp_pred_x0", "dp_last_error", "dp_version", "dp_group_norm_workspace",
        "dp_gemm_workspace", "dp_conv_fwd_workspace", "dp_conv_dgrad_workspace", "dp_flash_attn_bwd_workspace"}


class Recorder:
    def __init__(self, lib):
        self._lib = lib
        self.calls = []
        self.on = False

    def __getattr__(self, name):
        f = getattr(self._lib, name)
        if not self.on or not name.startswith("dp_") or name in SKIP:
            return f

        def call(*args):
            saved = []
            for a in args:
                obj = getattr(a, "_obj", None)
                if obj is not None and isinstance(obj, ctypes.Structure):
                    saved.append(("struct", type(obj).from_buffer_copy(obj)))
                else:
                    saved.append(("val", a))
            self.calls.append((name, saved))
            return f(*args)
        return call


def signature(name, saved):
    if saved and saved[0][0] == "struct":
        s = saved[0][1]
        if name == "dp_gemm":
            return (f"gemm {s.M}x{s.N}x{s.K}{'a' if s.a_mn_major else ''}{'b' if s.b_mn_major else ''}"
                    f"{'+acc' if s.out_mode else ''}{'+bias' if s.bias else ''}{'+res' if s.Res else ''}"
                    f"x{max(1, s.batch1) * max(1, s.batch2)}"), 2.0 * s.M * s.N * s.K * max(1, s.batch1) * max(1, s.batch2)
        if name.startswith("dp_conv"):
            if name == "dp_conv_wgrad":
                fl = 2.0 * s.N * s.P * s.Q * s.K * s.R * s.S * s.C
            elif name == "dp_conv_dgrad":
                fl = 2.0 * s.N * s.H * s.W * s.C * s.R * s.S * s.K
            else:
                fl = 2.0 * s.N * s.P * s.Q * s.K * s.R * s.S * s.C
            return f"{name[3:]} {s.N}x{s.H}x{s.W}x{s.C}->{s.K} r{s.R}s{s.stride} pq{s.P}x{s.Q}", fl
        if name.startswith("dp_flash"):
            fl = 4.0 * s.B * s.heads * s.N * s.Nk * s.head_dim * (0.5 if s.causal else 1.0)
            if "bwd" in name:
                fl *= 2.5
            return f"{name[3:]} B{s.B} h{s.heads} N{s.N} Nk{s.Nk}{' causal' if s.causal else ''}", fl
    ints = [v for k, v in saved[:-1] if k == "val" and isinstance(v, int) and abs(v) < 10 ** 7]
    return f"{name[3:]} {ints[:6]}", 0.0


def _args(saved, sh, keep):
    args = []
    for k, v in saved:
        if k == "struct":
            c = type(v).from_buffer_copy(v)
            keep.append(c)
            args.append(ctypes.byref(c))
        else:
            args.append(v)
    args[-1] = sh
    return args


def time_call(name, saved, reps=10):
    """Device time of one recorded call: `reps` copies captured in one CUDA graph, replayed."""
    stream = torch.cuda.Stream()
    lib = _lib._lib
    keep = []
    fn = getattr(lib, name)
    with torch.cuda.stream(stream):
        for _ in range(2):
            if fn(*_args(saved, stream.cuda_stream, keep)):
                raise RuntimeError(f"{name}: {lib.dp_last_error().decode()}")
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        for _ in range(reps):
            fn(*_args(saved, stream.cuda_stream, keep))
    g.replay()
    torch.cuda.synchronize()
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0.record()
    g.replay()
    s1.record()
    torch.cuda.synchronize()
    return s0.elapsed_time(s1) / reps


def cublas_time(M, N, K, a_mn, b_mn, reps=20):
    A = torch.randn((K, M) if a_mn else (M, K), device="cuda").bfloat16()
    B = torch.randn((K, N) if b_mn else (N, K), device="cuda").bfloat16()
    Aop = A.t() if a_mn else A
    Bop = B if b_mn else B.t()
    out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    for _ in range(3):
        torch.matmul(Aop, Bop, out=out)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps):
            torch.matmul(Aop, Bop, out=out)
    g.replay()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    g.replay()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--batch", type=int, default=32)
    ap.add_argument("--top", type=int, default=70)
    ap.add_argument("--cublas", action="store_true")
    ap.add_argument("--json", default=None)
    args = ap.parse_args()
    tr = engine.Trainer.create(args.config, world=1, rank=0, S=1, M=1, D=1, world_batch=args.batch)
    tr.prefetch(6)
    for _ in range(3):
        tr.step()
    torch.cuda.synchronize()
    lib = _lib.lib()
    rec = Recorder(lib)
    _lib._lib = rec
    rec.on = True
    tr.step()
    torch.cuda.synchronize()
    rec.on = False
    _lib._lib = lib
    calls = rec.calls
    agg = defaultdict(lambda: [0.0, 0, 0.0])
    per_sig = {}
    for name, saved in calls:
        sig, fl = signature(name, saved)
        if sig not in per_sig:
            per_sig[sig] = time_call(name, saved)
        a = agg[sig]
        a[0] += per_sig[sig]
        a[1] += 1
        a[2] += fl
    times = [v[0] for v in agg.values()]
    total = float("nan")
    ssum = sum(times)
    print(f"{len(calls)} recorded libdpipe calls, {len(per_sig)} signatures; sum of isolated per-call device "
          f"times {ssum:.2f} ms")
    fam = defaultdict(lambda: [0.0, 0, 0.0])
    for sig, (t, n, fl) in agg.items():
        f = fam[sig.split(" ")[0]]
        f[0] += t
        f[1] += n
        f[2] += fl
    print("-- by kernel family")
    for k, (t, n, fl) in sorted(fam.items(), key=lambda kv: -kv[1][0]):
        tf = f"{fl / t / 1e9:7.1f} TF/s" if fl else ""
        print(f"{t:8.3f} ms {n:5d}x {tf}  {k}")
    print("-- by signature")
    rows = []
    for sig, (t, n, fl) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:args.top]:
        tf = fl / t / 1e9 if fl else 0.0
        extra = ""
        row = dict(sig=sig, ms=t, launches=n, us_each=1e3 * t / n, tflops=tf)
        if args.cublas and sig.startswith("gemm ") and sig.endswith("x1"):
            import re
            mm = re.match(r"gemm (\d+)x(\d+)x(\d+)(a?)(b?)", sig)
            M, N, K = int(mm.group(1)), int(mm.group(2)), int(mm.group(3))
            a_mn, b_mn = bool(mm.group(4)), bool(mm.group(5))
            cb = cublas_time(M, N, K, a_mn, b_mn)
            row["cublas_us"] = 1e3 * cb
            extra = f"  cuBLAS {1e3 * cb:7.1f} us ({row['us_each'] / (1e3 * cb):4.2f}x)"
        rows.append(row)
        print(f"{t:8.3f} ms {n:4d}x {1e3 * t / n:8.1f} us {tf:7.1f} TF/s  {sig}{extra}")
    if args.json:
        with open(args.json, "w") as f:
            json.dump(dict(total_ms=total, sum_ms=ssum, rows=rows,
                           families={k: dict(ms=v[0], launches=v[1], flops=v[2]) for k, v in fam.items()}), f)


if __name__ == "__main__":
    main()
