"""Per-signature device time of the tensor-core contractions of one training step, on FRESH buffers.

Records every dp_gemm / dp_conv_{fwd,dgrad,wgrad} call of one steady-state step (argument structs copied),
then for each distinct signature allocates new operands sized from the struct (so nothing depends on the
step's freed memory), times `reps` back-to-back calls in a CUDA graph and weights by the signature's count.
Prints the signatures sorted by their gap to the measured bf16 peak (where the step's GEMM time goes).

  python tools/sig_replay.py [--config c2] [--top 40] [--json out.json]
"""
import argparse
import ctypes
import json
import os
import sys
from collections import OrderedDict

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2405_01248_b200 import _lib, engine  # noqa: E402

NAMES = ("dp_gemm", "dp_conv_fwd", "dp_conv_dgrad", "dp_conv_wgrad")
PEAK = 1401.7


class Recorder:
    def __init__(self, lib):
        self._lib = lib
        self.calls = []

    def __getattr__(self, name):
        f = getattr(self._lib, name)
        if name not in NAMES:
            return f

        def call(ptr, stream):
            obj = ptr._obj
            self.calls.append((name, type(obj).from_buffer_copy(obj)))
            return f(ptr, stream)
        return call


def sig_of(name, s):
    if name == "dp_gemm":
        b = max(1, s.batch1) * max(1, s.batch2)
        key = (name, s.M, s.N, s.K, s.batch1, s.batch2, s.a_mn_major, s.b_mn_major, s.out_mode, s.d_dtype,
               bool(s.bias), bool(s.Res), s.dtype, s.a_ld, s.b_ld, s.d_ld, s.a_bs1, s.a_bs2, s.b_bs1, s.b_bs2,
               s.d_bs1, s.d_bs2)
        label = (f"gemm {s.M}x{s.N}x{s.K}{' aMN' if s.a_mn_major else ''}{' bMN' if s.b_mn_major else ''}"
                 f"{' +acc' if s.out_mode else ''}{' +res' if s.Res else ''}{' x' + str(b) if b > 1 else ''}")
        return key, label, 2.0 * s.M * s.N * s.K * b
    fl = {"dp_conv_fwd": 2.0 * s.N * s.P * s.Q * s.K * s.R * s.S * s.C,
          "dp_conv_dgrad": 2.0 * s.N * s.H * s.W * s.C * s.R * s.S * s.K,
          "dp_conv_wgrad": 2.0 * s.N * s.P * s.Q * s.K * s.R * s.S * s.C}[name]
    key = (name, s.N, s.H, s.W, s.C, s.K, s.R, s.S, s.stride, s.pad_h, s.pad_w, s.P, s.Q, bool(s.bias), bool(s.Res),
           s.out_mode, s.dtype)
    label = f"{name[3:]} {s.N}x{s.H}x{s.W}x{s.C}->{s.K} r{s.R} s{s.stride} pq{s.P}x{s.Q}{' +res' if s.Res else ''}"
    return key, label, fl


def _buf(nbytes, keep):
    t = torch.empty(max(16, int(nbytes)) // 2 + 64, device="cuda", dtype=torch.bfloat16).normal_()
    keep.append(t)
    return t.data_ptr()


def fresh(name, s, keep):
    """A copy of the struct pointing at new buffers of sufficient size."""
    c = type(s).from_buffer_copy(s)
    esz = 2
    if name == "dp_gemm":
        b1, b2 = max(1, s.batch1), max(1, s.batch2)
        rows_a = s.K if s.a_mn_major else s.M
        rows_b = s.K if s.b_mn_major else s.N
        span = lambda ld, rows, bs1, bs2: (ld * rows + bs1 * (b1 - 1) + bs2 * (b2 - 1) + 64) * esz  # noqa: E731
        c.A = _buf(span(s.a_ld, rows_a, s.a_bs1, s.a_bs2), keep)
        c.B = _buf(span(s.b_ld, rows_b, s.b_bs1, s.b_bs2), keep)
        dsz = 4 if s.d_dtype == _lib.DP_F32 else 2
        c.D = _buf(span(s.d_ld, s.M, s.d_bs1, s.d_bs2) * dsz // 2, keep)
        if s.bias:
            c.bias = _buf(s.N * 4 + 64, keep)
        if s.Res:
            c.Res = _buf(span(s.r_ld, s.M, s.r_bs1, s.r_bs2), keep)
        if s.workspace:
            c.workspace = _buf(s.workspace_bytes, keep)
        return c
    xs = (s.N * s.H * s.W * s.C) * esz
    ws = (s.K * s.R * s.S * s.C) * 4
    ys = (s.N * s.P * s.Q * s.K) * 4
    big = max(xs, ws, ys) + 4096
    c.x, c.w, c.y = _buf(big, keep), _buf(big, keep), _buf(big, keep)
    if s.bias:
        c.bias = _buf(s.K * 4 + 64, keep)
    if s.Res:
        c.Res = _buf(big, keep)
    if s.workspace:
        c.workspace = _buf(s.workspace_bytes, keep)
    return c


def time_sig(lib, name, s, reps=10):
    keep = []
    c = fresh(name, s, keep)
    fn = getattr(lib, name)
    stream = torch.cuda.Stream()
    with torch.cuda.stream(stream):
        for _ in range(2):
            if fn(ctypes.byref(c), stream.cuda_stream):
                raise RuntimeError(f"{name}: {lib.dp_last_error().decode()}")
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        for _ in range(reps):
            fn(ctypes.byref(c), stream.cuda_stream)
    g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    g.replay()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--top", type=int, default=40)
    ap.add_argument("--json", default=None)
    args = ap.parse_args()
    tr = engine.Trainer.create(args.config, world=1, rank=0, S=1, M=1, D=1, world_batch=32)
    tr.prefetch(6)
    for _ in range(3):
        tr.step()
    torch.cuda.synchronize()
    lib = _lib.lib()
    rec = Recorder(lib)
    _lib._lib = rec
    tr.step()
    torch.cuda.synchronize()
    _lib._lib = lib
    agg = OrderedDict()
    for name, s in rec.calls:
        key, label, fl = sig_of(name, s)
        if key not in agg:
            agg[key] = dict(name=name, s=s, label=label, flops=fl, n=0)
        agg[key]["n"] += 1
    rows = []
    for key, v in agg.items():
        ms = time_sig(lib, v["name"], v["s"])
        ideal = v["flops"] / (PEAK * 1e9)
        rows.append(dict(label=v["label"], n=v["n"], us=ms * 1e3, tflops=v["flops"] / ms / 1e9,
                         total_ms=ms * v["n"], gap_ms=(ms - ideal) * v["n"]))
    tot = sum(r["total_ms"] for r in rows)
    gap = sum(r["gap_ms"] for r in rows)
    fl = sum(v["flops"] * v["n"] for v in agg.values())
    print(f"{len(rec.calls)} contractions, {len(rows)} signatures: {tot:.2f} ms (graph-timed, warm), "
          f"{fl / tot / 1e9:.0f} TF/s; gap to {PEAK} TF/s: {gap:.2f} ms")
    for r in sorted(rows, key=lambda r: -r["gap_ms"])[:args.top]:
        print(f"{r['gap_ms']:7.3f} ms gap {r['total_ms']:7.3f} ms {r['n']:3d}x {r['us']:8.1f} us {r['tflops']:7.1f} TF/s  {r['label']}")
    if args.json:
        with open(args.json, "w") as f:
            json.dump(dict(total_ms=tot, gap_ms=gap, rows=rows), f)


if __name__ == "__main__":
    main()
