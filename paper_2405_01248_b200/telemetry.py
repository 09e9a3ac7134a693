"""Launch accounting and live per-kernel timing for bench.py.

* every libdpipe entry point reports through `_lib.check`, which counts the kernels it
  launched (`launches`) — the bench's `gpu_launches` claim;
* when `timer.active`, the GEMM/conv wrappers bracket their launch with CUDA events on the
  launching stream and record (family, algorithmic FLOPs) so bench.py can compute the
  dominant kernel's achieved TFLOP/s over the timed region.
"""

from __future__ import annotations

from collections import Counter

import torch

launches = Counter()


class _Timer:
    def __init__(self):
        self.active = False
        self.records = []

    def start(self):
        self.records = []
        self.active = True

    def stop(self):
        self.active = False
        torch.cuda.synchronize()
        out = {}
        for fam, flops, a, b in self.records:
            ms = a.elapsed_time(b)
            f = out.setdefault(fam, dict(launches=0, flops=0.0, ms=0.0))
            f["launches"] += 1
            f["flops"] += flops
            f["ms"] += ms
        self.records = []
        return out


timer = _Timer()


def timed(family, flops, fn):
    if not timer.active:
        return fn()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    r = fn()
    b.record()
    timer.records.append((family, flops, a, b))
    return r


def count(what, n=1):
    launches[what] += n


def total_launches():
    return sum(launches.values())


def reset():
    launches.clear()
