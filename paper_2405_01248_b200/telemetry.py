"""Launch accounting and live per-kernel timing for bench.py.

* every libdpipe entry point reports through `_lib.check`, which counts the kernels it
  launched (`launches`) — the bench's `gpu_launches` claim;
* when `timer.active`, every libdpipe call is bracketed by CUDA events on the launching
  stream (`_lib.lib()` hands out a timing proxy) and recorded under a family name: the
  tensor-core GEMM/conv wrappers record their algorithmic FLOPs under "tcgen05_gemm[.site]"
  (site = attn / conv_fwd / conv_dgrad / conv_wgrad / linear), every other entry point under
  its own name. bench.py turns this into the per-family breakdown and the roofline line.
"""

from __future__ import annotations

import contextlib
import threading
from collections import Counter

import torch

launches = Counter()
SHAPES = False  # label GEMM launches by shape (tools/step_breakdown.py)
_site = threading.local()


class _Timer:
    def __init__(self):
        self.active = False
        self.records = []
        self.depth = 0
        self.pool = []  # pre-created timing events (event creation kept off the timed path)

    def event(self):
        return self.pool.pop() if self.pool else torch.cuda.Event(enable_timing=True)

    def start(self, reserve=0):
        self.records = []
        if len(self.pool) < reserve:
            self.pool.extend(torch.cuda.Event(enable_timing=True) for _ in range(reserve - len(self.pool)))
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
            self.pool.extend((a, b))
        self.records = []
        return out


timer = _Timer()


@contextlib.contextmanager
def site(name):
    """Label the GEMM launches issued inside the block (e.g. 'attn')."""
    prev = getattr(_site, "name", None)
    _site.name = name
    try:
        yield
    finally:
        _site.name = prev


def timed(family, flops, fn, sub=None):
    if not timer.active:
        return fn()
    s = getattr(_site, "name", None) or sub
    fam = f"{family}.{s}" if s else family
    a = timer.event()
    b = timer.event()
    a.record()
    timer.depth += 1
    try:
        r = fn()
    finally:
        timer.depth -= 1
    b.record()
    timer.records.append((fam, flops, a, b))
    return r


class TimedLib:
    """Proxy over the ctypes library: times every entry point not already inside `timed`."""

    def __init__(self, lib):
        self._lib = lib

    def __getattr__(self, name):
        f = getattr(self._lib, name)
        if not callable(f) or timer.depth > 0 or name in ("dp_last_error", "dp_version",
                                                         "dp_group_norm_workspace", "dp_gemm_workspace",
                                                         "dp_conv_fwd_workspace", "dp_conv_dgrad_workspace",
                                                         "dp_flash_attn_bwd_workspace"):
            return f

        def call(*args):
            return timed(name, 0.0, lambda: f(*args))
        return call


def count(what, n=1):
    launches[what] += n


def total_launches():
    return sum(launches.values())


def reset():
    launches.clear()
