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


_raw_stream = getattr(torch._C, "_cuda_getCurrentRawStream", None)
_cur_device = getattr(torch._C, "_cuda_getDevice", None)


def _stream_ptr():
    if _raw_stream is not None and _cur_device is not None:
        return _raw_stream(_cur_device())
    return torch.cuda.current_stream().cuda_stream


class _Timer:
    """Event pairs from libdpipe's native pool (dp_timing_record: one C call per record on the
    launching stream; the torch Event path cost enough host time per record to make the bracketed
    pass host-bound, so brackets measured launch latency rather than kernels)."""

    def __init__(self):
        self.active = False
        self.records = []
        self.depth = 0
        self.next = 0
        self.capacity = 0

    @staticmethod
    def _lib():
        from . import _lib

        return _lib.lib()  # the raw handle: called while the timer is still inactive

    def event(self):
        i = self.next
        if i >= self.capacity:  # grow the native pool (event creation is host-side only)
            cap = max(2 * self.capacity, 1024)
            if self.native.dp_timing_events(cap) != 0:
                raise RuntimeError("dp_timing_events failed")
            self.capacity = cap
        self.next += 1
        return i

    def record(self, i):
        self.native.dp_timing_record(i, _stream_ptr())

    def start(self, reserve=0):
        self.records = []
        self.active = False
        self.native = self._lib()
        if reserve > self.capacity:
            if self.native.dp_timing_events(reserve) != 0:
                raise RuntimeError("dp_timing_events failed")
            self.capacity = reserve
        self.next = 0
        self.active = True

    def stop(self):
        self.active = False
        torch.cuda.synchronize()
        out = {}
        for fam, flops, a, b in self.records:
            ms = self.native.dp_timing_elapsed(a, b)
            f = out.setdefault(fam, dict(launches=0, flops=0.0, ms=0.0))
            f["launches"] += 1
            f["flops"] += flops
            f["ms"] += ms
        self.records = []
        self.next = 0
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
    timer.record(a)
    timer.depth += 1
    try:
        r = fn()
    finally:
        timer.depth -= 1
    timer.record(b)
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
