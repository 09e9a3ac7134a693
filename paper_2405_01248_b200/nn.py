"""Layer library of the executor: flat parameter stores and autograd Functions
whose forward/backward run only libdpipe kernels (ops.py).

Design (B200-first, not a port):
* Every trainable stage owns ONE flat fp32 master buffer, one flat fp32 grad
  buffer and the AdamW moments; the compute copy (bf16 for the SD configs,
  the master itself for fp32) is a second flat buffer. Weight gradients are
  accumulated by the wgrad GEMM epilogue straight into the fp32 grad views,
  so gradient allreduce and AdamW are single flat launches per stage.
* Weights are therefore not torch leaves; each Function receives its layer
  and writes `param.g` itself. A per-stage "grad anchor" (a 1-element tensor
  with requires_grad) is threaded into every parameterised Function so that
  torch's autograd engine records branches whose activations carry no grad
  (time embedding from t, cross-attention K/V from the frozen context).
* Activations: NHWC for convolutions, [B, L, C] rows for transformers (the
  NHWC tensor viewed as [B, H*W, C] — no permutes on the hot path).

Reference semantics: the paper trains diffusion backbones with frozen
encoders; layer shapes follow SD v2.1 / DiT.
"""

from __future__ import annotations

import math
import os
import threading
import zlib

import torch

from . import ops, telemetry
from ._lib import DP_ACT_GELU, DP_ACT_GELU_TANH, DP_ACT_SILU

_ALIGN = 64  # elements; keeps every view 128-byte aligned for TMA
FLASH_ATTENTION = True  # bf16 head-dim-64 attention through the fused tcgen05 kernels


# ============================================================================ parameters

class Param:
    __slots__ = ("name", "shape", "fp32", "init", "offset", "numel", "w", "g", "master", "wt", "wt_fn",
                 "flip_args")

    def __init__(self, name, shape, fp32, init):
        self.name = name
        self.shape = tuple(shape)
        self.fp32 = fp32
        self.init = init
        self.numel = math.prod(self.shape)
        self.offset = None
        self.w = None       # compute view (bf16 weights, or fp32)
        self.g = None       # fp32 grad view (None when frozen)
        self.master = None  # fp32 master view
        self.wt = None      # cached flip-transposed bf16 copy for dgrad (ops.cached_flip)
        self.wt_fn = None   # recomputes wt in place from w
        self.flip_args = None  # (w, wt, K, R, S, C) when wt is a plain flip of w (batched refresh)


# flip-transposed weight copies for dgrad are cached and refreshed right after each AdamW update
# of their parameter (on the optimizer's stream, off the backward's critical path); DP_FLIP_CACHE=0
# flips inside every dgrad instead (the A/B reference)
FLIP_CACHE = os.environ.get("DP_FLIP_CACHE", "1") != "0"


class ParamStore:
    """Flat parameter storage for one stage (trainable) or one frozen component."""

    def __init__(self, dtype=torch.float32, trainable=True):
        self.dtype = dtype
        self.trainable = trainable
        self.params: dict[str, Param] = {}
        self.master = self.grad = self.compute = self.exp_avg = self.exp_avg_sq = None
        self.step = 0
        self.flip_params = []  # params holding a cached wt, refreshed after their AdamW update

    def register_flip(self, p):
        self.flip_params.append(p)

    def refresh_flips(self, lo, hi):
        """Recompute the cached dgrad weight copies of the params inside the flat range [lo, hi)
        (call right after updating it, on the same stream)."""
        jobs = []
        for p in self.flip_params:
            if lo <= p.offset < hi:
                if p.flip_args is not None and FLIP_BATCH:
                    jobs.append(p.flip_args)
                else:
                    p.wt_fn(p.wt)
        ops.flip_batch(jobs)

    def add(self, name, shape, fp32=False, init="w"):
        if name in self.params:
            raise KeyError(f"duplicate parameter {name}")
        p = Param(name, shape, fp32 or self.dtype == torch.float32, init)
        self.params[name] = p
        return p

    def numel(self):
        return sum(p.numel for p in self.params.values())

    def materialize(self, device, seed=0, state=None, order_key=None):
        """Allocate the flat buffers and fill them: from `state` (name -> fp32 tensor) when
        given, else from the deterministic initialiser (same values the CPU oracle uses).
        `order_key(param)` orders the flat layout (stable), e.g. by owning layer."""
        off = 0
        plist = list(self.params.values())
        if order_key is not None:
            plist = sorted(plist, key=order_key)
        for p in plist:
            p.offset = off
            off += -(-p.numel // _ALIGN) * _ALIGN
        total = max(off, _ALIGN)
        for p in plist:
            p.wt = p.wt_fn = None
        self.flip_params = []
        self.master = torch.zeros(total, device=device, dtype=torch.float32)
        if self.dtype != torch.float32:
            self.compute = torch.zeros(total, device=device, dtype=self.dtype)
        else:
            self.compute = self.master
        if self.trainable:
            self.grad = torch.zeros(total, device=device, dtype=torch.float32)
            self.exp_avg = torch.zeros(total, device=device, dtype=torch.float32)
            self.exp_avg_sq = torch.zeros(total, device=device, dtype=torch.float32)
        init = state if state is not None else init_state(self.param_specs(), seed)
        for p in self.params.values():
            sl = slice(p.offset, p.offset + p.numel)
            p.master = self.master[sl].view(p.shape)
            p.master.copy_(init[p.name].reshape(p.shape))
            p.w = p.master if p.fp32 else self.compute[sl].view(p.shape)
            p.g = self.grad[sl].view(p.shape) if self.trainable else None
        if self.compute is not self.master:
            ops.cast(self.master, self.dtype, out=self.compute)
        return self

    def param_specs(self):
        return [(p.name, p.shape, p.init) for p in self.params.values()]

    def state_dict(self):
        return {p.name: p.master.detach().float().cpu().clone() for p in self.params.values()}

    def grads(self):
        return {p.name: p.g.detach().float().cpu().clone() for p in self.params.values()}

    def zero_grad(self, rng=None):
        if self.grad is not None:
            lo, hi = rng if rng is not None else (0, self.grad.numel())
            self.grad[lo:hi].zero_()

    def adamw_begin(self, betas=(0.9, 0.999), **_):
        """Chunked AdamW, part 1: advance the step counter (host and device) once per iteration."""
        self.step += 1
        if getattr(self, "step_dev", None) is None:
            self.step_dev = torch.zeros(1, device=self.master.device, dtype=torch.int32)
            self.bc_dev = torch.zeros(2, device=self.master.device, dtype=torch.float32)
        ops.adamw_advance(self.step_dev, self.bc_dev, betas[0], betas[1])

    def adamw_apply(self, rng, lr=1e-4, betas=(0.9, 0.999), eps=1e-8, weight_decay=0.01, grad_scale=1.0,
                    max_ctas=0, zero_grad=False):
        """(zero_grad: the kernel clears the gradient slice after reading it — no separate fill.)"""
        """Chunked AdamW, part 2: update the flat slice `rng` with this iteration's corrections."""
        lo, hi = rng
        if hi <= lo:
            return
        ops.adamw_apply(self.master[lo:hi], self.grad[lo:hi], self.exp_avg[lo:hi], self.exp_avg_sq[lo:hi],
                        None if self.compute is self.master else self.compute[lo:hi],
                        lr, betas[0], betas[1], eps, weight_decay, self.bc_dev, grad_scale, max_ctas,
                        zero_grad)
        self.refresh_flips(lo, hi)

    def adamw_step(self, lr=1e-4, betas=(0.9, 0.999), eps=1e-8, weight_decay=0.01, grad_scale=1.0,
                   rng=None):
        """One AdamW step over the flat slice `rng` (default: everything). The step counter and
        the bias corrections live on the device so the update is CUDA-graph replayable."""
        self.step += 1
        lo, hi = rng if rng is not None else (0, self.master.numel())
        if hi <= lo:
            return
        if self.master.is_cuda:
            if getattr(self, "step_dev", None) is None:
                self.step_dev = torch.zeros(1, device=self.master.device, dtype=torch.int32)
                self.bc_dev = torch.zeros(2, device=self.master.device, dtype=torch.float32)
            ops.adamw_dev(self.master[lo:hi], self.grad[lo:hi], self.exp_avg[lo:hi], self.exp_avg_sq[lo:hi],
                          None if self.compute is self.master else self.compute[lo:hi],
                          lr, betas[0], betas[1], eps, weight_decay, self.step_dev, self.bc_dev, grad_scale)
            self.refresh_flips(lo, hi)
            return
        ops.adamw(self.master[lo:hi], self.grad[lo:hi], self.exp_avg[lo:hi], self.exp_avg_sq[lo:hi],
                  None if self.compute is self.master else self.compute[lo:hi],
                  lr, betas[0], betas[1], eps, weight_decay, self.step, grad_scale)


def _name_seed(name: str, seed: int) -> int:
    return (zlib.crc32(name.encode()) * 1000003 + seed) & 0x7FFFFFFF


def init_state(specs, seed=0):
    """Deterministic CPU initialiser shared by the executor and the CPU oracle.

    w: N(0, 1/fan_in); b: 0.02 N(0,1); g (norm scale): 1 + 0.02 N(0,1); e (embedding): 0.02 N(0,1).
    Zero-initialised layers of the original recipes (adaLN-Zero, zero convs) get the small
    random init too so that their gradients are non-trivial in parity tests.
    """
    out = {}
    for name, shape, kind in specs:
        g = torch.Generator().manual_seed(_name_seed(name, seed))
        t = torch.randn(*shape, generator=g, dtype=torch.float32)
        if kind == "w":
            fan_in = math.prod(shape[1:]) if len(shape) > 1 else shape[0]
            t = t / math.sqrt(fan_in)
        elif kind == "b":
            t = t * 0.02
        elif kind == "g":
            t = 1.0 + 0.02 * t
        elif kind == "e":
            t = t * 0.02
        elif kind == "z":
            t = t * 1e-3
        out[name] = t
    return out


# ============================================================================ grad anchor

_tls = threading.local()


def current_anchor():
    return getattr(_tls, "anchor", None)


class grad_anchor:
    """Context manager installing the per-stage grad anchor (see module doc)."""

    def __init__(self, enabled=True, device="cuda"):
        self.enabled = enabled
        self.device = device

    def __enter__(self):
        self.prev = current_anchor()
        _tls.anchor = (torch.zeros(1, device=self.device, requires_grad=True)
                       if self.enabled else None)
        return _tls.anchor

    def __exit__(self, *exc):
        _tls.anchor = self.prev
        return False


def _c(t):
    return t if t.is_contiguous() else t.contiguous()


# ============================================================================ Functions

def _flip_cache(layer):
    """(store, weight param) when the layer's dgrad may reuse a cached flip-transposed weight: a
    trainable store refreshes it after each AdamW update, a frozen one never changes it."""
    return (layer.store, layer.weight) if FLIP_CACHE else None


class _LinearFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, anchor, residual, layer):
        K = x.shape[-1]
        x2 = _c(x).view(-1, K)
        W = layer.weight
        N = W.shape[0]
        out = torch.empty(*x.shape[:-1], N, device=x.device, dtype=x.dtype)
        ops.linear(x2, W.w, bias=None if layer.bias is None else layer.bias.w,
                   residual=None if residual is None else _c(residual).view(-1, N),
                   out=out.view(-1, N))
        ctx.save_for_backward(x2)
        ctx.layer = layer
        ctx.has_res = residual is not None
        return out

    @staticmethod
    def backward(ctx, dy):
        (x2,) = ctx.saved_tensors
        layer = ctx.layer
        W = layer.weight
        N = W.shape[0]
        dy2 = _c(dy).view(-1, N)
        dx = None
        if ctx.needs_input_grad[0]:
            dx = ops.linear_dgrad(dy2, W.w, cache=_flip_cache(layer)).view(*dy.shape[:-1], W.shape[1])
        if W.g is not None:
            ops.linear_wgrad(dy2, x2, W.g)
        if layer.bias is not None and layer.bias.g is not None and not layer.bias_grad_by_row:
            ops.bias_grad(dy2, layer.bias.g)
        return dx, None, (dy if ctx.has_res else None), None


# bf16 transformer FF: the ff1 GEMM writes both its pre-activation h (kept for the backward) and
# GEGLU(h) from one epilogue (no separate GEGLU pass re-reading h); DP_FUSED_GEGLU=0: unfused
FUSED_GEGLU = os.environ.get("DP_FUSED_GEGLU", "1") != "0"
# the ff2 input gradient applying the GEGLU backward in its epilogue (DP_FUSED_GEGLU_BWD=1) measured slower
# than the dgrad GEMM + the vectorised GEGLU-backward kernel (140 vs 125 us at 32768x320: the epilogue's
# per-row reads of h), so it is off by default
FUSED_GEGLU_BWD = os.environ.get("DP_FUSED_GEGLU_BWD", "0") != "0"
# ff1's bias gradient accumulated by the GEGLU-backward pass (DP_GEGLU_BIAS_DB=0: separate pass, A/B)
GEGLU_BIAS_DB = os.environ.get("DP_GEGLU_BIAS_DB", "1") != "0"
# cached dgrad weight copies refreshed by one batched launch per optimizer slice (DP_FLIP_BATCH=0: per param)
FLIP_BATCH = os.environ.get("DP_FLIP_BATCH", "1") != "0"


class _LinearGegluFn(torch.autograd.Function):
    """y = GEGLU(x @ W^T + b): forward in one GEMM, backward = GEGLU backward then the linear's."""

    @staticmethod
    def forward(ctx, x, anchor, layer):
        K = x.shape[-1]
        x2 = _c(x).view(-1, K)
        W = layer.weight
        h, y = ops.linear_geglu(x2, W.w, layer.bias.w)
        ctx.save_for_backward(x2, h)
        ctx.layer = layer
        return y.view(*x.shape[:-1], W.shape[0] // 2)

    @staticmethod
    def backward(ctx, dy):
        x2, h = ctx.saved_tensors
        layer = ctx.layer
        W = layer.weight
        db = layer.bias.g if (layer.bias is not None and GEGLU_BIAS_DB) else None
        dh = ops.geglu_bwd(h, _c(dy).view(h.shape[0], -1), db=db)
        dx = None
        if ctx.needs_input_grad[0]:
            dx = ops.linear_dgrad(dh, W.w, cache=_flip_cache(layer)).view(*dy.shape[:-1], W.shape[1])
        if W.g is not None:
            ops.linear_wgrad(dh, x2, W.g)
        if layer.bias is not None and layer.bias.g is not None and db is None:
            ops.bias_grad(dh, layer.bias.g)
        return dx, None, None


class _FeedForwardGegluFn(torch.autograd.Function):
    """out = ff2(GEGLU(ff1(x))) + residual, three GEMMs and no elementwise pass: ff1's epilogue writes
    the pre-activation h and GEGLU(h); in the backward ff2's input-gradient GEMM applies the GEGLU
    backward in its epilogue (reading h) and hands dh straight to ff1's backward."""

    @staticmethod
    def forward(ctx, x, anchor, residual, ff1, ff2):
        K = x.shape[-1]
        x2 = _c(x).view(-1, K)
        h, y = ops.linear_geglu(x2, ff1.weight.w, ff1.bias.w)
        N2 = ff2.weight.shape[0]
        out = torch.empty(*x.shape[:-1], N2, device=x.device, dtype=x.dtype)
        ops.linear(y, ff2.weight.w, bias=ff2.bias.w,
                   residual=None if residual is None else _c(residual).view(-1, N2), out=out.view(-1, N2))
        ctx.save_for_backward(x2, h, y)
        ctx.layers = (ff1, ff2)
        ctx.has_res = residual is not None
        return out

    @staticmethod
    def backward(ctx, dout):
        x2, h, y = ctx.saved_tensors
        ff1, ff2 = ctx.layers
        N2 = ff2.weight.shape[0]
        d2 = _c(dout).view(-1, N2)
        if ff2.weight.g is not None:
            ops.linear_wgrad(d2, y, ff2.weight.g)
        if ff2.bias.g is not None:
            ops.bias_grad(d2, ff2.bias.g)
        db1 = None
        if FUSED_GEGLU_BWD:
            dh = ops.linear_dgrad_geglu(d2, ff2.weight.w, h, cache=_flip_cache(ff2))
        else:
            # ff1's bias gradient in the GEGLU-backward pass (no separate re-read of dh)
            db1 = ff1.bias.g if GEGLU_BIAS_DB else None
            dh = ops.geglu_bwd(h, ops.linear_dgrad(d2, ff2.weight.w, cache=_flip_cache(ff2)), db=db1)
        dx = None
        if ctx.needs_input_grad[0]:
            dx = ops.linear_dgrad(dh, ff1.weight.w, cache=_flip_cache(ff1)).view(*dout.shape[:-1], x2.shape[1])
        if ff1.weight.g is not None:
            ops.linear_wgrad(dh, x2, ff1.weight.g)
        if ff1.bias.g is not None and db1 is None:
            ops.bias_grad(dh, ff1.bias.g)
        return dx, None, (dout if ctx.has_res else None), None, None


def feed_forward_geglu(x, ff1, ff2, residual=None):
    """ff2(GEGLU(ff1(x))) (+ residual): the fused three-GEMM path for bf16 (see _FeedForwardGegluFn),
    the layer-by-layer composition otherwise."""
    F = ff1.weight.shape[0] // 2
    rows = x.numel() // x.shape[-1]
    if (FUSED_GEGLU and x.dtype == torch.bfloat16 and x.is_cuda and ff1.bias is not None and ff2.bias is not None
            and F % 64 == 0 and x.shape[-1] % 8 == 0 and rows >= 1024 and ff2.weight.shape[1] == F):
        return _FeedForwardGegluFn.apply(x, _anchor(), residual, ff1, ff2)
    return ff2(geglu(ff1(x)), residual=residual)


# frozen (no-grad) bf16 MLPs: GELU in the fc1 GEMM epilogue (DP_GELU_EPI=0: separate activation pass)
GELU_EPI = os.environ.get("DP_GELU_EPI", "1") != "0"


def linear_gelu(x, layer):
    """gelu_erf(layer(x)): one GEMM with the activation in its epilogue when no gradient is recorded
    (frozen encoders), the linear + activation pair otherwise."""
    N = layer.weight.shape[0]
    if (GELU_EPI and not torch.is_grad_enabled() and x.dtype == torch.bfloat16 and x.is_cuda
            and layer.bias is not None and N % 128 == 0 and x.shape[-1] % 8 == 0):
        K = x.shape[-1]
        y = ops.linear_gelu(_c(x).view(-1, K), layer.weight.w, layer.bias.w)
        return y.view(*x.shape[:-1], N)
    return gelu(layer(x))


def linear_geglu(x, layer):
    """GEGLU(layer(x)) for an nn.Linear with bias and an even output width."""
    F = layer.weight.shape[0] // 2
    if (FUSED_GEGLU and x.dtype == torch.bfloat16 and x.is_cuda and layer.bias is not None
            and F % 64 == 0 and x.shape[-1] % 8 == 0 and x.numel() // x.shape[-1] >= 128):
        return _LinearGegluFn.apply(x, _anchor(), layer)
    return geglu(layer(x))


# convs whose output feeds a GroupNorm can accumulate its statistics in the GEMM epilogue (Conv2d.gn_stats =
# G) so that the GroupNorm reads its input once. Measured on c2 (VAE convs): 627 vs 632-635 samples/s with
# and without -- the epilogue's per-chunk reductions and atomics cost more than the statistics pass they
# replace (that pass already runs near HBM bandwidth on the large maps), so it is off by default
# (DP_GN_STATS=1: on)
GN_STATS = os.environ.get("DP_GN_STATS", "0") != "0"


def _lib_gn_slots():
    return 16  # DP_GN_SLOTS (include/dpipe.h)


def _gn_sums_of(x, G):
    s = getattr(x, "_dp_gn", None)
    return s[0] if (s is not None and s[1] == G) else None


class _ConvFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, anchor, residual, layer):
        x = _c(x)
        hw = layer.out_hw(x)
        G = layer.gn_stats
        sums = None
        if (GN_STATS and G and x.dtype == torch.bfloat16 and x.is_cuda and (hw[0] * hw[1]) % 32 == 0
                and layer.weight.shape[0] % (4 * G) == 0 and x.shape[-1] % 64 == 0):
            sums = torch.empty(_lib_gn_slots(), x.shape[0], G, 2, device=x.device, dtype=torch.float32)
        y = ops.conv2d(x, layer.weight.w, stride=layer.stride, pad=layer.pad, out_hw=hw,
                       bias=None if layer.bias is None else layer.bias.w,
                       residual=None if residual is None else _c(residual), gn_sums=sums, gn_groups=G)
        if sums is not None:
            y._dp_gn = (sums, G)
        ctx.save_for_backward(x)
        ctx.layer = layer
        ctx.has_res = residual is not None
        return y

    @staticmethod
    def backward(ctx, dy):
        (x,) = ctx.saved_tensors
        layer = ctx.layer
        dy = _c(dy)
        dx = None
        if ctx.needs_input_grad[0]:
            dx = ops.conv2d_dgrad(dy, layer.weight.w, x.shape, stride=layer.stride, pad=layer.pad,
                                  cache=_flip_cache(layer))
        if layer.weight.g is not None:
            ops.conv2d_wgrad(dy, x, layer.weight.g, stride=layer.stride, pad=layer.pad)
        if layer.bias is not None and layer.bias.g is not None and not layer.bias_grad_by_row:
            ops.bias_grad(dy, layer.bias.g)
        return dx, None, (dy if ctx.has_res else None), None


class _GroupNormFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, anchor, layer):
        x = _c(x)
        y, mean, rstd = ops.group_norm(x, layer.gamma.w, layer.beta.w, layer.groups, layer.eps, layer.silu,
                                       sums=_gn_sums_of(x, layer.groups))
        ctx.save_for_backward(x, mean, rstd)
        ctx.layer = layer
        return y

    @staticmethod
    def backward(ctx, dy):
        x, mean, rstd = ctx.saved_tensors
        L = ctx.layer
        dx = ops.group_norm_bwd(x, _c(dy), L.gamma.w, L.beta.w, mean, rstd, L.groups, L.silu,
                                dgamma=L.gamma.g, dbeta=L.beta.g)
        return dx, None, None


class _LayerNormFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, anchor, layer):
        x = _c(x)
        g = None if layer.gamma is None else layer.gamma.w
        b = None if layer.beta is None else layer.beta.w
        y, mean, rstd = ops.layer_norm(x, g, b, layer.eps)
        ctx.save_for_backward(x, mean, rstd)
        ctx.layer = layer
        return y

    @staticmethod
    def backward(ctx, dy):
        x, mean, rstd = ctx.saved_tensors
        L = ctx.layer
        dx = ops.layer_norm_bwd(x, _c(dy), None if L.gamma is None else L.gamma.w, mean, rstd,
                                dgamma=None if L.gamma is None else L.gamma.g,
                                dbeta=None if L.beta is None else L.beta.g)
        return dx, None, None


def _identity_grad(g):
    """Gradient of a fork's identity output as a contiguous buffer the norm backward may add into
    (autograd hands the consumer's gradient over; every kernel that read it is already enqueued on
    this stream, so accumulating in place is ordered after them)."""
    return None if g is None else (g if g.is_contiguous() else g.contiguous())


class _GroupNormForkFn(torch.autograd.Function):
    """(GroupNorm(x), x) for an x with a second consumer (residual / skip): both gradients reach one
    backward and the GroupNorm backward kernel adds its dx into the identity branch's gradient
    instead of autograd summing the two with a separate elementwise kernel."""

    @staticmethod
    def forward(ctx, x, anchor, layer):
        ctx.set_materialize_grads(False)
        xc = _c(x)
        y, mean, rstd = ops.group_norm(xc, layer.gamma.w, layer.beta.w, layer.groups, layer.eps, layer.silu,
                                       sums=_gn_sums_of(xc, layer.groups))
        ctx.save_for_backward(xc, mean, rstd)
        ctx.layer = layer
        return y, x.view_as(x)

    @staticmethod
    def backward(ctx, dy, dres):
        x, mean, rstd = ctx.saved_tensors
        L = ctx.layer
        if dy is None:
            return dres, None, None
        dx = ops.group_norm_bwd(x, _c(dy), L.gamma.w, L.beta.w, mean, rstd, L.groups, L.silu,
                                dgamma=L.gamma.g, dbeta=L.beta.g, accumulate_into=_identity_grad(dres))
        return dx.view_as(x), None, None


class _LayerNormForkFn(torch.autograd.Function):
    """(LayerNorm(x), x): as _GroupNormForkFn for the transformer's pre-norm residual stream."""

    @staticmethod
    def forward(ctx, x, anchor, layer):
        ctx.set_materialize_grads(False)
        xc = _c(x)
        g = None if layer.gamma is None else layer.gamma.w
        b = None if layer.beta is None else layer.beta.w
        y, mean, rstd = ops.layer_norm(xc, g, b, layer.eps)
        ctx.save_for_backward(xc, mean, rstd)
        ctx.layer = layer
        return y, x.view_as(x)

    @staticmethod
    def backward(ctx, dy, dres):
        x, mean, rstd = ctx.saved_tensors
        L = ctx.layer
        if dy is None:
            return dres, None, None
        dx = ops.layer_norm_bwd(x, _c(dy), None if L.gamma is None else L.gamma.w, mean, rstd,
                                dgamma=None if L.gamma is None else L.gamma.g,
                                dbeta=None if L.beta is None else L.beta.g,
                                accumulate_into=_identity_grad(dres))
        return dx.view_as(x), None, None


class _LayerNormModFn(torch.autograd.Function):
    """adaLN: y = LN(x) * (1 + mod[b, scale_off:+C]) + mod[b, shift_off:+C]."""

    @staticmethod
    def forward(ctx, x, mod, shift_off, scale_off, eps):
        x = _c(x)
        B = mod.shape[0]
        rps = x.numel() // x.shape[-1] // B
        y, mean, rstd = ops.layer_norm(x, None, None, eps, mod=mod, mod_ld=mod.stride(0),
                                       shift_off=shift_off, scale_off=scale_off, rows_per_sample=rps)
        ctx.save_for_backward(x, mod, mean, rstd)
        ctx.meta = (shift_off, scale_off, rps)
        return y

    @staticmethod
    def backward(ctx, dy):
        x, mod, mean, rstd = ctx.saved_tensors
        shift_off, scale_off, rps = ctx.meta
        dmod = torch.zeros_like(mod)
        dx = ops.layer_norm_bwd(x, _c(dy), None, mean, rstd, mod=mod, mod_ld=mod.stride(0),
                                shift_off=shift_off, scale_off=scale_off, rows_per_sample=rps,
                                dmod=dmod, dmod_ld=dmod.stride(0))
        return dx, dmod, None, None, None


class _GateResidualFn(torch.autograd.Function):
    """y = x + mod[b, off:off+C] * h   (adaLN-Zero gate)."""

    @staticmethod
    def forward(ctx, x, mod, off, h):
        x, h = _c(x), _c(h)
        B = mod.shape[0]
        rps = x.numel() // x.shape[-1] // B
        g = mod[:, off:]
        y = ops.gate_residual(x, g, mod.stride(0), h, rps)
        ctx.save_for_backward(mod, h)
        ctx.meta = (off, rps)
        return y

    @staticmethod
    def backward(ctx, dy):
        mod, h = ctx.saved_tensors
        off, rps = ctx.meta
        dy = _c(dy)
        dmod = torch.zeros_like(mod)
        dh = ops.gate_residual_bwd(dy, mod[:, off:], mod.stride(0), h, dmod[:, off:], dmod.stride(0),
                                   mod.shape[0], rps)
        return dy, dmod, None, dh


class _ActFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, op):
        x = _c(x)
        ctx.save_for_backward(x)
        ctx.op = op
        return ops.act(x, op)

    @staticmethod
    def backward(ctx, dy):
        (x,) = ctx.saved_tensors
        return ops.act_bwd(x, _c(dy), ctx.op), None


class _GegluFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x):
        x = _c(x)
        ctx.save_for_backward(x)
        return ops.geglu(x)

    @staticmethod
    def backward(ctx, dy):
        (x,) = ctx.saved_tensors
        return ops.geglu_bwd(x, _c(dy))


class _AddFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, a, b):
        return ops.axpby(_c(a), _c(b))

    @staticmethod
    def backward(ctx, dy):
        return dy, dy


class _RowBiasFn(torch.autograd.Function):
    """y = x + e[b] broadcast over the pixels/tokens of sample b."""

    @staticmethod
    def forward(ctx, x, e, bias, e_bias):
        x = _c(x)
        B = e.shape[0]
        rps = x.numel() // x.shape[-1] // B
        ctx.meta = (B, rps)
        ctx.biases = (bias, e_bias)
        return ops.row_bias(x, e, rps)

    @staticmethod
    def backward(ctx, dy):
        B, rps = ctx.meta
        dy = _c(dy)
        # the producing conv's and the temb projection's bias gradients (both = sum of dy over every row)
        # from the same per-sample sums
        db, db2 = (b.g if b is not None else None for b in ctx.biases)
        return dy, ops.row_bias_bwd(dy, B, rps, db=db, db2=db2), None, None


class _ConcatFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, a, b):
        ctx.Ca = a.shape[-1]
        return ops.concat_last(_c(a), _c(b))

    @staticmethod
    def backward(ctx, dy):
        dy = _c(dy)
        Ca = ctx.Ca
        da = torch.empty(*dy.shape[:-1], Ca, device=dy.device, dtype=dy.dtype)
        db = torch.empty(*dy.shape[:-1], dy.shape[-1] - Ca, device=dy.device, dtype=dy.dtype)
        ops.split_last(dy, Ca, da, db)
        return da, db


class _AddConstFn(torch.autograd.Function):
    """y[b] = x[b] + const (const broadcast over the batch; e.g. fixed 2-D sin-cos positions)."""

    @staticmethod
    def forward(ctx, x, const):
        x = _c(x)
        B = x.shape[0]
        flat = x.view(B, -1)
        y = ops.row_bias(flat, const.view(1, -1).expand(1, flat.shape[1]), B)
        return y.view(x.shape)

    @staticmethod
    def backward(ctx, dy):
        return dy, None


class _SpaceToDepthFn(torch.autograd.Function):
    """NHWC [B,H,W,C] <-> [B,H/p,W/p,p*p*C] with patch channel order (i, j, c)."""

    @staticmethod
    def forward(ctx, x, p, inverse):
        ctx.meta = (p, inverse)
        return ops.space_to_depth(_c(x), p, inverse)

    @staticmethod
    def backward(ctx, dy):
        p, inverse = ctx.meta
        return ops.space_to_depth(_c(dy), p, not inverse), None, None


class _Upsample2xFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x):
        return ops.upsample2x(_c(x))

    @staticmethod
    def backward(ctx, dy):
        return ops.upsample2x_bwd(_c(dy))


class _AttentionFn(torch.autograd.Function):
    """Multi-head attention composed of batched tensor-core GEMMs and the softmax kernel.

    self-attention: q_t is a fused [B, N, 3C] qkv tensor and kv_t is None;
    cross-attention: q_t is [B, N, C], kv_t a fused [B, Nk, 2C] tensor.
    Scores/probabilities live in [B, h, N, ld] buffers with ld = Nk rounded up to 8
    (TMA row-stride alignment; the padding columns are never read).
    """

    @staticmethod
    def forward(ctx, q_t, kv_t, heads, causal):
        with telemetry.site("attn"):
            return _AttentionFn._fwd(ctx, q_t, kv_t, heads, causal)

    @staticmethod
    def backward(ctx, do):
        with telemetry.site("attn"):
            return _AttentionFn._bwd(ctx, do)

    @staticmethod
    def _fwd(ctx, q_t, kv_t, heads, causal):
        q_t = _c(q_t)
        kv_t = None if kv_t is None else _c(kv_t)
        B, N = q_t.shape[0], q_t.shape[1]
        if kv_t is None:
            C = q_t.shape[2] // 3
            src_k, Nk, k_off, v_off, kv_ld = q_t, N, C, 2 * C, 3 * C
            q_ld = 3 * C
        else:
            C = q_t.shape[2]
            src_k, Nk, k_off, v_off, kv_ld = kv_t, kv_t.shape[1], 0, C, 2 * C
            q_ld = C
        hd = C // heads
        scale = 1.0 / math.sqrt(hd)
        dev, dt = q_t.device, q_t.dtype
        # causal masking exists in the fused forward only: used where no gradient flows back
        # (the frozen CLIP text encoder); a trainable causal attention keeps the explicit path
        grad_needed = ctx.needs_input_grad[0] or ctx.needs_input_grad[1]
        if FLASH_ATTENTION and dt == torch.bfloat16 and hd == 64 and not (causal and grad_needed):
            # fused tcgen05 attention: no score / probability tensors in HBM
            o = torch.empty(B, N, C, device=dev, dtype=dt)
            lse = torch.empty(B, heads, N, device=dev, dtype=torch.float32)
            kp = src_k.view(-1)[k_off:]
            vp = src_k.view(-1)[v_off:]
            ops.flash_attn_fwd(q_t, kp, vp, o, B=B, N=N, Nk=Nk, heads=heads, q_ld=q_ld, kv_ld=kv_ld,
                               o_ld=C, scale=scale, lse=lse, causal=causal)
            ctx.save_for_backward(q_t, src_k if kv_t is not None else q_t, o, lse)
            ctx.meta = (kv_t is None, heads, B, N, Nk, C, hd, q_ld, kv_ld, k_off, v_off, scale)
            ctx.flash = True
            return o
        ctx.flash = False
        ld = -(-Nk // 8) * 8
        S = torch.empty(B, heads, N, ld, device=dev, dtype=torch.float32)
        P = torch.empty(B, heads, N, ld, device=dev, dtype=dt)
        o = torch.empty(B, N, C, device=dev, dtype=dt)
        qp = q_t  # q at offset 0 in both layouts
        kp = src_k.view(-1)[k_off:]
        vp = src_k.view(-1)[v_off:]
        # S[b,h] = Q_bh K_bh^T (unscaled; the softmax applies `scale`)
        ops.gemm(qp, kp, S, M=N, N=Nk, K=hd, a_ld=q_ld, b_ld=kv_ld, d_ld=ld, batch=(heads, B),
                 a_bs=(hd, N * q_ld), b_bs=(hd, Nk * kv_ld), d_bs=(N * ld, heads * N * ld))
        ops.softmax(S, P, scale, Nk, causal=causal, Lq=N)
        # O[b, :, h*hd:] = P_bh V_bh   (V MN-major)
        ops.gemm(P, vp, o, M=N, N=hd, K=Nk, a_ld=ld, b_ld=kv_ld, b_mn=True, d_ld=C, batch=(heads, B),
                 a_bs=(N * ld, heads * N * ld), b_bs=(hd, Nk * kv_ld), d_bs=(hd, N * C))
        ctx.save_for_backward(q_t, src_k if kv_t is not None else q_t, P)
        ctx.meta = (kv_t is None, heads, B, N, Nk, C, hd, ld, q_ld, kv_ld, k_off, v_off, scale)
        return o

    @staticmethod
    def _bwd(ctx, do):
        if ctx.flash:
            q_t, src_k, o, lse = ctx.saved_tensors
            self_attn, heads, B, N, Nk, C, hd, q_ld, kv_ld, k_off, v_off, scale = ctx.meta
            do = _c(do)
            dq_t = torch.empty_like(q_t)
            dkv_t = dq_t if self_attn else torch.empty_like(src_k)
            ops.flash_attn_bwd(q_t, src_k.view(-1)[k_off:], src_k.view(-1)[v_off:], o, do, dq_t,
                               dkv_t.view(-1)[k_off:], dkv_t.view(-1)[v_off:], lse, B=B, N=N, Nk=Nk,
                               heads=heads, q_ld=q_ld, kv_ld=kv_ld, o_ld=C, do_ld=C, dq_ld=q_ld,
                               dkv_ld=kv_ld, scale=scale)
            if self_attn:
                return dq_t, None, None, None
            return dq_t, dkv_t, None, None
        q_t, src_k, P = ctx.saved_tensors
        self_attn, heads, B, N, Nk, C, hd, ld, q_ld, kv_ld, k_off, v_off, scale = ctx.meta
        do = _c(do)
        dev, dt = do.device, do.dtype
        dq_t = torch.empty_like(q_t)
        dkv_t = dq_t if self_attn else torch.empty_like(src_k)
        kp = src_k.view(-1)[k_off:]
        vp = src_k.view(-1)[v_off:]
        dkp = dkv_t.view(-1)[k_off:]
        dvp = dkv_t.view(-1)[v_off:]
        # dV = P^T dO : M=Nk, N=hd, K=N
        ops.gemm(P, do, dvp, M=Nk, N=hd, K=N, a_ld=ld, a_mn=True, b_ld=C, b_mn=True, d_ld=kv_ld,
                 batch=(heads, B), a_bs=(N * ld, heads * N * ld), b_bs=(hd, N * C), d_bs=(hd, Nk * kv_ld))
        # dP = dO V^T : M=N, N=Nk, K=hd (fp32)
        dP = torch.empty(B, heads, N, ld, device=dev, dtype=torch.float32)
        ops.gemm(do, vp, dP, M=N, N=Nk, K=hd, a_ld=C, b_ld=kv_ld, d_ld=ld, batch=(heads, B),
                 a_bs=(hd, N * C), b_bs=(hd, Nk * kv_ld), d_bs=(N * ld, heads * N * ld))
        dS = torch.empty(B, heads, N, ld, device=dev, dtype=dt)
        ops.softmax_bwd(P, dP, dS, scale, Nk)
        del dP
        # dQ = dS K : M=N, N=hd, K=Nk (K MN-major)
        ops.gemm(dS, kp, dq_t, M=N, N=hd, K=Nk, a_ld=ld, b_ld=kv_ld, b_mn=True, d_ld=q_ld,
                 batch=(heads, B), a_bs=(N * ld, heads * N * ld), b_bs=(hd, Nk * kv_ld), d_bs=(hd, N * q_ld))
        # dK = dS^T Q : M=Nk, N=hd, K=N
        ops.gemm(dS, q_t, dkp, M=Nk, N=hd, K=N, a_ld=ld, a_mn=True, b_ld=q_ld, b_mn=True, d_ld=kv_ld,
                 batch=(heads, B), a_bs=(N * ld, heads * N * ld), b_bs=(hd, N * q_ld), d_bs=(hd, Nk * kv_ld))
        if self_attn:
            return dq_t, None, None, None
        return dq_t, dkv_t, None, None


# ============================================================================ layer API

def _anchor():
    return current_anchor()


class Linear:
    def __init__(self, store, name, fin, fout, bias=True, init="w"):
        self.store = store
        self.weight = store.add(f"{name}.weight", (fout, fin), init=init)
        self.bias = store.add(f"{name}.bias", (fout,), fp32=True, init="b") if bias else None
        # True when the output feeds only a per-sample row bias whose backward produces this bias gradient
        self.bias_grad_by_row = False

    def __call__(self, x, residual=None):
        return _LinearFn.apply(x, _anchor(), residual, self)


class Conv2d:
    """NHWC conv, weights [K, R, S, C]; `pad` = (top, left); symmetric unless out_hw given."""

    def __init__(self, store, name, cin, cout, k=3, stride=1, pad=None, bias=True, init="w",
                 asym=False):
        self.k, self.stride = k, stride
        self.pad = (0, 0) if asym else ((k // 2, k // 2) if pad is None else pad)
        self.asym = asym
        self.store = store
        self.weight = store.add(f"{name}.weight", (cout, k, k, cin), init=init)
        self.bias = store.add(f"{name}.bias", (cout,), fp32=True, init="b") if bias else None
        self.gn_stats = 0  # GroupNorm groups of the output's consumer (statistics in the conv epilogue)
        # True when the output's only consumer is a per-sample row bias (ResBlock conv1 + temb) whose
        # backward also produces this conv's bias gradient (add_row_bias(..., bias=...))
        self.bias_grad_by_row = False

    def out_hw(self, x):
        H, W = x.shape[1], x.shape[2]
        if self.asym:  # SD-VAE downsample: pad (0,1,0,1) then 3x3 stride 2
            return ((H + 1 - self.k) // 2 + 1, (W + 1 - self.k) // 2 + 1)
        return (ops.conv_out_size(H, self.k, self.stride, self.pad[0], self.pad[0]),
                ops.conv_out_size(W, self.k, self.stride, self.pad[1], self.pad[1]))

    def __call__(self, x, residual=None):
        return _ConvFn.apply(x, _anchor(), residual, self)


class GroupNorm:
    def __init__(self, store, name, C, groups=32, eps=1e-6, silu=False):
        self.groups, self.eps, self.silu = groups, eps, silu
        self.gamma = store.add(f"{name}.weight", (C,), fp32=True, init="g")
        self.beta = store.add(f"{name}.bias", (C,), fp32=True, init="b")

    def __call__(self, x):
        return _GroupNormFn.apply(x, _anchor(), self)

    def fork(self, x):
        """(GroupNorm(x), x-alias): use the alias for x's other consumer (residual / skip)."""
        return _GroupNormForkFn.apply(x, _anchor(), self)


class LayerNorm:
    def __init__(self, store, name, C, eps=1e-5, affine=True):
        self.eps = eps
        self.gamma = store.add(f"{name}.weight", (C,), fp32=True, init="g") if affine else None
        self.beta = store.add(f"{name}.bias", (C,), fp32=True, init="b") if affine else None

    def __call__(self, x):
        return _LayerNormFn.apply(x, _anchor(), self)

    def fork(self, x):
        """(LayerNorm(x), x-alias): use the alias for x's other consumer (the residual add)."""
        return _LayerNormForkFn.apply(x, _anchor(), self)


def ln_modulate(x, mod, shift_off, scale_off, eps=1e-6):
    return _LayerNormModFn.apply(x, mod, shift_off, scale_off, eps)


def gate_residual(x, mod, off, h):
    return _GateResidualFn.apply(x, mod, off, h)


def silu(x):
    return _ActFn.apply(x, DP_ACT_SILU)


def gelu(x, tanh=False):
    return _ActFn.apply(x, DP_ACT_GELU_TANH if tanh else DP_ACT_GELU)


def geglu(x):
    return _GegluFn.apply(x)


def add(a, b):
    return _AddFn.apply(a, b)


# DP_ROW_BIAS_DB=0: ResBlock conv1's bias gradient by its own pass over dy (A/B)
ROW_BIAS_DB = os.environ.get("DP_ROW_BIAS_DB", "1") != "0"


def add_row_bias(x, e, bias=None, e_bias=None):
    """x + e[sample]; `bias` / `e_bias` (Params whose layers have bias_grad_by_row set: the layer that
    produced x / e) each also receive sum(dy) over every row in the backward."""
    return _RowBiasFn.apply(x, e, bias, e_bias)


def concat(a, b):
    return _ConcatFn.apply(a, b)


def upsample2x(x):
    return _Upsample2xFn.apply(x)


def add_const(x, const):
    return _AddConstFn.apply(x, const)


def space_to_depth(x, p):
    return _SpaceToDepthFn.apply(x, p, False)


def depth_to_space(x, p):
    return _SpaceToDepthFn.apply(x, p, True)


def attention(q_t, kv_t, heads, causal=False):
    return _AttentionFn.apply(q_t, kv_t, heads, causal)


class SelfAttention:
    """Fused qkv projection -> attention -> out projection (+ residual in the epilogue)."""

    def __init__(self, store, name, C, heads, qkv_bias=False, causal=False):
        self.heads, self.causal = heads, causal
        self.qkv = Linear(store, f"{name}.qkv", C, 3 * C, bias=qkv_bias)
        self.out = Linear(store, f"{name}.out", C, C)

    def __call__(self, x, residual=None):
        o = attention(self.qkv(x), None, self.heads, self.causal)
        return self.out(o, residual=residual)


class CrossAttention:
    def __init__(self, store, name, C, ctx_dim, heads):
        self.heads = heads
        self.q = Linear(store, f"{name}.q", C, C, bias=False)
        self.kv = Linear(store, f"{name}.kv", ctx_dim, 2 * C, bias=False)
        self.out = Linear(store, f"{name}.out", C, C)

    def __call__(self, x, ctx, residual=None):
        o = attention(self.q(x), self.kv(ctx), self.heads)
        return self.out(o, residual=residual)
