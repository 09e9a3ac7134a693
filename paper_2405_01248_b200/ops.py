"""Torch-facing wrappers over the libdpipe C ABI (no autograd here).

Every function takes/returns torch CUDA tensors, launches on the current
torch stream, and raises when the native library is missing: there is no
eager-PyTorch or CPU fallback on the product path.
"""

from __future__ import annotations

import ctypes

import torch

from . import _lib, telemetry
from ._lib import DP_BF16, DP_F32, DP_OUT_ATOMIC_ADD, DP_OUT_STORE, DpConvArgs, DpGemmArgs, check

_DT = {torch.float32: DP_F32, torch.bfloat16: DP_BF16}


def dtype_code(t: torch.Tensor) -> int:
    try:
        return _DT[t.dtype]
    except KeyError:
        raise TypeError(f"unsupported dtype {t.dtype}") from None


_raw_stream = getattr(torch._C, "_cuda_getCurrentRawStream", None)
_cur_device = getattr(torch._C, "_cuda_getDevice", None)


def _stream() -> int:
    """cudaStream_t of torch's current stream on the current device. The C accessors skip the
    public current_stream() path (device-index normalisation, availability checks, a Stream
    object per call), which was a quarter of the host time per launch."""
    if _raw_stream is not None and _cur_device is not None:
        return _raw_stream(_cur_device())
    return torch.cuda.current_stream().cuda_stream


def _ptr(t):
    return None if t is None else t.data_ptr()


def _require_cuda(*ts):
    for t in ts:
        if t is not None and not t.is_cuda:
            raise ValueError("libdpipe ops need CUDA tensors (no CPU fallback on the product path)")


# ---------------------------------------------------------------------------- GEMM

def gemm(A, B, D, *, M, N, K, a_ld, b_ld, d_ld, a_mn=False, b_mn=False,
         batch=(1, 1), a_bs=(0, 0), b_bs=(0, 0), d_bs=(0, 0),
         bias=None, residual=None, r_ld=None, r_bs=None, alpha=1.0, accumulate=False,
         split_k=0):
    """D[z](m,n) = alpha * sum_k A[z](m,k) B[z](n,k) (+bias[n]) (+residual[z](m,n)).

    Raw-stride interface mirroring DpGemmArgs; A and B must share a dtype
    (bf16 -> tcgen05 tensor cores, fp32 -> fp32 SIMT path).
    """
    _require_cuda(A, B, D, bias, residual)
    if A.dtype != B.dtype:
        raise TypeError("A and B must share a dtype")
    if bias is not None and bias.dtype != torch.float32:
        raise TypeError("bias must be fp32")
    args = DpGemmArgs()
    args.M, args.N, args.K = M, N, K
    args.batch1, args.batch2 = batch
    args.dtype = dtype_code(A)
    args.A, args.a_ld, (args.a_bs1, args.a_bs2), args.a_mn_major = _ptr(A), a_ld, a_bs, int(a_mn)
    args.B, args.b_ld, (args.b_bs1, args.b_bs2), args.b_mn_major = _ptr(B), b_ld, b_bs, int(b_mn)
    args.D, args.d_dtype, args.d_ld, (args.d_bs1, args.d_bs2) = _ptr(D), dtype_code(D), d_ld, d_bs
    args.out_mode = DP_OUT_ATOMIC_ADD if accumulate else DP_OUT_STORE
    args.bias = _ptr(bias)
    args.Res = _ptr(residual)
    args.r_ld = d_ld if r_ld is None else r_ld
    args.r_bs1, args.r_bs2 = d_bs if r_bs is None else r_bs
    args.alpha = alpha
    args.split_k = split_k
    ws = _splitk_ws(args, "dp_gemm_workspace", A.device)
    fam = "tcgen05_gemm" if A.dtype == torch.bfloat16 else "simt_gemm"
    flops = 2.0 * M * N * K * max(1, batch[0]) * max(1, batch[1])
    telemetry.timed(fam, flops, lambda: check(_lib.lib().dp_gemm(ctypes.byref(args), _stream()), "dp_gemm",
                                              2 if ws is not None else 1),
                    sub=f"linear {M}x{N}x{K}{'a' if a_mn else ''}{'b' if b_mn else ''}x{batch[0] * batch[1]}"
                    if telemetry.SHAPES else "linear")
    return D


def _splitk_ws(args, query, device):
    """fp32 workspace that lets an under-filled bf16 launch split K over every SM (the C ABI
    decides and sizes it; kernels never allocate). Returns the tensor (kept alive by the
    caller until the launch is enqueued) or None."""
    if args.dtype != DP_BF16:
        return None
    nbytes = getattr(_lib.lib(), query)(ctypes.byref(args))
    if nbytes <= 0:
        return None
    ws = torch.empty(nbytes // 4, device=device, dtype=torch.float32)
    args.workspace = ws.data_ptr()
    args.workspace_bytes = nbytes
    return ws


def linear(x, w, bias=None, residual=None, out=None):
    """y[M,N] = x[M,K] @ w[N,K]^T (+bias) (+residual)."""
    M, K = x.shape
    N = w.shape[0]
    if out is None:
        out = torch.empty(M, N, device=x.device, dtype=x.dtype)
    return gemm(x, w, out, M=M, N=N, K=K, a_ld=x.stride(0), b_ld=w.stride(0), d_ld=out.stride(0),
                bias=bias, residual=residual)


def linear_gelu(x, w, bias, out=None):
    """y[M,N] = gelu_erf(x @ w^T + bias) in one tensor-core GEMM (GELU in the epilogue, no separate
    activation pass); bf16, K-major operands, N % 128 == 0 (the frozen text encoders' MLP fc1)."""
    _require_cuda(x, w, bias)
    M, K = x.shape
    N = w.shape[0]
    y = torch.empty(M, N, device=x.device, dtype=x.dtype) if out is None else out
    args = DpGemmArgs()
    args.M, args.N, args.K = M, N, K
    args.batch1, args.batch2 = 1, 1
    args.dtype = dtype_code(x)
    args.A, args.a_ld, args.a_bs1, args.a_bs2, args.a_mn_major = _ptr(x), x.stride(0), 0, 0, 0
    args.B, args.b_ld, args.b_bs1, args.b_bs2, args.b_mn_major = _ptr(w), w.stride(0), 0, 0, 0
    args.D, args.d_dtype, args.d_ld, args.d_bs1, args.d_bs2 = _ptr(y), dtype_code(y), y.stride(0), 0, 0
    args.out_mode = DP_OUT_STORE
    args.bias = _ptr(bias)
    args.Res = None
    args.r_ld, args.r_bs1, args.r_bs2 = y.stride(0), 0, 0
    args.alpha = 1.0
    args.split_k = 0
    args.geglu_mode = 3
    telemetry.timed("tcgen05_gemm", 2.0 * M * N * K,
                    lambda: check(_lib.lib().dp_gemm(ctypes.byref(args), _stream()), "dp_gemm"),
                    sub=f"linear {M}x{N}x{K} gelu" if telemetry.SHAPES else "linear")
    return y


def linear_geglu(x, w, bias, h_out=None, y_out=None):
    """h[M,2F] = x @ w^T + bias (the GEGLU pre-activation, stored for the backward) and
    y[M,F] = h[:, :F] * gelu_erf(h[:, F:]) in ONE tensor-core GEMM (the epilogue writes both);
    bf16, K-major operands, F % 64 == 0."""
    _require_cuda(x, w, bias)
    M, K = x.shape
    N = w.shape[0]
    F = N // 2
    h = torch.empty(M, N, device=x.device, dtype=x.dtype) if h_out is None else h_out
    y = torch.empty(M, F, device=x.device, dtype=x.dtype) if y_out is None else y_out
    args = DpGemmArgs()
    args.M, args.N, args.K = M, N, K
    args.batch1, args.batch2 = 1, 1
    args.dtype = dtype_code(x)
    args.A, args.a_ld, args.a_bs1, args.a_bs2, args.a_mn_major = _ptr(x), x.stride(0), 0, 0, 0
    args.B, args.b_ld, args.b_bs1, args.b_bs2, args.b_mn_major = _ptr(w), w.stride(0), 0, 0, 0
    args.D, args.d_dtype, args.d_ld, args.d_bs1, args.d_bs2 = _ptr(h), dtype_code(h), h.stride(0), 0, 0
    args.out_mode = DP_OUT_STORE
    args.bias = _ptr(bias)
    args.Res = None
    args.r_ld, args.r_bs1, args.r_bs2 = h.stride(0), 0, 0
    args.alpha = 1.0
    args.split_k = 0
    args.geglu_out = _ptr(y)
    args.geglu_ld = y.stride(0)
    args.geglu_mode = 1
    telemetry.timed("tcgen05_gemm", 2.0 * M * N * K,
                    lambda: check(_lib.lib().dp_gemm(ctypes.byref(args), _stream()), "dp_gemm"),
                    sub=f"linear {M}x{N}x{K} geglu" if telemetry.SHAPES else "linear")
    return h, y


def linear_dgrad_geglu(dy, w, h, cache=None):
    """dh[M,2F] = GEGLU'(h) applied to (dy[M,N] @ w[N,F]): the input gradient of the FF output projection
    and the GEGLU backward in one GEMM (its epilogue reads h = [a | g] and writes both halves of dh)."""
    M, N = dy.shape
    F = w.shape[1]
    dh = torch.empty(M, 2 * F, device=dy.device, dtype=dy.dtype)

    def make(dst):
        wt = torch.empty(F, N, device=w.device, dtype=w.dtype) if dst is None else dst
        check(_lib.lib().dp_conv_weight_flip(dtype_code(w), _ptr(w), _ptr(wt), N, 1, 1, F, _stream()),
              "dp_conv_weight_flip")
        return wt
    wt = cached_flip(cache, make, lambda wt_: (w, wt_, N, 1, 1, F))
    args = DpGemmArgs()
    args.M, args.N, args.K = M, F, N
    args.batch1, args.batch2 = 1, 1
    args.dtype = dtype_code(dy)
    args.A, args.a_ld, args.a_bs1, args.a_bs2, args.a_mn_major = _ptr(dy), dy.stride(0), 0, 0, 0
    args.B, args.b_ld, args.b_bs1, args.b_bs2, args.b_mn_major = _ptr(wt), N, 0, 0, 0
    args.D, args.d_dtype, args.d_ld, args.d_bs1, args.d_bs2 = _ptr(dh), dtype_code(dh), dh.stride(0), 0, 0
    args.out_mode = DP_OUT_STORE
    args.bias = None
    args.Res = None
    args.r_ld, args.r_bs1, args.r_bs2 = dh.stride(0), 0, 0
    args.alpha = 1.0
    args.split_k = 0
    args.geglu_out = _ptr(h)
    args.geglu_ld = h.stride(0)
    args.geglu_mode = 2
    telemetry.timed("tcgen05_gemm", 2.0 * M * N * F,
                    lambda: check(_lib.lib().dp_gemm(ctypes.byref(args), _stream()), "dp_gemm"),
                    sub=f"linear {M}x{F}x{N}b geglu-bwd" if telemetry.SHAPES else "linear")
    return dh


def cached_flip(cache, make, flip_args=None):
    """The flip-transposed weight for a dgrad: `make(dst)` writes it from the current weights.
    cache = (store, param) keeps one persistent copy per parameter, refreshed by the store right
    after each AdamW update of that parameter (nn.ParamStore.refresh_flips); None flips now.
    flip_args(wt) -> (w, K, R, S, C) when the copy is a plain flip of the parameter's own bf16 view
    (no channel padding): those refreshes are batched into one launch per optimizer slice."""
    if cache is None:
        return make(None)
    store, p = cache
    if p.wt is None:
        p.wt = make(None)
        p.wt_fn = make
        p.flip_args = None if flip_args is None else flip_args(p.wt)
        store.register_flip(p)
    return p.wt


def flip_batch(jobs):
    """Refresh cached dgrad weight copies: jobs = [(w, wt, K, R, S, C)], one launch per 48 jobs."""
    if not jobs:
        return
    arr = (_lib.DpFlipJob * len(jobs))()
    for i, (w, wt, K, R, S, C) in enumerate(jobs):
        arr[i].w, arr[i].wt, arr[i].K, arr[i].R, arr[i].S, arr[i].C = _ptr(w), _ptr(wt), K, R, S, C
    check(_lib.lib().dp_conv_weight_flip_batch(arr, len(jobs), _stream()), "dp_conv_weight_flip_batch",
          (len(jobs) + 47) // 48)


def linear_dgrad(dy, w, out=None, cache=None):
    """dx[M,K] = dy[M,N] @ w[N,K]. bf16 with a K-dim multiple of 8: the weight is transposed once
    (tiled flip-transpose kernel, K x N x 2 B) so that B is K-major and the GEMM can use CTA pairs and
    32-column tile widths (MN-major B is restricted to 64-column boxes on single CTAs)."""
    M, N = dy.shape
    K = w.shape[1]
    if out is None:
        out = torch.empty(M, K, device=dy.device, dtype=dy.dtype)
    if dy.dtype == torch.bfloat16 and K % 8 == 0 and N % 8 == 0 and w.is_contiguous() and M >= 1024:
        def make(dst):
            wt = torch.empty(K, N, device=w.device, dtype=w.dtype) if dst is None else dst
            check(_lib.lib().dp_conv_weight_flip(dtype_code(w), _ptr(w), _ptr(wt), N, 1, 1, K, _stream()),
                  "dp_conv_weight_flip")
            return wt
        wt = cached_flip(cache, make, (lambda wt_: (w, wt_, N, 1, 1, K)) if w.dtype == torch.bfloat16 else None)
        return gemm(dy, wt, out, M=M, N=K, K=N, a_ld=dy.stride(0), b_ld=N, d_ld=out.stride(0))
    return gemm(dy, w, out, M=M, N=K, K=N, a_ld=dy.stride(0), b_ld=w.stride(0), b_mn=True,
                d_ld=out.stride(0))


def linear_wgrad(dy, x, dw):
    """dw[N,K] (fp32) += dy[M,N]^T @ x[M,K]."""
    M, N = dy.shape
    K = x.shape[1]
    return gemm(dy, x, dw, M=N, N=K, K=M, a_ld=dy.stride(0), a_mn=True, b_ld=x.stride(0),
                b_mn=True, d_ld=dw.stride(0), accumulate=True)


# ---------------------------------------------------------------------------- conv (NHWC)

def conv_out_size(H, R, stride, pad_lo, pad_hi):
    return (H + pad_lo + pad_hi - R) // stride + 1


def _conv_args(x, w, y, stride, pad, P, Q, bias=None, residual=None, accumulate=False,
               alpha=1.0):
    N, H, W, C = x.shape
    K, R, S, _ = w.shape
    a = DpConvArgs()
    a.dtype = dtype_code(x)
    a.N, a.H, a.W, a.C = N, H, W, C
    a.K, a.R, a.S = K, R, S
    a.stride, a.pad_h, a.pad_w = stride, pad[0], pad[1]
    a.P, a.Q = P, Q
    a.x, a.w, a.y = _ptr(x), _ptr(w), _ptr(y)
    a.bias, a.Res = _ptr(bias), _ptr(residual)
    a.alpha = alpha
    a.out_mode = DP_OUT_ATOMIC_ADD if accumulate else DP_OUT_STORE
    a.split_k = 0
    return a


def _tiles(P, Q, pixels):
    if Q >= pixels:
        return Q % pixels == 0
    if pixels % Q:
        return False
    if P * Q >= pixels:
        return (P * Q) % pixels == 0
    return pixels % (P * Q) == 0


def _pad_last(t, mult=64):
    """Zero-pad the channel (last) dim to a multiple of `mult` (small convs such as the U-Net's
    4-channel conv_in/conv_out go through the same tensor-core implicit GEMM)."""
    C = t.shape[-1]
    pad = -C % mult
    if not pad:
        return t
    return concat_last(t.contiguous(), None, pad)  # the concat kernel writes the zero channels itself


def _pad_first(w, mult=64):
    K = w.shape[0]
    pad = -K % mult
    if not pad:
        return w
    out = torch.zeros(K + pad, *w.shape[1:], device=w.device, dtype=w.dtype)
    out[:K].copy_(w)
    return out


def _take_last(t, C):
    if t.shape[-1] == C:
        return t
    out = torch.empty(*t.shape[:-1], C, device=t.device, dtype=t.dtype)
    split_last(t, C, out, None)
    return out


def conv2d(x, w, *, stride=1, pad=(1, 1), out_hw=None, bias=None, residual=None, out=None, gn_sums=None,
           gn_groups=0):
    """NHWC conv: x [N,H,W,C], w [K,R,S,C] -> y [N,P,Q,K].

    pad is (top, left); bottom/right padding is implied by out_hw (default:
    symmetric padding). bf16: tcgen05 implicit GEMM (channels zero-padded to 64 when
    needed); fp32 (parity config): im2col + fp32 GEMM.
    """
    _require_cuda(x, w, bias, residual)
    N, H, W, C = x.shape
    K, R, S, C2 = w.shape
    assert C == C2, (x.shape, w.shape)
    if out_hw is None:
        out_hw = (conv_out_size(H, R, stride, pad[0], pad[0]), conv_out_size(W, S, stride, pad[1], pad[1]))
    P, Q = out_hw
    if out is None:
        out = torch.empty(N, P, Q, K, device=x.device, dtype=x.dtype)
    if R == 1 and S == 1 and stride == 1 and pad == (0, 0):
        return linear(x.reshape(-1, C), w.reshape(K, C), bias=bias,
                      residual=None if residual is None else residual.reshape(-1, K),
                      out=out.view(-1, K)).view(N, P, Q, K)
    if x.dtype == torch.bfloat16 and stride in (1, 2) and _tiles(P, Q, 128):
        xp, wp = _pad_last(x), _pad_last(w)
        Cp = xp.shape[-1]
        a = _conv_args(xp, wp, out, stride, pad, P, Q, bias, residual)
        if gn_sums is not None:  # GroupNorm statistics of the output for its consumer (conv epilogue)
            a.gn_sums, a.gn_groups = _ptr(gn_sums), gn_groups
        ws = None if gn_sums is not None else _splitk_ws(a, "dp_conv_fwd_workspace", x.device)
        telemetry.timed("tcgen05_gemm", 2.0 * N * P * Q * K * R * S * C,
                        lambda: check(_lib.lib().dp_conv_fwd(ctypes.byref(a), _stream()), "dp_conv_fwd",
                                      2 if ws is not None else 1),
                        sub=f"conv_fwd {N}x{H}x{W}x{C}->{K} r{R}s{stride}" if telemetry.SHAPES else "conv_fwd")
        return out
    cols = im2col(x, R, S, stride, pad, P, Q)
    linear(cols, w.reshape(K, -1), bias=bias,
           residual=None if residual is None else residual.reshape(-1, K), out=out.view(-1, K))
    return out


def im2col(x, R, S, stride, pad, P, Q):
    N, H, W, C = x.shape
    cols = torch.empty(N * P * Q, R * S * C, device=x.device, dtype=x.dtype)
    check(_lib.lib().dp_im2col(dtype_code(x), _ptr(x), _ptr(cols), N, H, W, C, R, S, stride,
                               pad[0], pad[1], P, Q, _stream()), "dp_im2col")
    return cols


def col2im(cols, dx, R, S, stride, pad, P, Q):
    N, H, W, C = dx.shape
    check(_lib.lib().dp_col2im(dtype_code(dx), _ptr(cols), _ptr(dx), N, H, W, C, R, S, stride,
                               pad[0], pad[1], P, Q, _stream()), "dp_col2im")
    return dx


def conv2d_dgrad(dy, w, x_shape, *, stride=1, pad=(1, 1), cache=None):
    """dx [N,H,W,C] of y = conv2d(x, w). bf16: implicit GEMM over dy (zero-dilated for
    stride 2) with the weights read tap-flipped in place (dp_conv_dgrad)."""
    _require_cuda(dy, w)
    N, P, Q, K = dy.shape
    K2, R, S, C = w.shape
    _, H, W, _ = x_shape
    if R == 1 and S == 1 and stride == 1 and pad == (0, 0):
        return linear_dgrad(dy.reshape(-1, K), w.reshape(K, C), cache=cache).view(N, H, W, C)
    if dy.dtype == torch.bfloat16 and _tiles(H, W, 128) and N * H * W < 8192:
        # small feature maps (U-Net 8x8 / 4x4 levels): the weights dominate the traffic, read
        # them tap-flipped in place (MN-major B_DGRAD operand mode, no transposed copy)
        src = _pad_last(dy)
        Kp = src.shape[-1]
        wp = _pad_first(_pad_last(w))
        Cp = wp.shape[-1]
        if stride > 1:
            dil = torch.empty(N, P * stride, Q * stride, Kp, device=dy.device, dtype=dy.dtype)
            check(_lib.lib().dp_dilate(dtype_code(dy), _ptr(src), _ptr(dil), N, P, Q, Kp, stride,
                                       _stream()), "dp_dilate")
            src = dil
        dx = torch.empty(N, H, W, Cp, device=dy.device, dtype=dy.dtype)
        a = _conv_args(dx, wp, dx, 1, pad, src.shape[1], src.shape[2])
        a.x = _ptr(src)
        ws = _splitk_ws(a, "dp_conv_dgrad_workspace", dy.device)
        telemetry.timed("tcgen05_gemm", 2.0 * N * H * W * C * R * S * K,
                        lambda: check(_lib.lib().dp_conv_dgrad(ctypes.byref(a), _stream()), "dp_conv_dgrad",
                                      2 if ws is not None else 1),
                        sub=f"conv_dgrad {N}x{H}x{W}x{C}<-{K} r{R}" if telemetry.SHAPES else "conv_dgrad")
        return _take_last(dx, C)
    if dy.dtype == torch.bfloat16 and _tiles(H, W, 128):
        # dx = conv(dy (zero-dilated for stride 2), flip-transposed w, pad R-1-pad): the forward
        # implicit GEMM with K-major weights (CTA pairs, 32-column tile widths) instead of the
        # MN-major B_DGRAD operand mode (64-column boxes, single CTAs)
        src = _pad_last(dy)
        Kp = src.shape[-1]
        wp = _pad_first(_pad_last(w))
        Cp = wp.shape[-1]
        if stride > 1:
            dil = torch.empty(N, P * stride, Q * stride, Kp, device=dy.device, dtype=dy.dtype)
            check(_lib.lib().dp_dilate(dtype_code(dy), _ptr(src), _ptr(dil), N, P, Q, Kp, stride,
                                       _stream()), "dp_dilate")
            src = dil
        def make(dst):
            wpp = _pad_first(_pad_last(w))  # the current weights (a refresh re-reads them)
            wt = torch.empty(Cp, R, S, Kp, device=w.device, dtype=w.dtype) if dst is None else dst
            check(_lib.lib().dp_conv_weight_flip(dtype_code(wpp), _ptr(wpp), _ptr(wt), Kp, R, S, Cp,
                                                 _stream()), "dp_conv_weight_flip")
            return wt
        plain = Kp == K and Cp == C  # no channel padding: the copy is a flip of the parameter view itself
        wt = cached_flip(cache, make, (lambda wt_: (w, wt_, K, R, S, C)) if plain else None)
        dx = torch.empty(N, H, W, Cp, device=dy.device, dtype=dy.dtype)
        a = _conv_args(src, wt, dx, 1, (R - 1 - pad[0], S - 1 - pad[1]), H, W)
        ws = _splitk_ws(a, "dp_conv_fwd_workspace", dy.device)
        telemetry.timed("tcgen05_gemm", 2.0 * N * H * W * C * R * S * K,
                        lambda: check(_lib.lib().dp_conv_fwd(ctypes.byref(a), _stream()), "dp_conv_fwd",
                                      2 if ws is not None else 1),
                        sub=f"conv_dgrad {N}x{H}x{W}x{C}<-{K} r{R}" if telemetry.SHAPES else "conv_dgrad")
        return _take_last(dx, C)
    dcols = linear_dgrad(dy.reshape(-1, K), w.reshape(K, -1))
    dx = torch.zeros(N, H, W, C, device=dy.device, dtype=dy.dtype)
    return col2im(dcols, dx, R, S, stride, pad, P, Q)


def conv2d_wgrad(dy, x, dw, *, stride=1, pad=(1, 1)):
    """dw [K,R,S,C] (fp32, accumulated) += wgrad of y = conv2d(x, w)."""
    _require_cuda(dy, x, dw)
    N, P, Q, K = dy.shape
    _, H, W, C = x.shape
    _, R, S, _ = dw.shape
    if R == 1 and S == 1 and stride == 1 and pad == (0, 0):
        return linear_wgrad(dy.reshape(-1, K), x.reshape(-1, C), dw.view(K, C))
    if dy.dtype == torch.bfloat16 and _tiles(P, Q, 64):
        dyp, xp = _pad_last(dy), _pad_last(x)
        Kp, Cp = dyp.shape[-1], xp.shape[-1]
        tgt = dw if (Kp == K and Cp == C) else torch.zeros(Kp, R, S, Cp, device=dw.device,
                                                           dtype=torch.float32)
        a = _conv_args(xp, tgt, tgt, stride, pad, P, Q, accumulate=True)
        a.w = _ptr(dyp)  # wgrad reads dy through the `w` slot (see dpipe.h)
        a.K, a.R, a.S = Kp, R, S
        telemetry.timed("tcgen05_gemm", 2.0 * N * P * Q * K * R * S * C,
                        lambda: check(_lib.lib().dp_conv_wgrad(ctypes.byref(a), _stream()), "dp_conv_wgrad"),
                        sub=f"conv_wgrad {N}x{H}x{W}x{C}->{K} r{R}" if telemetry.SHAPES else "conv_wgrad")
        if tgt is not dw:
            dw.add_(tgt[:K, :, :, :C])
        return dw
    cols = im2col(x, R, S, stride, pad, P, Q)
    return linear_wgrad(dy.reshape(-1, K), cols, dw.view(K, -1))


# ---------------------------------------------------------------------------- elementwise / norm

def _L():
    return _lib.lib()


def act(x, op, out=None):
    out = torch.empty_like(x) if out is None else out
    check(_L().dp_act_fwd(op, dtype_code(x), _ptr(x), _ptr(out), x.numel(), _stream()), "dp_act_fwd")
    return out


def act_bwd(x, dy, op, dx=None, accumulate=False):
    dx = torch.empty_like(x) if dx is None else dx
    check(_L().dp_act_bwd(op, dtype_code(x), _ptr(x), _ptr(dy), _ptr(dx), x.numel(), int(accumulate),
                          _stream()), "dp_act_bwd")
    return dx


def geglu(x):
    rows, F2 = x.numel() // x.shape[-1], x.shape[-1]
    y = torch.empty(*x.shape[:-1], F2 // 2, device=x.device, dtype=x.dtype)
    check(_L().dp_geglu_fwd(dtype_code(x), _ptr(x), _ptr(y), rows, F2 // 2, _stream()), "dp_geglu_fwd")
    return y


def geglu_bwd(x, dy, db=None):
    """dx = GEGLU'(x) dy; with db (fp32 [2F]) also db += column sums of dx (the bias gradient of the
    projection that produced x, fused into the same pass)."""
    rows, F2 = x.numel() // x.shape[-1], x.shape[-1]
    dx = torch.empty_like(x)
    if db is not None:
        check(_L().dp_geglu_bwd_db(dtype_code(x), _ptr(x), _ptr(dy), _ptr(dx), rows, F2 // 2, _ptr(db),
                                   _stream()), "dp_geglu_bwd_db")
        return dx
    check(_L().dp_geglu_bwd(dtype_code(x), _ptr(x), _ptr(dy), _ptr(dx), rows, F2 // 2, _stream()),
          "dp_geglu_bwd")
    return dx


def axpby(a, b, alpha=1.0, beta=1.0, out=None):
    out = torch.empty_like(a) if out is None else out
    check(_L().dp_axpby(dtype_code(a), _ptr(a), _ptr(b), _ptr(out), a.numel(), alpha, beta, _stream()),
          "dp_axpby")
    return out


def gate_residual(x, g, g_ld, h, rows_per_sample):
    C = x.shape[-1]
    y = torch.empty_like(x)
    check(_L().dp_gate_residual_fwd(dtype_code(x), _ptr(x), _ptr(g), g_ld, _ptr(h), _ptr(y),
                                    x.numel() // C, C, rows_per_sample, _stream()), "dp_gate_residual_fwd")
    return y


def gate_residual_bwd(dy, g, g_ld, h, dg, dg_ld, B, rows_per_sample):
    C = dy.shape[-1]
    dh = torch.empty_like(dy)
    check(_L().dp_gate_residual_bwd(dtype_code(dy), _ptr(dy), _ptr(g), g_ld, _ptr(h), _ptr(dh), _ptr(dg),
                                    dg_ld, B, C, rows_per_sample, _stream()), "dp_gate_residual_bwd")
    return dh


def q_sample(x0, noise, t, sqrt_ab, sqrt_1mab, out=None):
    out = torch.empty_like(x0) if out is None else out
    check(_L().dp_q_sample(dtype_code(x0), _ptr(x0), _ptr(noise), _ptr(t), _ptr(sqrt_ab), _ptr(sqrt_1mab),
                           _ptr(out), x0.numel(), x0.numel() // x0.shape[0], _stream()), "dp_q_sample")
    return out


def pred_x0(xt, eps, t, sqrt_ab, sqrt_1mab, out=None):
    out = torch.empty_like(xt) if out is None else out
    check(_L().dp_pred_x0(dtype_code(xt), _ptr(xt), _ptr(eps), _ptr(t), _ptr(sqrt_ab), _ptr(sqrt_1mab),
                          _ptr(out), xt.numel(), xt.numel() // xt.shape[0], _stream()), "dp_pred_x0")
    return out


def mse(pred, target, loss_acc, scale, dpred=None):
    check(_L().dp_mse(dtype_code(pred), _ptr(pred), _ptr(target), _ptr(dpred), _ptr(loss_acc), pred.numel(),
                      scale, _stream()), "dp_mse")
    return dpred


def timestep_embed(t, dim, dtype, max_period=10000.0):
    out = torch.empty(t.shape[0], dim, device=t.device, dtype=dtype)
    check(_L().dp_timestep_embed(_DT[dtype], _ptr(t), _ptr(out), t.shape[0], dim, max_period, _stream()),
          "dp_timestep_embed")
    return out


def embed(ids, table, pos=None):
    B, L = ids.shape
    C = table.shape[1]
    out = torch.empty(B, L, C, device=ids.device, dtype=table.dtype)
    check(_L().dp_embed(dtype_code(table), _ptr(ids), _ptr(table), _ptr(pos), _ptr(out), B * L, L, C,
                        _stream()), "dp_embed")
    return out


def concat_last(a, b, Cb=None):
    """cat([a, b], -1) over row-major tensors; b None -> zeros of width Cb."""
    Ca = a.shape[-1]
    Cb = b.shape[-1] if b is not None else Cb
    rows = a.numel() // Ca
    out = torch.empty(*a.shape[:-1], Ca + Cb, device=a.device, dtype=a.dtype)
    check(_L().dp_concat(dtype_code(a), _ptr(a), _ptr(b), _ptr(out), rows, Ca, Cb, _stream()), "dp_concat")
    return out


def split_last(src, Ca, a=None, b=None, acc_a=False, acc_b=False):
    C = src.shape[-1]
    rows = src.numel() // C
    check(_L().dp_split(dtype_code(src), _ptr(src), _ptr(a), _ptr(b), rows, Ca, C - Ca, int(acc_a),
                        int(acc_b), _stream()), "dp_split")
    return a, b


def upsample2x(x):
    N, H, W, C = x.shape
    y = torch.empty(N, 2 * H, 2 * W, C, device=x.device, dtype=x.dtype)
    check(_L().dp_upsample2x(dtype_code(x), _ptr(x), _ptr(y), N, H, W, C, _stream()), "dp_upsample2x")
    return y


def upsample2x_bwd(dy):
    N, H2, W2, C = dy.shape
    dx = torch.empty(N, H2 // 2, W2 // 2, C, device=dy.device, dtype=dy.dtype)
    check(_L().dp_upsample2x_bwd(dtype_code(dy), _ptr(dy), _ptr(dx), N, H2 // 2, W2 // 2, C, _stream()),
          "dp_upsample2x_bwd")
    return dx


def cast(x, dtype, out=None):
    out = torch.empty(x.shape, device=x.device, dtype=dtype) if out is None else out
    check(_L().dp_cast(dtype_code(x), _DT[dtype], _ptr(x), _ptr(out), x.numel(), _stream()), "dp_cast")
    return out


def bias_grad(dy, db):
    C = dy.shape[-1]
    check(_L().dp_bias_grad(dtype_code(dy), _ptr(dy), _ptr(db), dy.numel() // C, C, _stream()),
          "dp_bias_grad")


def adamw(param, grad, exp_avg, exp_avg_sq, param_bf16, lr, beta1, beta2, eps, weight_decay, step,
          grad_scale=1.0):
    check(_L().dp_adamw(_ptr(param), _ptr(grad), _ptr(exp_avg), _ptr(exp_avg_sq), _ptr(param_bf16),
                        param.numel(), lr, beta1, beta2, eps, weight_decay, step, grad_scale, _stream()),
          "dp_adamw")


def adamw_dev(param, grad, exp_avg, exp_avg_sq, param_bf16, lr, beta1, beta2, eps, weight_decay,
              step_dev, bc_dev, grad_scale=1.0):
    check(_L().dp_adamw_dev(_ptr(param), _ptr(grad), _ptr(exp_avg), _ptr(exp_avg_sq), _ptr(param_bf16),
                            param.numel(), lr, beta1, beta2, eps, weight_decay, _ptr(step_dev), _ptr(bc_dev),
                            grad_scale, _stream()), "dp_adamw_dev", 2)


def adamw_advance(step_dev, bc_dev, beta1, beta2):
    check(_L().dp_adamw_advance(_ptr(step_dev), beta1, beta2, _ptr(bc_dev), _stream()), "dp_adamw_advance")


def adamw_apply(param, grad, exp_avg, exp_avg_sq, param_bf16, lr, beta1, beta2, eps, weight_decay, bc_dev,
                grad_scale=1.0, max_ctas=0, zero_grad=False):
    check(_L().dp_adamw_apply(_ptr(param), _ptr(grad), _ptr(exp_avg), _ptr(exp_avg_sq), _ptr(param_bf16),
                              param.numel(), lr, beta1, beta2, eps, weight_decay, _ptr(bc_dev), grad_scale,
                              max_ctas, int(zero_grad), _stream()), "dp_adamw_apply")


_GN_WS = {}


def _gn_ws(device, nbytes):
    """GroupNorm partial-statistics scratch, one buffer per (device, stream): the forward and backward
    pass statistics between their two kernels through it, so kernels on the fill stream (frozen VAE
    GroupNorms in bubbles) and on the compute stream (U-Net) must never share one. The buffer is
    allocated on (and, when it grows, released to) the pool of the stream that uses it, so the caching
    allocator orders the reuse of a replaced buffer after that stream's pending kernels."""
    key = (device, _stream())
    ws = _GN_WS.get(key)
    if ws is None or ws.numel() * 4 < nbytes:
        ws = torch.empty((nbytes + 3) // 4 + 1024, device=device, dtype=torch.float32)
        _GN_WS[key] = ws
    return ws


def group_norm(x, gamma, beta, G, eps, silu, sums=None):
    """x NHWC [N,H,W,C] (or [N,L,C]); returns y, mean, rstd. sums: the producer's per-(sample, group)
    {sum, sum of squares} (conv2d gn_sums): one pass over x instead of two."""
    N, C = x.shape[0], x.shape[-1]
    HW = x.numel() // (N * C)
    y = torch.empty_like(x)
    mean = torch.empty(N, G, device=x.device, dtype=torch.float32)
    rstd = torch.empty_like(mean)
    if sums is not None:
        check(_L().dp_group_norm_fwd_sums(dtype_code(x), _ptr(x), _ptr(gamma), _ptr(beta), _ptr(y), _ptr(mean),
                                          _ptr(rstd), N, HW, C, G, eps, int(silu), _ptr(sums), _stream()),
              "dp_group_norm_fwd_sums")
        return y, mean, rstd
    ws = _gn_ws(x.device, _L().dp_group_norm_workspace(N, HW, G))
    check(_L().dp_group_norm_fwd(dtype_code(x), _ptr(x), _ptr(gamma), _ptr(beta), _ptr(y), _ptr(mean),
                                 _ptr(rstd), N, HW, C, G, eps, int(silu), _ptr(ws), _stream()),
          "dp_group_norm_fwd", 2)
    return y, mean, rstd


def group_norm_bwd(x, dy, gamma, beta, mean, rstd, G, silu, dgamma=None, dbeta=None, accumulate_into=None):
    """dx of GroupNorm(+SiLU); accumulate_into: add dx into this contiguous tensor in the kernel
    (a second consumer's gradient of x) and return it."""
    N, C = x.shape[0], x.shape[-1]
    HW = x.numel() // (N * C)
    dx = torch.empty_like(x) if accumulate_into is None else accumulate_into
    ws = _gn_ws(x.device, _L().dp_group_norm_workspace(N, HW, G))
    check(_L().dp_group_norm_bwd(dtype_code(x), _ptr(x), _ptr(dy), _ptr(gamma), _ptr(beta), _ptr(mean),
                                 _ptr(rstd), _ptr(dx), _ptr(dgamma), _ptr(dbeta), N, HW, C, G, int(silu),
                                 int(accumulate_into is not None), _ptr(ws), _stream()), "dp_group_norm_bwd", 2)
    return dx


def layer_norm(x, gamma, beta, eps, mod=None, mod_ld=0, shift_off=0, scale_off=0, rows_per_sample=1):
    C = x.shape[-1]
    rows = x.numel() // C
    y = torch.empty_like(x)
    mean = torch.empty(rows, device=x.device, dtype=torch.float32)
    rstd = torch.empty_like(mean)
    check(_L().dp_layer_norm_fwd(dtype_code(x), _ptr(x), _ptr(gamma), _ptr(beta), _ptr(mod), mod_ld,
                                 shift_off, scale_off, rows_per_sample, _ptr(y), _ptr(mean), _ptr(rstd),
                                 rows, C, eps, _stream()), "dp_layer_norm_fwd")
    return y, mean, rstd


def rms_norm(x, gamma, y, eps):
    """T5 RMSNorm forward (frozen encoders): y = x * rsqrt(mean(x^2) + eps) * gamma."""
    C = x.shape[-1]
    check(_L().dp_rms_norm_fwd(dtype_code(x), _ptr(x), _ptr(gamma), _ptr(y), x.numel() // C, C, eps,
                               _stream()), "dp_rms_norm_fwd")
    return y


def layer_norm_bwd(x, dy, gamma, mean, rstd, dgamma=None, dbeta=None, mod=None, mod_ld=0, shift_off=0,
                   scale_off=0, rows_per_sample=1, dmod=None, dmod_ld=0, accumulate_into=None):
    C = x.shape[-1]
    rows = x.numel() // C
    dx = torch.empty_like(x) if accumulate_into is None else accumulate_into
    check(_L().dp_layer_norm_bwd(dtype_code(x), _ptr(x), _ptr(dy), _ptr(gamma), _ptr(mod), mod_ld,
                                 shift_off, scale_off, rows_per_sample, _ptr(mean), _ptr(rstd), _ptr(dx),
                                 _ptr(dgamma), _ptr(dbeta), _ptr(dmod), dmod_ld, rows, C,
                                 int(accumulate_into is not None), _stream()),
          "dp_layer_norm_bwd", 1 + int(gamma is not None and dgamma is not None) + int(mod is not None and dmod is not None))
    return dx


def softmax(S, P, scale, cols, causal=False, Lq=1):
    """S fp32 / P [..., ld] row-major with `cols` valid columns per row."""
    ld = S.shape[-1]
    rows = S.numel() // ld
    check(_L().dp_softmax_fwd(dtype_code(P), _ptr(S), _ptr(P), rows, cols, ld, scale, int(causal), Lq,
                              _stream()), "dp_softmax_fwd")
    return P


def softmax_bwd(P, dP, dS, scale, cols):
    ld = dP.shape[-1]
    rows = dP.numel() // ld
    check(_L().dp_softmax_bwd(dtype_code(P), _ptr(P), _ptr(dP), _ptr(dS), rows, cols, ld, scale, _stream()),
          "dp_softmax_bwd")
    return dS


def row_bias(x, e, rows_per_sample):
    """y = x + e[b] broadcast over the rows of sample b (e [B, >=C] with row stride e.stride(0))."""
    C = x.shape[-1]
    y = torch.empty_like(x)
    check(_L().dp_row_bias_fwd(dtype_code(x), _ptr(x), _ptr(e), e.stride(0), _ptr(y), x.numel() // C, C,
                               rows_per_sample, _stream()), "dp_row_bias_fwd")
    return y


def row_bias_bwd(dy, B, rows_per_sample, db=None, db2=None):
    """de[b] = sum of dy over sample b; with db / db2 (fp32 [C]) also db += sum of dy over all rows and
    db2 += the same (the bias gradients of the layers that produced x and e, from the same per-sample sums)."""
    C = dy.shape[-1]
    de = torch.empty(B, C, device=dy.device, dtype=dy.dtype)
    if db is not None or db2 is not None:
        check(_L().dp_row_bias_bwd_db(dtype_code(dy), _ptr(dy), _ptr(de), C, B, C, rows_per_sample, _ptr(db),
                                      _ptr(db2), _stream()), "dp_row_bias_bwd_db")
        return de
    check(_L().dp_row_bias_bwd(dtype_code(dy), _ptr(dy), _ptr(de), C, B, C, rows_per_sample, _stream()),
          "dp_row_bias_bwd")
    return de


def space_to_depth(x, p, inverse=False):
    """NHWC space-to-depth by p (patch channel order (i, j, c)); inverse = depth-to-space."""
    if not inverse:
        N, H, W, C = x.shape
        out = torch.empty(N, H // p, W // p, p * p * C, device=x.device, dtype=x.dtype)
        Hs, Ws, Cs = H, W, C
    else:
        N, h, w, PC = x.shape
        C = PC // (p * p)
        out = torch.empty(N, h * p, w * p, C, device=x.device, dtype=x.dtype)
        Hs, Ws, Cs = h * p, w * p, C
    check(_L().dp_space_to_depth(dtype_code(x), _ptr(x), _ptr(out), N, Hs, Ws, Cs, p, int(inverse), _stream()),
          "dp_space_to_depth")
    return out


def _attn_args(q, k, v, o, B, N, Nk, heads, q_ld, kv_ld, o_ld, scale, lse):
    a = _lib.DpAttnArgs()
    a.dtype = DP_BF16
    a.B, a.N, a.Nk, a.heads, a.head_dim = B, N, Nk, heads, 64
    a.q, a.k, a.v, a.o = _ptr(q), _ptr(k), _ptr(v), _ptr(o)
    a.q_ld, a.q_bs = q_ld, N * q_ld
    a.kv_ld, a.kv_bs = kv_ld, Nk * kv_ld
    a.o_ld, a.o_bs = o_ld, N * o_ld
    a.scale = scale
    a.lse = _ptr(lse)
    return a


def flash_attn_fwd(q, k, v, o, *, B, N, Nk, heads, q_ld, kv_ld, o_ld, scale, lse=None, causal=False):
    """Fused attention forward (bf16, head dim 64). q/k/v/o are base pointers of
    [B, N(k), heads*64] column views with token strides *_ld (elements). causal (N == Nk, forward
    only): key j > query i masked."""
    a = _attn_args(q, k, v, o, B, N, Nk, heads, q_ld, kv_ld, o_ld, scale, lse)
    a.causal = int(causal)
    flops = 4.0 * B * heads * 64 * (N * (N + 1) / 2 if causal else N * Nk)
    telemetry.timed("tcgen05_gemm", flops,
                    lambda: check(_L().dp_flash_attn_fwd(ctypes.byref(a), _stream()), "dp_flash_attn_fwd"),
                    sub="flash_fwd")
    return o


def _fa_bwd_launches(B, N, Nk, heads):
    """Kernels dp_flash_attn_bwd launches: D prep + backward, the dQ cast unless one key tile
    (dQ stored directly), the dK/dV casts when query tiles are split (mirrors fa_bwd_qsplit)."""
    nkt = -(-Nk // 128)
    split = nkt * heads * B < 2 * 148 and -(-N // 128) >= 2
    return 2 + (0 if nkt == 1 else 1) + (2 if split else 0)


def flash_attn_bwd(q, k, v, o, do, dq, dk, dv, lse, *, B, N, Nk, heads, q_ld, kv_ld, o_ld, do_ld, dq_ld,
                   dkv_ld, scale):
    a = _attn_args(q, k, v, o, B, N, Nk, heads, q_ld, kv_ld, o_ld, scale, lse)
    ws = torch.empty(_L().dp_flash_attn_bwd_workspace(ctypes.byref(a)) // 4, device=o.device, dtype=torch.float32)
    flops = 10.0 * B * heads * N * Nk * 64  # S, dP, dV, dK, dQ recomputation + products
    telemetry.timed("tcgen05_gemm", flops,
                    lambda: check(_L().dp_flash_attn_bwd(ctypes.byref(a), _ptr(do), do_ld, _ptr(dq), dq_ld,
                                                         _ptr(dk), _ptr(dv), dkv_ld, _ptr(ws), _stream()),
                                  "dp_flash_attn_bwd", _fa_bwd_launches(B, N, Nk, heads)), sub="flash_bwd")
