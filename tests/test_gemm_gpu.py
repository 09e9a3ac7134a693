"""GEMM / implicit-conv kernels vs a plain PyTorch fp32 reference (GPU)."""

import pytest
import torch
import torch.nn.functional as F

pytestmark = pytest.mark.gpu


def _ops():
    from paper_2405_01248_b200 import ops

    return ops


def _rel(a, b):
    return ((a.float() - b.float()).norm() / (b.float().norm() + 1e-12)).item()


@pytest.mark.parametrize("M,N,K", [(128, 64, 64), (300, 200, 136), (1024, 1024, 1024),
                                   (4096, 320, 2880), (77, 1024, 1024), (512, 1280, 5120)])
def test_linear_bf16(M, N, K):
    ops = _ops()
    g = torch.Generator(device="cuda").manual_seed(M * 7 + N)
    x = torch.randn(M, K, device="cuda", generator=g).bfloat16()
    w = torch.randn(N, K, device="cuda", generator=g).bfloat16()
    b = torch.randn(N, device="cuda", generator=g)
    y = ops.linear(x, w, bias=b)
    ref = x.float() @ w.float().t() + b
    assert _rel(y, ref) < 1e-2


@pytest.mark.parametrize("M,N,K", [(256, 192, 320), (300, 200, 136), (2048, 640, 640)])
def test_linear_grads_bf16(M, N, K):
    ops = _ops()
    g = torch.Generator(device="cuda").manual_seed(3)
    x = torch.randn(M, K, device="cuda", generator=g).bfloat16()
    w = torch.randn(N, K, device="cuda", generator=g).bfloat16()
    dy = torch.randn(M, N, device="cuda", generator=g).bfloat16()
    dx = ops.linear_dgrad(dy, w)
    assert _rel(dx, dy.float() @ w.float()) < 1e-2
    dw = torch.zeros(N, K, device="cuda")
    ops.linear_wgrad(dy, x, dw)
    ops.linear_wgrad(dy, x, dw)  # accumulates
    assert _rel(dw, 2 * dy.float().t() @ x.float()) < 1e-2


def test_residual_epilogue():
    ops = _ops()
    x = torch.randn(256, 128, device="cuda").bfloat16()
    w = torch.randn(64, 128, device="cuda").bfloat16()
    r = torch.randn(256, 64, device="cuda").bfloat16()
    y = ops.linear(x, w, residual=r)
    assert _rel(y, x.float() @ w.float().t() + r.float()) < 1e-2


@pytest.mark.parametrize("B,H,N,Nk", [(2, 5, 1024, 1024), (3, 4, 256, 77)])
def test_batched_attention_shapes(B, H, N, Nk):
    ops = _ops()
    C = H * 64
    q = torch.randn(B, N, C, device="cuda").bfloat16()
    k = torch.randn(B, Nk, C, device="cuda").bfloat16()
    v = torch.randn(B, Nk, C, device="cuda").bfloat16()
    s = torch.empty(B, H, N, Nk, device="cuda", dtype=torch.float32)
    # S[b,h] = Q_bh K_bh^T : z1 = head, z2 = batch
    ops.gemm(q, k, s, M=N, N=Nk, K=64, a_ld=C, b_ld=C, d_ld=Nk, batch=(H, B),
             a_bs=(64, N * C), b_bs=(64, Nk * C), d_bs=(N * Nk, H * N * Nk), alpha=0.125)
    qh = q.float().view(B, N, H, 64).transpose(1, 2)
    kh = k.float().view(B, Nk, H, 64).transpose(1, 2)
    vh = v.float().view(B, Nk, H, 64).transpose(1, 2)
    ref = qh @ kh.transpose(-1, -2) * 0.125
    assert _rel(s, ref) < 1e-2
    p = torch.softmax(ref, -1).bfloat16().contiguous()
    o = torch.empty(B, N, C, device="cuda", dtype=torch.bfloat16)
    if Nk % 8 == 0:
        # O[b, n, h*64:] = P_bh V_bh  (V is MN-major: [Nk][64] with row stride C)
        ops.gemm(p, v, o, M=N, N=64, K=Nk, a_ld=Nk, b_ld=C, b_mn=True, d_ld=C, batch=(H, B),
                 a_bs=(N * Nk, H * N * Nk), b_bs=(64, Nk * C), d_bs=(64, N * C))
        ref_o = (p.float() @ vh).transpose(1, 2).reshape(B, N, C)
        assert _rel(o, ref_o) < 1e-2


def test_fp32_simt_gemm():
    ops = _ops()
    x = torch.randn(77, 96, device="cuda")
    w = torch.randn(50, 96, device="cuda")
    y = ops.linear(x, w)
    assert _rel(y, x @ w.t()) < 1e-5
    dw = torch.zeros(50, 96, device="cuda")
    dy = torch.randn(77, 50, device="cuda")
    ops.linear_wgrad(dy, x, dw)
    assert _rel(dw, dy.t() @ x) < 1e-5


def _conv_ref(x, w, stride, pad, out_hw):
    # x NHWC, w KRSC -> NHWC, using explicit asymmetric padding
    N, H, W, C = x.shape
    K, R, S, _ = w.shape
    P, Q = out_hw
    pad_b = (P - 1) * stride + R - H - pad[0]
    pad_r = (Q - 1) * stride + S - W - pad[1]
    xp = F.pad(x.permute(0, 3, 1, 2).float(), (pad[1], max(pad_r, 0), pad[0], max(pad_b, 0)))
    y = F.conv2d(xp, w.permute(0, 3, 1, 2).float(), stride=stride)
    return y[:, :, :P, :Q].permute(0, 2, 3, 1)


@pytest.mark.parametrize("N,H,C,K,stride,pad", [
    (2, 32, 64, 128, 1, (1, 1)),
    (4, 32, 320, 320, 1, (1, 1)),
    (8, 16, 128, 192, 1, (1, 1)),
    (16, 8, 128, 64, 1, (1, 1)),
    (32, 4, 64, 128, 1, (1, 1)),
    (2, 32, 128, 128, 2, (1, 1)),
    (2, 64, 128, 128, 2, (0, 0)),
    (1, 256, 64, 64, 1, (1, 1)),
    (4, 32, 4, 320, 1, (1, 1)),      # U-Net conv_in (channels zero-padded to 64)
    (4, 32, 320, 4, 1, (1, 1)),      # U-Net conv_out (4 filters)
    (2, 64, 8, 128, 1, (1, 1)),      # VAE conv_in (RGB padded to 8)
    (2, 16, 192, 320, 1, (1, 1)),    # C not a multiple of 64
    (4, 16, 640, 640, 1, (1, 1)),    # swapped weight gradient (K % 128 == 0): U-Net 16x16 level
    (3, 8, 1280, 1280, 1, (1, 1)),   # 8x8 level, pairs of BN 256
    (5, 4, 2560, 1280, 1, (1, 1)),   # 4x4 level, 2560-channel concat input
    (2, 16, 640, 640, 2, (1, 1)),    # strided downsample (swapped wgrad with element strides)
])
def test_conv_implicit(N, H, C, K, stride, pad):
    ops = _ops()
    g = torch.Generator(device="cuda").manual_seed(H + C)
    x = torch.randn(N, H, H, C, device="cuda", generator=g).bfloat16()
    w = (torch.randn(K, 3, 3, C, device="cuda", generator=g) * 0.05).bfloat16()
    P = ops.conv_out_size(H, 3, stride, pad[0], 1 if stride == 2 else pad[0])
    out_hw = (P, P)
    y = ops.conv2d(x, w, stride=stride, pad=pad, out_hw=out_hw)
    ref = _conv_ref(x, w, stride, pad, out_hw)
    assert _rel(y, ref) < 1e-2
    # backward
    dy = torch.randn_like(y)
    xr = x.float().permute(0, 3, 1, 2).requires_grad_(True)
    wr = w.float().permute(0, 3, 1, 2).requires_grad_(True)
    pad_b = (P - 1) * stride + 3 - H - pad[0]
    yr = F.conv2d(F.pad(xr, (pad[1], max(pad_b, 0), pad[0], max(pad_b, 0))), wr, stride=stride)
    yr = yr[:, :, :P, :P]
    yr.backward(dy.float().permute(0, 3, 1, 2))
    dx = ops.conv2d_dgrad(dy, w, x.shape, stride=stride, pad=pad)
    assert _rel(dx, xr.grad.permute(0, 2, 3, 1)) < 1e-2
    dw = torch.zeros(K, 3, 3, C, device="cuda")
    ops.conv2d_wgrad(dy, x, dw, stride=stride, pad=pad)
    assert _rel(dw, wr.grad.permute(0, 2, 3, 1)) < 1e-2


def test_conv_small_channels_fp32():
    ops = _ops()
    x = torch.randn(2, 16, 16, 8, device="cuda")
    w = torch.randn(32, 3, 3, 8, device="cuda")
    y = ops.conv2d(x, w, stride=1, pad=(1, 1))
    assert _rel(y, _conv_ref(x, w, 1, (1, 1), (16, 16))) < 1e-5


@pytest.mark.parametrize("M,N,K", [(32, 1280, 1280), (512, 1280, 11520), (200, 640, 2560)])
def test_splitk_bf16_linear(M, N, K):
    """Under-filled bf16 launches take the fp32 split-K / stream-K workspace path (the C ABI
    asks for a workspace) and finish bias + residual in the reduction pass."""
    ops = _ops()
    from paper_2405_01248_b200 import _lib
    import ctypes
    g = torch.Generator(device="cuda").manual_seed(M + N + K)
    x = torch.randn(M, K, device="cuda", generator=g).bfloat16()
    w = torch.randn(N, K, device="cuda", generator=g).bfloat16()
    b = torch.randn(N, device="cuda", generator=g)
    r = torch.randn(M, N, device="cuda", generator=g).bfloat16()
    a = _lib.DpGemmArgs()
    a.M, a.N, a.K, a.batch1, a.batch2, a.dtype = M, N, K, 1, 1, _lib.DP_BF16
    a.A, a.B, a.D = x.data_ptr(), w.data_ptr(), r.data_ptr()
    a.a_ld = a.b_ld = K
    a.d_ld = a.r_ld = N
    a.d_dtype = _lib.DP_BF16
    a.Res = r.data_ptr()
    ws = _lib.lib().dp_gemm_workspace(ctypes.byref(a))
    assert ws in (0, 4 * M * N)
    if M <= 256:  # a handful of tiles: always split
        assert ws == 4 * M * N
    y = ops.linear(x, w, bias=b, residual=r)
    ref = x.float() @ w.float().t() + b + r.float()
    assert _rel(y, ref) < 1e-2


@pytest.mark.parametrize("N,H,C,K", [(32, 4, 1280, 1280), (8, 8, 640, 1280)])
def test_splitk_conv_fwd_dgrad(N, H, C, K):
    ops = _ops()
    g = torch.Generator(device="cuda").manual_seed(H * C)
    x = torch.randn(N, H, H, C, device="cuda", generator=g).bfloat16()
    w = (torch.randn(K, 3, 3, C, device="cuda", generator=g) * 0.05).bfloat16()
    b = torch.randn(K, device="cuda", generator=g)
    r = torch.randn(N, H, H, K, device="cuda", generator=g).bfloat16()
    y = ops.conv2d(x, w, bias=b, residual=r)
    xr = x.float().permute(0, 3, 1, 2)
    wr = w.float().permute(0, 3, 1, 2)
    ref = F.conv2d(xr, wr, b, padding=1).permute(0, 2, 3, 1) + r.float()
    assert _rel(y, ref) < 1e-2
    dy = torch.randn(N, H, H, K, device="cuda", generator=g).bfloat16()
    dx = ops.conv2d_dgrad(dy, w, x.shape)
    ref_dx = torch.nn.grad.conv2d_input(xr.shape, wr, dy.float().permute(0, 3, 1, 2), padding=1)
    assert _rel(dx, ref_dx.permute(0, 2, 3, 1)) < 1e-2


@pytest.mark.parametrize("N,H,W,C,K", [(2, 4, 256, 128, 128), (1, 3, 128, 256, 256), (2, 2, 128, 128, 320),
                                       (1, 5, 384, 64, 192)])
def test_conv_halo_strips(N, H, W, C, K):
    """3x3 stride-1 convs whose 128-pixel tiles lie inside one image row use one input strip per
    filter row (three row-shifted tap views of it): must equal the reference conv."""
    ops = _ops()
    g = torch.Generator(device="cuda").manual_seed(C + K + W)
    x = torch.randn(N, H, W, C, device="cuda", generator=g).bfloat16()
    w = (torch.randn(K, 3, 3, C, device="cuda", generator=g) * 0.05).bfloat16()
    b = torch.randn(K, device="cuda", generator=g)
    y = ops.conv2d(x, w, bias=b)
    ref = F.conv2d(x.float().permute(0, 3, 1, 2), w.float().permute(0, 3, 1, 2), b, padding=1).permute(0, 2, 3, 1)
    assert _rel(y, ref) < 1e-2


@pytest.mark.parametrize("M,N,K", [(4096, 320, 2880), (8192, 640, 2560), (2048, 960, 1280), (512, 320, 4096)])
def test_linear_bn320(M, N, K):
    """N = 320 / 640 / 960 with long K: CTA pairs with two N = 160 MMAs per k-step (BN 320)."""
    ops = _ops()
    g = torch.Generator(device="cuda").manual_seed(M + N)
    x = torch.randn(M, K, device="cuda", generator=g).bfloat16()
    w = torch.randn(N, K, device="cuda", generator=g).bfloat16()
    b = torch.randn(N, device="cuda", generator=g)
    r = torch.randn(M, N, device="cuda", generator=g).bfloat16()
    y = ops.linear(x, w, bias=b, residual=r)
    assert _rel(y, x.float() @ w.float().t() + b + r.float()) < 1e-2


@pytest.mark.parametrize("N,H,C,K", [(8, 32, 320, 320), (8, 16, 640, 640), (4, 32, 640, 320)])
def test_conv_bn320_fwd_dgrad(N, H, C, K):
    ops = _ops()
    g = torch.Generator(device="cuda").manual_seed(C * K)
    x = torch.randn(N, H, H, C, device="cuda", generator=g).bfloat16()
    w = (torch.randn(K, 3, 3, C, device="cuda", generator=g) * 0.05).bfloat16()
    y = ops.conv2d(x, w)
    xr, wr = x.float().permute(0, 3, 1, 2), w.float().permute(0, 3, 1, 2)
    assert _rel(y, F.conv2d(xr, wr, padding=1).permute(0, 2, 3, 1)) < 1e-2
    dy = torch.randn(N, H, H, K, device="cuda", generator=g).bfloat16()
    dx = ops.conv2d_dgrad(dy, w, x.shape)
    ref = torch.nn.grad.conv2d_input(xr.shape, wr, dy.float().permute(0, 3, 1, 2), padding=1)
    assert _rel(dx, ref.permute(0, 2, 3, 1)) < 1e-2


@pytest.mark.parametrize("M,C", [(32768, 320), (8192, 640), (2048, 1280), (300, 320), (1000, 64)])
def test_linear_geglu_epilogue(M, C):
    """ff1 GEMM with the GEGLU epilogue: pre-activation h (bf16, as the unfused GEMM stores it) and
    y = a * gelu(g) from one launch, vs the unfused GEMM + GEGLU kernel and an fp32 torch reference;
    the fused FF layer's gradients vs the unfused layer."""
    ops = _ops()
    g = torch.Generator(device="cuda").manual_seed(M + C)
    x = torch.randn(M, C, device="cuda", generator=g).bfloat16()
    w = (torch.randn(8 * C, C, device="cuda", generator=g) / C ** 0.5).bfloat16()
    b = torch.randn(8 * C, device="cuda", generator=g) * 0.1
    h, y = ops.linear_geglu(x, w, b)
    h_ref = ops.linear(x, w, bias=b)
    y_ref = ops.geglu(h_ref)
    assert _rel(h, h_ref) < 2e-3 and _rel(y, y_ref) < 5e-3
    hf = x.float() @ w.float().t() + b
    yf = hf[:, :4 * C] * F.gelu(hf[:, 4 * C:])
    assert _rel(y, yf) < 1e-2


def test_linear_geglu_layer_grads():
    """The fused FF layer (nn.linear_geglu) against the unfused layer: output and all gradients."""
    from paper_2405_01248_b200 import nn
    torch.manual_seed(0)
    C, M = 320, 4096
    store = nn.ParamStore(torch.bfloat16)
    lin = nn.Linear(store, "ff", C, 8 * C)
    store.materialize("cuda", seed=3)
    x = torch.randn(M, C, device="cuda").bfloat16().requires_grad_(True)
    dy = torch.randn(M, 4 * C, device="cuda").bfloat16()
    outs = []
    for fused in (True, False):
        nn.FUSED_GEGLU = fused
        store.zero_grad()
        xi = x.detach().clone().requires_grad_(True)
        with nn.grad_anchor(device="cuda"):
            y = nn.linear_geglu(xi, lin)
            y.backward(dy)
        outs.append((y.detach().float(), xi.grad.float(), lin.weight.g.clone(), lin.bias.g.clone()))
    nn.FUSED_GEGLU = True
    for a, b in zip(outs[0], outs[1]):
        assert _rel(a, b) < 5e-3


@pytest.mark.parametrize("M,C", [(4096, 320), (2048, 640), (1024, 1280)])
def test_feed_forward_geglu_fused(M, C):
    """The fused feed-forward (ff1 GEGLU epilogue + ff2 dgrad GEGLU-backward epilogue) against the
    layer-by-layer composition: output, input / residual gradients, all four parameter gradients."""
    from paper_2405_01248_b200 import nn
    torch.manual_seed(M + C)
    store = nn.ParamStore(torch.bfloat16)
    ff1 = nn.Linear(store, "ff1", C, 8 * C)
    ff2 = nn.Linear(store, "ff2", 4 * C, C)
    store.materialize("cuda", seed=5)
    x = torch.randn(M, C, device="cuda").bfloat16()
    r = torch.randn(M, C, device="cuda").bfloat16()
    dy = torch.randn(M, C, device="cuda").bfloat16()
    outs = []
    for fused in (True, False):
        nn.FUSED_GEGLU = fused
        store.zero_grad()
        xi = x.clone().requires_grad_(True)
        ri = r.clone().requires_grad_(True)
        with nn.grad_anchor(device="cuda"):
            y = nn.feed_forward_geglu(xi, ff1, ff2, residual=ri)
            y.backward(dy)
        outs.append([y.detach().float(), xi.grad.float(), ri.grad.float(), ff1.weight.g.clone(), ff1.bias.g.clone(),
                     ff2.weight.g.clone(), ff2.bias.g.clone()])
    nn.FUSED_GEGLU = True
    for a, b in zip(outs[0], outs[1]):
        assert _rel(a, b) < 1e-2


def test_flip_batch_matches_single_flips():
    """Batched refresh of the cached dgrad weight copies (one launch for many parameters, more jobs than one
    launch holds) equals the per-parameter flip kernel."""
    ops = _ops()
    from paper_2405_01248_b200 import _lib
    import ctypes
    shapes = [(1280, 1, 1, 320), (320, 3, 3, 640), (640, 3, 3, 640), (64, 1, 1, 8)] * 13
    jobs, refs = [], []
    for i, (K, R, S, C) in enumerate(shapes):
        w = torch.randn(K, R, S, C, device="cuda").bfloat16()
        wt = torch.empty(C, R, S, K, device="cuda", dtype=torch.bfloat16)
        ref = torch.empty_like(wt)
        ops.check(_lib.lib().dp_conv_weight_flip(ops.dtype_code(w), w.data_ptr(), ref.data_ptr(), K, R, S, C,
                                                 ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)), "flip")
        jobs.append((w, wt, K, R, S, C))
        refs.append(ref)
    ops.flip_batch(jobs)
    torch.cuda.synchronize()
    for (w, wt, *_), ref in zip(jobs, refs):
        assert torch.equal(wt, ref)


@pytest.mark.parametrize("N,H,C,K,stride", [(2, 64, 128, 128, 1), (2, 32, 256, 256, 1), (3, 16, 512, 512, 1),
                                            (2, 64, 128, 128, 2), (2, 32, 128, 512, 1)])
def test_conv_groupnorm_statistics_epilogue(N, H, C, K, stride):
    """GroupNorm statistics accumulated by the conv epilogue (VAE convs): the sums match the stored output,
    and the one-pass GroupNorm from them matches the two-pass GroupNorm."""
    ops = _ops()
    g = torch.Generator(device="cuda").manual_seed(H + C + K)
    x = torch.randn(N, H, H, C, device="cuda", generator=g).bfloat16()
    w = (torch.randn(K, 3, 3, C, device="cuda", generator=g) * 0.05).bfloat16()
    b = torch.randn(K, device="cuda", generator=g)
    G = 32
    P = H // stride
    sums = torch.empty(16, N, G, 2, device="cuda")  # DP_GN_SLOTS partial tables
    y = ops.conv2d(x, w, stride=stride, pad=(1, 1), out_hw=(P, P), bias=b, gn_sums=sums, gn_groups=G)
    y_ref = ops.conv2d(x, w, stride=stride, pad=(1, 1), out_hw=(P, P), bias=b)
    assert _rel(y, y_ref) < 1e-2  # (the unfused launch may split K: rounding differs)
    yf = y.float().view(N, P * P, G, K // G)
    ref = torch.stack([yf.sum((1, 3)), (yf * yf).sum((1, 3))], -1)
    assert _rel(sums.sum(0), ref) < 1e-4
    gam = torch.randn(K, device="cuda") * 0.1 + 1
    bet = torch.randn(K, device="cuda") * 0.1
    a1, m1, r1 = ops.group_norm(y, gam, bet, G, 1e-6, True, sums=sums)
    a2, m2, r2 = ops.group_norm(y, gam, bet, G, 1e-6, True)
    assert _rel(m1, m2) < 1e-4 and _rel(r1, r2) < 1e-3 and _rel(a1, a2) < 1e-2


@pytest.mark.parametrize("M,N,K", [(2464, 4096, 1024), (200, 4096, 1024), (300, 384, 136), (1000, 256, 64)])
def test_linear_gelu_epilogue(M, N, K):
    """Frozen-MLP fc1 with GELU (erf) in the GEMM epilogue vs the unfused GEMM + activation kernel and an
    fp32 torch reference; nn.linear_gelu takes the fused path only without autograd."""
    ops = _ops()
    from paper_2405_01248_b200 import nn
    g = torch.Generator(device="cuda").manual_seed(M + N + K)
    x = torch.randn(M, K, device="cuda", generator=g).bfloat16()
    w = (torch.randn(N, K, device="cuda", generator=g) / K ** 0.5).bfloat16()
    b = torch.randn(N, device="cuda", generator=g) * 0.1
    y = ops.linear_gelu(x, w, b)
    y_ref = ops.act(ops.linear(x, w, bias=b), nn.DP_ACT_GELU)
    assert _rel(y, y_ref) < 5e-3
    yf = F.gelu(x.float() @ w.float().t() + b)
    assert _rel(y, yf) < 1e-2
