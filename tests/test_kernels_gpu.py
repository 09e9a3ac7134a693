"""libdpipe norm / elementwise / attention / optimizer kernels vs plain PyTorch fp32
references of the same ops (GPU). Tolerances: fp32 1e-5 relative, bf16 2e-2."""

import math

import pytest
import torch
import torch.nn.functional as F

pytestmark = pytest.mark.gpu

DT = [torch.float32, torch.bfloat16]


def _tol(dt):
    return 2e-5 if dt == torch.float32 else 2e-2


def _rel(a, b):
    return ((a.float() - b.float()).norm() / (b.float().norm() + 1e-12)).item()


@pytest.mark.parametrize("dt", DT)
@pytest.mark.parametrize("N,H,C,G,silu", [(2, 16, 64, 32, False), (3, 8, 320, 32, True),
                                          (2, 32, 128, 32, True), (1, 4, 2560, 32, True),
                                          (2, 4, 4096, 32, True), (4, 32, 320, 32, True),
                                          (3, 16, 640, 32, False), (2, 64, 256, 32, True)])
def test_group_norm(dt, N, H, C, G, silu):
    from paper_2405_01248_b200 import ops
    x = (torch.randn(N, H, H, C, device="cuda") * 2 + 0.5).to(dt)
    g = torch.randn(C, device="cuda") * 0.1 + 1
    b = torch.randn(C, device="cuda") * 0.1
    y, mean, rstd = ops.group_norm(x, g, b, G, 1e-6, silu)
    xr = x.float().permute(0, 3, 1, 2).requires_grad_(True)
    gr, br = g.clone().requires_grad_(True), b.clone().requires_grad_(True)
    yr = F.group_norm(xr, G, gr, br, 1e-6)
    if silu:
        yr = F.silu(yr)
    assert _rel(y, yr.permute(0, 2, 3, 1)) < _tol(dt)
    dy = torch.randn_like(y)
    yr.backward(dy.float().permute(0, 3, 1, 2))
    dg = torch.zeros(C, device="cuda")
    db = torch.zeros(C, device="cuda")
    dx = ops.group_norm_bwd(x, dy, g, b, mean, rstd, G, silu, dg, db)
    tol = _tol(dt) * (1 if dt == torch.float32 else 2)
    assert _rel(dx, xr.grad.permute(0, 2, 3, 1)) < tol
    assert _rel(dg, gr.grad) < tol
    assert _rel(db, br.grad) < tol


@pytest.mark.parametrize("dt", DT)
@pytest.mark.parametrize("rows,C", [(77, 1024), (300, 320), (64, 256), (10, 1280), (32768, 320), (8192, 640),
                                    (2048, 1280), (333, 640)])
def test_layer_norm_affine(dt, rows, C):
    from paper_2405_01248_b200 import ops
    x = (torch.randn(rows, C, device="cuda") * 3 - 1).to(dt)
    g = torch.randn(C, device="cuda") * 0.1 + 1
    b = torch.randn(C, device="cuda") * 0.1
    y, mean, rstd = ops.layer_norm(x, g, b, 1e-5)
    xr = x.float().requires_grad_(True)
    gr, br = g.clone().requires_grad_(True), b.clone().requires_grad_(True)
    yr = F.layer_norm(xr, (C,), gr, br, 1e-5)
    assert _rel(y, yr) < _tol(dt)
    dy = torch.randn_like(y)
    yr.backward(dy.float())
    dg = torch.zeros(C, device="cuda")
    db = torch.zeros(C, device="cuda")
    dx = ops.layer_norm_bwd(x, dy, g, mean, rstd, dgamma=dg, dbeta=db)
    assert _rel(dx, xr.grad) < 2 * _tol(dt)
    assert _rel(dg, gr.grad) < 2 * _tol(dt)
    assert _rel(db, br.grad) < 2 * _tol(dt)


@pytest.mark.parametrize("rows,C", [(1000, 320), (257, 640), (99, 1280)])
def test_layer_norm_bwd_accumulate_no_affine(rows, C):
    """Backward accumulated into an existing gradient (norm forks) and the affine-free form (bf16 row groups)."""
    from paper_2405_01248_b200 import ops
    x = (torch.randn(rows, C, device="cuda") * 2 + 0.5).bfloat16()
    y, mean, rstd = ops.layer_norm(x, None, None, 1e-6)
    xr = x.float().requires_grad_(True)
    yr = F.layer_norm(xr, (C,), eps=1e-6)
    assert _rel(y, yr) < _tol(torch.bfloat16)
    dy = torch.randn_like(y)
    yr.backward(dy.float())
    base = torch.randn_like(x)
    acc = base.clone()
    ops.layer_norm_bwd(x, dy, None, mean, rstd, accumulate_into=acc)
    assert _rel(acc, base.float() + xr.grad) < 2 * _tol(torch.bfloat16)


@pytest.mark.parametrize("dt", DT)
def test_layer_norm_modulated(dt):
    from paper_2405_01248_b200 import nn
    B, L, D = 3, 64, 256
    x = torch.randn(B, L, D, device="cuda").to(dt).requires_grad_(True)
    mod = (torch.randn(B, 6 * D, device="cuda") * 0.3).to(dt).requires_grad_(True)
    y = nn.ln_modulate(x, mod, 3 * D, 4 * D)
    xr = x.detach().float().requires_grad_(True)
    mr = mod.detach().float().requires_grad_(True)
    yr = F.layer_norm(xr, (D,), eps=1e-6) * (1 + mr[:, None, 4 * D:5 * D]) + mr[:, None, 3 * D:4 * D]
    assert _rel(y, yr) < _tol(dt)
    dy = torch.randn_like(y)
    y.backward(dy)
    yr.backward(dy.float())
    assert _rel(x.grad, xr.grad) < 2 * _tol(dt)
    assert _rel(mod.grad, mr.grad) < 2 * _tol(dt)


@pytest.mark.parametrize("dt", DT)
@pytest.mark.parametrize("B,N,Nk,C,heads,causal,cross", [(2, 256, 256, 256, 4, False, False),
                                                          (2, 77, 77, 128, 2, True, False),
                                                          (2, 256, 77, 320, 5, False, True),
                                                          (1, 64, 16, 512, 1, False, True)])
def test_attention(dt, B, N, Nk, C, heads, causal, cross):
    from paper_2405_01248_b200 import nn
    if cross:
        q = (torch.randn(B, N, C, device="cuda")).to(dt).requires_grad_(True)
        kv = (torch.randn(B, Nk, 2 * C, device="cuda")).to(dt).requires_grad_(True)
        o = nn.attention(q, kv, heads)
        qr, kvr = q.detach().float().requires_grad_(True), kv.detach().float().requires_grad_(True)
        Q, K, V = qr, kvr[..., :C], kvr[..., C:]
    else:
        q = (torch.randn(B, N, 3 * C, device="cuda")).to(dt).requires_grad_(True)
        o = nn.attention(q, None, heads, causal)
        qr = q.detach().float().requires_grad_(True)
        Q, K, V = qr[..., :C], qr[..., C:2 * C], qr[..., 2 * C:]
    hd = C // heads

    def sp(t, n):
        return t.reshape(B, n, heads, hd).transpose(1, 2)

    ref = F.scaled_dot_product_attention(sp(Q, N), sp(K, Nk), sp(V, Nk), is_causal=causal)
    ref = ref.transpose(1, 2).reshape(B, N, C)
    assert _rel(o, ref) < _tol(dt) * 2
    do = torch.randn_like(o)
    o.backward(do)
    ref.backward(do.float())
    assert _rel(q.grad, qr.grad) < _tol(dt) * 3
    if cross:
        assert _rel(kv.grad, kvr.grad) < _tol(dt) * 3


@pytest.mark.parametrize("dt", DT)
def test_eltwise_family(dt):
    from paper_2405_01248_b200 import nn, ops
    x = torch.randn(4, 33, 64, device="cuda").to(dt).requires_grad_(True)
    for fn, ref in [(nn.silu, F.silu), (lambda t: nn.gelu(t), F.gelu),
                    (lambda t: nn.gelu(t, tanh=True), lambda t: F.gelu(t, approximate="tanh"))]:
        y = fn(x)
        xr = x.detach().float().requires_grad_(True)
        yr = ref(xr)
        assert _rel(y, yr) < _tol(dt)
        dy = torch.randn_like(y)
        x.grad = None
        y.backward(dy)
        yr.backward(dy.float())
        assert _rel(x.grad, xr.grad) < 2 * _tol(dt)
    g = torch.randn(4, 10, 128, device="cuda").to(dt).requires_grad_(True)
    y = nn.geglu(g)
    gr = g.detach().float().requires_grad_(True)
    a, b = gr.chunk(2, -1)
    yr = a * F.gelu(b)
    assert _rel(y, yr) < _tol(dt)
    dy = torch.randn_like(y)
    y.backward(dy)
    yr.backward(dy.float())
    assert _rel(g.grad, gr.grad) < 2 * _tol(dt)
    # per-sample bias and its gradient
    h = torch.randn(3, 8, 8, 64, device="cuda").to(dt).requires_grad_(True)
    e = torch.randn(3, 64, device="cuda").to(dt).requires_grad_(True)
    y = nn.add_row_bias(h, e)
    assert _rel(y, h.float() + e.float()[:, None, None, :]) < _tol(dt)
    y.backward(torch.ones_like(y))
    assert _rel(e.grad, torch.full((3, 64), 64.0, device="cuda")) < _tol(dt)
    # U-Net widths, a one-vector row, and a row of a prime number of 16-byte vectors above 256
    # (no channel-block width in [8, 256] divides it: ADVICE r1, CV = 257 had produced zeros)
    for C in (320, 1280, 8, 257 * (4 if dt == torch.float32 else 8)):
        h = torch.randn(4, 16, 16, C, device="cuda").to(dt).requires_grad_(True)
        e = torch.randn(4, C, device="cuda").to(dt).requires_grad_(True)
        y = nn.add_row_bias(h, e)
        assert _rel(y, h.float() + e.float()[:, None, None, :]) < _tol(dt)
        g = torch.randn_like(y)
        y.backward(g)
        assert _rel(e.grad, g.float().sum((1, 2))) < _tol(dt)
    # space_to_depth round trip
    z = torch.randn(2, 8, 8, 4, device="cuda").to(dt)
    assert torch.equal(ops.space_to_depth(ops.space_to_depth(z, 2), 2, inverse=True), z)
    ref = z.view(2, 4, 2, 4, 2, 4).permute(0, 1, 3, 2, 4, 5).reshape(2, 4, 4, 16)
    assert torch.equal(ops.space_to_depth(z, 2), ref)
    # upsample
    u = torch.randn(2, 4, 4, 64, device="cuda").to(dt)
    up = ops.upsample2x(u)
    assert torch.equal(up, u.repeat_interleave(2, 1).repeat_interleave(2, 2))
    assert _rel(ops.upsample2x_bwd(up), 4 * u.float()) < _tol(dt)
    for C in (64, 3):  # 16-byte channel vectors / scalar path
        u = torch.randn(2, 4, 5, C, device="cuda").to(dt)
        assert torch.equal(ops.upsample2x(u), u.repeat_interleave(2, 1).repeat_interleave(2, 2))
        g = torch.randn(2, 8, 10, C, device="cuda").to(dt)
        ref = g.float().view(2, 4, 2, 5, 2, C).sum((2, 4))
        assert _rel(ops.upsample2x_bwd(g), ref) < _tol(dt)


def test_adamw_matches_torch():
    from paper_2405_01248_b200 import ops
    n = 1000003
    p = torch.randn(n, device="cuda")
    g = torch.randn(n, device="cuda")
    m = torch.zeros(n, device="cuda")
    v = torch.zeros(n, device="cuda")
    pb = torch.empty(n, device="cuda", dtype=torch.bfloat16)
    pr = p.clone().requires_grad_(True)
    opt = torch.optim.AdamW([pr], lr=1e-3, betas=(0.9, 0.999), eps=1e-8, weight_decay=0.01)
    for step in range(1, 4):
        ops.adamw(p, g, m, v, pb, 1e-3, 0.9, 0.999, 1e-8, 0.01, step)
        pr.grad = g.clone()
        opt.step()
    assert _rel(p, pr.detach()) < 1e-6
    assert torch.equal(pb, p.bfloat16())


@pytest.mark.parametrize("dt", DT)
def test_q_sample_mse(dt):
    from paper_2405_01248_b200 import diffusion, ops
    sab, s1m = [t.cuda() for t in diffusion.noise_schedule()]
    x0 = torch.randn(4, 8, 8, 4, device="cuda").to(dt)
    nz = torch.randn_like(x0)
    t = torch.tensor([0, 10, 500, 999], device="cuda")
    xt = ops.q_sample(x0, nz, t, sab, s1m)
    ref = sab[t][:, None, None, None] * x0.float() + s1m[t][:, None, None, None] * nz.float()
    assert _rel(xt, ref) < _tol(dt)
    back = ops.pred_x0(xt, nz, t, sab, s1m)
    assert _rel(back, x0.float()) < 5 * _tol(dt)
    loss = torch.zeros(1, device="cuda")
    dp = torch.empty_like(x0)
    ops.mse(xt, nz, loss, 0.25, dp)
    refl = 0.25 * ((xt.float() - nz.float()) ** 2).sum()
    assert abs(loss.item() - refl.item()) <= 1e-4 * refl.item()
    assert _rel(dp, 0.5 * (xt.float() - nz.float())) < _tol(dt)


@pytest.mark.parametrize("B,N,Nk,C,heads,cross", [(2, 1024, 1024, 320, 5, False), (3, 256, 256, 640, 10, False),
                                                  (2, 64, 64, 1280, 20, False), (4, 16, 16, 1280, 20, False),
                                                  (2, 1024, 77, 320, 5, True), (2, 200, 77, 128, 2, True),
                                                  (1, 300, 300, 128, 2, False)])
def test_flash_attention_vs_torch(B, N, Nk, C, heads, cross):
    """The fused tcgen05 attention (fwd + bwd) vs fp32 PyTorch SDPA."""
    from paper_2405_01248_b200 import nn
    assert nn.FLASH_ATTENTION
    g = torch.Generator(device="cuda").manual_seed(N + Nk)
    if cross:
        q = torch.randn(B, N, C, device="cuda", generator=g).bfloat16().requires_grad_(True)
        kv = torch.randn(B, Nk, 2 * C, device="cuda", generator=g).bfloat16().requires_grad_(True)
        o = nn.attention(q, kv, heads)
        qr, kvr = q.detach().float().requires_grad_(True), kv.detach().float().requires_grad_(True)
        Q, K, V = qr, kvr[..., :C], kvr[..., C:]
    else:
        q = torch.randn(B, N, 3 * C, device="cuda", generator=g).bfloat16().requires_grad_(True)
        o = nn.attention(q, None, heads)
        qr = q.detach().float().requires_grad_(True)
        Q, K, V = qr[..., :C], qr[..., C:2 * C], qr[..., 2 * C:]

    def sp(t, n):
        return t.reshape(B, n, heads, 64).transpose(1, 2)

    ref = F.scaled_dot_product_attention(sp(Q, N), sp(K, Nk), sp(V, Nk)).transpose(1, 2).reshape(B, N, C)
    assert _rel(o, ref) < 2e-2
    do = torch.randn_like(o)
    o.backward(do)
    ref.backward(do.float())
    assert _rel(q.grad, qr.grad) < 3e-2
    if cross:
        assert _rel(kv.grad, kvr.grad) < 3e-2


@pytest.mark.parametrize("N,ramp", [(1024, 6.0), (4096, 3.0), (1000, 12.0)])
def test_flash_attention_growing_max(N, ramp):
    """Keys whose norm grows along the sequence: the running row max rises by far more than the forward's
    lazy-rescale threshold (2^8) across key tiles, so the O-in-TMEM rescale path runs; also the 4096-token
    (512 px level-0) shape. Forward and backward vs fp32 PyTorch SDPA."""
    from paper_2405_01248_b200 import nn
    B, C, heads = 1, 128, 2
    g = torch.Generator(device="cuda").manual_seed(N)
    base = torch.randn(B, N, 3 * C, device="cuda", generator=g)
    gain = 1.0 + ramp * torch.arange(N, device="cuda", dtype=torch.float32) / N
    base[..., C:2 * C] *= gain[None, :, None]
    base[..., :C] *= 2.0
    q = base.bfloat16().requires_grad_(True)
    o = nn.attention(q, None, heads)
    qr = q.detach().float().requires_grad_(True)
    Q, K, V = (qr[..., i * C:(i + 1) * C].reshape(B, N, heads, 64).transpose(1, 2) for i in range(3))
    ref = F.scaled_dot_product_attention(Q, K, V).transpose(1, 2).reshape(B, N, C)
    assert _rel(o, ref) < 2e-2
    do = torch.randn_like(o)
    o.backward(do)
    ref.backward(do.float())
    assert _rel(q.grad, qr.grad) < 3e-2


@pytest.mark.parametrize("B,N,C,heads", [(4, 77, 1024, 16), (2, 300, 128, 2), (1, 1024, 320, 5)])
def test_flash_attention_causal_forward(B, N, C, heads):
    """Causal fused forward (frozen CLIP text encoder: no gradient) vs fp32 PyTorch SDPA."""
    from paper_2405_01248_b200 import nn
    g = torch.Generator(device="cuda").manual_seed(N)
    q = torch.randn(B, N, 3 * C, device="cuda", generator=g).bfloat16()
    with torch.no_grad():
        o = nn.attention(q, None, heads, True)
    Q, K, V = (q.float()[..., i * C:(i + 1) * C].reshape(B, N, heads, 64).transpose(1, 2) for i in range(3))
    ref = F.scaled_dot_product_attention(Q, K, V, is_causal=True).transpose(1, 2).reshape(B, N, C)
    assert _rel(o, ref) < 2e-2


@pytest.mark.parametrize("dt", DT)
@pytest.mark.parametrize("rows,C", [(32768, 320), (8192, 640), (2048, 1280), (512, 2560), (100, 8), (77, 1024)])
def test_bias_grad(dt, rows, C):
    """db += column sums of dy (bias gradients of linears / convs) vs fp32 torch."""
    from paper_2405_01248_b200 import ops
    dy = torch.randn(rows, C, device="cuda").to(dt)
    db = torch.randn(C, device="cuda")
    ref = db + dy.float().sum(0)
    ops.bias_grad(dy, db)
    assert _rel(db, ref) < 1e-4


@pytest.mark.parametrize("dt", DT)
@pytest.mark.parametrize("Ca,Cb,zeros", [(3, 5, True), (4, 60, True), (4, 4, False), (320, 320, False),
                                         (5, 6, False)])
def test_concat_last(dt, Ca, Cb, zeros):
    """Channel concat (U-Net skips, self-conditioning input, zero channel padding) vs torch.cat."""
    from paper_2405_01248_b200 import ops
    a = torch.randn(7, 9, Ca, device="cuda").to(dt)
    b = None if zeros else torch.randn(7, 9, Cb, device="cuda").to(dt)
    out = ops.concat_last(a, b, Cb)
    ref = torch.cat([a, torch.zeros(7, 9, Cb, device="cuda", dtype=dt) if zeros else b], -1)
    assert torch.equal(out, ref)


@pytest.mark.parametrize("dt", DT)
@pytest.mark.parametrize("rows,F", [(32768, 1280), (8192, 2560), (2048, 5120), (512, 5120), (100, 64), (77, 40)])
def test_geglu_bwd_bias_fused(dt, rows, F):
    """GEGLU backward with the FF input projection's bias gradient fused (db += column sums of dx) vs
    fp32 torch autograd; dx identical to the unfused kernel."""
    from paper_2405_01248_b200 import ops
    g = torch.Generator(device="cuda").manual_seed(rows + F)
    x = torch.randn(rows, 2 * F, device="cuda", generator=g).to(dt)
    dy = torch.randn(rows, F, device="cuda", generator=g).to(dt)
    db0 = torch.randn(2 * F, device="cuda", generator=g)
    db = db0.clone()
    dx = ops.geglu_bwd(x, dy, db=db)
    assert torch.equal(dx, ops.geglu_bwd(x, dy))
    xr = x.float().requires_grad_(True)
    a, gg = xr[:, :F], xr[:, F:]
    (a * torch.nn.functional.gelu(gg)).backward(dy.float())
    tol = 1e-4 if dt == torch.float32 else 2e-2
    assert _rel(dx, xr.grad) < tol
    assert _rel(db - db0, dx.float().sum(0)) < 1e-4


@pytest.mark.parametrize("dt", DT)
@pytest.mark.parametrize("B,rps,C", [(32, 1024, 320), (32, 256, 640), (32, 64, 1280), (32, 16, 1280), (3, 7, 12),
                                     (2, 5, 2056)])
def test_row_bias_bwd_conv_bias(dt, B, rps, C):
    """Per-sample row-bias backward that also accumulates the producing conv's bias gradient
    (db += sum of dy over all rows) vs fp32 torch; de identical to the plain kernel."""
    from paper_2405_01248_b200 import ops
    g = torch.Generator(device="cuda").manual_seed(B * rps + C)
    dy = torch.randn(B * rps, C, device="cuda", generator=g).to(dt)
    db0 = torch.randn(C, device="cuda", generator=g)
    db = db0.clone()
    db2 = -db0
    de = ops.row_bias_bwd(dy, B, rps, db=db, db2=db2)
    assert torch.equal(de, ops.row_bias_bwd(dy, B, rps))
    assert _rel(de, dy.float().view(B, rps, C).sum(1)) < (1e-5 if dt == torch.float32 else 1e-2)
    assert _rel(db - db0, dy.float().sum(0)) < 1e-4
    assert _rel(db2 + db0, dy.float().sum(0)) < 1e-4  # the temb projection's bias gradient (same sums)
