"""fp32 CPU restatement of the executor's model components (TEST INFRASTRUCTURE).

Every function takes the flat name -> fp32 tensor parameter dict `P` produced by
paper_2405_01248_b200.nn.init_state / ParamStore.state_dict and recomputes the
component with plain torch.nn.functional ops (no libdpipe). Layouts follow the
executor's canonical ones (NHWC activations, conv weights [K, R, S, C]) and are
converted to torch's NCHW inside each op. Param names mirror networks.py.
"""

from __future__ import annotations

import math

import torch
import torch.nn.functional as F


# ----------------------------------------------------------------------------- primitives

def linear(P, name, x, bias=True):
    y = x @ P[f"{name}.weight"].t()
    if bias and f"{name}.bias" in P:
        y = y + P[f"{name}.bias"]
    return y


def conv(P, name, x, stride=1, pad=None, asym=False):
    w = P[f"{name}.weight"]
    k = w.shape[1]
    xp = x.permute(0, 3, 1, 2)
    if asym:
        xp = F.pad(xp, (0, 1, 0, 1))
        padding = 0
    else:
        padding = k // 2 if pad is None else pad
    y = F.conv2d(xp, w.permute(0, 3, 1, 2), P.get(f"{name}.bias"), stride=stride, padding=padding)
    return y.permute(0, 2, 3, 1)


def group_norm(P, name, x, groups=32, eps=1e-6, silu=False):
    shape = x.shape
    B, C = shape[0], shape[-1]
    xp = x.reshape(B, -1, C).permute(0, 2, 1)
    y = F.group_norm(xp, groups, P[f"{name}.weight"], P[f"{name}.bias"], eps)
    y = y.permute(0, 2, 1).reshape(shape)
    return F.silu(y) if silu else y


def layer_norm(P, name, x, eps=1e-5):
    C = x.shape[-1]
    if name is None:
        return F.layer_norm(x, (C,), None, None, eps)
    return F.layer_norm(x, (C,), P[f"{name}.weight"], P[f"{name}.bias"], eps)


def modulate(x, shift, scale):
    return x * (1 + scale[:, None, :]) + shift[:, None, :]


def mha(q, k, v, heads, causal=False):
    B, N, C = q.shape
    Nk = k.shape[1]
    hd = C // heads
    qh = q.view(B, N, heads, hd).transpose(1, 2)
    kh = k.view(B, Nk, heads, hd).transpose(1, 2)
    vh = v.view(B, Nk, heads, hd).transpose(1, 2)
    s = (qh @ kh.transpose(-1, -2)) / math.sqrt(hd)
    if causal:
        mask = torch.ones(N, Nk, dtype=torch.bool).triu(1)
        s = s.masked_fill(mask, float("-inf"))
    o = torch.softmax(s, -1) @ vh
    return o.transpose(1, 2).reshape(B, N, C)


def self_attention(P, name, x, heads, causal=False):
    C = x.shape[-1]
    qkv = linear(P, f"{name}.qkv", x)
    o = mha(qkv[..., :C], qkv[..., C:2 * C], qkv[..., 2 * C:], heads, causal)
    return linear(P, f"{name}.out", o)


def cross_attention(P, name, x, ctx, heads):
    C = x.shape[-1]
    q = linear(P, f"{name}.q", x)
    kv = linear(P, f"{name}.kv", ctx)
    o = mha(q, kv[..., :C], kv[..., C:], heads)
    return linear(P, f"{name}.out", o)


def timestep_embedding(t, dim, max_period=10000.0):
    half = dim // 2
    k = torch.arange(half, dtype=torch.float32)
    freqs = torch.exp(-math.log(max_period) * k / half)
    args = t.float()[:, None] * freqs[None]
    return torch.cat([torch.cos(args), torch.sin(args)], -1)


def sincos_2d(D, h, w):
    def one(dim, pos):
        om = torch.arange(dim // 2, dtype=torch.float64) / (dim / 2.0)
        om = 1.0 / 10000 ** om
        out = pos.reshape(-1, 1).double() * om.reshape(1, -1)
        return torch.cat([torch.sin(out), torch.cos(out)], dim=1)
    gy, gx = torch.meshgrid(torch.arange(h, dtype=torch.float64), torch.arange(w, dtype=torch.float64),
                            indexing="ij")
    return torch.cat([one(D // 2, gx), one(D // 2, gy)], dim=1).float()


def depth_to_space(y, p):
    B, h, w, PC = y.shape
    C = PC // (p * p)
    return y.view(B, h, w, p, p, C).permute(0, 1, 3, 2, 4, 5).reshape(B, h * p, w * p, C)


# ----------------------------------------------------------------------------- components

def resblock(P, p, x, temb=None, eps=1e-6):
    h = conv(P, f"{p}.conv1", group_norm(P, f"{p}.norm1", x, eps=eps, silu=True))
    if temb is not None:
        h = h + linear(P, f"{p}.emb_proj", F.silu(temb))[:, None, None, :]
    sk = x if f"{p}.skip.weight" not in P else conv(P, f"{p}.skip", x)
    return conv(P, f"{p}.conv2", group_norm(P, f"{p}.norm2", h, eps=eps, silu=True)) + sk


def vae_encoder(P, img, ch, mult, n_res, zc=4, scale=0.18215):
    h = conv(P, "conv_in", img)
    for lvl, m in enumerate(mult):
        for r in range(n_res):
            h = resblock(P, f"down.{lvl}.res.{r}", h)
        if lvl != len(mult) - 1:
            h = conv(P, f"down.{lvl}.downsample", h, stride=2, asym=True)
    h = resblock(P, "mid.res1", h)
    B, H, W, C = h.shape
    a = group_norm(P, "mid.attn.norm", h).reshape(B, H * W, C)
    h = (self_attention(P, "mid.attn.attn", a, 1) + h.reshape(B, H * W, C)).reshape(B, H, W, C)
    h = resblock(P, "mid.res2", h)
    y = conv(P, "conv_out", group_norm(P, "norm_out", h, silu=True))
    return y[..., :zc] * scale


def text_encoder(P, ids, heads, layers, gelu_tanh=False):
    h = P["token_embedding"][ids] + P["position_embedding"][None]
    for i in range(layers):
        p = f"layers.{i}"
        h = self_attention(P, f"{p}.attn", layer_norm(P, f"{p}.ln1", h), heads, causal=True) + h
        m = linear(P, f"{p}.mlp.fc1", layer_norm(P, f"{p}.ln2", h))
        m = F.gelu(m, approximate="tanh" if gelu_tanh else "none")
        h = linear(P, f"{p}.mlp.fc2", m) + h
    ctx = layer_norm(P, "ln_final", h)
    return ctx, ctx.mean(1)


def dit(P, x, t, ctx, pooled, D=256, heads=4, depth=4, patch=2, cout=4, freq_dim=256):
    B, H, W, _ = x.shape
    g = H // patch
    h = conv(P, "x_embed", x, stride=patch, pad=0).reshape(B, g * g, D) + sincos_2d(D, g, g)[None]
    temb = linear(P, "t_embed.mlp2", F.silu(linear(P, "t_embed.mlp1", timestep_embedding(t, freq_dim))))
    c = linear(P, "y_embed", pooled) + temb
    for i in range(depth):
        p = f"blocks.{i}"
        mod = linear(P, f"{p}.adaLN", F.silu(c))
        sh1, sc1, g1, sh2, sc2, g2 = mod.chunk(6, -1)
        a = self_attention(P, f"{p}.attn", modulate(layer_norm(None, None, h, 1e-6), sh1, sc1), heads)
        h = h + g1[:, None, :] * a
        h = cross_attention(P, f"{p}.cross", layer_norm(P, f"{p}.norm_cross", h, 1e-6), ctx, heads) + h
        m = linear(P, f"{p}.mlp.fc1", modulate(layer_norm(None, None, h, 1e-6), sh2, sc2))
        m = linear(P, f"{p}.mlp.fc2", F.gelu(m, approximate="tanh"))
        h = h + g2[:, None, :] * m
    mod = linear(P, "final.adaLN", F.silu(c))
    sh, sc = mod.chunk(2, -1)
    y = linear(P, "final.linear", modulate(layer_norm(None, None, h, 1e-6), sh, sc))
    return depth_to_space(y.reshape(B, g, g, patch * patch * cout), patch)


def spatial_transformer(P, p, x, ctx, head_dim=64):
    B, H, W, C = x.shape
    heads = C // head_dim
    x2 = x.reshape(B, H * W, C)
    h = linear(P, f"{p}.proj_in", group_norm(P, f"{p}.norm", x).reshape(B, H * W, C))
    h = self_attention(P, f"{p}.attn1", layer_norm(P, f"{p}.ln1", h), heads) + h
    h = cross_attention(P, f"{p}.attn2", layer_norm(P, f"{p}.ln2", h), ctx, heads) + h
    a, gt = linear(P, f"{p}.ff.proj", layer_norm(P, f"{p}.ln3", h)).chunk(2, -1)
    h = linear(P, f"{p}.ff.out", a * F.gelu(gt)) + h
    return (linear(P, f"{p}.proj_out", h) + x2).reshape(B, H, W, C)


def sd_unet(P, x, t, ctx, mc=320, mult=(1, 2, 4, 4), n_res=2, attn_levels=(0, 1, 2)):
    temb = linear(P, "time_embed.2", F.silu(linear(P, "time_embed.0", timestep_embedding(t, mc))))
    h = conv(P, "input_blocks.0", x)
    skips = [h]
    idx = 1
    for lvl, m in enumerate(mult):
        for r in range(n_res):
            h = resblock(P, f"input_blocks.{idx}.res", h, temb, eps=1e-5)
            if lvl in attn_levels:
                h = spatial_transformer(P, f"input_blocks.{idx}.tr", h, ctx)
            skips.append(h)
            idx += 1
        if lvl != len(mult) - 1:
            h = conv(P, f"input_blocks.{idx}.down", h, stride=2)
            skips.append(h)
            idx += 1
    h = resblock(P, "middle.res1", h, temb, eps=1e-5)
    h = spatial_transformer(P, "middle.tr", h, ctx)
    h = resblock(P, "middle.res2", h, temb, eps=1e-5)
    oidx = 0
    for lvl, m in list(enumerate(mult))[::-1]:
        for r in range(n_res + 1):
            h = torch.cat([h, skips.pop()], -1)
            h = resblock(P, f"output_blocks.{oidx}.res", h, temb, eps=1e-5)
            if lvl in attn_levels:
                h = spatial_transformer(P, f"output_blocks.{oidx}.tr", h, ctx)
            if lvl != 0 and r == n_res:
                B, H, W, C = h.shape
                h = h[:, :, None, :, None, :].expand(B, H, 2, W, 2, C).reshape(B, 2 * H, 2 * W, C)
                h = conv(P, f"output_blocks.{oidx}.up", h)
            oidx += 1
    return conv(P, "out.conv", group_norm(P, "out.norm", h, eps=1e-5, silu=True))


# ----------------------------------------------------------------------------- C3 / C4 / C5

def sd_unet_encoder(P, x, t, ctx, mc=320, mult=(1, 2, 4, 4), n_res=2, attn_levels=(0, 1, 2)):
    """Input blocks + middle block of sd_unet: returns (h, skips, temb)."""
    temb = linear(P, "time_embed.2", F.silu(linear(P, "time_embed.0", timestep_embedding(t, mc))))
    h = conv(P, "input_blocks.0", x)
    skips = [h]
    idx = 1
    for lvl, m in enumerate(mult):
        for r in range(n_res):
            h = resblock(P, f"input_blocks.{idx}.res", h, temb, eps=1e-5)
            if lvl in attn_levels:
                h = spatial_transformer(P, f"input_blocks.{idx}.tr", h, ctx)
            skips.append(h)
            idx += 1
        if lvl != len(mult) - 1:
            h = conv(P, f"input_blocks.{idx}.down", h, stride=2)
            skips.append(h)
            idx += 1
    h = resblock(P, "middle.res1", h, temb, eps=1e-5)
    h = spatial_transformer(P, "middle.tr", h, ctx)
    h = resblock(P, "middle.res2", h, temb, eps=1e-5)
    return h, skips, temb


def sd_unet_decoder(P, h, skips, temb, ctx, mult=(1, 2, 4, 4), n_res=2, attn_levels=(0, 1, 2)):
    skips = list(skips)
    oidx = 0
    for lvl, m in list(enumerate(mult))[::-1]:
        for r in range(n_res + 1):
            h = torch.cat([h, skips.pop()], -1)
            h = resblock(P, f"output_blocks.{oidx}.res", h, temb, eps=1e-5)
            if lvl in attn_levels:
                h = spatial_transformer(P, f"output_blocks.{oidx}.tr", h, ctx)
            if lvl != 0 and r == n_res:
                B, H, W, C = h.shape
                h = h[:, :, None, :, None, :].expand(B, H, 2, W, 2, C).reshape(B, 2 * H, 2 * W, C)
                h = conv(P, f"output_blocks.{oidx}.up", h)
            oidx += 1
    return conv(P, "out.conv", group_norm(P, "out.norm", h, eps=1e-5, silu=True))


HINT = ((3, 16, 1), (16, 16, 1), (16, 32, 2), (32, 32, 1), (32, 96, 2), (96, 96, 1), (96, 256, 2))


def controlnet(Pc, Pl, x, hint, t, ctx, locked_h, locked_skips, locked_temb, mc=320, mult=(1, 2, 4, 4),
               n_res=2, attn_levels=(0, 1, 2)):
    """ControlNet v1.0 branch (params Pc) + locked SD decoder (params Pl) consuming the locked
    encoder outputs (h, skips, temb) plus the zero-conv residuals."""
    temb = linear(Pc, "time_embed.2", F.silu(linear(Pc, "time_embed.0", timestep_embedding(t, mc))))
    g = hint
    for j, (_, _, s) in enumerate(HINT):
        g = F.silu(conv(Pc, f"input_hint_block.{2 * j}", g, stride=s, pad=1))
    g = conv(Pc, f"input_hint_block.{2 * len(HINT)}", g)
    h = conv(Pc, "input_blocks.0", x) + g
    res = [conv(Pc, "zero_convs.0", h, pad=0)]
    idx = 1
    for lvl, m in enumerate(mult):
        for r in range(n_res):
            h = resblock(Pc, f"input_blocks.{idx}.res", h, temb, eps=1e-5)
            if lvl in attn_levels:
                h = spatial_transformer(Pc, f"input_blocks.{idx}.tr", h, ctx)
            res.append(conv(Pc, f"zero_convs.{idx}", h, pad=0))
            idx += 1
        if lvl != len(mult) - 1:
            h = conv(Pc, f"input_blocks.{idx}.down", h, stride=2)
            res.append(conv(Pc, f"zero_convs.{idx}", h, pad=0))
            idx += 1
    h = resblock(Pc, "middle.res1", h, temb, eps=1e-5)
    h = spatial_transformer(Pc, "middle.tr", h, ctx)
    h = resblock(Pc, "middle.res2", h, temb, eps=1e-5)
    mid = conv(Pc, "middle_block_out", h, pad=0)
    skips = [a + b for a, b in zip(locked_skips, res)]
    return sd_unet_decoder(Pl, locked_h + mid, skips, locked_temb, ctx, mult, n_res, attn_levels)


def t5_buckets(L, num_buckets=32, max_distance=128):
    """T5 bidirectional relative-position bucket of (query i, key j) (HF T5Attention._relative_position_bucket)."""
    rel = torch.arange(L)[None, :] - torch.arange(L)[:, None]
    nb = num_buckets // 2
    ret = (rel > 0).long() * nb
    n = rel.abs()
    max_exact = nb // 2
    large = max_exact + (torch.log(n.float().clamp(min=1) / max_exact) / math.log(max_distance / max_exact)
                         * (nb - max_exact)).long()
    large = large.clamp(max=nb - 1)
    return ret + torch.where(n < max_exact, n, large)


def rms_norm(x, g, eps=1e-6):
    return x * torch.rsqrt((x * x).mean(-1, keepdim=True) + eps) * g


def t5_encoder(P, ids, heads=16, layers=24):
    h = P["shared"][ids]
    B, L, D = h.shape
    hd = D // heads
    bias = P["rel_bias"][t5_buckets(L)].permute(2, 0, 1)[None]  # [1, H, L, L]
    for i in range(layers):
        p = f"block.{i}"
        qkv = rms_norm(h, P[f"{p}.ln1.weight"]) @ P[f"{p}.attn.qkv.weight"].t()
        q, k, v = [a.reshape(B, L, heads, hd).transpose(1, 2) for a in qkv.split(D, -1)]
        s = q @ k.transpose(-1, -2) + bias          # T5: no 1/sqrt(d) scaling
        o = (torch.softmax(s, -1) @ v).transpose(1, 2).reshape(B, L, D)
        h = o @ P[f"{p}.attn.o.weight"].t() + h
        a, gt = (rms_norm(h, P[f"{p}.ln2.weight"]) @ P[f"{p}.ff.wi.weight"].t()).chunk(2, -1)
        h = (a * F.gelu(gt)) @ P[f"{p}.ff.wo.weight"].t() + h
    return rms_norm(h, P["final_ln.weight"])


def image_pyramid(img, f=4):
    """(img_sr, base x0 = f x f average pool, nearest f x upsample of it)."""
    B, H, W, C = img.shape
    lo = img.reshape(B, H // f, f, W // f, f, C).mean((2, 4))
    up = lo[:, :, None, :, None, :].expand(B, H // f, f, W // f, f, C).reshape(B, H, W, C)
    return img, lo, up
