"""Model components of the pipelined diffusion training step, written as
ordered LAYER lists because that is the unit the planner partitions and fills
(reference profile.py:76-130: a component is a list of LayerCost; stages are
contiguous layer ranges, partitioner.py:69-84; fills run whole layers or
partial batches of one layer, filler.py:35-54).

Every layer maps a *live-set* dict of tensors to the next live-set dict. For a
trainable backbone the live set crossing a stage cut is exactly what the
stage-boundary P2P carries (hidden state, U-Net skip stack, conditioning
vectors, frozen context, loss target). Frozen components map their inputs
(images / token ids) to their outputs (latents / context) the same way.

Components:
  TinyDiT, TinyVAEEncoder, TinyTextEncoder   -- config C1 (BASELINE.json configs[0])
  SDUNet, SDVAEEncoder, CLIPTextEncoder      -- config C2 (configs[1], SD v2.1 shapes)
All activations NHWC / [B, L, C]; kernels from nn.py (libdpipe only).
"""

from __future__ import annotations

import math

import torch

from . import nn, ops


def sincos_2d(D, h, w):
    """Fixed 2-D sin-cos position embedding [h*w, D] (DiT's get_2d_sincos_pos_embed)."""
    def one(dim, pos):
        om = torch.arange(dim // 2, dtype=torch.float64) / (dim / 2.0)
        om = 1.0 / 10000 ** om
        out = pos.reshape(-1, 1).double() * om.reshape(1, -1)
        return torch.cat([torch.sin(out), torch.cos(out)], dim=1)
    gy, gx = torch.meshgrid(torch.arange(h, dtype=torch.float64), torch.arange(w, dtype=torch.float64),
                            indexing="ij")
    emb = torch.cat([one(D // 2, gx), one(D // 2, gy)], dim=1)
    return emb.float()


class Component:
    """An ordered list of layers over one flat parameter store."""

    name = "component"

    def __init__(self, dtype, trainable):
        self.dtype = dtype
        self.store = nn.ParamStore(dtype, trainable)
        self.layers = []       # callables state -> state
        self.layer_names = []
        self.layer_prefixes = []

    def add_layer(self, name, fn, prefixes=None):
        self.layer_names.append(name)
        self.layers.append(fn)
        self.layer_prefixes.append(tuple(prefixes) if prefixes is not None else (name,))

    def layer_of_param(self, pname):
        hits = [i for i, prefs in enumerate(self.layer_prefixes)
                if any(pname == p or pname.startswith(p + ".") for p in prefs)]
        if len(hits) != 1:
            raise KeyError(f"parameter {pname} maps to layers {hits} of {self.name}")
        return hits[0]

    def materialize(self, device, seed=0, state=None):
        """Allocate parameters ordered by layer so every stage [lo, hi) owns one contiguous
        slice of the flat master/grad/moment buffers."""
        self.device = torch.device(device)
        self.store.materialize(device, seed, state, order_key=lambda p: self.layer_of_param(p.name))
        self._post_materialize()
        return self

    def stage_slice(self, lo, hi):
        """[start, end) element range of layers [lo, hi) in the flat buffers (per-layer ranges
        are computed once: this is called per layer group on the backward's critical path)."""
        rng = getattr(self, "_layer_rng", None)
        if rng is None:
            rng = {}
            for p in self.store.params.values():
                j = self.layer_of_param(p.name)
                a, b = rng.get(j, (p.offset, p.offset + p.numel))
                rng[j] = (min(a, p.offset), max(b, p.offset + p.numel))
            self._layer_rng = rng
        parts = [rng[j] for j in range(lo, hi) if j in rng]
        if not parts:
            return (0, 0)
        start = min(a for a, _ in parts)
        end = max(b for _, b in parts)
        end = -(-end // nn._ALIGN) * nn._ALIGN
        return (start, end)

    def _post_materialize(self):
        pass

    def run(self, state, lo=0, hi=None):
        hi = len(self.layers) if hi is None else hi
        for fn in self.layers[lo:hi]:
            state = fn(state)
        return state


# ============================================================================ C1: tiny DiT

class TinyDiT(Component):
    """DiT with adaLN-Zero blocks plus cross-attention to the text context.

    Input live set: x [B, H, W, Cin] (x_t concat self-cond estimate), t [B] int64,
    ctx [B, Lt, Dt], pooled [B, Dt], noise [B, H, W, Cout] (loss target).
    Layers: embed, block_0..block_{n-1}, final. Output: state["out"] eps [B, H, W, Cout].
    """

    name = "dit"

    def __init__(self, dtype=torch.float32, img=32, cin=8, cout=4, patch=2, D=256, heads=4, depth=4,
                 ctx_dim=256, freq_dim=256):
        super().__init__(dtype, trainable=True)
        s = self.store
        self.img, self.cin, self.cout, self.patch, self.D, self.heads = img, cin, cout, patch, D, heads
        self.freq_dim = freq_dim
        self.tokens = (img // patch) ** 2
        self.x_embed = nn.Conv2d(s, "x_embed", cin, D, k=patch, stride=patch, pad=(0, 0))
        self.t_mlp1 = nn.Linear(s, "t_embed.mlp1", freq_dim, D)
        self.t_mlp2 = nn.Linear(s, "t_embed.mlp2", D, D)
        self.y_proj = nn.Linear(s, "y_embed", ctx_dim, D)
        self.blocks = []
        for i in range(depth):
            p = f"blocks.{i}"
            blk = dict(
                ada=nn.Linear(s, f"{p}.adaLN", D, 6 * D, init="z"),
                attn=nn.SelfAttention(s, f"{p}.attn", D, heads, qkv_bias=True),
                norm_x=nn.LayerNorm(s, f"{p}.norm_cross", D, eps=1e-6),
                xattn=nn.CrossAttention(s, f"{p}.cross", D, ctx_dim, heads),
                fc1=nn.Linear(s, f"{p}.mlp.fc1", D, 4 * D),
                fc2=nn.Linear(s, f"{p}.mlp.fc2", 4 * D, D),
            )
            self.blocks.append(blk)
        self.final_ada = nn.Linear(s, "final.adaLN", D, 2 * D, init="z")
        self.final_lin = nn.Linear(s, "final.linear", D, patch * patch * cout, init="z")
        self.add_layer("embed", self._embed, ("x_embed", "t_embed", "y_embed"))
        for i in range(depth):
            self.add_layer(f"block_{i}", self._make_block(i), (f"blocks.{i}",))
        self.add_layer("final", self._final, ("final",))

    def _post_materialize(self):
        g = self.img // self.patch
        self.pos = sincos_2d(self.D, g, g).to(self.device, self.dtype).contiguous()

    def _embed(self, st):
        x = st["x"]
        B = x.shape[0]
        h = self.x_embed(x).view(B, self.tokens, self.D)
        h = nn.add_const(h, self.pos)
        temb = self.t_mlp2(nn.silu(self.t_mlp1(ops.timestep_embed(st["t"], self.freq_dim, self.dtype))))
        c = self.y_proj(st["pooled"], residual=temb)
        out = {k: v for k, v in st.items() if k not in ("x", "t", "pooled")}
        out["h"], out["c"] = h, c
        return out

    def _make_block(self, i):
        blk = self.blocks[i]
        D = self.D

        def block(st):
            h, c = st["h"], st["c"]
            mod = blk["ada"](nn.silu(c))  # [B, 6D]: shift1 scale1 gate1 shift2 scale2 gate2
            a = blk["attn"](nn.ln_modulate(h, mod, 0, D))
            h = nn.gate_residual(h, mod, 2 * D, a)
            h = blk["xattn"](blk["norm_x"](h), st["ctx"], residual=h)
            m = blk["fc2"](nn.gelu(blk["fc1"](nn.ln_modulate(h, mod, 3 * D, 4 * D)), tanh=True))
            h = nn.gate_residual(h, mod, 5 * D, m)
            out = dict(st)
            out["h"] = h
            return out

        return block

    def _final(self, st):
        h, c = st["h"], st["c"]
        B = h.shape[0]
        mod = self.final_ada(nn.silu(c))
        y = self.final_lin(nn.ln_modulate(h, mod, 0, self.D))
        g = self.img // self.patch
        eps = nn.depth_to_space(y.view(B, g, g, self.patch * self.patch * self.cout), self.patch)
        out = {k: v for k, v in st.items() if k not in ("h", "c", "ctx")}
        out["out"] = eps
        return out


# ============================================================================ shared blocks

class ResBlock:
    """GN+SiLU -> conv3x3 (+ temb) -> GN+SiLU -> conv3x3 + skip (1x1 when channels change)."""

    def __init__(self, s, p, cin, cout, temb_dim=None, groups=32, eps=1e-6):
        self.n1 = nn.GroupNorm(s, f"{p}.norm1", cin, groups, eps, silu=True)
        self.c1 = nn.Conv2d(s, f"{p}.conv1", cin, cout, 3)
        self.emb = nn.Linear(s, f"{p}.emb_proj", temb_dim, cout) if temb_dim else None
        self.n2 = nn.GroupNorm(s, f"{p}.norm2", cout, groups, eps, silu=True)
        self.c2 = nn.Conv2d(s, f"{p}.conv2", cout, cout, 3, init="z")
        self.skip = nn.Conv2d(s, f"{p}.skip", cin, cout, 1) if cin != cout else None
        # conv1's bias gradient comes from the temb row bias's per-sample sums (no separate pass)
        self.c1.bias_grad_by_row = self.emb is not None and nn.ROW_BIAS_DB
        if self.emb is not None:
            self.emb.bias_grad_by_row = nn.ROW_BIAS_DB  # its bias gradient = sum_b de[b]: the same sums

    def __call__(self, x, temb_act=None):
        hn, x = self.n1.fork(x)  # x's skip-path gradient is accumulated in the GroupNorm backward
        h = self.c1(hn)
        if self.emb is not None:
            by_row = self.c1.bias_grad_by_row
            h = nn.add_row_bias(h, self.emb(temb_act), bias=self.c1.bias if by_row else None,
                                e_bias=self.emb.bias if by_row else None)
        sk = x if self.skip is None else self.skip(x)
        return self.c2(self.n2(h), residual=sk)


class VAEAttn:
    """VAE mid-block single-head spatial self-attention (head dim = C)."""

    def __init__(self, s, p, C, groups=32):
        self.norm = nn.GroupNorm(s, f"{p}.norm", C, groups, 1e-6)
        self.attn = nn.SelfAttention(s, f"{p}.attn", C, 1, qkv_bias=True)

    def __call__(self, x):
        B, H, W, C = x.shape
        h = self.norm(x).view(B, H * W, C)
        return self.attn(h, residual=x.view(B, H * W, C)).view(B, H, W, C)


class VAEEncoderBase(Component):
    """SD-style VAE encoder (frozen): conv_in, per level [ResBlock x n, Downsample],
    mid (Res, Attn, Res), GN+SiLU+conv_out -> posterior mean * scale_factor."""

    name = "vae"

    def __init__(self, dtype, ch, mult, n_res, zc=4, in_ch=3, scale=0.18215, attn_mid=True,
                 pad_in=0):
        super().__init__(dtype, trainable=False)
        s = self.store
        self.zc, self.scale, self.in_ch = zc, scale, in_ch + pad_in
        self.conv_in = nn.Conv2d(s, "conv_in", self.in_ch, ch, 3)
        self.add_layer("conv_in", self._conv_in)
        self._blocks, self._downs = [], []
        cin = ch
        for lvl, m in enumerate(mult):
            cout = ch * m
            for r in range(n_res):
                blk = ResBlock(s, f"down.{lvl}.res.{r}", cin, cout)
                self._blocks.append(blk)
                self.add_layer(f"down.{lvl}.res.{r}", self._res(blk))
                cin = cout
            if lvl != len(mult) - 1:
                ds = nn.Conv2d(s, f"down.{lvl}.downsample", cin, cin, 3, stride=2, asym=True)
                self._downs.append(ds)
                self.add_layer(f"down.{lvl}.downsample", self._conv(ds))
        m1 = ResBlock(s, "mid.res1", cin, cin)
        self._blocks.append(m1)
        self.add_layer("mid.res1", self._res(m1))
        if attn_mid:
            at = VAEAttn(s, "mid.attn", cin)
            self.add_layer("mid.attn", lambda st, at=at: {"h": at(st["h"])})
        m2 = ResBlock(s, "mid.res2", cin, cin)
        self._blocks.append(m2)
        self.add_layer("mid.res2", self._res(m2))
        self.norm_out = nn.GroupNorm(s, "norm_out", cin, 32, 1e-6, silu=True)
        self.conv_out = nn.Conv2d(s, "conv_out", cin, 2 * zc, 3)
        self.add_layer("out", self._out, ("norm_out", "conv_out"))
        self.pad_in = pad_in
        # convs whose output a 32-group GroupNorm reads directly accumulate its statistics in their epilogue:
        # conv_in and the downsamples (the next block's norm1), every block's conv1 (its norm2) and conv2 (the
        # next block's norm1 / the mid attention's norm / norm_out; wasted only before a downsample)
        for cv in [self.conv_in] + self._downs + [c for b in self._blocks for c in (b.c1, b.c2)]:
            cv.gn_stats = 32

    def _conv_in(self, st):
        img = st["images"].to(self.dtype)
        if self.pad_in:
            img = ops.concat_last(img, torch.zeros(*img.shape[:-1], self.pad_in, device=img.device,
                                                   dtype=img.dtype))
        return {"h": self.conv_in(img)}

    @staticmethod
    def _res(blk):
        return lambda st: {"h": blk(st["h"])}

    @staticmethod
    def _conv(cv):
        return lambda st: {"h": cv(st["h"])}

    def _out(self, st):
        y = self.conv_out(self.norm_out(st["h"]))  # [B, h, w, 2 zc] = (mean, logvar)
        mean = torch.empty(*y.shape[:-1], self.zc, device=y.device, dtype=y.dtype)
        ops.split_last(y, self.zc, mean, None)
        return {"latent": ops.axpby(mean, None, alpha=self.scale)}


class TinyVAEEncoder(VAEEncoderBase):
    def __init__(self, dtype=torch.float32):
        super().__init__(dtype, ch=64, mult=(1, 2, 4), n_res=1, zc=4)


class TextEncoderBase(Component):
    """Pre-LN causal transformer text encoder (frozen): token+position embedding,
    `layers` blocks (LN, causal MHA, LN, MLP GELU), final LN -> ctx and mean-pooled."""

    name = "text"

    def __init__(self, dtype, vocab, L, D, heads, layers, mlp=4, gelu_tanh=False):
        super().__init__(dtype, trainable=False)
        s = self.store
        self.L, self.D = L, D
        self.tok = s.add("token_embedding", (vocab, D), init="e")
        self.pos = s.add("position_embedding", (L, D), init="e")
        self.add_layer("embed", lambda st: {"h": ops.embed(st["ids"], self.tok.w, self.pos.w)},
                       ("token_embedding", "position_embedding"))
        for i in range(layers):
            p = f"layers.{i}"
            blk = dict(
                ln1=nn.LayerNorm(s, f"{p}.ln1", D),
                attn=nn.SelfAttention(s, f"{p}.attn", D, heads, qkv_bias=True, causal=True),
                ln2=nn.LayerNorm(s, f"{p}.ln2", D),
                fc1=nn.Linear(s, f"{p}.mlp.fc1", D, mlp * D),
                fc2=nn.Linear(s, f"{p}.mlp.fc2", mlp * D, D),
            )
            self.add_layer(p, self._make_block(blk, gelu_tanh))
        self.ln_final = nn.LayerNorm(s, "ln_final", D)
        self.add_layer("final", self._final, ("ln_final",))

    @staticmethod
    def _make_block(blk, gelu_tanh):
        def block(st):
            h = st["h"]
            h = blk["attn"](blk["ln1"](h), residual=h)
            x = blk["ln2"](h)
            a = nn.gelu(blk["fc1"](x), tanh=True) if gelu_tanh else nn.linear_gelu(x, blk["fc1"])
            h = blk["fc2"](a, residual=h)
            return {"h": h}
        return block

    def _final(self, st):
        ctx = self.ln_final(st["h"])
        B, L, D = ctx.shape
        pooled = ops.axpby(ops.row_bias_bwd(ctx, B, L), None, alpha=1.0 / L)
        return {"ctx": ctx, "pooled": pooled}


class TinyTextEncoder(TextEncoderBase):
    def __init__(self, dtype=torch.float32):
        super().__init__(dtype, vocab=1000, L=16, D=256, heads=4, layers=2)


# ============================================================================ C2: SD v2.1 shapes

class SDVAEEncoder(VAEEncoderBase):
    """SD v2.1 VAE encoder: ch 128, mult (1,2,4,4), 2 ResBlocks per level, z=4.
    The RGB input is zero-padded to 8 channels so conv_in rows are 16-byte aligned."""

    def __init__(self, dtype=torch.bfloat16):
        super().__init__(dtype, ch=128, mult=(1, 2, 4, 4), n_res=2, zc=4, pad_in=5)


class CLIPTextEncoder(TextEncoderBase):
    """OpenCLIP ViT-H/14 text tower as used by SD v2.1 ("penultimate"): 23 of 24
    blocks, width 1024, 16 heads, 77 tokens, GELU MLP, then ln_final."""

    def __init__(self, dtype=torch.bfloat16, layers=23):
        super().__init__(dtype, vocab=49408, L=77, D=1024, heads=16, layers=layers)


class SpatialTransformer:
    """GN -> proj_in (linear) -> [LN, self-attn, LN, cross-attn, LN, GEGLU FF] -> proj_out + x."""

    def __init__(self, s, p, C, ctx_dim, head_dim=64):
        heads = C // head_dim
        self.norm = nn.GroupNorm(s, f"{p}.norm", C, 32, 1e-6)
        self.proj_in = nn.Linear(s, f"{p}.proj_in", C, C)
        self.ln1 = nn.LayerNorm(s, f"{p}.ln1", C)
        self.attn1 = nn.SelfAttention(s, f"{p}.attn1", C, heads)
        self.ln2 = nn.LayerNorm(s, f"{p}.ln2", C)
        self.attn2 = nn.CrossAttention(s, f"{p}.attn2", C, ctx_dim, heads)
        self.ln3 = nn.LayerNorm(s, f"{p}.ln3", C)
        self.ff1 = nn.Linear(s, f"{p}.ff.proj", C, 8 * C)
        self.ff2 = nn.Linear(s, f"{p}.ff.out", 4 * C, C)
        self.proj_out = nn.Linear(s, f"{p}.proj_out", C, C, init="z")

    def __call__(self, x, ctx):
        B, H, W, C = x.shape
        # pre-norm forks: each norm's backward adds into its residual branch's gradient
        xn, x = self.norm.fork(x)
        x2 = x.view(B, H * W, C)
        h = self.proj_in(xn.view(B, H * W, C))
        a, h = self.ln1.fork(h)
        h = self.attn1(a, residual=h)
        a, h = self.ln2.fork(h)
        h = self.attn2(a, ctx, residual=h)
        a, h = self.ln3.fork(h)
        h = nn.feed_forward_geglu(a, self.ff1, self.ff2, residual=h)
        return self.proj_out(h, residual=x2).view(B, H, W, C)


class SDUNet(Component):
    """SD v2.1 U-Net (865M): model_channels 320, mult (1,2,4,4), 2 ResBlocks per level,
    attention at the first three levels (head dim 64, linear proj, depth 1), context 1024.

    Planner layers (26): in.0 (conv_in + time embedding), in.1..in.11 (ResBlock[+Transformer]
    or Downsample), mid, out.0..out.11 (concat skip, ResBlock[+Transformer][+Upsample]), final.
    Live set: h, skips s0..s11 (the not-yet-consumed input-block outputs), temb, ctx, noise.
    """

    name = "unet"

    def __init__(self, dtype=torch.bfloat16, cin=4, cout=4, mc=320, mult=(1, 2, 4, 4), n_res=2,
                 attn_levels=(0, 1, 2), ctx_dim=1024, head_dim=64, trainable=True, name=None):
        super().__init__(dtype, trainable=trainable)
        if name:
            self.name = name
        s = self.store
        self.in_mods, self.out_mods = [], []  # per layer: the modules (reused by ControlNet)
        self.mc = mc
        ted = 4 * mc
        self.ted = ted
        self.t1 = nn.Linear(s, "time_embed.0", mc, ted)
        self.t2 = nn.Linear(s, "time_embed.2", ted, ted)
        self.conv_in = nn.Conv2d(s, "input_blocks.0", cin, mc, 3)
        self.add_layer("in.0", self._in0, ("time_embed", "input_blocks.0"))
        chans = [mc]
        ch = mc
        idx = 1
        for lvl, m in enumerate(mult):
            for r in range(n_res):
                res = ResBlock(s, f"input_blocks.{idx}.res", ch, m * mc, ted, eps=1e-5)
                ch = m * mc
                tr = SpatialTransformer(s, f"input_blocks.{idx}.tr", ch, ctx_dim, head_dim) \
                    if lvl in attn_levels else None
                self.add_layer(f"in.{idx}", self._in_block(res, tr, idx), (f"input_blocks.{idx}",))
                self.in_mods.append(("res", res, tr))
                chans.append(ch)
                idx += 1
            if lvl != len(mult) - 1:
                ds = nn.Conv2d(s, f"input_blocks.{idx}.down", ch, ch, 3, stride=2)
                self.add_layer(f"in.{idx}", self._down(ds, idx), (f"input_blocks.{idx}",))
                self.in_mods.append(("down", ds, None))
                chans.append(ch)
                idx += 1
        self.n_skips = idx
        mres1 = ResBlock(s, "middle.res1", ch, ch, ted, eps=1e-5)
        mtr = SpatialTransformer(s, "middle.tr", ch, ctx_dim, head_dim)
        mres2 = ResBlock(s, "middle.res2", ch, ch, ted, eps=1e-5)
        self.add_layer("mid", self._mid(mres1, mtr, mres2), ("middle",))
        self.mid_mods = (mres1, mtr, mres2)
        self.chans = list(chans)
        oidx = 0
        skip_i = idx - 1
        for lvl, m in list(enumerate(mult))[::-1]:
            for r in range(n_res + 1):
                sc = chans[skip_i]
                res = ResBlock(s, f"output_blocks.{oidx}.res", ch + sc, m * mc, ted, eps=1e-5)
                ch = m * mc
                tr = SpatialTransformer(s, f"output_blocks.{oidx}.tr", ch, ctx_dim, head_dim) \
                    if lvl in attn_levels else None
                up = nn.Conv2d(s, f"output_blocks.{oidx}.up", ch, ch, 3) \
                    if (lvl != 0 and r == n_res) else None
                self.add_layer(f"out.{oidx}", self._out_block(res, tr, up, skip_i),
                               (f"output_blocks.{oidx}",))
                self.out_mods.append((res, tr, up, skip_i))
                skip_i -= 1
                oidx += 1
        self.norm_out = nn.GroupNorm(s, "out.norm", ch, 32, 1e-5, silu=True)
        self.conv_out = nn.Conv2d(s, "out.conv", ch, cout, 3, init="z")
        self.add_layer("final", self._final, ("out",))

    def _in0(self, st):
        # the live set carries SiLU(temb): every ResBlock's embedding projection reads the activated
        # time embedding, so it is computed once here instead of once per block
        temb = nn.silu(self.t2(nn.silu(self.t1(ops.timestep_embed(st["t"], self.mc, self.dtype)))))
        h = self.conv_in(st["x"])
        out = {k: v for k, v in st.items() if k not in ("x", "t", "pooled")}
        out["h"], out["temb"], out["s0"] = h, temb, h
        return out

    @staticmethod
    def _in_block(res, tr, idx):
        def f(st):
            h = res(st["h"], st["temb"])
            if tr is not None:
                h = tr(h, st["ctx"])
            out = dict(st)
            out["h"], out[f"s{idx}"] = h, h
            return out
        return f

    @staticmethod
    def _down(ds, idx):
        def f(st):
            h = ds(st["h"])
            out = dict(st)
            out["h"], out[f"s{idx}"] = h, h
            return out
        return f

    @staticmethod
    def _mid(r1, tr, r2):
        def f(st):
            ta = st["temb"]
            h = r2(tr(r1(st["h"], ta), st["ctx"]), ta)
            out = dict(st)
            out["h"] = h
            return out
        return f

    @staticmethod
    def _out_block(res, tr, up, skip_i):
        def f(st):
            out = {k: v for k, v in st.items() if k != f"s{skip_i}"}
            h = nn.concat(st["h"], st[f"s{skip_i}"])
            h = res(h, st["temb"])
            if tr is not None:
                h = tr(h, st["ctx"])
            if up is not None:
                h = up(nn.upsample2x(h))
            out["h"] = h
            return out
        return f

    def _final(self, st):
        eps = self.conv_out(self.norm_out(st["h"]))
        out = {k: v for k, v in st.items() if k not in ("h", "temb", "ctx")}
        out["out"] = eps
        return out


# ============================================================================ C3: ControlNet v1.0

class HintImage(Component):
    """Frozen pre-processing of the ControlNet condition: the raw hint map -> compute dtype.
    (ControlNet v1.0 trains on hint maps produced by a frozen detector; the synthetic hint is
    already a map, so the detector is the identity here.)"""

    name = "hint"

    def __init__(self, dtype=torch.bfloat16):
        super().__init__(dtype, trainable=False)
        self.add_layer("hint", lambda st: {"hint": ops.cast(st["hint"], self.dtype)}, ())

    def layer_of_param(self, pname):
        return 0


class LockedUNetEncoder:
    """The locked (frozen) SD U-Net's input blocks + middle block as a FROZEN component of the
    ControlNet configuration: it consumes the VAE latent and the text
    context (frozen dependencies vae->enc, text->enc) plus the batch's t and noise,
    and produces the decoder's inputs (skip stack lk_s*, middle output lk_h, time embedding
    lk_temb). It shares its parameter store with the locked decoder inside the backbone."""

    def __init__(self, unet: "SDUNet"):
        self.unet = unet
        self.name = unet.name
        self.store = unet.store
        self.dtype = unet.dtype
        self.sqrt_ab = self.sqrt_1mab = None   # noise-schedule tables (set by the config builder)
        n = unet.n_skips
        self.layers = [self._l0] + [self._block(i) for i in range(1, n)] + [self._mid]
        self.layer_names = ["lk.in.0"] + [f"lk.in.{i}" for i in range(1, n)] + ["lk.mid"]

    def materialize(self, device, seed=0, state=None):
        self.unet.materialize(device, seed, state)
        return self

    def _l0(self, st):
        u = self.unet
        xt = ops.q_sample(st["latent"], st["noise"], st["t"], self.sqrt_ab, self.sqrt_1mab)
        temb = nn.silu(u.t2(nn.silu(u.t1(ops.timestep_embed(st["t"], u.mc, u.dtype)))))  # SiLU(temb), as SDUNet
        h = u.conv_in(xt)
        return {"h": h, "temb": temb, "ctx": st["ctx"], "lk_s0": h}

    def _block(self, i):
        kind, m, tr = self.unet.in_mods[i - 1]

        def f(st):
            if kind == "down":
                h = m(st["h"])
            else:
                h = m(st["h"], st["temb"])
                if tr is not None:
                    h = tr(h, st["ctx"])
            out = dict(st)
            out["h"], out[f"lk_s{i}"] = h, h
            return out
        return f

    def _mid(self, st):
        r1, tr, r2 = self.unet.mid_mods
        ta = st["temb"]
        h = r2(tr(r1(st["h"], ta), st["ctx"]), ta)
        out = {k: v for k, v in st.items() if k.startswith("lk_s")}
        out["lk_h"], out["lk_temb"] = h, st["temb"]
        return out


class ControlNet(Component):
    """ControlNet v1.0 training backbone: the trainable ControlNet branch (hint encoder, a copy
    of the U-Net input blocks + middle block, zero 1x1 convs on every skip and on the middle
    output) followed by the LOCKED SD U-Net decoder (frozen weights: input gradients only, no
    weight gradients) that consumes the locked encoder's frozen outputs plus the ControlNet
    residuals. One backbone chain, per SURVEY Appendix B.2.

    Planner layers: c.in, c.1..c.11, c.mid, lk.out.0..lk.out.11, lk.final (26).
    Live set: ch / ctemb (branch), c0..c11, cmid (residuals), lk_* (locked encoder outputs),
    ctx, noise, then h through the decoder."""

    name = "controlnet"
    HINT = ((3, 16, 1), (16, 16, 1), (16, 32, 2), (32, 32, 1), (32, 96, 2), (96, 96, 1), (96, 256, 2))

    def __init__(self, locked: SDUNet, dtype=torch.bfloat16, cin=4, ctx_dim=1024, head_dim=64,
                 attn_levels=(0, 1, 2), mult=(1, 2, 4, 4), n_res=2):
        super().__init__(dtype, trainable=True)
        s = self.store
        self.locked = locked
        mc = locked.mc
        self.mc = mc
        ted = 4 * mc
        self.t1 = nn.Linear(s, "time_embed.0", mc, ted)
        self.t2 = nn.Linear(s, "time_embed.2", ted, ted)
        self.conv_in = nn.Conv2d(s, "input_blocks.0", cin, mc, 3)
        self.hint = []
        for j, (a, b, st_) in enumerate(self.HINT):
            self.hint.append(nn.Conv2d(s, f"input_hint_block.{2 * j}", a, b, 3, stride=st_))
        self.hint_out = nn.Conv2d(s, f"input_hint_block.{2 * len(self.HINT)}", 256, mc, 3, init="z")
        self.zero = [nn.Conv2d(s, "zero_convs.0", mc, mc, 1, pad=(0, 0), init="z")]
        self.add_layer("c.in", self._cin, ("time_embed", "input_blocks.0", "input_hint_block", "zero_convs.0"))
        ch = mc
        idx = 1
        for lvl, m in enumerate(mult):
            for r in range(n_res):
                res = ResBlock(s, f"input_blocks.{idx}.res", ch, m * mc, ted, eps=1e-5)
                ch = m * mc
                tr = SpatialTransformer(s, f"input_blocks.{idx}.tr", ch, ctx_dim, head_dim) \
                    if lvl in attn_levels else None
                z = nn.Conv2d(s, f"zero_convs.{idx}", ch, ch, 1, pad=(0, 0), init="z")
                self.add_layer(f"c.{idx}", self._cblock(res, tr, z, idx), (f"input_blocks.{idx}", f"zero_convs.{idx}"))
                idx += 1
            if lvl != len(mult) - 1:
                ds = nn.Conv2d(s, f"input_blocks.{idx}.down", ch, ch, 3, stride=2)
                z = nn.Conv2d(s, f"zero_convs.{idx}", ch, ch, 1, pad=(0, 0), init="z")
                self.add_layer(f"c.{idx}", self._cdown(ds, z, idx), (f"input_blocks.{idx}", f"zero_convs.{idx}"))
                idx += 1
        mres1 = ResBlock(s, "middle.res1", ch, ch, ted, eps=1e-5)
        mtr = SpatialTransformer(s, "middle.tr", ch, ctx_dim, head_dim)
        mres2 = ResBlock(s, "middle.res2", ch, ch, ted, eps=1e-5)
        mz = nn.Conv2d(s, "middle_block_out", ch, ch, 1, pad=(0, 0), init="z")
        self.add_layer("c.mid", self._cmid(mres1, mtr, mres2, mz), ("middle", "middle_block_out"))
        for j, (res, tr, up, skip_i) in enumerate(locked.out_mods):
            self.add_layer(f"lk.out.{j}", self._dec(j, res, tr, up, skip_i), ())
        self.add_layer("lk.final", self._final, ())

    def layer_of_param(self, pname):
        return Component.layer_of_param(self, pname)

    def _cin(self, st):
        temb = nn.silu(self.t2(nn.silu(self.t1(ops.timestep_embed(st["t"], self.mc, self.dtype)))))  # SiLU(temb)
        g = st["hint"]
        for cv in self.hint:
            g = nn.silu(cv(g))
        h = self.conv_in(st["x"], residual=self.hint_out(g))
        out = {k: v for k, v in st.items() if k not in ("x", "t", "pooled", "hint")}
        out["ch"], out["ctemb"], out["c0"] = h, temb, self.zero[0](h)
        return out

    @staticmethod
    def _cblock(res, tr, z, idx):
        def f(st):
            h = res(st["ch"], st["ctemb"])
            if tr is not None:
                h = tr(h, st["ctx"])
            out = dict(st)
            out["ch"], out[f"c{idx}"] = h, z(h)
            return out
        return f

    @staticmethod
    def _cdown(ds, z, idx):
        def f(st):
            h = ds(st["ch"])
            out = dict(st)
            out["ch"], out[f"c{idx}"] = h, z(h)
            return out
        return f

    @staticmethod
    def _cmid(r1, tr, r2, z):
        def f(st):
            ta = st["ctemb"]
            h = r2(tr(r1(st["ch"], ta), st["ctx"]), ta)
            out = {k: v for k, v in st.items() if k not in ("ch", "ctemb")}
            out["cmid"] = z(h)
            return out
        return f

    @staticmethod
    def _dec(j, res, tr, up, skip_i):
        def f(st):
            drop = {f"lk_s{skip_i}", f"c{skip_i}"} | ({"lk_h", "cmid"} if j == 0 else set())
            out = {k: v for k, v in st.items() if k not in drop}
            h = nn.add(st["lk_h"], st["cmid"]) if j == 0 else st["h"]
            h = nn.concat(h, nn.add(st[f"lk_s{skip_i}"], st[f"c{skip_i}"]))
            h = res(h, st["lk_temb"])
            if tr is not None:
                h = tr(h, st["ctx"])
            if up is not None:
                h = up(nn.upsample2x(h))
            out["h"] = h
            return out
        return f

    def _final(self, st):
        u = self.locked
        eps = u.conv_out(u.norm_out(st["h"]))
        out = {k: v for k, v in st.items() if k not in ("h", "lk_temb", "ctx")}
        out["out"] = eps
        return out


# ============================================================================ C4: cascaded model

def t5_buckets(L, num_buckets=32, max_distance=128):
    """T5 bidirectional relative-position buckets [L, L] (query i, key j)."""
    ctx = torch.arange(L)[:, None]
    mem = torch.arange(L)[None, :]
    rel = mem - ctx
    nb = num_buckets // 2
    ret = (rel > 0).long() * nb
    n = rel.abs()
    max_exact = nb // 2
    large = max_exact + (torch.log(n.float().clamp(min=1) / max_exact) / math.log(max_distance / max_exact)
                         * (nb - max_exact)).long()
    large = large.clamp(max=nb - 1)
    return ret + torch.where(n < max_exact, n, large)


class T5Encoder(Component):
    """T5 v1.1-large-shaped text encoder (frozen): shared token embedding; per block RMSNorm ->
    self-attention with the relative-position bias of block 0 (no 1/sqrt(d) scaling) ->
    residual, RMSNorm -> gated-GELU FF -> residual; final RMSNorm -> ctx [B, L, D].
    Attention runs as QK^T GEMM with the position bias fused as an fp32 residual (batch stride
    0) in the GEMM epilogue, row softmax, P.V GEMM."""

    name = "t5"

    def __init__(self, dtype=torch.bfloat16, vocab=32128, L=128, D=1024, heads=16, layers=24, ff=2816):
        super().__init__(dtype, trainable=False)
        s = self.store
        self.L, self.D, self.heads, self.ff = L, D, heads, ff
        self.tok = s.add("shared", (vocab, D), init="e")
        self.rel = s.add("rel_bias", (32, heads), fp32=True, init="e")
        self.blocks = []
        for i in range(layers):
            p = f"block.{i}"
            blk = dict(ln1=s.add(f"{p}.ln1.weight", (D,), fp32=True, init="g"),
                       qkv=nn.Linear(s, f"{p}.attn.qkv", D, 3 * D, bias=False),
                       o=nn.Linear(s, f"{p}.attn.o", D, D, bias=False),
                       ln2=s.add(f"{p}.ln2.weight", (D,), fp32=True, init="g"),
                       wi=nn.Linear(s, f"{p}.ff.wi", D, 2 * ff, bias=False),
                       wo=nn.Linear(s, f"{p}.ff.wo", ff, D, bias=False))
            self.blocks.append(blk)
            pre = (p, "shared", "rel_bias") if i == 0 else (p,)
            if i == layers - 1:
                pre = pre + ("final_ln",)
            self.add_layer(p, self._make_block(i, layers), pre)
        self.final_ln = s.add("final_ln.weight", (D,), fp32=True, init="g")

    def _post_materialize(self):
        # the position bias is a function of the frozen table only: expand it once (init time)
        L = self.L
        self.ld = -(-L // 8) * 8
        idx = t5_buckets(L).to(self.rel.w.device)
        bias = torch.zeros(self.heads, L, self.ld, device=self.rel.w.device, dtype=torch.float32)
        bias[:, :, :L] = self.rel.w.float()[idx].permute(2, 0, 1)
        self.pos_bias = bias

    def _rms(self, x, g):
        y = torch.empty_like(x)
        ops.rms_norm(x, g.w, y, 1e-6)
        return y

    def _attn(self, x, blk):
        B, L, D = x.shape
        H, hd, ld = self.heads, D // self.heads, self.ld
        qkv = ops.linear(self._rms(x, blk["ln1"]).view(-1, D), blk["qkv"].weight.w)
        S = torch.empty(B, H, L, ld, device=x.device, dtype=torch.float32)
        ops.gemm(qkv, qkv.view(-1)[D:], S, M=L, N=L, K=hd, a_ld=3 * D, b_ld=3 * D, d_ld=ld, batch=(H, B),
                 a_bs=(hd, L * 3 * D), b_bs=(hd, L * 3 * D), d_bs=(L * ld, H * L * ld),
                 residual=self.pos_bias, r_ld=ld, r_bs=(L * ld, 0))
        P = torch.empty(B, H, L, ld, device=x.device, dtype=x.dtype)
        ops.softmax(S, P, 1.0, L)
        o = torch.empty(B, L, D, device=x.device, dtype=x.dtype)
        ops.gemm(P, qkv.view(-1)[2 * D:], o, M=L, N=hd, K=L, a_ld=ld, b_ld=3 * D, b_mn=True, d_ld=D,
                 batch=(H, B), a_bs=(L * ld, H * L * ld), b_bs=(hd, L * 3 * D), d_bs=(hd, L * D))
        return ops.linear(o.view(-1, D), blk["o"].weight.w, residual=x.view(-1, D)).view(B, L, D)

    def _make_block(self, i, n):
        blk = self.blocks[i]

        def f(st):
            x = ops.embed(st["ids"], self.tok.w) if i == 0 else st["h"]
            B, L, D = x.shape
            x = self._attn(x, blk)
            m = ops.geglu(ops.linear(self._rms(x, blk["ln2"]).view(-1, D), blk["wi"].weight.w))
            x = ops.linear(m, blk["wo"].weight.w, residual=x.view(-1, D)).view(B, L, D)
            if i == n - 1:
                return {"ctx": self._rms(x, self.final_ln)}
            return {"h": x}
        return f


class ImagePyramid(Component):
    """Frozen pre-processing of the cascaded model (CDM): the 256 px image is the x0 of the
    super-resolution pipe ("img_sr"); its 4x4 average pool is the 64 px x0 of the base pipe
    ("latent"); the nearest 4x upsample of that is the SR pipe's low-resolution condition
    ("lowres"). Average pooling = space-to-depth(4) + a constant [3, 48] averaging GEMM."""

    name = "pyramid"

    def __init__(self, dtype=torch.bfloat16, factor=4):
        super().__init__(dtype, trainable=False)
        self.f = factor
        self.add_layer("pool", self._pool, ())
        self.add_layer("lowres", self._lowres, ())

    def layer_of_param(self, pname):
        return 0

    def _post_materialize(self):
        f2 = self.f * self.f
        w = torch.zeros(3, f2 * 3)
        for c in range(3):
            w[c, c::3] = 1.0 / f2
        self.avg_w = w.to(self.device, self.dtype)

    def _pool(self, st):
        img = ops.cast(st["images"], self.dtype)
        B, H, W, _ = img.shape
        sd = ops.space_to_depth(img, self.f)            # [B, H/f, W/f, f*f*3]
        lo = ops.linear(sd.view(-1, sd.shape[-1]), self.avg_w).view(B, H // self.f, W // self.f, 3)
        return {"img_sr": img, "latent": lo}

    def _lowres(self, st):
        up = st["latent"]
        f = self.f
        while f > 1:
            up = ops.upsample2x(up)
            f //= 2
        return {"img_sr": st["img_sr"], "latent": st["latent"], "lowres": up}
