"""A tiny torch-op model with the executor's component interface, for CPU/gloo tests of the
multi-rank control plane (runtime.py + adapter.py): live sets with pass-through grad-carrying
entries (temb, a skip), a self-conditioning input, two frozen components (image and text
encoders). TEST-ONLY: the product runs networks.py components on B200."""

from __future__ import annotations

import math

import torch

from paper_2405_01248_b200.runtime import FrozenSpec, TrainModel

IMG, LAT, ZC, TL, VOCAB, HID = 8, 4, 2, 4, 11, 32


class FlatStore:
    """Parameters as views of one flat leaf tensor; autograd accumulates into flat.grad."""

    def __init__(self, shapes, seed, trainable=True):
        self.shapes = shapes
        self.offsets = {}
        off = 0
        for n, s in shapes.items():
            self.offsets[n] = (off, off + math.prod(s))
            off += math.prod(s)
        g = torch.Generator().manual_seed(seed)
        self.flat = (torch.randn(off, generator=g) * 0.3).requires_grad_(trainable)
        if trainable:
            self.flat.grad = torch.zeros(off)
            self.m = torch.zeros(off)
            self.v = torch.zeros(off)
        self.step = 0
        self.params = {}

    @property
    def grad(self):
        return self.flat.grad

    def w(self, n):
        a, b = self.offsets[n]
        return self.flat[a:b].view(self.shapes[n])

    def zero_grad(self, rng=None):
        lo, hi = rng if rng is not None else (0, self.flat.numel())
        self.flat.grad[lo:hi].zero_()

    def adamw_step(self, lr=1e-2, betas=(0.9, 0.999), eps=1e-8, weight_decay=0.01, grad_scale=1.0, rng=None):
        self.step += 1
        lo, hi = rng if rng is not None else (0, self.flat.numel())
        with torch.no_grad():
            p, g = self.flat[lo:hi], self.flat.grad[lo:hi] * grad_scale
            m, v = self.m[lo:hi], self.v[lo:hi]
            p.mul_(1 - lr * weight_decay)
            m.mul_(betas[0]).add_(g, alpha=1 - betas[0])
            v.mul_(betas[1]).addcmul_(g, g, value=1 - betas[1])
            bc1, bc2 = 1 - betas[0] ** self.step, 1 - betas[1] ** self.step
            p.addcdiv_(m / bc1, (v / bc2).sqrt() + eps, value=-lr)


class Backbone:
    name = "toy_backbone"

    def __init__(self, L=6, selfcond=True, seed=1):
        self.L = L
        cin = 2 * ZC if selfcond else ZC
        shapes = {"w_in": (LAT * LAT * cin, HID), "w_pool": (HID, HID), "w_t": (8, HID)}
        for j in range(1, L - 1):
            shapes[f"w{j}"] = (HID, HID)
        shapes["w_out"] = (HID, LAT * LAT * ZC)
        self.store = FlatStore(shapes, seed)
        self.layers = [self._l0] + [self._mid(j) for j in range(1, L - 1)] + [self._last]
        self.layer_names = [f"l{j}" for j in range(L)]
        # layer -> contiguous parameter slice (the executor's stage_slice contract)
        self._layer_params = {0: ["w_in", "w_pool", "w_t"], L - 1: ["w_out"]}
        for j in range(1, L - 1):
            self._layer_params[j] = [f"w{j}"]

    def stage_slice(self, lo, hi):
        names = [n for j in range(lo, hi) for n in self._layer_params[j]]
        a = min(self.store.offsets[n][0] for n in names)
        b = max(self.store.offsets[n][1] for n in names)
        return (a, b)

    def run(self, st, lo=0, hi=None):
        for fn in self.layers[lo:len(self.layers) if hi is None else hi]:
            st = fn(st)
        return st

    def _l0(self, st):
        s = self.store
        x = st["x"].reshape(st["x"].shape[0], -1)
        freqs = torch.arange(1, 9, dtype=torch.float32)
        temb = torch.sin(st["t"].float()[:, None] * freqs[None] / 100.0) @ s.w("w_t")
        pre = x @ s.w("w_in") + st["pooled"] @ s.w("w_pool") + temb
        if "hint" in st:  # output of a frozen component that depends on two others (ControlNet-like)
            pre = pre + st["hint"]
        h = torch.tanh(pre)
        out = {k: v for k, v in st.items() if k not in ("x", "t", "pooled", "hint")}
        out.update(h=h, temb=temb, s1=h)
        return out

    def _mid(self, j):
        def f(st):
            h = torch.tanh(st["h"] @ self.store.w(f"w{j}") + st["temb"] + st["ctx"].mean(1))
            out = dict(st)
            if j == self.L - 2:
                h = h + out.pop("s1")
            out["h"] = h
            return out
        return f

    def _last(self, st):
        B = st["h"].shape[0]
        eps = (st["h"] @ self.store.w("w_out")).view(B, LAT, LAT, ZC)
        out = {k: v for k, v in st.items() if k not in ("h", "temb", "ctx", "s1")}
        out["out"] = eps
        return out


class _Frozen:
    def __init__(self, name, shapes, layers, seed):
        self.name = name
        self.store = FlatStore(shapes, seed, trainable=False)
        self.layers = layers(self.store)


def _vae(s):
    return [lambda st: {"h": torch.tanh(st["images"].reshape(st["images"].shape[0], -1) @ s.w("v0"))},
            lambda st: {"h": torch.tanh(st["h"] @ s.w("v1"))},
            lambda st: {"latent": (st["h"] @ s.w("v2")).view(-1, LAT, LAT, ZC)}]


def _enc(s):
    return [lambda st: {"e": torch.tanh(st["latent"].reshape(st["latent"].shape[0], -1) @ s.w("e0")
                                        + st["pooled"] @ s.w("e1"))},
            lambda st: {"hint": st["e"] @ s.w("e2")}]


def _text(s):
    return [lambda st: {"e": s.w("emb")[st["ids"]]},
            lambda st: {"ctx": torch.tanh(st["e"] @ s.w("t1")),
                        "pooled": torch.tanh(st["e"] @ s.w("t1")).mean(1) @ s.w("tp")}]


class TorchOps:
    @staticmethod
    def q_sample(x0, noise, t, sab, s1m):
        return sab[t].view(-1, 1, 1, 1) * x0 + s1m[t].view(-1, 1, 1, 1) * noise

    @staticmethod
    def pred_x0(xt, eps, t, sab, s1m):
        return (xt - s1m[t].view(-1, 1, 1, 1) * eps) / sab[t].view(-1, 1, 1, 1)

    @staticmethod
    def mse(pred, target, loss_acc, scale, dpred):
        d = pred - target
        loss_acc += scale * (d * d).sum()
        dpred.copy_(2 * scale * d)

    @staticmethod
    def concat_last(a, b):
        return torch.cat([a, b], -1)


def build(selfcond=True, L=6, deps=False, two=False):
    from paper_2405_01248_b200.diffusion import noise_schedule

    bb = Backbone(L, selfcond)
    bbs = [bb, Backbone(L, selfcond, seed=11)] if two else None
    vae = _Frozen("vae", {"v0": (IMG * IMG * 3, 16), "v1": (16, 16), "v2": (16, LAT * LAT * ZC)}, _vae, 2)
    txt = _Frozen("text", {"emb": (VOCAB, 8), "t1": (8, HID), "tp": (HID, HID)}, _text, 3)
    frozen = [FrozenSpec(vae, ("images",)), FrozenSpec(txt, ("ids",))]
    if deps:
        enc = _Frozen("enc", {"e0": (LAT * LAT * ZC, HID), "e1": (HID, HID), "e2": (HID, HID)}, _enc, 4)
        frozen.append(FrozenSpec(enc, ()))
    sab, s1m = noise_schedule()
    m = TrainModel(bb, frozen, TorchOps, sab, s1m,
                   selfcond_channels=ZC if selfcond else 0,
                   adamw=dict(lr=1e-2, betas=(0.9, 0.999), eps=1e-8, weight_decay=0.01), backbones=bbs)
    m.selfcond_p = 0.5 if selfcond else 0.0
    m.frozen_deps = ((0, 2), (1, 2)) if deps else ()
    return m
