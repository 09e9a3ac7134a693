"""Diffusion-training ingredients shared by the executor and its tests:
the noise schedule (SD's scaled-linear betas, 1000 steps) and the seeded
synthetic batch source (SURVEY.md §8d "Synthetic inputs").

Every random stream is drawn on the CPU from its own torch.Generator so the
executor (any world size, any plan) and the CPU oracle see bit-identical
inputs: seed = ((1000 * config + iteration) * 8 + stream).
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

STREAM_IMAGES, STREAM_IDS, STREAM_T, STREAM_NOISE, STREAM_COIN = range(5)
STREAM_EXTRA0 = 5  # extra fields (ControlNet hint, second-pipe noise) use streams 5, 6, ...


def noise_schedule(T=1000, beta_start=0.00085, beta_end=0.012):
    """Scaled-linear betas (SD): returns fp32 (sqrt(abar), sqrt(1 - abar)) tables of length T."""
    betas = torch.linspace(beta_start ** 0.5, beta_end ** 0.5, T, dtype=torch.float64) ** 2
    abar = torch.cumprod(1.0 - betas, 0)
    return abar.sqrt().float(), (1.0 - abar).sqrt().float()


def _gen(config_id, iteration, stream):
    return torch.Generator().manual_seed(((1000 * config_id + iteration) * 8 + stream) & 0x7FFFFFFF)


@dataclass
class Batch:
    """One world batch (all samples of all DP groups), NHWC fp32 on the host."""

    images: torch.Tensor   # [WB, H, W, 3] ~ U[-1, 1]
    ids: torch.Tensor      # [WB, L] int64 in [0, vocab), last position = EOT (vocab - 1)
    t: torch.Tensor        # [WB] int64 in [0, T)
    noise: torch.Tensor    # [WB, h, w, zc] ~ N(0, 1)
    selfcond: bool         # per-iteration coin shared by all ranks
    extra: dict = None     # config-specific fields: "hint" (ControlNet), "noise_sr" (cascaded SR pipe)

    def slice(self, lo, hi):
        return Batch(self.images[lo:hi], self.ids[lo:hi], self.t[lo:hi], self.noise[lo:hi], self.selfcond,
                     {k: v[lo:hi] for k, v in (self.extra or {}).items()})

    def fields(self):
        return dict(images=self.images, ids=self.ids, t=self.t, noise=self.noise, **(self.extra or {}))


@dataclass(frozen=True)
class DataSpec:
    config_id: int
    world_batch: int
    image: int          # H = W of the RGB input
    latent: int         # h = w of the latent
    zc: int = 4
    text_len: int = 16
    vocab: int = 1000
    T: int = 1000
    selfcond_p: float = 0.0
    # extra per-sample fields: (name, kind, H, C) with kind "bernoulli" (ControlNet hint ~ B(0.1),
    # SURVEY.md §8d) or "noise" (N(0,1), e.g. the super-resolution pipe of a cascaded model)
    extra: tuple = ()


def make_batch(spec: DataSpec, iteration: int) -> Batch:
    WB = spec.world_batch
    g = _gen(spec.config_id, iteration, STREAM_IMAGES)
    images = torch.rand(WB, spec.image, spec.image, 3, generator=g) * 2 - 1
    g = _gen(spec.config_id, iteration, STREAM_IDS)
    ids = torch.randint(0, spec.vocab - 1, (WB, spec.text_len), generator=g)
    ids[:, -1] = spec.vocab - 1
    g = _gen(spec.config_id, iteration, STREAM_T)
    t = torch.randint(0, spec.T, (WB,), generator=g)
    g = _gen(spec.config_id, iteration, STREAM_NOISE)
    noise = torch.randn(WB, spec.latent, spec.latent, spec.zc, generator=g)
    g = _gen(spec.config_id, iteration, STREAM_COIN)
    coin = bool(torch.rand(1, generator=g).item() < spec.selfcond_p)
    extra = {}
    for i, (name, kind, H, C) in enumerate(spec.extra):
        g = _gen(spec.config_id, iteration, STREAM_EXTRA0 + i)
        if kind == "bernoulli":
            extra[name] = (torch.rand(WB, H, H, C, generator=g) < 0.1).float()
        elif kind == "noise":
            extra[name] = torch.randn(WB, H, H, C, generator=g)
        else:
            raise ValueError(kind)
    return Batch(images, ids, t, noise, coin, extra)
