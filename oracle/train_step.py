"""Sequential CPU fp32 oracle of the pipelined diffusion training step (TEST INFRASTRUCTURE).

Semantics: per iteration the frozen
encoders map the batch to latents (VAE posterior mean x 0.18215) and text context;
x_t = sqrt(abar_t) x0 + sqrt(1 - abar_t) eps; with the iteration's self-conditioning
coin, a no-grad forward on [x_t, 0] gives eps_sc and x0_sc = (x_t - sqrt(1-abar) eps_sc)
/ sqrt(abar), else x0_sc = 0; the backbone predicts eps from [x_t, x0_sc]; the loss is
the mean squared error over the whole world batch; AdamW updates the backbone.
Pipelining, bubble filling, partial batches and cross-iteration overlap do not change
this arithmetic — which is exactly what the parity tests check.
"""

from __future__ import annotations

import torch

from . import nets


def c1_forward(P, batch, sab, s1m):
    """Returns (loss, eps_pred, frozen outputs) for config c1 (tiny DiT)."""
    Pd, Pv, Pt = P["dit"], P["vae"], P["text"]
    img = batch.images.float()
    x0 = nets.vae_encoder(Pv, img, ch=64, mult=(1, 2, 4), n_res=1)
    ctx, pooled = nets.text_encoder(Pt, batch.ids, heads=4, layers=2)
    t = batch.t
    a = sab[t][:, None, None, None]
    b = s1m[t][:, None, None, None]
    noise = batch.noise.float()
    xt = a * x0 + b * noise
    if batch.selfcond:
        with torch.no_grad():
            eps_sc = nets.dit(Pd, torch.cat([xt, torch.zeros_like(xt)], -1), t, ctx, pooled)
            x0_sc = (xt - b * eps_sc) / a
    else:
        x0_sc = torch.zeros_like(xt)
    eps = nets.dit(Pd, torch.cat([xt, x0_sc], -1), t, ctx, pooled)
    loss = ((eps - noise) ** 2).mean()
    return loss, eps, dict(latent=x0, ctx=ctx, pooled=pooled)


def c2_forward(P, batch, sab, s1m, clip_layers=23):
    """Config c2 (SD v2.1 U-Net, frozen OpenCLIP-H text + SD VAE encoder, no self-cond)."""
    Pu, Pv, Pt = P["unet"], P["vae"], P["text"]
    img = batch.images.float()
    img = torch.cat([img, torch.zeros(*img.shape[:-1], 5)], -1)  # RGB zero-padded to 8 channels
    x0 = nets.vae_encoder(Pv, img, ch=128, mult=(1, 2, 4, 4), n_res=2)
    ctx, _ = nets.text_encoder(Pt, batch.ids, heads=16, layers=clip_layers)
    t = batch.t
    a = sab[t][:, None, None, None]
    b = s1m[t][:, None, None, None]
    noise = batch.noise.float()
    xt = a * x0 + b * noise
    eps = nets.sd_unet(Pu, xt, t, ctx)
    loss = ((eps - noise) ** 2).mean()
    return loss, eps, dict(latent=x0, ctx=ctx)


FORWARDS = {"c1": ("dit", c1_forward), "c2": ("unet", c2_forward)}


def train(config, params, batches, sab, s1m, adamw=dict(lr=1e-4, betas=(0.9, 0.999), eps=1e-8,
                                                         weight_decay=0.01), **kw):
    """Run len(batches) sequential iterations. params: {backbone|"vae"|"text": {name: fp32}}.
    Returns per-iteration losses, the backbone gradients of every iteration and the final
    backbone parameters."""
    bb, fwd = FORWARDS[config]
    P = {k: {n: v.detach().clone().float() for n, v in d.items()} for k, d in params.items()}
    for v in P[bb].values():
        v.requires_grad_(True)
    opt = torch.optim.AdamW(list(P[bb].values()), **adamw)
    losses, grads = [], []
    for batch in batches:
        opt.zero_grad(set_to_none=False)
        loss, _, _ = fwd(P, batch, sab, s1m, **kw)
        loss.backward()
        losses.append(loss.item())
        grads.append({n: v.grad.detach().clone() for n, v in P[bb].items()})
        opt.step()
    return losses, grads, {n: v.detach().clone() for n, v in P[bb].items()}
