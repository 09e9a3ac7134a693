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


def _q(x0, noise, t, sab, s1m):
    return sab[t][:, None, None, None] * x0 + s1m[t][:, None, None, None] * noise


def c3_forward(P, batch, sab, s1m, clip_layers=23):
    """ControlNet v1.0: frozen VAE / text / hint / locked U-Net encoder;
    the loss trains the ControlNet branch through the locked decoder."""
    img = batch.images.float()
    img = torch.cat([img, torch.zeros(*img.shape[:-1], 5)], -1)
    x0 = nets.vae_encoder(P["vae"], img, ch=128, mult=(1, 2, 4, 4), n_res=2)
    ctx, _ = nets.text_encoder(P["text"], batch.ids, heads=16, layers=clip_layers)
    noise = batch.noise.float()
    xt = _q(x0, noise, batch.t, sab, s1m)
    with torch.no_grad():
        lh, lskips, ltemb = nets.sd_unet_encoder(P["unet_locked"], xt, batch.t, ctx)
    hint = batch.extra["hint"].float()
    eps = nets.controlnet(P["controlnet"], P["unet_locked"], xt, hint, batch.t, ctx, lh, lskips, ltemb)
    loss = ((eps - noise) ** 2).mean()
    return loss, eps, dict(latent=x0, ctx=ctx)


CDM_BASE = dict(mc=192, mult=(1, 2, 3, 4), attn_levels=(1, 2, 3))
CDM_SR = dict(mc=128, mult=(1, 2, 4, 4), attn_levels=(3,))


def c4_forward(P, batch, sab, s1m, t5_layers=24, factor=4):
    """Cascaded model: base (64 px) and super-resolution (256 px, conditioned on the upsampled
    low-res image) U-Nets trained independently on shared frozen outputs;
    self-conditioning on both pipes when the iteration's coin is set; loss = sum of the two
    pipes' mean squared errors. Returns the summed loss (both backbones' params get grads)."""
    img = batch.images.float()
    img_sr, lo, up = nets.image_pyramid(img, factor)
    ctx = nets.t5_encoder(P["t5"], batch.ids, layers=t5_layers)
    t = batch.t
    a = sab[t][:, None, None, None]
    b = s1m[t][:, None, None, None]
    total = 0.0
    outs = []
    for name, x0, noise, cond, kw in (("unet_base", lo, batch.noise.float(), None, CDM_BASE),
                                      ("unet_sr", img_sr, batch.extra["noise_sr"].float(), up, CDM_SR)):
        xt = a * x0 + b * noise
        inp = xt if cond is None else torch.cat([xt, cond], -1)
        if batch.selfcond:
            with torch.no_grad():
                eps_sc = nets.sd_unet(P[name], torch.cat([inp, torch.zeros_like(xt)], -1), t, ctx, **kw)
                x0_sc = (xt - b * eps_sc) / a
        else:
            x0_sc = torch.zeros_like(xt)
        eps = nets.sd_unet(P[name], torch.cat([inp, x0_sc], -1), t, ctx, **kw)
        total = total + ((eps - noise) ** 2).mean()
        outs.append(eps)
    return total, outs, dict(latent=lo, ctx=ctx)


def c5_forward(P, batch, sab, s1m, clip_layers=23):
    """Scaled-up SD U-Net (model channels 512): same training step as c2."""
    img = batch.images.float()
    img = torch.cat([img, torch.zeros(*img.shape[:-1], 5)], -1)
    x0 = nets.vae_encoder(P["vae"], img, ch=128, mult=(1, 2, 4, 4), n_res=2)
    ctx, _ = nets.text_encoder(P["text"], batch.ids, heads=16, layers=clip_layers)
    noise = batch.noise.float()
    xt = _q(x0, noise, batch.t, sab, s1m)
    eps = nets.sd_unet(P["unet"], xt, batch.t, ctx, mc=512)
    loss = ((eps - noise) ** 2).mean()
    return loss, eps, dict(latent=x0, ctx=ctx)


FORWARDS.update({"c3": ("controlnet", c3_forward), "c5": ("unet", c5_forward)})


def grads_of(config, params, batch, sab, s1m, trainable, **kw):
    """Loss and gradients of one iteration (no optimizer state: for the big configs)."""
    fwd = {"c2": c2_forward, "c3": c3_forward, "c4": c4_forward, "c5": c5_forward}[config]
    P = {k: {n: v.detach().clone().float() for n, v in d.items()} for k, d in params.items()}
    for name in trainable:
        for v in P[name].values():
            v.requires_grad_(True)
    loss, _, _ = fwd(P, batch, sab, s1m, **kw)
    loss.backward()
    return loss.item(), {name: {n: v.grad.detach().clone() for n, v in P[name].items()} for name in trainable}
