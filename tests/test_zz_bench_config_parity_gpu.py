"""Parity at the BENCHMARKED configuration (VERDICT r1 "next" #1): config c2 exactly as
`bench.py` runs it at N=1 — world batch 32, the full 23-layer OpenCLIP-H text encoder,
cross-iteration filling (has_next=True: each iteration runs the frozen encoders of the NEXT batch),
the optimizer overlapped with the final backward (layer-group AdamW on a side stream, driven by
gradient hooks) and the cached flip-transposed dgrad weights — against the fp32 CPU oracle
(oracle/train_step.py) on identical inputs and initial weights, over 2 iterations.

Compared, with the bf16 tolerances of BASELINE.json north_star (rtol 2e-2):
  * per-iteration loss: |loss - ref| <= 2e-2 |ref|;
  * per-iteration flat gradient (captured per AdamW chunk, before the update): relative L2 < 2e-2;
  * encoder outputs, directly: VAE latents and CLIP context of batch 0 (warm-up pass) and of
    batch 1 (produced by iteration 0's fills / tail): relative L2 < 2e-2, elementwise
    |d| <= 2e-2 |ref| + 2e-2 max|ref| (bf16 activations through 23 transformer layers);
  * post-step parameters after 2 AdamW steps: the update delta (p - p0) against the oracle's,
    cosine similarity > 0.98 and relative L2 < 0.2 (AdamW's m / sqrt(v) amplifies bf16 gradient
    noise on near-zero gradient elements, whose update is ~lr x sign), and the parameters
    themselves elementwise within 2e-2 |ref| + 2 lr.
Also one full-width c3 (512 px ControlNet) and c5 (2.2B U-Net) iteration at world batch 2 with the
same path (has_next, overlap on): loss and per-backbone flat-gradient relative L2.

Each case runs in its own process with a timeout and one retry: full-size iterations with per-slice
gradient snapshots have intermittently hung in a device synchronize (never seen in the bench
or in snapshot-free runs), and a hang must fail this test, not stall the whole -m gpu session."""

import os
import subprocess
import sys

import pytest
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

pytestmark = pytest.mark.gpu
ITERS = 2
LR = 1e-4


def _rel(a, b):
    return ((a - b).norm() / b.norm().clamp_min(1e-30)).item()


def _frozen(tr, ready, n):
    m = tr.ex.frozen_for(ready, 0, n)
    return {k: v.float().cpu() for k, v in m.items()}


def _isolated(*args, timeout=600):
    """Run one case of this file in a fresh process (own CUDA context); retry once after a timeout."""
    cmd = [sys.executable, os.path.abspath(__file__), *args]
    for attempt in range(2):
        try:
            r = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, cwd=ROOT)
        except subprocess.TimeoutExpired:
            print(f"{args}: attempt {attempt} timed out after {timeout} s (killed)")
            continue
        assert r.returncode == 0, (r.stdout[-4000:], r.stderr[-4000:])
        print(r.stdout[-3000:])
        return
    pytest.fail(f"{args}: timed out twice")


def test_c2_bench_config_matches_oracle():
    _isolated("c2")


@pytest.mark.parametrize("cfg", ["c3", "c5"])
def test_full_width_config_iteration_matches_oracle(cfg):
    _isolated(cfg)


def _c2_body():
    from oracle import nets, train_step
    from paper_2405_01248_b200 import diffusion, engine, nn

    wb = 32  # bench.py --per-gpu-batch default, N = 1
    tr = engine.Trainer.create("c2", world=1, rank=0, S=1, M=1, D=1, world_batch=wb)
    assert tr.ex.overlap_sync and nn.FLIP_CACHE
    m = tr.model
    assert len(m.frozen[1].component.layers) >= 23
    tr.ex.grad_snapshots = []
    tr.prefetch(ITERS + 1)  # device-resident batches built before the first step, as bench.py's value pass
    p0 = m.backbone.store.master.detach().float().cpu().clone()
    losses, grads, enc = [], [], []
    for i in range(ITERS):
        loss = tr.step(has_next=True)
        losses.append(loss.item())
        grads.append(tr.ex.take_grad_snapshots()[0])
        if i == 0:
            enc.append(_frozen(tr, tr.ex.frozen_cur, wb))   # batch 0 (warm-up pass)
            enc.append(_frozen(tr, tr.ex.frozen_ready, wb))  # batch 1 (iteration 0's fills / tail)
    assert tr.ex._ovl_top, "overlapped optimizer did not run"
    p1 = m.backbone.store.master.detach().float().cpu()

    torch.set_num_threads(max(1, torch.get_num_threads()))
    params = {c.name: nn.init_state(c.store.param_specs(), 0)
              for c in [m.backbone] + [f.component for f in m.frozen]}
    sab, s1m = diffusion.noise_schedule()
    batches = [diffusion.make_batch(tr.data_spec, i) for i in range(ITERS)]
    ref_losses, ref_grads, ref_params = train_step.train("c2", params, batches, sab, s1m)

    report = []
    for i in range(ITERS):
        assert abs(losses[i] - ref_losses[i]) <= 2e-2 * abs(ref_losses[i]), (i, losses, ref_losses)
        ref_flat = torch.zeros_like(grads[i])
        for p in m.backbone.store.params.values():
            ref_flat[p.offset:p.offset + p.numel] = ref_grads[i][p.name].reshape(-1)
        e = _rel(grads[i], ref_flat)
        report.append(("grad", i, e))
        assert e < 2e-2, report

    # encoder outputs: the oracle's VAE / CLIP on the same batches
    Pv = {k: v.float() for k, v in params["vae"].items()}
    Pt = {k: v.float() for k, v in params["text"].items()}
    for i, got in enumerate(enc):
        b = batches[i] if i < len(batches) else diffusion.make_batch(tr.data_spec, i)
        img = torch.cat([b.images.float(), torch.zeros(*b.images.shape[:-1], 5)], -1)
        with torch.no_grad():
            lat = nets.vae_encoder(Pv, img, ch=128, mult=(1, 2, 4, 4), n_res=2)
            ctx, _ = nets.text_encoder(Pt, b.ids, heads=16, layers=23)
        for name, ref in (("latent", lat), ("ctx", ctx)):
            g = got[name].reshape(ref.shape)
            e = _rel(g, ref)
            report.append((name, i, e))
            assert e < 2e-2, report
            tol = 2e-2 * ref.abs() + 2e-2 * ref.abs().max()
            assert bool(((g - ref).abs() <= tol).all()), (name, i, (g - ref).abs().max().item())

    # post-step parameters
    ref_p = torch.zeros_like(p1)
    for p in m.backbone.store.params.values():
        ref_p[p.offset:p.offset + p.numel] = ref_params[p.name].reshape(-1)
    d_got, d_ref = p1 - p0, ref_p - p0
    cos = (torch.dot(d_got.double(), d_ref.double()) / (d_got.double().norm() * d_ref.double().norm())).item()
    report.append(("update_cos", cos, _rel(d_got, d_ref)))
    assert cos > 0.98 and _rel(d_got, d_ref) < 0.2, report
    # elementwise: AdamW's bias-corrected step is bounded by |m_hat| / sqrt(v_hat) <= 1.0014 at
    # t <= 2 (Cauchy-Schwarz over the EMA weights), so two runs that agree up to bf16 gradient
    # noise can differ by at most 2 steps x 2 runs x 1.0014 lr on elements whose gradient sign
    # flips; everything else must sit inside 2e-2 |ref| + 2 lr, and such flips must be rare
    dev = (p1 - ref_p).abs()
    outside = (dev > 2e-2 * ref_p.abs() + 2 * LR).float().mean().item()
    report.append(("param_outside_2lr_frac", outside, dev.max().item()))
    assert bool((dev <= 2e-2 * ref_p.abs() + 4.01 * LR).all()), report
    assert outside < 1e-2, report
    print("c2 bench-config parity:", report)


_FULL_WIDTH = {"c3": (("controlnet",), dict(clip_layers=23)), "c5": (("unet",), dict(clip_layers=23))}


def _full_width_body(cfg, bb_names, kw):
    from oracle import train_step
    from paper_2405_01248_b200 import diffusion, engine, nn

    tr = engine.Trainer.create(cfg, world=1, rank=0, S=1, M=1, D=1, world_batch=2)
    tr.ex.grad_snapshots = []
    tr.prefetch(2)  # device-resident batches built before the first step, as bench.py's value pass
    batch = diffusion.make_batch(tr.data_spec, 0)
    loss = tr.step(has_next=True).item()
    snaps = tr.ex.take_grad_snapshots()
    assert tr.ex._ovl_top, "overlapped optimizer did not run"
    m = tr.model
    comps = list(m.backbones) + [f.component for f in m.frozen]
    params = {c.name: nn.init_state(c.store.param_specs(), 0) for c in comps}
    sab, s1m = diffusion.noise_schedule()
    torch.set_num_threads(max(1, torch.get_num_threads()))
    ref_loss, ref_grads = train_step.grads_of(cfg, params, batch, sab, s1m, [b.name for b in m.backbones], **kw)
    assert abs(loss - ref_loss) <= 2e-2 * abs(ref_loss), (loss, ref_loss)
    for bi, g in snaps.items():
        bb = m.backbones[bi]
        assert bb.name in bb_names
        ref_flat = torch.zeros_like(g)
        for p in bb.store.params.values():
            ref_flat[p.offset:p.offset + p.numel] = ref_grads[bb.name][p.name].reshape(-1)
        e = _rel(g, ref_flat)
        assert e < 2e-2, (cfg, bb.name, e)


if __name__ == "__main__":
    sys.path.insert(0, ROOT)
    case = sys.argv[1]
    if torch.cuda.is_available():
        torch.backends.cuda.matmul.allow_tf32 = False
        torch.backends.cudnn.allow_tf32 = False
    if case == "c2":
        _c2_body()
    else:
        _full_width_body(case, *_FULL_WIDTH[case])
    print(case, "ok")
