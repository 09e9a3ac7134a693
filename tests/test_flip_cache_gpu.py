"""Cached flip-transposed dgrad weights (refreshed after each AdamW update on the optimizer stream)
== flipping inside every dgrad, over several c2 training steps: same losses and parameter updates up to
the nondeterminism of fp32 atomic accumulation (stream-K wgrad)."""

import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("cfg", ["c2", "c3"])
def test_flip_cache_matches_uncached(cfg):
    from paper_2405_01248_b200 import engine, nn

    def run(cache):
        old = nn.FLIP_CACHE
        nn.FLIP_CACHE = cache
        try:
            tr = engine.Trainer.create(cfg, world=1, rank=0, S=1, M=1, D=1, world_batch=4, small=True)
            p0 = tr.model.backbones[0].store.master.clone()
            losses = [tr.step().item() for _ in range(4)]
            cached = sum(p.wt is not None for p in tr.model.backbones[0].store.params.values())
            return losses, tr.model.backbones[0].store.master.clone() - p0, cached
        finally:
            nn.FLIP_CACHE = old

    lc, dc, nc = run(True)
    lu, du, nu = run(False)
    assert nc > 0 and nu == 0
    for a, b in zip(lc, lu):
        assert abs(a - b) <= 1e-3 * abs(b), (lc, lu)
    assert ((dc - du).norm() / du.norm()).item() < 5e-2
