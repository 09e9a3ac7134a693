"""CUDA-graph replay of the single-GPU c2 iteration == eager iterations: same losses, and the
same parameter updates up to the nondeterminism of fp32 atomic accumulation (split-K /
stream-K wgrad), which AdamW's sign-like first steps amplify for near-zero gradients."""

import pytest
import torch

pytestmark = pytest.mark.gpu


def test_graph_replay_matches_eager():
    from paper_2405_01248_b200 import engine

    def run(graph):
        tr = engine.Trainer.create("c2", world=1, rank=0, S=1, M=1, D=1, world_batch=4, small=True)
        p0 = tr.model.backbone.store.master.clone()
        losses = [tr.step().item()]
        if graph:
            tr.enable_cuda_graph()
        for _ in range(3):
            losses.append(tr.step().item())
        return losses, tr.model.backbone.store.master.clone() - p0

    le, de = run(False)
    lg, dg = run(True)
    for a, b in zip(le, lg):
        assert abs(a - b) <= 1e-3 * abs(b), (le, lg)
    assert ((de - dg).norm() / de.norm()).item() < 5e-2
