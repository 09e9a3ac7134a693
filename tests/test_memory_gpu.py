"""Memory-feasibility model: the predicted per-device bytes of a plan must track the
measured peak of the same training step on B200 (within the model's stated accuracy)."""

import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("cfg,kw", [("c2", dict(small=True)), ("c1", {})])
def test_predicted_memory_tracks_measured_peak(cfg, kw):
    import gc

    from paper_2405_01248_b200 import engine, memory

    gc.collect()
    torch.cuda.synchronize()
    base = torch.cuda.memory_allocated()
    tr = engine.Trainer.create(cfg, world=1, rank=0, S=1, M=1, D=1, world_batch=8, **kw)
    tr.step()
    torch.cuda.synchronize()
    torch.cuda.reset_peak_memory_stats()
    tr.step()
    torch.cuda.synchronize()
    peak = torch.cuda.max_memory_allocated() - base
    pred = tr.memory_report()[0]
    assert 0.6 * peak < pred < 1.6 * peak, (pred / 2**30, peak / 2**30)
    # the budget check passes for this plan and fails for an absurdly small budget
    memory.check_plan(tr.ex.prog0, tr.model, [[0.0] * len(b.layers) for b in tr.model.backbones])
    with pytest.raises(MemoryError):
        memory.check_plan(tr.ex.prog0, tr.model, [[0.0] * len(b.layers) for b in tr.model.backbones], budget=1)
