"""The numerics oracle's text encoders pinned to transformers' CLIPTextModel / T5EncoderModel
(tests/golden/make_encoder_golden.py documents the weight mapping). Two legs:
  * the committed fixtures (HF outputs generated here with transformers 5.5.0), always;
  * a live comparison against transformers when it is importable.
The U-Net, VAE, ControlNet and DiT restatements cannot be pinned this way: diffusers / open_clip
are not available offline."""

import os

import pytest
import torch

from oracle import nets

HERE = os.path.dirname(os.path.abspath(__file__))
FIX = os.path.join(HERE, "golden", "encoder_cases.pt")
RTOL = 1e-5


def _run(case):
    c, P, ids = case["cfg"], case["P"], case["ids"]
    if case["kind"] == "clip":
        ctx, _ = nets.text_encoder(P, ids, c["heads"], c["layers"])
        return ctx
    return nets.t5_encoder(P, ids, heads=c["heads"], layers=c["layers"])


def _check(case):
    with torch.no_grad():
        got = _run(case)
    ref = case["out"]
    assert got.shape == ref.shape
    err = (got - ref).abs().max().item()
    assert err <= RTOL * ref.abs().max().item() + 1e-6, (case["kind"], case["cfg"], err)


def test_encoder_fixtures_match_oracle():
    data = torch.load(FIX, weights_only=False)
    kinds = [c["kind"] for c in data["cases"]]
    assert kinds.count("clip") >= 2 and kinds.count("t5") >= 2
    for case in data["cases"]:
        _check(case)


def test_encoder_oracle_matches_transformers_live():
    pytest.importorskip("transformers")
    import importlib.util
    import sys

    spec = importlib.util.spec_from_file_location("make_encoder_golden", os.path.join(HERE, "golden",
                                                                                     "make_encoder_golden.py"))
    mod = importlib.util.module_from_spec(spec)
    sys.modules["make_encoder_golden"] = mod
    spec.loader.exec_module(mod)
    for case in mod.build_cases():
        _check(case)


def test_t5_bucket_function_matches_transformers():
    tr = pytest.importorskip("transformers")
    from transformers.models.t5.modeling_t5 import T5Attention

    for L in (8, 77, 128, 300):
        rel = torch.arange(L)[None, :] - torch.arange(L)[:, None]
        ref = T5Attention._relative_position_bucket(rel, bidirectional=True, num_buckets=32, max_distance=128)
        assert torch.equal(nets.t5_buckets(L), ref), (L, tr.__version__)
