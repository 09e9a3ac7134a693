"""Pins the numerics oracle's frozen text encoders to the published implementations
(VERDICT r1 "next" #2): oracle/nets.text_encoder against transformers'
CLIPTextModel (OpenCLIP ViT-H/14's text tower has the same pre-LN causal layout: token +
position embedding, per layer LN -> causal MHA (q/k/v/out with bias, 1/sqrt(hd) scaling) ->
residual, LN -> fc1 -> GELU -> fc2 -> residual, final LayerNorm), and oracle/nets.t5_encoder
against transformers' T5EncoderModel (shared embedding, RMSNorm without mean subtraction,
no-bias q/k/v/o without 1/sqrt(d) scaling, relative-position bias from block 0 shared by every
block, gated-GELU feed-forward, final RMSNorm).

Weight mapping (HF -> oracle parameter dict):
  CLIP  q_proj/k_proj/v_proj -> attn.qkv (rows [q; k; v]); out_proj -> attn.out;
        layer_norm1/2 -> ln1/ln2; mlp.fc1/fc2 -> mlp.fc1/fc2; final_layer_norm -> ln_final
  T5    shared -> shared; SelfAttention.q/k/v -> attn.qkv; .o -> attn.o;
        block.0 relative_attention_bias [buckets, heads] -> rel_bias;
        DenseReluDense.wi_1 (linear half) / wi_0 (activated half) -> ff.wi rows [wi_1; wi_0];
        wo -> ff.wo; layer[0/1].layer_norm -> ln1/ln2; final_layer_norm -> final_ln
The executor's T5 uses exact (erf) GELU in its gated feed-forward, so the HF model is built
with dense_act_fn="gelu" (T5 v1.1 ships "gelu_new", the tanh approximation).

Writes tests/golden/encoder_cases.pt: tiny seeded configurations with their HF weights (as
oracle parameter dicts), token ids and HF outputs, so the pin is also checked where transformers
is absent. Run from the repo root:  python tests/golden/make_encoder_golden.py
"""

from __future__ import annotations

import os

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "encoder_cases.pt")

CLIP_CASES = [dict(d=64, heads=4, layers=2, ffn=256, vocab=97, L=16, B=2, seed=11),
              dict(d=96, heads=3, layers=3, ffn=160, vocab=50, L=9, B=3, seed=12)]
T5_CASES = [dict(d=64, heads=4, layers=2, ffn=128, vocab=101, L=16, B=2, seed=21, buckets=32, max_dist=128),
            dict(d=48, heads=2, layers=3, ffn=96, vocab=64, L=40, B=2, seed=22, buckets=32, max_dist=128)]


def clip_hf(c):
    from transformers import CLIPTextConfig, CLIPTextModel

    torch.manual_seed(c["seed"])
    cfg = CLIPTextConfig(vocab_size=c["vocab"], hidden_size=c["d"], intermediate_size=c["ffn"],
                         num_hidden_layers=c["layers"], num_attention_heads=c["heads"],
                         max_position_embeddings=c["L"], hidden_act="gelu", layer_norm_eps=1e-5,
                         attention_dropout=0.0)
    m = CLIPTextModel(cfg).eval()
    # HF's init leaves biases / LN affine at 0 / 1: randomise them so the mapping is exercised
    with torch.no_grad():
        for n, p in m.named_parameters():
            if n.endswith("bias") or "norm" in n:
                p.add_(0.1 * torch.randn_like(p))
    return m


def clip_to_oracle(m):
    sd = {k: v.detach().clone().float() for k, v in m.state_dict().items()}
    t = "text_model."
    P = {"token_embedding": sd[t + "embeddings.token_embedding.weight"],
         "position_embedding": sd[t + "embeddings.position_embedding.weight"],
         "ln_final.weight": sd[t + "final_layer_norm.weight"], "ln_final.bias": sd[t + "final_layer_norm.bias"]}
    i = 0
    while f"{t}encoder.layers.{i}.self_attn.q_proj.weight" in sd:
        h, p = f"{t}encoder.layers.{i}.", f"layers.{i}."
        a = h + "self_attn."
        P[p + "attn.qkv.weight"] = torch.cat([sd[a + f"{x}_proj.weight"] for x in "qkv"])
        P[p + "attn.qkv.bias"] = torch.cat([sd[a + f"{x}_proj.bias"] for x in "qkv"])
        P[p + "attn.out.weight"], P[p + "attn.out.bias"] = sd[a + "out_proj.weight"], sd[a + "out_proj.bias"]
        for hn, on in (("layer_norm1", "ln1"), ("layer_norm2", "ln2"), ("mlp.fc1", "mlp.fc1"), ("mlp.fc2", "mlp.fc2")):
            P[p + on + ".weight"], P[p + on + ".bias"] = sd[h + hn + ".weight"], sd[h + hn + ".bias"]
        i += 1
    return P


def t5_hf(c):
    from transformers import T5Config, T5EncoderModel

    torch.manual_seed(c["seed"])
    cfg = T5Config(vocab_size=c["vocab"], d_model=c["d"], d_kv=c["d"] // c["heads"], d_ff=c["ffn"],
                   num_layers=c["layers"], num_heads=c["heads"], relative_attention_num_buckets=c["buckets"],
                   relative_attention_max_distance=c["max_dist"], feed_forward_proj="gated-gelu",
                   dropout_rate=0.0, layer_norm_epsilon=1e-6)
    cfg.dense_act_fn = "gelu"  # exact GELU, as the executor's gated feed-forward computes it
    m = T5EncoderModel(cfg).eval()
    with torch.no_grad():
        for n, p in m.named_parameters():
            if "layer_norm" in n:
                p.add_(0.1 * torch.randn_like(p))
    return m


def t5_to_oracle(m):
    sd = {k: v.detach().clone().float() for k, v in m.state_dict().items()}
    P = {"shared": sd["shared.weight"], "final_ln.weight": sd["encoder.final_layer_norm.weight"],
         "rel_bias": sd["encoder.block.0.layer.0.SelfAttention.relative_attention_bias.weight"]}
    i = 0
    while f"encoder.block.{i}.layer.0.SelfAttention.q.weight" in sd:
        h, p = f"encoder.block.{i}.layer.", f"block.{i}."
        P[p + "attn.qkv.weight"] = torch.cat([sd[h + f"0.SelfAttention.{x}.weight"] for x in "qkv"])
        P[p + "attn.o.weight"] = sd[h + "0.SelfAttention.o.weight"]
        P[p + "ln1.weight"] = sd[h + "0.layer_norm.weight"]
        P[p + "ln2.weight"] = sd[h + "1.layer_norm.weight"]
        P[p + "ff.wi.weight"] = torch.cat([sd[h + "1.DenseReluDense.wi_1.weight"],
                                           sd[h + "1.DenseReluDense.wi_0.weight"]])
        P[p + "ff.wo.weight"] = sd[h + "1.DenseReluDense.wo.weight"]
        i += 1
    return P


def make_ids(c):
    g = torch.Generator().manual_seed(1000 + c["seed"])
    return torch.randint(0, c["vocab"], (c["B"], c["L"]), generator=g)


def build_cases():
    cases = []
    with torch.no_grad():
        for c in CLIP_CASES:
            m, ids = clip_hf(c), make_ids(c)
            out = m(input_ids=ids).last_hidden_state.float()
            cases.append(dict(kind="clip", cfg=c, P=clip_to_oracle(m), ids=ids, out=out))
        for c in T5_CASES:
            m, ids = t5_hf(c), make_ids(c)
            out = m(input_ids=ids).last_hidden_state.float()
            cases.append(dict(kind="t5", cfg=c, P=t5_to_oracle(m), ids=ids, out=out))
    return cases


if __name__ == "__main__":
    import transformers

    cases = build_cases()
    torch.save({"transformers": transformers.__version__, "torch": torch.__version__, "cases": cases}, OUT)
    print(f"wrote {OUT}: {len(cases)} cases (transformers {transformers.__version__})")
