"""Golden vectors that pin the model oracle (oracle/model_ref.py) to an independent Llama / Qwen2
implementation: HF transformers (5.5.0 in this image) LlamaForCausalLM / Qwen2ForCausalLM in fp32,
loaded with the library's deterministic weights (oracle.model_ref.generate_weights).

For each model: the last-position logits of a 24-token prompt, then 3 greedy decode steps through
HF's KV cache (logits of each). Written to tests/golden/hf_logits.npz.

    python tests/golden/make_hf_golden.py
"""
from __future__ import annotations

import pathlib
import sys

import numpy as np
import torch

REPO = pathlib.Path(__file__).resolve().parents[2]
sys.path.insert(0, str(REPO))

from oracle import model_ref as mr  # noqa: E402

# (name, dims, weight seed): the tiny preset (config 1) and a Qwen2-shaped tiny model with QKV bias
# and GQA group 5 (the group of Qwen2.5-14B).
CASES = [
    ("llama_tiny", mr.preset("tiny"), 11),
    ("qwen2_tiny", mr.Dims(2, 320, 5, 1, 64, 640, 1024, 1, 1.0e6, 1e-6), 5),
]
PROMPT_LEN, N_DECODE = 24, 3


def hf_model(d: mr.Dims, w: dict):
    from transformers import LlamaConfig, LlamaForCausalLM, Qwen2Config, Qwen2ForCausalLM
    common = dict(vocab_size=d.vocab, hidden_size=d.d_model, intermediate_size=d.ffn_dim,
                  num_hidden_layers=d.n_layers, num_attention_heads=d.n_heads, num_key_value_heads=d.n_kv_heads,
                  rms_norm_eps=d.rms_eps, rope_theta=d.rope_theta, max_position_embeddings=4096,
                  tie_word_embeddings=False, hidden_act="silu", torch_dtype=torch.float32)
    if d.qkv_bias:
        assert d.n_heads * d.head_dim == d.d_model, "HF Qwen2 ties head_dim to hidden_size / heads"
        model = Qwen2ForCausalLM(Qwen2Config(**common, use_sliding_window=False))
    else:
        model = LlamaForCausalLM(LlamaConfig(**common, head_dim=d.head_dim, attention_bias=False, mlp_bias=False))
    model = model.eval().float()
    H, Hk, dh = d.n_heads, d.n_kv_heads, d.head_dim
    sd = {"model.embed_tokens.weight": w["embed"], "lm_head.weight": w["lm_head"], "model.norm.weight": w["final_norm"]}
    for l, L in enumerate(w["layers"]):
        p = f"model.layers.{l}."
        sd[p + "self_attn.q_proj.weight"] = L["qkv"][: H * dh]
        sd[p + "self_attn.k_proj.weight"] = L["qkv"][H * dh:(H + Hk) * dh]
        sd[p + "self_attn.v_proj.weight"] = L["qkv"][(H + Hk) * dh:]
        if d.qkv_bias:
            sd[p + "self_attn.q_proj.bias"] = L["qkv_bias"][: H * dh]
            sd[p + "self_attn.k_proj.bias"] = L["qkv_bias"][H * dh:(H + Hk) * dh]
            sd[p + "self_attn.v_proj.bias"] = L["qkv_bias"][(H + Hk) * dh:]
        sd[p + "self_attn.o_proj.weight"] = L["o"]
        sd[p + "mlp.gate_proj.weight"] = L["gate"]
        sd[p + "mlp.up_proj.weight"] = L["up"]
        sd[p + "mlp.down_proj.weight"] = L["down"]
        sd[p + "input_layernorm.weight"] = L["attn_norm"]
        sd[p + "post_attention_layernorm.weight"] = L["mlp_norm"]
    missing, unexpected = model.load_state_dict({k: v.contiguous() for k, v in sd.items()}, strict=False)
    assert not unexpected and all("rotary" in k for k in missing), (missing, unexpected)
    return model


@torch.no_grad()
def hf_greedy(model, prompt, n_new):
    ids = torch.tensor([prompt])
    out = model(input_ids=ids, use_cache=True)
    logits, past = [out.logits[0, -1].clone()], out.past_key_values
    toks = []
    for i in range(n_new):
        t = int(torch.argmax(logits[-1]))
        toks.append(t)
        if i + 1 == n_new:
            break
        out = model(input_ids=torch.tensor([[t]]), past_key_values=past, use_cache=True)
        past = out.past_key_values
        logits.append(out.logits[0, -1].clone())
    return toks, torch.stack(logits)


def main():
    torch.manual_seed(0)
    res = {}
    for name, d, seed in CASES:
        w = mr.generate_weights(d, seed)
        prompt = mr.prompt_tokens(seed, 1, PROMPT_LEN, d.vocab)
        toks, lg = hf_greedy(hf_model(d, w), prompt, N_DECODE + 1)
        res[f"{name}_prompt"] = np.array(prompt, dtype=np.int32)
        res[f"{name}_tokens"] = np.array(toks, dtype=np.int32)
        res[f"{name}_logits"] = lg.numpy().astype(np.float32)
        print(name, toks, float(lg.std()))
    np.savez_compressed(pathlib.Path(__file__).with_name("hf_logits.npz"), **res)


if __name__ == "__main__":
    main()
