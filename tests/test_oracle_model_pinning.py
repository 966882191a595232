"""Pins the model oracle (oracle/model_ref.py) to an independent Llama / Qwen2 implementation.

The reference has no model arithmetic, so the oracle restates our spec. Here its
pure-fp32 mode (round_bf16=False) is checked against HF transformers 5.5.0 LlamaForCausalLM /
Qwen2ForCausalLM in fp32 with identical weights: golden logits in tests/golden/hf_logits.npz
(made by tests/golden/make_hf_golden.py), plus a live HF comparison when transformers imports.
This covers RMSNorm, the half-split RoPE with theta, the GQA head mapping (q head h -> kv head
h // G, groups 2 and 5), QKV bias, SwiGLU, the untied LM head, the KV cache and greedy argmax.
The bf16 storage points of the default mode are the GPU's (checked by the -m gpu tests).
"""
import pathlib

import numpy as np
import pytest
import torch

from oracle import model_ref as mr

GOLD = np.load(pathlib.Path(__file__).parent / "golden" / "hf_logits.npz")
CASES = {
    "llama_tiny": (mr.preset("tiny"), 11),
    "qwen2_tiny": (mr.Dims(2, 320, 5, 1, 64, 640, 1024, 1, 1.0e6, 1e-6), 5),
}
ATOL = 2e-4  # fp32 vs fp32 (different summation order, RoPE table in fp64 vs fp32)


@pytest.mark.parametrize("name", sorted(CASES))
def test_oracle_fp32_matches_hf_golden(name):
    d, seed = CASES[name]
    prompt = GOLD[f"{name}_prompt"].tolist()
    assert prompt == mr.prompt_tokens(seed, 1, len(prompt), d.vocab)
    model = mr.RefModel(d, mr.generate_weights(d, seed), round_bf16=False)
    toks, lg = model.generate(prompt, len(GOLD[f"{name}_tokens"]))
    assert toks == GOLD[f"{name}_tokens"].tolist()
    err = float((lg - torch.from_numpy(GOLD[f"{name}_logits"])).abs().max())
    assert err < ATOL, err


@pytest.mark.parametrize("name", sorted(CASES))
def test_bf16_storage_points_stay_close_to_fp32(name):
    """The default (GPU-matching) mode differs from pure fp32 only by bf16 storage rounding."""
    d, seed = CASES[name]
    prompt = GOLD[f"{name}_prompt"].tolist()
    w = mr.generate_weights(d, seed)
    _, lg16 = mr.RefModel(d, w).generate(prompt, 1)
    ref = torch.from_numpy(GOLD[f"{name}_logits"][0])
    assert float((lg16[0] - ref).abs().max()) < 0.05 * float(ref.std())


def test_oracle_matches_live_hf():
    pytest.importorskip("transformers")
    import sys
    sys.path.insert(0, str(pathlib.Path(__file__).parent / "golden"))
    import make_hf_golden as mk
    d, seed = CASES["qwen2_tiny"]
    w = mr.generate_weights(d, seed)
    prompt = mr.prompt_tokens(seed, 9, 37, d.vocab)
    toks, lg = mk.hf_greedy(mk.hf_model(d, w), prompt, 2)
    otoks, olg = mr.RefModel(d, w, round_bf16=False).generate(prompt, 2)
    assert toks == otoks
    assert float((lg - olg).abs().max()) < ATOL
