"""Parity at the exact step shapes bench.py measures ("parity-test the shapes you
benchmark"), on layer-reduced models (2 layers, every other dimension as benchmarked):

* config 2 (bench.py default): Llama-3-8B shapes, one step = a 512-token prefill chunk over a
  512-token paged prefix + 64 decodes at context 1024 (T = 576 rows), with the concurrent
  prefill | decode attention SM split active (attn_pf_sms > 0), plus the decode-only step of the
  same 64 decodes (T = 64: small token tiles, stream-K residual GEMMs);
* config 5 (bench.py --model qwen2_5_14b --prefill 1024 --prefix 4096 --decode 32 --ctx 8192):
  Qwen2.5-14B shapes (QKV bias, GQA group 5), a 1024-token chunk over a 4096-token prefix + 32
  decodes at context 8192.

Decode contexts repeat a few distinct prompts (the oracle cost is per distinct prompt); every
decode row has its own request id, pages and sampled row. Tolerances: tests/test_gpu_step.py.
"""
import pytest
import torch

from oracle import model_ref as mr
from test_gpu_step import Follower, check_row

pytestmark = pytest.mark.gpu


def run_bench_step(model_name, seed, P, prefix, D, ctx, distinct, max_ctx):
    from paper_2508_01989_b200 import Instance
    d = mr.preset(model_name)
    torch.set_num_threads(max(1, torch.get_num_threads()))
    with Instance(model_name, weight_seed=seed, kv_pool_tokens=(D + 2) * (ctx + 64) + prefix + P + 4096,
                  max_step_tokens=max(P + D, 2048), max_seqs=D + 8, max_context=max_ctx) as inst:
        model = mr.RefModel(d, mr.weights_from_device(inst, d), max_pos=max_ctx)
        prompt = mr.prompt_tokens(seed, 0, prefix + P, d.vocab)
        for s in range(0, prefix, 2048):
            inst.step(prefill=[(0, s, prompt[s:min(prefix, s + 2048)], False)])
        ctxs = [mr.prompt_tokens(seed, 1000 + j, ctx, d.vocab) for j in range(distinct)]
        dec_tok = [mr.prompt_tokens(seed, 2000 + j, 1, d.vocab)[0] for j in range(distinct)]
        for rid in range(1, D + 1):
            toks = ctxs[(rid - 1) % distinct]
            for s in range(0, ctx, 2048):
                inst.step(prefill=[(rid, s, toks[s:s + 2048], False)])
        decode = [(rid, ctx, dec_tok[(rid - 1) % distinct]) for rid in range(1, D + 1)]
        out = inst.step(prefill=[(0, prefix, prompt[prefix:], True)], decode=decode, keep_logits=True)
        dec_only = inst.step(decode=[(rid, ctx + 1, int(out.sampled[rid])) for rid in range(1, D + 1)],
                             keep_logits=True)
    # oracle
    fp = Follower(model, prompt)
    near = int(check_row(int(out.sampled[0]), out.logits[0], fp.ref_logits()))
    fol = []
    for j in range(distinct):
        f = Follower(model, ctxs[j])
        f.feed([dec_tok[j]])
        fol.append(f)
    for rid in range(1, D + 1):
        near += int(check_row(int(out.sampled[rid]), out.logits[rid], fol[(rid - 1) % distinct].ref_logits()))
    # decode-only step: rows sharing a context fed the same sampled token share the oracle state
    fed = {}
    for rid in range(1, D + 1):
        j = (rid - 1) % distinct
        key = (j, int(out.sampled[rid]))
        if key not in fed:
            f = Follower.__new__(Follower)
            f.model = model
            f.cache = [{"k": c["k"].clone(), "v": c["v"].clone()} for c in fol[j].cache]
            f.pos = fol[j].pos
            f.feed([key[1]])
            fed[key] = f
        near += int(check_row(int(dec_only.sampled[rid - 1]), dec_only.logits[rid - 1], fed[key].ref_logits()))
    return out, near


def test_config2_bench_step_llama_shape():
    out, near = run_bench_step("llama3_8b:L2", 3, P=512, prefix=512, D=64, ctx=1024, distinct=8, max_ctx=2048)
    assert out.attn_pf_sms > 0, "the concurrent prefill | decode attention split was not active"
    assert near <= 129 // 4


def test_config5_bench_step_qwen_shape():
    out, near = run_bench_step("qwen2_5_14b:L2", 5, P=1024, prefix=4096, D=32, ctx=8192, distinct=2, max_ctx=8256)
    assert out.attn_pf_sms > 0
    assert near <= 65 // 4


def test_odd_step_shapes_llama():
    """Off-bench sizes through the same path: a mixed step of T = 260 rows (2 token tiles of 160,
    one ragged) and a decode-only step of T = 100 rows (one 128-token tile, 28 padded rows) --
    the direct ws GEMM units with fused epilogues at token tiles the bench shapes do not hit."""
    out, near = run_bench_step("llama3_8b:L2", 11, P=160, prefix=256, D=100, ctx=512, distinct=4, max_ctx=1024)
    assert near <= 201 // 4
