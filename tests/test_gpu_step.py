"""The hybrid step through the C ABI (tc_step_launch / tc_step_wait) vs the CPU oracle
(oracle/model_ref.py; its fp32 mode is pinned to HF transformers by test_oracle_model_pinning.py).

Stated tolerances (from the measured budget of tools/parity_budget.py,
profiles/r02/parity_budget_*.json):
  * logits: max |gpu - oracle| <= LOGIT_REL * std(oracle logits) + LOGIT_ABS. The oracle emulates
    every bf16 storage point of the GPU path; what remains is fp32 accumulation order (split-K
    partials are reduced in arrival order), bf16 rounding of the unnormalised attention
    probabilities against a running max, and exp2 approximations.
  * greedy tokens: a GPU token g may differ from the oracle's token r only where that is
    consistent with the logit bound, i.e. oracle[r] - oracle[g] <= 2 * logit_tol; the oracle then
    continues from the GPU token (teacher forcing). Logits are checked on every sampled row.
"""
import numpy as np
import pytest
import torch

from oracle import model_ref as mr

pytestmark = pytest.mark.gpu

LOGIT_REL, LOGIT_ABS = 0.08, 0.01


def logit_tol(ref):
    return LOGIT_REL * float(ref.std()) + LOGIT_ABS


def check_row(gpu_token, gpu_logits, ref):
    """Returns True when the tokens differ (an allowed near-tie)."""
    tol = logit_tol(ref)
    gpu = torch.as_tensor(gpu_logits)
    err = (gpu - ref).abs().max().item()
    assert err <= tol, f"max |dlogit| {err:.4f} > {tol:.4f}"
    assert int(torch.argmax(gpu)) == gpu_token, "sampled id is not the argmax of the returned logits"
    ref_tok = int(torch.argmax(ref))
    if ref_tok == gpu_token:
        return False
    gap = float(ref[ref_tok] - ref[gpu_token])
    assert gap <= 2 * tol, f"token mismatch {gpu_token} vs {ref_tok}: oracle gap {gap:.4f} > 2 x tol {tol:.4f}"
    return True


class Follower:
    """Oracle decoder for one request, teacher-forced on GPU tokens."""

    def __init__(self, model, prompt):
        self.model, self.cache, self.pos = model, model.new_cache(), 0
        self.x = None
        self.feed(prompt)
        self.near_ties = 0

    def feed(self, toks):
        self.x = self.model.forward(list(toks), self.pos, self.cache)
        self.pos += len(toks)

    def ref_logits(self):
        return self.model.logits(self.x[-1:])[0]

    def check(self, gpu_token, gpu_logits):
        self.near_ties += check_row(gpu_token, gpu_logits, self.ref_logits())


@pytest.fixture(scope="module")
def tiny():
    from paper_2508_01989_b200 import Instance
    inst = Instance("tiny", weight_seed=11, kv_pool_tokens=1 << 15, max_step_tokens=2048, max_seqs=64,
                    max_context=4096)
    d = mr.preset("tiny")
    model = mr.RefModel(d, mr.generate_weights(d, 11))
    yield inst, model
    inst.close()


def test_tiny_weights_bitexact_with_oracle_init(tiny):
    inst, model = tiny
    d = mr.preset("tiny")
    np.testing.assert_array_equal(inst.weight("L1.qkv"), mr.gen_bits(11, mr.tid_layer(1, 0), 512, 256, mr.LIN_SCALE, 0.0))
    np.testing.assert_array_equal(inst.weight("embed"), mr.gen_bits(11, mr.TID_EMBED, d.vocab, d.d_model, np.float32(1), 0.0))
    gu = inst.weight("L0.gate_up").reshape(d.ffn_dim // 64, 2, 64, d.d_model)
    np.testing.assert_array_equal(gu[:, 1].reshape(d.ffn_dim, -1),
                                  mr.gen_bits(11, mr.tid_layer(0, 3), d.ffn_dim, d.d_model, mr.LIN_SCALE, 0.0))


def test_tiny_chunked_prefill_then_decode(tiny):
    inst, model = tiny
    rid = 1
    prompt = mr.prompt_tokens(11, rid, 37, 1024)
    inst.step(prefill=[(rid, 0, prompt[:16], False)])
    out = inst.step(prefill=[(rid, 16, prompt[16:], True)], keep_logits=True)
    f = Follower(model, prompt)
    f.check(int(out.sampled[0]), out.logits[0])
    tok, pos = int(out.sampled[0]), 37
    for _ in range(12):
        f.feed([tok])
        out = inst.step(decode=[(rid, pos, tok)], keep_logits=True)
        f.check(int(out.sampled[0]), out.logits[0])
        tok, pos = int(out.sampled[0]), pos + 1
    inst.kv_release(rid)


def test_tiny_mixed_batches(tiny):
    """Several requests at different phases share steps; a chunk spans two prompts."""
    inst, model = tiny
    rng = np.random.default_rng(5)
    reqs = {}
    for rid in range(10, 16):
        n = int(rng.integers(5, 300))
        reqs[rid] = {"prompt": mr.prompt_tokens(11, rid, n, 1024), "done": 0, "tok": None, "pos": 0}
    followers = {}
    chunk = 128
    for it in range(60):
        prefill, decode = [], []
        budget = chunk
        for rid, r in reqs.items():
            if r["tok"] is not None:
                decode.append((rid, r["pos"], r["tok"]))
        for rid, r in reqs.items():
            left = len(r["prompt"]) - r["done"]
            if left > 0 and budget > 0:
                take = min(left, budget)
                prefill.append((rid, r["done"], r["prompt"][r["done"]:r["done"] + take], take == left))
                budget -= take
        if not prefill and not decode:
            break
        out = inst.step(prefill=prefill, decode=decode, keep_logits=True)
        k = 0
        for rid, pos0, toks, want in prefill:
            reqs[rid]["done"] += len(toks)
            if want:
                r = reqs[rid]
                followers[rid] = Follower(model, r["prompt"])
                followers[rid].check(int(out.sampled[k]), out.logits[k])
                r["tok"], r["pos"] = int(out.sampled[k]), len(r["prompt"])
                k += 1
        for rid, pos, tok in decode:
            f = followers[rid]
            f.feed([tok])
            f.check(int(out.sampled[k]), out.logits[k])
            reqs[rid]["tok"], reqs[rid]["pos"] = int(out.sampled[k]), pos + 1
            k += 1
    assert len(followers) == len(reqs)
    for rid in reqs:
        inst.kv_release(rid)


@pytest.mark.parametrize("lengths", [(3500,), (1, 15, 16, 17, 33, 700, 3500), tuple(range(1, 60, 3))])
def test_tiny_decode_page_stream_splits(tiny, lengths):
    """Decode attention work split (attn_decode): contexts of 1..3500 tokens in one step; a lone
    3500-token request is cut across > 32 CTAs (multi-part global merge), short ones share CTAs."""
    inst, model = tiny
    reqs = {}
    for k, n in enumerate(lengths):
        rid = 200 + k
        prompt = mr.prompt_tokens(11, rid, n, 1024)
        for s0 in range(0, n, 2048):
            out = inst.step(prefill=[(rid, s0, prompt[s0:s0 + 2048], s0 + 2048 >= n)], keep_logits=True)
        reqs[rid] = [Follower(model, prompt), int(out.sampled[0]), n]
        reqs[rid][0].check(reqs[rid][1], out.logits[0])
    for _ in range(2):
        dec = [(rid, r[2], r[1]) for rid, r in reqs.items()]
        o = inst.step(decode=dec, keep_logits=True)
        for k, (rid, pos, tok) in enumerate(dec):
            f = reqs[rid][0]
            f.feed([tok])
            f.check(int(o.sampled[k]), o.logits[k])
            reqs[rid][1], reqs[rid][2] = int(o.sampled[k]), pos + 1
    for rid in reqs:
        inst.kv_release(rid)


def test_kv_pages_released_and_reused(tiny):
    inst, _ = tiny
    _, free0 = inst.kv_stats()
    inst.step(prefill=[(99, 0, list(range(40)), True)])
    n, free1 = inst.kv_stats(99)
    assert n == 3 and free1 == free0 - 3
    inst.kv_release(99)
    assert inst.kv_stats(99) == (0, free0)


def test_error_paths(tiny):
    from paper_2508_01989_b200.runtime import TaichiError
    inst, _ = tiny
    with pytest.raises(TaichiError, match="token id out of range"):
        inst.step(prefill=[(5, 0, [5000], True)])
    with pytest.raises(TaichiError, match="empty step"):
        inst.step()
    inst.kv_release(5)


def test_tiny_migration_between_instances(tiny):
    """Init-style migration (P-heavy -> D-heavy) on one GPU: pages are byte-identical and the
    destination continues the exact greedy trajectory."""
    from paper_2508_01989_b200 import Instance
    src, model = tiny
    dst = Instance("tiny", weight_seed=11, kv_pool_tokens=1 << 14, max_step_tokens=512, max_seqs=16, max_context=4096)
    rid = 77
    prompt = mr.prompt_tokens(11, rid, 150, 1024)
    out = src.step(prefill=[(rid, 0, prompt, True)], keep_logits=True)
    src_pages = src.kv_pages(rid)
    before = src.read_pages(src_pages)
    src.migrate_to(dst, rid, len(prompt))
    ms, nbytes = src.migrate_wait()
    assert src.kv_stats(rid)[0] == 0
    dst_pages = dst.kv_pages(rid)
    assert len(dst_pages) == len(src_pages) and nbytes == len(src_pages) * before.shape[1]
    np.testing.assert_array_equal(dst.read_pages(dst_pages), before)
    f = Follower(model, prompt)
    f.check(int(out.sampled[0]), out.logits[0])
    tok, pos = int(out.sampled[0]), len(prompt)
    for _ in range(6):
        f.feed([tok])
        o = dst.step(decode=[(rid, pos, tok)], keep_logits=True)
        f.check(int(o.sampled[0]), o.logits[0])
        tok, pos = int(o.sampled[0]), pos + 1
    dst.close()


def test_migration_round_trip_during_inflight_step(tiny):
    """A request degrades and back-flows while a step that decodes it is still in flight on the
    source (the engine then commits that step's token, engine.hpp:461-493). Whole held pages move,
    so the row the in-flight step writes (here the first row of a fresh page) survives the round
    trip and decoding continues on the exact greedy trajectory."""
    from paper_2508_01989_b200 import Instance
    src, model = tiny
    dst = Instance("tiny", weight_seed=11, kv_pool_tokens=1 << 14, max_step_tokens=512, max_seqs=16, max_context=4096)
    rid = 78
    prompt = mr.prompt_tokens(11, rid, 32, 1024)  # footprint 33: the next row (32) opens page 3
    out = src.step(prefill=[(rid, 0, prompt, True)], keep_logits=True)
    f = Follower(model, prompt)
    f.check(int(out.sampled[0]), out.logits[0])
    tok, pos = int(out.sampled[0]), len(prompt)
    src.launch(decode=[(rid, pos, tok)], keep_logits=True)  # writes row 32, not yet waited
    src.migrate_to(dst, rid, pos)              # degrade: footprint - 1 rows requested
    src.migrate_wait()
    dst.migrate_to(src, rid, pos)              # backflow before the step completes
    dst.migrate_wait()
    o = src.wait()
    f.feed([tok])
    f.check(int(o.sampled[0]), o.logits[0])
    tok, pos = int(o.sampled[0]), pos + 1
    for _ in range(4):
        f.feed([tok])
        o = src.step(decode=[(rid, pos, tok)], keep_logits=True)
        f.check(int(o.sampled[0]), o.logits[0])
        tok, pos = int(o.sampled[0]), pos + 1
    src.kv_release(rid)
    dst.close()


@pytest.fixture(scope="module")
def llama_l2():
    from paper_2508_01989_b200 import Instance
    inst = Instance("llama3_8b:L2", weight_seed=3, kv_pool_tokens=1 << 15, max_step_tokens=1024, max_seqs=64,
                    max_context=8192)
    d = mr.preset("llama3_8b:L2")
    model = mr.RefModel(d, mr.weights_from_device(inst, d), max_pos=8192)
    yield inst, model
    inst.close()


def test_llama_shape_prefill_decode_long_context(llama_l2):
    """Llama-3-8B layer shapes (2 layers): 1000-token prompt in 512 chunks, then split-KV decode."""
    inst, model = llama_l2
    rid = 5
    prompt = mr.prompt_tokens(3, rid, 1000, 128256)
    inst.step(prefill=[(rid, 0, prompt[:512], False)])
    out = inst.step(prefill=[(rid, 512, prompt[512:], True)], keep_logits=True)
    f = Follower(model, prompt)
    f.check(int(out.sampled[0]), out.logits[0])
    tok, pos = int(out.sampled[0]), 1000
    for _ in range(4):
        f.feed([tok])
        o = inst.step(decode=[(rid, pos, tok)], keep_logits=True)
        f.check(int(o.sampled[0]), o.logits[0])
        tok, pos = int(o.sampled[0]), pos + 1
    inst.kv_release(rid)


def test_llama_shape_mixed_step(llama_l2):
    """One step = a prefill chunk spanning two prompts + 20 decodes (M = 150 rows)."""
    inst, model = llama_l2
    prompts = {rid: mr.prompt_tokens(3, rid, 40 + 3 * rid, 128256) for rid in range(100, 120)}
    follow = {}
    toks = {}
    for rid, p in prompts.items():
        o = inst.step(prefill=[(rid, 0, p, True)], keep_logits=True)
        toks[rid] = int(o.sampled[0])
        follow[rid] = Follower(model, p)
        follow[rid].check(toks[rid], o.logits[0])
    a = mr.prompt_tokens(3, 500, 70, 128256)
    b = mr.prompt_tokens(3, 501, 60, 128256)
    decode = [(rid, len(p), toks[rid]) for rid, p in prompts.items()]
    out = inst.step(prefill=[(500, 0, a, True), (501, 0, b[:40], False)], decode=decode, keep_logits=True)
    fa = Follower(model, a)
    fa.check(int(out.sampled[0]), out.logits[0])
    for k, (rid, pos, tok) in enumerate(decode):
        follow[rid].feed([tok])
        follow[rid].check(int(out.sampled[1 + k]), out.logits[1 + k])
    for rid in list(prompts) + [500, 501]:
        inst.kv_release(rid)


def test_qwen_shape_bias_and_group5():
    """Qwen2.5-14B layer shapes (2 layers, vocab 152064): QKV bias, GQA group 5 (40 q / 8 kv heads)."""
    from paper_2508_01989_b200 import Instance
    with Instance("qwen2_5_14b:L2", weight_seed=5, kv_pool_tokens=1 << 14, max_step_tokens=2048, max_seqs=32,
                  max_context=4096) as inst:
        d = mr.preset("qwen2_5_14b:L2")
        model = mr.RefModel(d, mr.weights_from_device(inst, d), max_pos=4096)
        prompts = {rid: mr.prompt_tokens(5, rid, 300 + 97 * rid, d.vocab) for rid in range(3)}
        out = inst.step(prefill=[(rid, 0, p, True) for rid, p in prompts.items()], keep_logits=True)
        follow = {}
        for k, (rid, p) in enumerate(prompts.items()):
            follow[rid] = Follower(model, p)
            follow[rid].check(int(out.sampled[k]), out.logits[k])
        toks = {rid: int(out.sampled[k]) for k, rid in enumerate(prompts)}
        pos = {rid: len(p) for rid, p in prompts.items()}
        for _ in range(3):
            dec = [(rid, pos[rid], toks[rid]) for rid in prompts]
            o = inst.step(decode=dec, keep_logits=True)
            for k, (rid, _, tok) in enumerate(dec):
                follow[rid].feed([tok])
                follow[rid].check(int(o.sampled[k]), o.logits[k])
                toks[rid] = int(o.sampled[k])
                pos[rid] += 1
