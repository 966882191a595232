"""Asynchronous KV migration (K11, tc_kv_migrate_async) and the shared per-GPU KV pool.

The reference prices a transfer as its own event (engine.hpp:388-413, cost_model.hpp:81-85); the
paper decouples the copy from the instances' iterations. Here the copy runs on the source's
high-priority copy stream; nothing blocks the host, several copies are in flight at once, the
destination's next step orders after the copy on the GPU, and source pages are quarantined until
the copy has read them. Tokens after migration are checked against the oracle (tolerances:
tests/test_gpu_step.py).
"""
import numpy as np
import pytest
import torch

from oracle import model_ref as mr
from test_gpu_step import Follower

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def model():
    d = mr.preset("tiny")
    return mr.RefModel(d, mr.generate_weights(d, 11), max_pos=4096)


def make(**kw):
    from paper_2508_01989_b200 import Instance
    args = dict(weight_seed=11, kv_pool_tokens=1 << 14, max_step_tokens=2048, max_seqs=64, max_context=4096)
    args.update(kw)
    return Instance("tiny", **args)


def test_many_async_migrations_in_flight_then_immediate_steps(model):
    """8 requests prefilled on src, all migrated at once without any host wait, then decoded on dst
    right away (the step orders after each copy on the GPU) while src keeps stepping."""
    src, dst = make(), make()
    prompts = {rid: mr.prompt_tokens(11, rid, 50 + 37 * rid, 1024) for rid in range(1, 9)}
    first = {}
    for rid, p in prompts.items():
        o = src.step(prefill=[(rid, 0, p, True)], keep_logits=True)
        first[rid] = int(o.sampled[0])
    before = {rid: src.read_pages(src.kv_pages(rid)) for rid in prompts}
    evs = [src.migrate_async(dst, rid, len(p)) for rid, p in prompts.items()]
    # src keeps working on another request while the copies run; its pages must not alias
    other = mr.prompt_tokens(11, 99, 300, 1024)
    src.launch(prefill=[(99, 0, other, True)])
    dec = [(rid, len(p), first[rid]) for rid, p in prompts.items()]
    out = dst.step(decode=dec, keep_logits=True)
    src.wait()
    for ev in evs:
        ms, nbytes = ev.wait()
        assert ms > 0 and nbytes > 0
        ev.close()
    for k, (rid, pos, tok) in enumerate(dec):
        f = Follower(model, prompts[rid])
        f.feed([tok])
        f.check(int(out.sampled[k]), out.logits[k])
        got = dst.read_pages(dst.kv_pages(rid))
        # rows written before the migration are byte-identical (the decode appended row `pos`)
        row_bytes = got.shape[1] // 16
        n_full = pos // 16
        np.testing.assert_array_equal(got[:n_full], before[rid][:n_full])
        assert src.kv_stats(rid)[0] == 0
    src.close()
    dst.close()


def test_source_pages_quarantined_until_copy_done(model):
    """A tiny source pool: the pages a migration frees are reused only after the copy read them, so
    a prefill launched right after the migration cannot overwrite KV still in transit."""
    src, dst = make(kv_pool_tokens=320), make()
    p = mr.prompt_tokens(11, 7, 300, 1024)                  # 19 of the 20 pages
    o = src.step(prefill=[(7, 0, p, True)], keep_logits=True)
    before = src.read_pages(src.kv_pages(7))
    ev = src.migrate_async(dst, 7, len(p))
    q = mr.prompt_tokens(11, 8, 300, 1024)
    src.step(prefill=[(8, 0, q, True)])                    # needs the quarantined pages back
    ev.wait()
    np.testing.assert_array_equal(dst.read_pages(dst.kv_pages(7)), before)
    f = Follower(model, p)
    f.check(int(o.sampled[0]), o.logits[0])
    tok = int(o.sampled[0])
    f.feed([tok])
    o2 = dst.step(decode=[(7, len(p), tok)], keep_logits=True)
    f.check(int(o2.sampled[0]), o2.logits[0])
    ev.close()
    src.close()
    dst.close()


def test_release_during_inbound_copy_and_shared_pool():
    """Two instances on one KV pool: one free list; a request released on the destination while its
    inbound copy may still run returns its pages only after the copy."""
    a = make(kv_pool_tokens=1 << 12)
    b = make(share_kv_pool=a, share_weights=a)
    _, free0 = a.kv_stats()
    assert b.kv_stats()[1] == free0
    a.step(prefill=[(1, 0, list(range(200)), True)])
    assert b.kv_stats()[1] == free0 - 13
    ev = a.migrate_async(b, 1, 200)
    b.kv_release(1)
    ev.wait()
    ev.close()
    assert a.kv_stats()[1] == free0 and b.kv_stats(1)[0] == 0
    b.close()
    assert a.kv_stats()[1] == free0
    a.close()


def test_migration_ping_pong_chain_without_host_waits(model):
    """A -> B -> A -> B with no waits between: each copy orders after the previous inbound copy."""
    a, b = make(), make()
    p = mr.prompt_tokens(11, 3, 129, 1024)
    o = a.step(prefill=[(3, 0, p, True)], keep_logits=True)
    before = a.read_pages(a.kv_pages(3))
    evs = [a.migrate_async(b, 3, len(p)), None, None]
    evs[1] = b.migrate_async(a, 3, len(p))
    evs[2] = a.migrate_async(b, 3, len(p))
    tok = int(o.sampled[0])
    o2 = b.step(decode=[(3, len(p), tok)], keep_logits=True)
    for e in evs:
        e.wait()
        e.close()
    np.testing.assert_array_equal(b.read_pages(b.kv_pages(3))[:len(p) // 16], before[:len(p) // 16])
    f = Follower(model, p)
    f.feed([tok])
    f.check(int(o2.sampled[0]), o2.logits[0])
    a.close()
    b.close()


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2, reason="needs 2 GPUs (NVLink P2P)")
def test_cross_gpu_migration_over_nvlink(model):
    """Instances on GPUs 0 and 1: the copy kernel on GPU 0 stores into GPU 1's pool over NVLink."""
    a, b = make(device=0), make(device=1)
    p = mr.prompt_tokens(11, 5, 1000, 1024)
    o = a.step(prefill=[(5, 0, p, True)], keep_logits=True)
    before = a.read_pages(a.kv_pages(5))
    ev = a.migrate_async(b, 5, len(p))
    ms, nbytes = ev.wait()
    ev.close()
    np.testing.assert_array_equal(b.read_pages(b.kv_pages(5)), before)
    tok = int(o.sampled[0])
    o2 = b.step(decode=[(5, len(p), tok)], keep_logits=True)
    f = Follower(model, p)
    f.feed([tok])
    f.check(int(o2.sampled[0]), o2.logits[0])
    a.close()
    b.close()


@pytest.mark.parametrize("page_bytes,n_pages", [(2 << 20, 37), (3 << 20, 5), (16 * 2 * 2 * 64 * 2, 300), (65536 + 4096, 9)])
def test_copy_pages_kernel_bytes(page_bytes, n_pages):
    """K11's copy kernel (tc_copy_pages, the same slice loop as the migration kernel) moves whole
    pages byte-exactly for page sizes that are, and are not, multiples of its 64 KiB slice."""
    from paper_2508_01989_b200 import runtime
    g = torch.Generator(device="cpu").manual_seed(page_bytes + n_pages)
    pool_pages = 2 * n_pages + 3
    src = torch.randint(-2**31, 2**31 - 1, (pool_pages, page_bytes // 4), generator=g, dtype=torch.int32).cuda()
    dst = torch.zeros_like(src)
    sp = torch.randperm(pool_pages, generator=g)[:n_pages].to(torch.int32)
    dp = torch.randperm(pool_pages, generator=g)[:n_pages].to(torch.int32)
    spd, dpd = sp.cuda(), dp.cuda()
    runtime.copy_pages(src.data_ptr(), dst.data_ptr(), spd.data_ptr(), dpd.data_ptr(), n_pages, page_bytes,
                       torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    ref = torch.zeros_like(src)
    ref[dp.long().cuda()] = src[sp.long().cuda()]
    assert torch.equal(dst, ref)
