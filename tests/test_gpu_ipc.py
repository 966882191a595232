"""Cross-process KV migration (tc_kv_pool_export / tc_kv_pool_import / tc_kv_push_pages).

One TaiChi instance per GPU means one process per GPU: the flowing-decode migration of a
request's KV (engine.hpp:388-413 degrade / backflow, :510-525 init; priced by
cost_model.hpp:81-85) crosses a process boundary. The destination exports its pool as a CUDA IPC
handle and reserves pages; the source maps the pool and pushes whole pages with the same copy
kernel as in-process migration, its stores going over NVLink to the peer GPU.

This box has one GPU, so the two processes share it (a same-GPU IPC mapping: the identical code
path minus the NVLink hop); the 2-GPU variant runs where two GPUs are visible. The copied pages
must be byte-identical, and the destination must decode the next token of the migrated request
exactly as the source would have (oracle check, tolerances of tests/test_gpu_step.py).
"""
import multiprocessing as mp

import numpy as np
import pytest
import torch

from oracle import model_ref as mr

pytestmark = pytest.mark.gpu

KW = dict(weight_seed=13, kv_pool_tokens=1 << 13, max_step_tokens=1024, max_seqs=16, max_context=2048)


def _destination(device, conn):
    """Destination process: reserve pages for the request, export the pool, wait for the push,
    then decode the next token on the pushed KV and return the pages + the decode output."""
    from paper_2508_01989_b200 import Instance
    with Instance("tiny", device=device, **KW) as dst:
        rid, n_tokens = conn.recv()
        dst.kv_reserve(rid, n_tokens + 1)  # +1: the decode appends row n_tokens
        conn.send((dst.export_pool(), [int(p) for p in dst.kv_pages(rid)]))
        pos, tok = conn.recv()  # the push has completed
        pages = dst.read_pages(dst.kv_pages(rid))
        out = dst.step(decode=[(rid, pos, tok)], keep_logits=True)
        conn.send((pages, int(out.sampled[0]), np.asarray(out.logits[0])))
        conn.recv()


def _push_roundtrip(dst_device):
    from paper_2508_01989_b200 import Instance, RemotePool
    ctx = mp.get_context("spawn")
    here, there = ctx.Pipe()
    proc = ctx.Process(target=_destination, args=(dst_device, there))
    proc.start()
    try:
        d = mr.preset("tiny")
        model = mr.RefModel(d, mr.generate_weights(d, 13), max_pos=2048)
        prompt = mr.prompt_tokens(13, 5, 333, d.vocab)
        rid = 5
        with Instance("tiny", device=0, **KW) as src:
            first = int(src.step(prefill=[(rid, 0, prompt, True)]).sampled[0])
            src_pages = [int(p) for p in src.kv_pages(rid)]
            here.send((rid, len(prompt)))
            exported, dst_pages = here.recv()
            assert len(dst_pages) >= len(src_pages)
            remote = RemotePool(exported, device=0)
            ev = src.push_pages(remote, src_pages, dst_pages[:len(src_pages)])
            ms, nbytes = ev.wait()
            ev.close()
            assert nbytes == len(src_pages) * exported["page_bytes"] and ms > 0
            want = src.read_pages(src_pages)
            here.send((len(prompt), first))
            got_pages, tok, logits = here.recv()
            remote.close()
        np.testing.assert_array_equal(got_pages[:len(src_pages)], want)
        # the destination continues the request exactly as the source would have
        ref_tokens, ref_logits = model.generate(prompt, 2)
        assert first == ref_tokens[0]
        err = float(np.abs(logits - ref_logits[1].numpy()).max())
        assert err <= 0.05 * float(ref_logits[1].std()) + 0.02, err
        assert tok == ref_tokens[1]
        here.send(None)
    finally:
        proc.join(timeout=120)
        if proc.is_alive():
            proc.kill()
    assert proc.exitcode == 0


def test_ipc_push_same_gpu(cuda_ok):
    _push_roundtrip(0)


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs 2 GPUs (NVLink P2P)")
def test_ipc_push_across_gpus(cuda_ok):
    _push_roundtrip(1)
