#!/usr/bin/env python3
"""Attention microbench on a layer-reduced model (tools only): per-layer device time of the
attention phase (decode-only and mixed steps of BASELINE config 2) for each variant in
--variants ("ENV=a,ENV2=b ENV=c ..."), each in its own process (the library reads its A/B
switches once per process), interleaved --rounds times so box drift hits every variant alike.

  python tools/attn_bench.py --variants "TC_DEC_CFG=4:4 TC_DEC_CFG=6:4" --rounds 2
"""
import argparse
import json
import os
import pathlib
import statistics
import subprocess
import sys

REPO = pathlib.Path(__file__).resolve().parents[1]


def worker(args):
    sys.path.insert(0, str(REPO))
    import numpy as np
    from paper_2508_01989_b200 import Instance
    D, ctx, P, prefix = args.decode, args.ctx, args.prefill, args.prefix
    inst = Instance(f"{args.model}:L{args.layers}", device=0, weight_seed=1,
                    kv_pool_tokens=(D + 2) * (ctx + 64) + prefix + P + 4096, max_step_tokens=max(P + D, 512),
                    max_seqs=D + 8, max_context=max(ctx, prefix + P) + 64)
    V = inst.dims.vocab
    rng = np.random.default_rng(0)
    prompt = rng.integers(0, V, prefix + P).tolist()
    for s in range(0, prefix, 512):
        inst.step(prefill=[(0, s, prompt[s:min(prefix, s + 512)], False)])
    for rid in range(1, D + 1):
        toks = rng.integers(0, V, ctx).tolist()
        for s in range(0, ctx, 512):
            inst.step(prefill=[(rid, s, toks[s:s + 512], False)])
    dec = [(rid, ctx, int(rng.integers(0, V))) for rid in range(1, D + 1)]
    mixed = [(0, prefix, prompt[prefix:prefix + P], True)]
    out = {}
    for name, kw in (("decode_only", dict(decode=dec)), ("mixed", dict(prefill=mixed, decode=dec))):
        for _ in range(3):
            inst.step(**kw)
        inst.set_profiling(True)
        attn, step = [], []
        for _ in range(args.steps):
            o = inst.step(**kw)
            attn.append(inst.phase_ms("attn") / args.layers)
            step.append(o.gpu_ms)
        inst.set_profiling(False)
        out[name] = {"attn_ms_per_layer": statistics.median(attn), "step_ms": statistics.median(step),
                     "pf_sms": o.attn_pf_sms if hasattr(o, "attn_pf_sms") else None}
    d = inst.dims
    kv_bytes = D * (ctx + 1) * 2 * d.n_kv_heads * d.head_dim * 2
    for v in out.values():
        v["decode_kv_gb_s"] = kv_bytes / (v["attn_ms_per_layer"] * 1e-3) / 1e9
    print(json.dumps(out))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--variants", default="TC_DEC_CFG=4:4")
    ap.add_argument("--rounds", type=int, default=2)
    ap.add_argument("--model", default="llama3_8b")
    ap.add_argument("--layers", type=int, default=2)
    ap.add_argument("--decode", type=int, default=64)
    ap.add_argument("--ctx", type=int, default=1024)
    ap.add_argument("--prefill", type=int, default=512)
    ap.add_argument("--prefix", type=int, default=512)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--worker", action="store_true")
    args = ap.parse_args()
    if args.worker:
        return worker(args)
    res = {}
    for r in range(args.rounds):
        for v in args.variants.split():
            env = dict(os.environ)
            for kv in v.split(","):
                k, _, val = kv.partition("=")
                env[k] = val
            cmd = [sys.executable, __file__, "--worker"] + [f"--{k}={getattr(args, k)}" for k in
                                                           ("model", "layers", "decode", "ctx", "prefill", "prefix", "steps")]
            p = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600)
            try:
                j = json.loads(p.stdout.strip().splitlines()[-1])
            except (IndexError, json.JSONDecodeError):
                j = {"error": p.stderr[-400:]}
            res.setdefault(v, []).append(j)
            print(v, json.dumps(j), flush=True)
    summ = {}
    for v, runs in res.items():
        ok = [x for x in runs if "error" not in x]
        if ok:
            summ[v] = {k: round(statistics.median(x[k]["attn_ms_per_layer"] for x in ok) * 1e3, 2) for k in ok[0]}
    print("SUMMARY attn us/layer:", json.dumps(summ))


if __name__ == "__main__":
    main()
