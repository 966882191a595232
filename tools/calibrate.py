#!/usr/bin/env python3
"""Fit a B200 CalibrationProfile (cost_model.hpp:19-38) from measured hybrid steps.

Times the real step on one GPU over a (prefill tokens P, decode requests D) grid and fits the
reference's affine form t = base + pp * P + pd * (D - ref) by least squares; kv_bytes_per_token is
the model's (131072 for Llama-3-8B) and link_bandwidth_bytes_per_ms the measured NVLink peer
bandwidth (770 GB/s, B200_PROFILING.md) -- the P2P path cannot be measured on a 1-GPU box.
Writes the profile (config JSON 'profile' block) and the raw grid.

  python tools/calibrate.py --model llama3_8b --out profiles/r01/b200_calibration_llama3_8b.json
"""
import argparse
import json
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2508_01989_b200 import Instance  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="llama3_8b")
    ap.add_argument("--ctx", type=int, default=512, help="decode context length")
    ap.add_argument("--out", required=True)
    ap.add_argument("--repeats", type=int, default=5)
    args = ap.parse_args()
    Ps = [0, 64, 128, 256, 512, 1024]
    Ds = [1, 8, 16, 32, 64, 128]
    maxD, ctx = max(Ds), args.ctx
    inst = Instance(args.model, kv_pool_tokens=(maxD + 4) * (ctx + 64) + 4096, max_step_tokens=max(Ps) + maxD + 64,
                    max_seqs=maxD + 8, max_context=ctx + 2048)
    V = inst.dims.vocab
    rng = np.random.default_rng(0)
    for rid in range(1, maxD + 1):  # decode contexts
        toks = rng.integers(0, V, ctx).tolist()
        for s in range(0, ctx, 512):
            inst.step(prefill=[(rid, s, toks[s:s + 512], False)])
    prompt = rng.integers(0, V, max(Ps)).tolist()
    rows = []
    for P in Ps:
        for D in Ds:
            if P == 0 and D == 0:
                continue
            pre = [(0, 0, prompt[:P], True)] if P else []
            dec = [(rid, ctx, 7) for rid in range(1, D + 1)]
            ms = []
            for _ in range(args.repeats + 2):
                ms.append(inst.step(prefill=pre, decode=dec).gpu_ms)
            rows.append({"P": P, "D": D, "ms": float(np.median(ms[2:]))})
            print(rows[-1], flush=True)
    ref = 16
    A = np.array([[1.0, r["P"], r["D"] - ref] for r in rows])
    y = np.array([r["ms"] for r in rows])
    coef, *_ = np.linalg.lstsq(A, y, rcond=None)
    pred = A @ coef
    r2 = 1 - ((y - pred) ** 2).sum() / ((y - y.mean()) ** 2).sum()
    kv_per_tok = 2 * inst.dims.n_layers * inst.dims.n_kv_heads * inst.dims.head_dim * 2
    prof = {"base_iter_ms": float(coef[0]), "per_prefill_token_ms": float(coef[1]),
            "per_decode_req_ms": float(max(coef[2], 1e-4)), "ref_decode_batch": ref,
            "kv_bytes_per_token": int(kv_per_tok), "link_bandwidth_bytes_per_ms": 770e6}
    out = {"model": args.model, "decode_ctx": ctx, "profile": prof, "r2": float(r2),
           "max_rel_err": float(np.max(np.abs(pred - y) / y)), "grid": rows,
           "note": "least-squares fit of cost_model.hpp:43-53's affine form to measured B200 step device time; "
                   "link bandwidth = measured NVLink peer copy (770 GB/s, B200_PROFILING.md)"}
    json.dump(out, open(args.out, "w"), indent=1)
    print(json.dumps({k: out[k] for k in ("profile", "r2", "max_rel_err")}))


if __name__ == "__main__":
    main()
