#!/usr/bin/env python3
"""Microbenchmark of the tcgen05 GEMM (tc_gemm) on the hybrid-step shapes.
Times each (shape, tile width, split) with CUDA events over 20 back-to-back launches."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2508_01989_b200 import runtime  # noqa: E402

SHAPES = {  # name: (M, N, K, epilogue)
    "qkv": (576, 6144, 4096, 0), "o": (576, 4096, 4096, 2), "gate_up": (576, 28672, 4096, 3),
    "down": (576, 4096, 14336, 2), "lm_head": (65, 128256, 4096, 4),
    "qkv_d64": (64, 6144, 4096, 0), "o_d64": (64, 4096, 4096, 2), "gate_up_d64": (64, 28672, 4096, 3),
    "down_d64": (64, 4096, 14336, 2), "gate_up_1100": (1100, 28672, 4096, 3),
}
VARIANTS = [(0, 0), (256, 1), (256, 3), (256, 5), (512, 0), (1024, 0), (1024, 1), (1024, 2), (1024, 3), (1024, 5)]


def main():
    import os
    out = {}
    only = [x for x in os.environ.get("GEMM_SHAPES", "").split(",") if x]
    for name, (m, n, k, epi) in SHAPES.items():
        if only and name not in only:
            continue
        a = torch.randn(m, k, device="cuda", dtype=torch.bfloat16)
        b = torch.randn(n, k, device="cuda", dtype=torch.bfloat16) * 0.02
        o = torch.zeros(m, n // 2 if epi == 3 else n, device="cuda",
                        dtype=torch.float32 if epi in (2, 4) else torch.bfloat16)
        res = {}
        for bn, sp in VARIANTS:
            if n % (bn or 128):
                continue
            try:
                for _ in range(3):
                    runtime.gemm(a.data_ptr(), b.data_ptr(), o.data_ptr(), m, n, k, epi, None, bn, sp)
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(20):
                    runtime.gemm(a.data_ptr(), b.data_ptr(), o.data_ptr(), m, n, k, epi, None, bn, sp)
                e1.record()
                torch.cuda.synchronize()
                us = e0.elapsed_time(e1) / 20 * 1e3
            except Exception as ex:  # noqa: BLE001
                us = str(ex)[:60]
            res[f"bn{bn}_s{sp}"] = us
        # same-box comparison point (NOT our path): cuBLAS via torch.matmul on the same operands
        try:
            for _ in range(3):
                torch.matmul(a, b.t())
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(20):
                torch.matmul(a, b.t())
            e1.record()
            torch.cuda.synchronize()
            res["cublas_bf16"] = e0.elapsed_time(e1) / 20 * 1e3
        except Exception as ex:  # noqa: BLE001
            res["cublas_bf16"] = str(ex)[:60]
        flops = 2.0 * m * n * k
        best = min((v for kk, v in res.items() if isinstance(v, float) and kk != "cublas_bf16"), default=None)
        out[name] = {"M": m, "N": n, "K": k, "us": res, "best_tflops": flops / best / 1e6 if best else None}
        print(name, {k: (round(v, 1) if isinstance(v, float) else v) for k, v in res.items()},
              "best TF/s %.0f" % (flops / best / 1e6), flush=True)
    json.dump(out, open(os.environ.get("GEMM_BENCH_OUT", "gpurun_out/gemm_bench.json"), "w"), indent=1)


if __name__ == "__main__":
    main()
