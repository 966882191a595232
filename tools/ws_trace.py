#!/usr/bin/env python3
"""Per-CTA timeline of the weight-stationary GEMM (TC_WS_TRACE=1 makes the library print a
%globaltimer summary per launch to stderr). Usage: TC_WS_TRACE=1 python tools/ws_trace.py"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2508_01989_b200 import runtime  # noqa: E402

SHAPES = {"qkv": (576, 6144, 4096, 0), "o": (576, 4096, 4096, 2), "gate_up": (576, 28672, 4096, 3),
          "down": (576, 4096, 14336, 2)}
for name, (m, n, k, epi) in SHAPES.items():
    a = torch.randn(m, k, device="cuda", dtype=torch.bfloat16)
    b = torch.randn(n, k, device="cuda", dtype=torch.bfloat16) * 0.02
    o = torch.zeros(m, n // 2 if epi == 3 else n, device="cuda", dtype=torch.float32 if epi == 2 else torch.bfloat16)
    for i in range(3):
        print(f"== {name} call {i}", file=sys.stderr, flush=True)
        runtime.gemm(a.data_ptr(), b.data_ptr(), o.data_ptr(), m, n, k, epi, None, 1024, 0)
    torch.cuda.synchronize()
