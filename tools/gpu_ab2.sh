#!/bin/bash
# gemm parity + microbench subset + bench
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 600 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_gemm.py > gpurun_out/ab2_gemm_tests.txt 2>&1; tail -15 gpurun_out/ab2_gemm_tests.txt
GEMM_SHAPES=${GEMM_SHAPES:-qkv,o,down,o_d64} timeout 600 python tools/gemm_bench.py 2>&1 | cut -c1-400
bash tools/gpu_ab.sh
