#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"; mkdir -p gpurun_out; export PYTHONUNBUFFERED=1
timeout 600 python -m pytest tests/test_gpu_gemm.py -q -x -p no:cacheprovider > gpurun_out/gpu_tests.txt 2>&1; tail -3 gpurun_out/gpu_tests.txt
timeout 600 python tools/gemm_bench.py 2>&1 | tail -12
