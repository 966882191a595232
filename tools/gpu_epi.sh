#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"; mkdir -p gpurun_out; export PYTHONUNBUFFERED=1
timeout 300 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_gemm.py > gpurun_out/epi_gemm_tests.txt 2>&1; echo "rc=$?"; tail -4 gpurun_out/epi_gemm_tests.txt
timeout 600 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_step.py > gpurun_out/epi_step_tests.txt 2>&1; echo "rc=$?"; tail -4 gpurun_out/epi_step_tests.txt
GEMM_SHAPES=qkv,o,gate_up,down timeout 300 python tools/gemm_bench.py 2>&1 | cut -c1-200
VARIANTS="TC_GEMM_WS=1" TESTS=tests/test_abi.py bash tools/gpu_ab.sh
bash tools/gpu_trace.sh 2>&1 | tail -36
