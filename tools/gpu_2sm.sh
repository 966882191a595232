#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"; mkdir -p gpurun_out; export PYTHONUNBUFFERED=1
# hard timeouts: a pairing bug in the 2-SM kernel would hang rather than fail
timeout 180 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_gemm.py -k 2sm > gpurun_out/gpu_tests_2sm.txt 2>&1; echo "2sm tests rc=$?"; tail -5 gpurun_out/gpu_tests_2sm.txt
if grep -q " passed" gpurun_out/gpu_tests_2sm.txt && ! grep -q "failed" gpurun_out/gpu_tests_2sm.txt; then
  timeout 300 python tools/gemm_bench.py 2>&1 | cut -c1-260 | tail -11
fi
