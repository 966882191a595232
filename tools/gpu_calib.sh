#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"; mkdir -p gpurun_out; export PYTHONUNBUFFERED=1
timeout 900 python -m pytest -m gpu -q -x -p no:cacheprovider tests/test_gpu_serve.py tests/test_gpu_step.py > gpurun_out/gpu_tests.txt 2>&1; tail -3 gpurun_out/gpu_tests.txt
timeout 900 python tools/calibrate.py --model llama3_8b --out gpurun_out/b200_calibration_llama3_8b.json 2>&1 | tail -3
