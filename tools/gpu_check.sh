#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"; mkdir -p gpurun_out; export PYTHONUNBUFFERED=1
timeout 900 python -m pytest -q -p no:cacheprovider -m gpu tests > gpurun_out/gpu_tests.txt 2>&1; tail -2 gpurun_out/gpu_tests.txt
VARIANTS="${VARIANTS:-TC_PDL=1}" bash tools/gpu_ab3.sh
