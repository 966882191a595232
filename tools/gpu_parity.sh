#!/bin/bash
# Parity evidence: step tests, bench-shape tests, logit error budget (Llama / Qwen shapes).
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"; mkdir -p gpurun_out; export PYTHONUNBUFFERED=1
timeout 1200 python -m pytest -q -p no:cacheprovider tests/test_gpu_step.py tests/test_gpu_bench_shapes.py -rA > gpurun_out/parity_tests.txt 2>&1; tail -15 gpurun_out/parity_tests.txt
timeout 600 python tools/parity_budget.py --out gpurun_out/budget_llama.json > gpurun_out/budget_llama.txt 2>&1; tail -c 500 gpurun_out/budget_llama.txt; echo
timeout 600 python tools/parity_budget.py --model qwen2_5_14b:L2 --seed 5 --n-req 12 --repeats 2 --out gpurun_out/budget_qwen.json > gpurun_out/budget_qwen.txt 2>&1; tail -c 500 gpurun_out/budget_qwen.txt; echo
