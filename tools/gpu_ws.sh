#!/bin/bash
# weight-stationary GEMM bring-up: gemm parity, step parity, microbench, bench A/B
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 600 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_gemm.py > gpurun_out/ws_gemm_tests.txt 2>&1; tail -5 gpurun_out/ws_gemm_tests.txt
timeout 900 python -m pytest -q -x -p no:cacheprovider -m gpu tests > gpurun_out/ws_all_tests.txt 2>&1; tail -5 gpurun_out/ws_all_tests.txt
timeout 600 python tools/gemm_bench.py > gpurun_out/ws_gemm_bench.txt 2>&1; cat gpurun_out/ws_gemm_bench.txt | cut -c1-400
for ws in 1 0; do
  TC_GEMM_WS=$ws timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_ws$ws.json 2> gpurun_out/bench_ws$ws.err
  python3 -c "
import json; d=json.load(open('gpurun_out/bench_ws$ws.json'))
print('ws=$ws', 'value', round(d['value']), 'ms', round(d['ms_per_step'],3), 'frac', round(d['step_roofline']['frac'],3))
print({k: round(v, 3) for k, v in d['step_roofline']['phase_ms'].items()})" || tail -5 gpurun_out/bench_ws$ws.err
done
