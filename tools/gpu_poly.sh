#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"; mkdir -p gpurun_out; export PYTHONUNBUFFERED=1
for v in TC_PF_POLY=0 TC_PF_POLY=1 TC_PF_POLY=2; do
  true || env $v timeout 300 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_step.py 2>&1 | tail -1
  for a in "--prefill 1024 --prefix 4096 --decode 0"; do
    env $v timeout 600 python bench.py --no-cpu-baseline $a > gpurun_out/bench_poly.json 2> gpurun_out/bench_poly.err
    python3 -c "
import json; d=json.load(open('gpurun_out/bench_poly.json'))
print('$v $a', 'value', round(d['value']), 'ms', round(d['ms_per_step'],3), 'attn', round(d['step_roofline']['phase_ms']['attn'],3))" || tail -3 gpurun_out/bench_poly.err
  done
done
