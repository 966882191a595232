#!/bin/bash
# A/B env variants on the mixed and the decode-only step
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"; mkdir -p gpurun_out; export PYTHONUNBUFFERED=1
for v in ${VARIANTS}; do
for a in "--prefill 512" "--prefill 0 --prefix 0"; do
  env $v timeout 600 python bench.py --no-cpu-baseline $a > gpurun_out/bench_ab3.json 2> gpurun_out/bench_ab3.err
  python3 -c "
import json; d=json.load(open('gpurun_out/bench_ab3.json'))
print('$v $a', 'value', round(d['value']), 'ms', round(d['ms_per_step'],3), 'frac', round(d['step_roofline']['frac'],3))
print('   ', {k: round(v, 3) for k, v in d['step_roofline']['phase_ms'].items()})" || tail -3 gpurun_out/bench_ab3.err
done; done
