#!/bin/bash
# quick A/B: step parity tests + bench (ws on / off) + optional extra command
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest -q -x -p no:cacheprovider -m gpu ${TESTS:-tests} > gpurun_out/ab_tests.txt 2>&1; tail -3 gpurun_out/ab_tests.txt
for v in ${VARIANTS:-"TC_GEMM_WS=1"}; do
  env $v timeout 600 python bench.py --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/bench_ab.json 2> gpurun_out/bench_ab.err
  python3 -c "
import json; d=json.load(open('gpurun_out/bench_ab.json'))
print('$v', 'value', round(d['value']), 'e2e', round(d['e2e']['value']), 'ms', round(d['ms_per_step'],3), 'frac', round(d['step_roofline']['frac'],3))
print({k: round(v, 3) for k, v in d['step_roofline']['phase_ms'].items()})
print('migration', d.get('migration'))" || tail -5 gpurun_out/bench_ab.err
done
