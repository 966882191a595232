#!/bin/bash
# iteration: GPU step tests + a list of bench configs (BENCHES, ';'-separated) + launch table of the first
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"; mkdir -p gpurun_out; export PYTHONUNBUFFERED=1
timeout ${TEST_TIMEOUT:-240} python -m pytest -q -x -p no:cacheprovider -m gpu ${TESTS:-tests/test_gpu_step.py} > gpurun_out/iter_tests.txt 2>&1; tail -${TEST_TAIL:-4} gpurun_out/iter_tests.txt
IFS=';' read -ra CFGS <<< "${BENCHES:-}"
for a in "${CFGS[@]}"; do
  timeout ${BENCH_TIMEOUT:-240} python bench.py --no-cpu-baseline $a > gpurun_out/b.json 2>gpurun_out/b.err || tail -5 gpurun_out/b.err
  python3 -c "
import json; d=json.loads(open('gpurun_out/b.json').read()); k=d['step_roofline']['kernels']
print('[$a]', round(d['value']), 'ms', round(d['ms_per_step'],3), 'frac', round(d['step_roofline']['frac'],3), {p: round(v,3) for p,v in d['step_roofline']['phase_ms'].items()}, 'attn bound', round(k['attn']['bound_ms'],3), 'dec-only', round(d['decode_only_step']['ms'],3))" 2>/dev/null
done
if [ -n "$LAUNCH" ]; then
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/launches_iter.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --profile-window $LAUNCH > /dev/null 2>&1
python3 tools/launch_table.py gpurun_out/launches_iter.csv
fi
