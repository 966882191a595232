#!/bin/bash
# decode attention iteration: parity tests + decode-only and mixed bench + launch list
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"; mkdir -p gpurun_out; export PYTHONUNBUFFERED=1
timeout 600 python -m pytest -q -x -p no:cacheprovider -m gpu tests/test_gpu_step.py > gpurun_out/step_tests.txt 2>&1; tail -15 gpurun_out/step_tests.txt
for a in "--prefill 0 --prefix 0 --decode 64 --ctx 1024" "--prefill 0 --prefix 0 --decode 16 --ctx 8192" ""; do
  timeout 600 python bench.py --no-cpu-baseline $a > gpurun_out/b.json 2>gpurun_out/b.err || tail -5 gpurun_out/b.err
  python3 -c "
import json; d=json.loads(open('gpurun_out/b.json').read()); k=d['step_roofline']['kernels']
print('[$a]', round(d['value']), 'ms', round(d['ms_per_step'],3), 'attn', round(d['step_roofline']['phase_ms']['attn'],3), 'attn bound', round(k['attn']['bound_ms'],3), 'dec-only', round(d['decode_only_step']['ms'],3))"
done
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/launches_dec.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --profile-window --prefill 0 --prefix 0 > /dev/null 2>&1
python3 tools/launch_table.py gpurun_out/launches_dec.csv
