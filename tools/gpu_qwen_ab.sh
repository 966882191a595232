#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"; mkdir -p gpurun_out; export PYTHONUNBUFFERED=1
for v in ${VARIANTS:-TC_PF_SMS=-1 TC_PF_SMS=0 TC_PF_SMS=24 TC_PF_SMS=48}; do
  env $v timeout 900 python bench.py --no-cpu-baseline --model qwen2_5_14b --prefill 1024 --prefix 4096 --decode 32 --ctx 8192 \
    --steps 10 --warmup 3 > gpurun_out/bench_qwen_ab.json 2> gpurun_out/bench_qwen_ab.err
  python3 -c "
import json; d=json.load(open('gpurun_out/bench_qwen_ab.json'))
print('$v', 'value', round(d['value']), 'ms', round(d['ms_per_step'],3), 'attn', round(d['step_roofline']['phase_ms']['attn'],3))" || tail -3 gpurun_out/bench_qwen_ab.err
done
