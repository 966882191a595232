#!/bin/bash
# decode-attention A/B: KV layout (slab / interleaved) x split merge (fused / separate kernel)
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"; mkdir -p gpurun_out; export PYTHONUNBUFFERED=1
for v in product kvil sepmerge kvil_sepmerge; do
  if [ $v = product ]; then unset TAICHI_B200_LIB; else export TAICHI_B200_LIB=paper_2508_01989_b200/lib/libtaichi_b200_$v.so; fi
  timeout 300 python -m pytest -q -x -p no:cacheprovider -m gpu tests/test_gpu_step.py -k "llama" > /dev/null 2>&1; echo "$v parity rc=$?"
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
    --log-file gpurun_out/launches_$v.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --profile-window > /dev/null 2>&1
  python3 tools/launch_summary.py gpurun_out/launches_$v.csv | grep -E "attn|total"
  timeout 300 python bench.py --no-cpu-baseline --steps 40 > gpurun_out/bench_$v.json 2>/dev/null
  python3 -c "
import json; d=json.loads(open('gpurun_out/bench_$v.json').read()); print('$v', round(d['value']), 'ms', round(d['ms_per_step'],3), 'attn', round(d['step_roofline']['phase_ms']['attn'],3), 'dec-only', round(d['decode_only_step']['ms'],3))"
done
