#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"; mkdir -p gpurun_out; export PYTHONUNBUFFERED=1
for v in product kvil product kvil; do
  if [ $v = product ]; then unset TAICHI_B200_LIB; else export TAICHI_B200_LIB=paper_2508_01989_b200/lib/libtaichi_b200_$v.so; fi
  timeout 600 python bench.py --no-cpu-baseline --steps 60 > gpurun_out/bench_$v.json 2>/dev/null
  python3 -c "
import json; d=json.loads(open('gpurun_out/bench_$v.json').read()); print('$v', round(d['value']), 'ms', round(d['ms_per_step'],3), 'dec', round(d['decode_only_step']['ms'],3), d['clocks']); print({k: round(v,3) for k,v in d['step_roofline']['phase_ms'].items()})"
done
unset TAICHI_B200_LIB
timeout 600 python tools/gemm_bench.py 2>&1 | cut -c1-230 | tail -11
