#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"; mkdir -p gpurun_out; export PYTHONUNBUFFERED=1
timeout 600 python -m pytest -m gpu -q -x -p no:cacheprovider tests/test_gpu_gemm.py tests/test_gpu_step.py > gpurun_out/gpu_tests.txt 2>&1; tail -3 gpurun_out/gpu_tests.txt
echo "== BK=32 (product)"; timeout 600 python tools/gemm_bench.py 2>&1 | cut -c1-200 | tail -11
cp gpurun_out/gemm_bench.json gpurun_out/gemm_bench_bk32.json
echo "== BK=64"; TAICHI_B200_LIB=paper_2508_01989_b200/lib/libtaichi_b200_bk64.so timeout 600 python tools/gemm_bench.py 2>&1 | cut -c1-200 | tail -11
cp gpurun_out/gemm_bench.json gpurun_out/gemm_bench_bk64.json
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err
python3 -c "
import json; d=json.loads(open('gpurun_out/bench.json').read()); print('value', d['value'], 'ms', d['ms_per_step'], 'frac', d['roofline']['frac']); print({k: round(v,3) for k,v in d['step_roofline']['phase_ms'].items()})"
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:attn_prefill -s 0 -c 1 \
  -o gpurun_out/prof_attn_prefill -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --profile-window > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:gemm_bf16_tcgen05 -s 2 -c 1 \
  -o gpurun_out/prof_gemm_gate_up_bk32 -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --profile-window > /dev/null 2>&1
ls gpurun_out/*.ncu-rep
