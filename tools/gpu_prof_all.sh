#!/bin/bash
# ncu --set full captures of the step's kernels inside a timed bench step (profile window) and of
# the KV migration copy; launch list of 2 timed steps.
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
mkdir -p gpurun_out
NCU="ncu --set full --clock-control none --import-source on"
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline"
timeout 900 $NCU --profile-from-start off -k regex:gemm_ws_2sm -s 0 -c 4 -o gpurun_out/prof_ws -f $B --profile-window > gpurun_out/prof_ws.txt 2>&1
timeout 900 $NCU --profile-from-start off -k regex:attn_ -s 0 -c 2 -o gpurun_out/prof_attn -f $B --profile-window > gpurun_out/prof_attn.txt 2>&1
timeout 900 $NCU -k regex:kv_copy_pages -s 12 -c 1 -o gpurun_out/prof_kvcopy -f $B > gpurun_out/prof_kvcopy.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/launches.csv $B --steps 2 --profile-window > gpurun_out/launches_bench.txt 2>&1
python3 tools/launch_summary.py gpurun_out/launches.csv | tail -14
ls -la gpurun_out/*.ncu-rep
