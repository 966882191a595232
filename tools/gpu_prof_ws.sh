#!/bin/bash
# ncu full capture of the first weight-stationary GEMM launches inside a timed step (qkv, o)
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
mkdir -p gpurun_out
timeout 1200 ncu --set full --clock-control none --import-source on --profile-from-start off \
  -k regex:gemm_ws_2sm -s 0 -c ${COUNT:-4} -o gpurun_out/prof_ws -f \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --profile-window > gpurun_out/prof_ws.txt 2>&1
tail -3 gpurun_out/prof_ws.txt; ls -la gpurun_out/prof_ws.ncu-rep
