#!/bin/bash
# Round-1 v7 goodput: recalibrate the cost model on the current kernels, then wall-clock SLO
# goodput for config 2 (1 aggregated instance) and config 3 (4P1024 + 4D256 emulated on one GPU).
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"; mkdir -p gpurun_out; export PYTHONUNBUFFERED=1
[ -n "$SKIP_CAL" ] || timeout 900 python tools/calibrate.py --model llama3_8b --out gpurun_out/b200_calibration_llama3_8b.json 2>&1 | tail -3
[ -n "$SKIP_C2" ] || timeout 1200 python tools/goodput.py --base configs/b200_c2_agg1.json --modes aggregation \
  --qps ${C2_QPS:-24,32,40,48,56} --seeds 0 --model llama3_8b --profile ${CAL:-gpurun_out/b200_calibration_llama3_8b.json} \
  --out gpurun_out/goodput_c2.json 2>&1 | tail -8
timeout 2400 python tools/goodput.py --base configs/b200_c3_4p4d.json --modes hybrid,aggregation,disaggregation \
  --qps ${C3_QPS:-120,160,200,240} --seeds 0 --model llama3_8b --pool-tokens ${POOL:-110000} \
  --profile ${CAL:-gpurun_out/b200_calibration_llama3_8b.json} --out gpurun_out/goodput_c3.json 2>&1 | tail -16
