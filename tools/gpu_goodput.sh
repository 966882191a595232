#!/bin/bash
# Wall-clock SLO goodput on B200 (Llama-3-8B-shaped): config 2 (1 aggregated instance) and config 3
# (4P1024 + 4D256, 8 instances emulated on one GPU with shared weights; same-device KV copies priced
# at the measured 770 GB/s NVLink peer bandwidth) for hybrid vs aggregation vs disaggregation.
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"; mkdir -p gpurun_out; export PYTHONUNBUFFERED=1
timeout 1500 python tools/goodput.py --base configs/b200_c2_agg1.json --modes aggregation \
  --qps ${C2_QPS:-4,8,12,16,20,24} --seeds 0 --model llama3_8b --out gpurun_out/goodput_c2.json 2>&1 | tail -12
timeout 3000 python tools/goodput.py --base configs/b200_c3_4p4d.json --modes hybrid,aggregation,disaggregation \
  --qps ${C3_QPS:-40,60,80,100,120} --seeds 0 --model llama3_8b --pool-tokens 110000 \
  --out gpurun_out/goodput_c3.json 2>&1 | tail -25
