#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"; mkdir -p gpurun_out; export PYTHONUNBUFFERED=1
timeout 2400 python tools/goodput.py --base configs/b200_c3_4p4d.json --modes hybrid \
  --qps 280,320,360,400 --seeds 0 --model llama3_8b --pool-tokens 140000 --slo 1704,6.39 \
  --profile profiles/r01/b200_calibration_llama3_8b_v3.json --out gpurun_out/goodput_c4_tight_tpot_hybrid.json 2>&1 | tail -6
