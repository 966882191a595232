#!/bin/bash
# Config 4 SLO sets on config 3's cluster (4P1024 + 4D256, time-shared on one B200): the paper's
# (16 s, 60 ms) tight-TPOT and (5 s, 250 ms) tight-TTFT sets, scaled like the balanced one
# ((6 s, 100 ms) -> (639.1 ms, 10.65 ms), factor 0.1065).
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"; mkdir -p gpurun_out; export PYTHONUNBUFFERED=1
CAL=profiles/r01/b200_calibration_llama3_8b_v3.json
timeout 2400 python tools/goodput.py --base configs/b200_c3_4p4d.json --modes hybrid,aggregation,disaggregation \
  --qps ${TPOT_QPS:-240,320,400,480} --seeds 0 --model llama3_8b --pool-tokens 140000 --slo 1704,6.39 \
  --profile $CAL --out gpurun_out/goodput_c4_tight_tpot.json 2>&1 | grep GOODPUT
timeout 2400 python tools/goodput.py --base configs/b200_c3_4p4d.json --modes hybrid,aggregation,disaggregation \
  --qps ${TTFT_QPS:-480,560,640,720} --seeds 0 --model llama3_8b --pool-tokens 140000 --slo 532.5,26.6 \
  --profile $CAL --out gpurun_out/goodput_c4_tight_ttft.json 2>&1 | grep GOODPUT
