#!/bin/bash
# quick GPU iteration: gpu tests + bench (+ optional launch list)
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest -m gpu -q -x -p no:cacheprovider ${TESTS:-tests} > gpurun_out/gpu_tests.txt 2>&1; tail -15 gpurun_out/gpu_tests.txt
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err
python3 - <<'PY'
import json
try:
    d = json.loads(open("gpurun_out/bench.json").read())
    print("value", d["value"], "ms", d["ms_per_step"], "frac", d["roofline"]["frac"], "step_frac", d["step_roofline"]["frac"])
    print({k: round(v, 3) for k, v in d["step_roofline"]["phase_ms"].items()})
except Exception as e:
    print("bench parse failed", e)
PY
if [ -n "$LAUNCHES" ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --profile-window > /dev/null 2>&1
  python3 tools/launch_summary.py gpurun_out/launches.csv
fi
