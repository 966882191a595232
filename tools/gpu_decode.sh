#!/bin/bash
# decode-only step: bench phases + launch list
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
ARGS=${ARGS:-"--prefill 0 --prefix 0 --decode 64 --ctx 1024"}
timeout 600 python bench.py --no-cpu-baseline $ARGS > gpurun_out/bench_dec.json 2> gpurun_out/bench_dec.err; tail -3 gpurun_out/bench_dec.err
python3 - <<'PY'
import json
d = json.loads(open("gpurun_out/bench_dec.json").read())
print("value", d["value"], "ms", d["ms_per_step"], "step_frac", d["step_roofline"]["frac"])
print({k: round(v, 3) for k, v in d["step_roofline"]["phase_ms"].items()})
print({k: round(v["bound_ms"], 3) for k, v in d["step_roofline"]["kernels"].items()})
PY
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/launches_dec.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --profile-window $ARGS > /dev/null 2>&1
python3 tools/launch_summary.py gpurun_out/launches_dec.csv
