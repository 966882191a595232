#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"; mkdir -p gpurun_out; export PYTHONUNBUFFERED=1
timeout 900 python -m pytest -q -p no:cacheprovider -m gpu tests > gpurun_out/gpu_tests.txt 2>&1; tail -2 gpurun_out/gpu_tests.txt
for a in "--prefill 512" "--prefill 0 --prefix 0"; do
  timeout 600 python bench.py --no-cpu-baseline $a > gpurun_out/bench_dec.json 2> gpurun_out/bench_dec.err
  python3 -c "
import json; d=json.load(open('gpurun_out/bench_dec.json'))
print('$a', 'value', round(d['value']), 'ms', round(d['ms_per_step'],3), 'frac', round(d['step_roofline']['frac'],3), 'bound', round(d['step_roofline']['bound_ms'],3))
print({k: round(v, 3) for k, v in d['step_roofline']['phase_ms'].items()})" || tail -3 gpurun_out/bench_dec.err
done
TC_WS_TRACE=1 timeout 600 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --prefill 0 --prefix 0 > /dev/null 2> gpurun_out/trace_dec.txt
python3 - <<'PY'
blocks=[];cur=None
for line in open("gpurun_out/trace_dec.txt"):
    if line.startswith("ws_trace"): cur=[line.rstrip()]; blocks.append(cur)
    elif cur is not None and line.startswith("  "): cur.append(line.rstrip())
m=[b for b in blocks if " M=64 " in b[0]]
print(len(m)); print("\n".join("\n".join(b) for b in m[3*128:3*128+4]))
PY
