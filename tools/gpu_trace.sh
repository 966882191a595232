#!/bin/bash
# ws GEMM timelines: isolated (microbench operands) and inside the bench step (last step's launches)
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"; mkdir -p gpurun_out; export PYTHONUNBUFFERED=1
TC_WS_TRACE=1 timeout 300 python tools/ws_trace.py > /dev/null 2> gpurun_out/trace_micro.txt
TC_WS_TRACE=1 timeout 600 python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2> gpurun_out/trace_step.txt
python3 - <<'PY'
import re
def blocks(path):
    out=[]; cur=None
    for line in open(path):
        if line.startswith("ws_trace"):
            cur=[line.rstrip()]; out.append(cur)
        elif cur is not None and line.startswith("  "):
            cur.append(line.rstrip())
    return out
m=blocks("gpurun_out/trace_micro.txt")
print("=== isolated (3rd call of each shape)")
for b in m[2::3]: print("\n".join(b))
s=blocks("gpurun_out/trace_step.txt")
print("=== in-step: launches", len(s), "-> layer 0..1 of the last timed step")
# mixed-step launches (M=576): 3 warm-up steps x 128, then the timed step
mixed=[b for b in s if " M=576 " in b[0]]
print("\n".join("\n".join(b) for b in mixed[3*128:3*128+8]))
PY
