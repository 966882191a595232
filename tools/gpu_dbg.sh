#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"; mkdir -p gpurun_out; export PYTHONUNBUFFERED=1
for d in 0 1 2 3; do
  echo "=== TC_WS_DBG=$d"
  TC_WS_DBG=$d TC_WS_TRACE=1 timeout 300 python tools/ws_trace.py > /dev/null 2> gpurun_out/trace_dbg$d.txt
  python3 - <<PY
blocks=[];cur=None
for line in open("gpurun_out/trace_dbg$d.txt"):
    if line.startswith("ws_trace"): cur=[line.rstrip()]; blocks.append(cur)
    elif cur is not None and line.startswith("  "): cur.append(line.rstrip())
for b in blocks[2::3][:2]:
    print(b[0][:60]); print("\n".join(x for x in b if any(k in x for k in ("last_mma","epi_start","c0_","c2_","c4_","epi_last"))))
PY
done
