#!/bin/bash
# ncu full captures of the decode-only step's top kernels
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"; mkdir -p gpurun_out; export PYTHONUNBUFFERED=1
ARGS=${ARGS:-"--prefill 0 --prefix 0 --decode 64 --ctx 1024"}
TAG=${TAG:-dec}
for k in ${KERNELS:-attn_decode}; do
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off \
  -k regex:$k -s ${SKIP:-2} -c 1 -o gpurun_out/prof_${TAG}_$k -f \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --profile-window $ARGS > gpurun_out/prof_${TAG}_$k.txt 2>&1
tail -2 gpurun_out/prof_${TAG}_$k.txt
done
ls -la gpurun_out/*.ncu-rep
