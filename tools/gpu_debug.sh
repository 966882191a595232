#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"; mkdir -p gpurun_out; export PYTHONUNBUFFERED=1
timeout 300 python bench.py --no-cpu-baseline --model llama3_8b:L2 --prefill 0 --prefix 0 --steps 3 --warmup 3 2>&1 | tail -3
timeout 300 python bench.py --no-cpu-baseline --model llama3_8b:L2 --steps 3 --warmup 3 2>&1 | tail -3
CUDA_LAUNCH_BLOCKING=1 timeout 300 python bench.py --no-cpu-baseline --model llama3_8b:L4 --prefill 0 --prefix 0 --steps 3 --warmup 3 2>&1 | tail -3
timeout 600 compute-sanitizer --tool memcheck --print-limit 5 python bench.py --no-cpu-baseline --model llama3_8b:L2 --prefill 0 --prefix 0 --steps 3 --warmup 3 --decode 8 --ctx 256 2>&1 | grep -v "^=========     " | head -40
