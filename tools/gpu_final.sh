#!/bin/bash
# Evidence refresh: GPU tests, smoke, default bench (with CPU baseline), reference arm, launch
# list, ncu captures of the ws GEMMs / attention / KV copy.
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"; mkdir -p gpurun_out; export PYTHONUNBUFFERED=1
nvidia-smi > gpurun_out/nvidia_smi.txt 2>&1
timeout 900 python -m pytest -q -p no:cacheprovider -m gpu tests > gpurun_out/gpu_tests.txt 2>&1; tail -2 gpurun_out/gpu_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; tail -1 gpurun_out/smoke.txt
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -c 400 gpurun_out/bench.json; echo
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; tail -c 300 gpurun_out/bench_ref.json; echo
bash tools/gpu_prof_all.sh
