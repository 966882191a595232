#!/bin/bash
# One GPU session: parity tests, smoke, bench, ncu launch list + full captures.
# Outputs land in gpurun_out/ (merged back by gpurun).
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
nvidia-smi > gpurun_out/nvidia_smi.txt 2>&1
lscpu > gpurun_out/lscpu.txt 2>&1; nproc >> gpurun_out/lscpu.txt
STAGES=${STAGES:-"tests smoke bench launches prof"}
for st in $STAGES; do
  case $st in
    tests) timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_tests.txt 2>&1; tail -5 gpurun_out/gpu_tests.txt ;;
    smoke) timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; tail -2 gpurun_out/smoke.txt ;;
    bench) timeout 900 python bench.py ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -c 600 gpurun_out/bench.json; tail -3 gpurun_out/bench.err ;;
    launches) timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
        --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --profile-window \
        > gpurun_out/launches_bench.txt 2>&1; wc -l gpurun_out/launches.csv ;;
    prof) timeout 1200 ncu --set full --clock-control none --import-source on --profile-from-start off \
        -k regex:gemm_bf16_tcgen05 -s 2 -c 1 -o gpurun_out/prof_gemm_gate_up -f \
        python bench.py --steps 1 --warmup 3 --no-cpu-baseline --profile-window > gpurun_out/prof_gemm.txt 2>&1
      timeout 1200 ncu --set full --clock-control none --import-source on --profile-from-start off \
        -k regex:attn_decode -s 0 -c 1 -o gpurun_out/prof_attn_decode -f \
        python bench.py --steps 1 --warmup 3 --no-cpu-baseline --profile-window > gpurun_out/prof_attn.txt 2>&1
      ls -la gpurun_out/*.ncu-rep ;;
  esac
done
echo ALLDONE
