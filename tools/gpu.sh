#!/bin/bash
# One parameterised GPU session (run on the B200 box: gpurun -- 'STAGES="tests bench" bash tools/gpu.sh').
# Every stage writes under gpurun_out/ (merged back by gpurun). Stages:
#   tests     all -m gpu tests                     smoke    __graft_entry__.smoke()
#   bench     default bench.py (config 2)          ref      bench.py --impl reference (driver's K/W)
#   qwen      config-5 bench line (Qwen2.5-14B)    dec      decode-only bench line (64 x 1k)
#   launches  ncu launch list of 2 timed steps (mixed and decode-only)
#   prof      ncu --set full of the step kernels ($PROF_K regex, default all step kernels)
#   san       compute-sanitizer racecheck / synccheck / memcheck on smoke()
#   ab        $VARIANTS (space-separated env assignments, comma-joined within one variant) on bench
#   calib     cost-model calibration on the current kernels -> gpurun_out/b200_calibration_$MODEL_$TAG.json
#   goodput   device-clock SLO goodput: GP_BASE config, GP_MODES, GP_QPS, GP_SEEDS (default 0,1,2), GP_SLO
#             (TTFT_ms,TPOT_ms override), GP_MODEL, GP_PROFILE (calibration JSON) -> gpurun_out/goodput_$TAG.json
#   cmd       $CMD (free-form)
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"; mkdir -p gpurun_out; export PYTHONUNBUFFERED=1
TAG=${TAG:-x}
nvidia-smi > gpurun_out/nvidia_smi.txt 2>&1
NCU="ncu --clock-control none"
B="python bench.py --no-cpu-baseline"
for st in ${STAGES:-tests smoke bench}; do
  echo "== $st"
  case $st in
    tests) timeout ${TEST_TIMEOUT:-1500} python -m pytest tests -m gpu -q -p no:cacheprovider -rA ${TEST_ARGS} > gpurun_out/gpu_tests_$TAG.txt 2>&1
      tail -4 gpurun_out/gpu_tests_$TAG.txt ;;
    smoke) timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.txt 2>&1; tail -2 gpurun_out/smoke_$TAG.txt ;;
    bench) timeout 900 python bench.py ${BENCH_ARGS} > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
      tail -c 300 gpurun_out/bench_$TAG.json; echo; tail -3 gpurun_out/bench_$TAG.err ;;
    ref) timeout 900 python bench.py --impl reference --steps ${REF_STEPS:-20} --warmup ${REF_WARMUP:-5} \
        > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err; tail -c 400 gpurun_out/bench_ref_$TAG.json; echo; tail -2 gpurun_out/bench_ref_$TAG.err ;;
    qwen) timeout 900 $B --model qwen2_5_14b --prefill 1024 --prefix 4096 --decode 32 --ctx 8192 ${QWEN_ARGS} \
        > gpurun_out/bench_qwen_$TAG.json 2> gpurun_out/bench_qwen_$TAG.err; tail -c 300 gpurun_out/bench_qwen_$TAG.json; echo ;;
    dec) timeout 900 $B --prefill 0 --prefix 0 > gpurun_out/bench_dec_$TAG.json 2> gpurun_out/bench_dec_$TAG.err
      tail -c 300 gpurun_out/bench_dec_$TAG.json; echo ;;
    launches) timeout 900 $NCU --metrics gpu__time_duration.sum --profile-from-start off --csv \
        --log-file gpurun_out/launches_$TAG.csv $B --steps 2 --warmup 3 --profile-window > gpurun_out/launches_$TAG.txt 2>&1
      python3 tools/launch_summary.py gpurun_out/launches_$TAG.csv > gpurun_out/launches_${TAG}_summary.txt 2>&1; tail -16 gpurun_out/launches_${TAG}_summary.txt
      timeout 900 $NCU --metrics gpu__time_duration.sum --profile-from-start off --csv \
        --log-file gpurun_out/launches_dec_$TAG.csv $B --prefill 0 --prefix 0 --steps 2 --warmup 3 --profile-window > gpurun_out/launches_dec_$TAG.txt 2>&1
      python3 tools/launch_summary.py gpurun_out/launches_dec_$TAG.csv > gpurun_out/launches_dec_${TAG}_summary.txt 2>&1; tail -16 gpurun_out/launches_dec_${TAG}_summary.txt ;;
    prof) timeout 1500 $NCU --set full --import-source on --profile-from-start off -k "regex:${PROF_K:-gemm_ws|attn_|rmsnorm}" \
        -s ${PROF_S:-0} -c ${PROF_C:-8} -o gpurun_out/prof_$TAG -f $B --steps 1 --warmup 3 --profile-window ${PROF_ARGS} > gpurun_out/prof_$TAG.txt 2>&1
      tail -3 gpurun_out/prof_$TAG.txt; ls -la gpurun_out/prof_$TAG.ncu-rep ;;
    san) for tool in racecheck synccheck memcheck; do
        timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool $tool --print-limit 20 python -c "import __graft_entry__ as g; g.smoke()" \
          > gpurun_out/san_${tool}_$TAG.txt 2>&1; echo "$tool rc=$?"; tail -3 gpurun_out/san_${tool}_$TAG.txt
      done ;;
    ab) for v in ${VARIANTS}; do
        n=$(echo "$v" | tr '=,/' '___')
        env ${v//,/ } timeout 600 $B ${BENCH_ARGS} > gpurun_out/ab_${TAG}_$n.json 2>&1
        echo "$v: $(python3 -c "import json,sys; j=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(round(j['value']), round(j['ms_per_step'],3), j.get('decode_only_step',{}) and round(j['decode_only_step']['ms'],3))" gpurun_out/ab_${TAG}_$n.json 2>&1 | tail -1)"
      done ;;
    calib) timeout 1200 python tools/calibrate.py --model ${MODEL:-llama3_8b} --out gpurun_out/b200_calibration_${MODEL:-llama3_8b}_$TAG.json 2>&1 | tail -3 ;;
    goodput) timeout ${GP_TIMEOUT:-3600} python tools/goodput.py --base ${GP_BASE:-configs/b200_c3_4p4d.json} \
        --modes ${GP_MODES:-hybrid,aggregation,disaggregation} --qps ${GP_QPS} --seeds ${GP_SEEDS:-0,1,2} \
        --model ${GP_MODEL:-llama3_8b} ${GP_PROFILE:+--profile $GP_PROFILE} ${GP_SLO:+--slo $GP_SLO} ${GP_ARGS} \
        --out gpurun_out/goodput_$TAG.json > gpurun_out/goodput_$TAG.txt 2>&1; grep GOODPUT gpurun_out/goodput_$TAG.txt ;;
    cmd) bash -c "$CMD" ;;
  esac
done
echo ALLDONE
