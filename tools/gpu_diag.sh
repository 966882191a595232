#!/bin/bash
# Parity diagnosis: logit error budget + determinism under A/B switches, sanitizer on the tiny step.
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"; mkdir -p gpurun_out; export PYTHONUNBUFFERED=1
for v in "" "TC_PDL=0" "TC_WS_SPLITS=1" "TC_PDL=0 TC_WS_SPLITS=1 TC_PF_SMS=0"; do
  tag=$(echo "base $v" | tr ' =' '__')
  env $v timeout 600 python tools/parity_budget.py --out gpurun_out/budget_$tag.json > gpurun_out/budget_$tag.txt 2>&1
  echo "== $v"; tail -c 600 gpurun_out/budget_$tag.txt; echo
done
timeout 600 python tools/parity_budget.py --model qwen2_5_14b:L2 --seed 5 --n-req 8 --repeats 2 --out gpurun_out/budget_qwen.json > gpurun_out/budget_qwen.txt 2>&1
echo "== qwen"; tail -c 600 gpurun_out/budget_qwen.txt; echo
for tool in racecheck synccheck memcheck; do
  timeout 600 /usr/local/cuda/bin/compute-sanitizer --tool $tool --print-limit 20 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/san_$tool.txt 2>&1
  echo "== $tool rc=$?"; tail -5 gpurun_out/san_$tool.txt
done
