cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 300 python -m pytest tests/test_gpu_gemm.py -q -x -p no:cacheprovider 2>&1 | tail -40 > gpurun_out/gemm_tests.txt
timeout 600 python -m pytest tests/test_gpu_step.py -q -p no:cacheprovider 2>&1 | tail -60 > gpurun_out/step_tests.txt
echo done
