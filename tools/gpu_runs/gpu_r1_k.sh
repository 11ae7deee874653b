cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gemm_gpu.py tests/test_attention_gpu.py -x -q > gpurun_out/pytest_sk.log 2>&1
timeout 300 python -m pytest tests/test_psd_gpu.py -x -q >> gpurun_out/pytest_sk.log 2>&1
timeout 300 python tools/kbench.py --json gpurun_out/kbench3.json > gpurun_out/kbench3.log 2>&1
timeout 300 python tools/prof_step.py 48 0 1 > gpurun_out/prof_step_single5.log 2>&1
timeout 300 python tools/prof_step.py 48 1 1 > gpurun_out/prof_step_dual5.log 2>&1
echo done
