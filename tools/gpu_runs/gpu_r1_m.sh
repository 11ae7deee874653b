cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_layers_gpu.py tests/test_psd_gpu.py tests/test_gemm_gpu.py -q > gpurun_out/pytest_m.log 2>&1
timeout 300 python tools/kbench.py --only gemm,attn,norm > gpurun_out/kbench4.log 2>&1
timeout 300 python tools/prof_step.py 48 0 1 > gpurun_out/prof_step_single6.log 2>&1
timeout 300 python tools/prof_step.py 48 1 1 > gpurun_out/prof_step_dual6.log 2>&1
echo done
