cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gemm_gpu.py -q -x > gpurun_out/x_pytest_gemm.log 2>&1
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/x_pytest.log 2>&1
PSD_GEMM_DSMEM=0 timeout 200 python tools/kbench.py --only gemmpf > gpurun_out/x_kb_nodsmem.log 2>&1
PSD_GEMM_DSMEM=1 timeout 200 python tools/kbench.py --only gemmpf > gpurun_out/x_kb_dsmem.log 2>&1
PSD_GEMM_DSMEM=0 timeout 300 python tools/prof_step.py 48 0 1 > gpurun_out/x_single_nodsmem.log 2>&1
PSD_GEMM_DSMEM=1 timeout 300 python tools/prof_step.py 48 0 1 > gpurun_out/x_single_dsmem.log 2>&1
PSD_GEMM_DSMEM=1 timeout 300 python tools/prof_step.py 48 1 1 > gpurun_out/x_dual_dsmem.log 2>&1
echo done
