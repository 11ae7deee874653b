cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gemm_gpu.py -q -x > gpurun_out/o_pytest_gemm.log 2>&1
timeout 600 python -m pytest tests -m gpu -q > gpurun_out/o_pytest.log 2>&1
PSD_GEMM_PAIR=0 timeout 200 python tools/kbench.py --only gemmpf > gpurun_out/o_kb_single.log 2>&1
PSD_GEMM_PAIR=1 timeout 200 python tools/kbench.py --only gemmpf > gpurun_out/o_kb_pair.log 2>&1
PSD_GEMM_PAIR=0 timeout 300 python tools/prof_step.py 48 0 1 > gpurun_out/o_step_single.log 2>&1
PSD_GEMM_PAIR=1 timeout 300 python tools/prof_step.py 48 0 1 > gpurun_out/o_step_pair.log 2>&1
echo done
