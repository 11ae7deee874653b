cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gemm_gpu.py -q -x > gpurun_out/ag_pytest.log 2>&1
KB_AUTO_ONLY=1 timeout 300 python tools/kbench.py --only gemmpart,gemmpf > gpurun_out/ag_kbench.log 2>&1
PSD_GEMM_TMA_STORE=0 KB_AUTO_ONLY=1 timeout 300 python tools/kbench.py --only gemmpart,gemmpf > gpurun_out/ag_kbench_off.log 2>&1
echo done
