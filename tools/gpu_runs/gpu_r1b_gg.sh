cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
PSD_GEMM_MW2=1 timeout 600 python -m pytest tests/test_gemm_gpu.py -q -x > gpurun_out/gg_pytest_mw2.log 2>&1
PSD_GEMM_MW2=0 timeout 300 python tools/kbench.py --only gemmmw > gpurun_out/gg_kb_mw1.log 2>&1
PSD_GEMM_MW2=1 timeout 300 python tools/kbench.py --only gemmmw > gpurun_out/gg_kb_mw2.log 2>&1
echo done
