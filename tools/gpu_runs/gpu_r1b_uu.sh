cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gemm_gpu.py -q -x > gpurun_out/uu_pytest.log 2>&1
timeout 300 python tools/sk_trace.py > gpurun_out/uu_trace.log 2>&1
timeout 300 python tools/kbench.py --only gemmgu,gemmpf,gemmnt > gpurun_out/uu_kbench.log 2>&1
PSD_GEMM_SK_DP=0 timeout 300 python tools/kbench.py --only gemmgu,gemmpf,gemmnt > gpurun_out/uu_kbench_off.log 2>&1
echo done
