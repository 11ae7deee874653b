cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gemm_gpu.py -q -x > gpurun_out/pp_pytest.log 2>&1
for i in 1 2; do timeout 300 python tools/kbench.py --only gemmgu,gemmpf >> gpurun_out/pp_kbench.log 2>&1; done
PSD_GEMM_TMA_STORE=0 timeout 300 python tools/kbench.py --only gemmgu,gemmpf > gpurun_out/pp_kbench_off.log 2>&1
timeout 300 python tools/sk_trace.py > gpurun_out/pp_trace.log 2>&1
echo done
