cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gemm_gpu.py -q -x > gpurun_out/rr_pytest.log 2>&1
timeout 300 python tools/sk_trace.py > gpurun_out/rr_trace.log 2>&1
timeout 300 python tools/kbench.py --only gemmgu,gemmpf >> gpurun_out/rr_kbench.log 2>&1
echo done
