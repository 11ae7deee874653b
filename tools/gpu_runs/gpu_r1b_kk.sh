cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gemm_gpu.py -q -x > gpurun_out/kk_pytest.log 2>&1
for i in 1 2; do timeout 300 python tools/kbench.py --only gemmgu,gemmpf >> gpurun_out/kk_kbench.log 2>&1; done
echo done
