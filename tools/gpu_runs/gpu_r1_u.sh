cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_pair_gpu.py tests/test_gemm_gpu.py tests/test_layers_gpu.py tests/test_psd_gpu.py -q > gpurun_out/pytest_u.log 2>&1
timeout 120 python tools/kbench.py --only gemmx > gpurun_out/kbench9.log 2>&1
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench5.log 2>&1
echo done
