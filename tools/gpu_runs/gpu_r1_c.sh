cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_psd_gpu.py -x -q > gpurun_out/pytest_psd.log 2>&1
timeout 300 python -m pytest tests/test_verify_gpu.py tests/test_gemm_gpu.py -x -q > gpurun_out/pytest_vg.log 2>&1
echo done
