cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gemm_gpu.py -q -x -k "trace or schedules" > gpurun_out/bf_pytest.log 2>&1
echo done
