cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gemm_gpu.py -x -q > gpurun_out/pytest_gemm.log 2>&1
timeout 300 python -m pytest tests/test_verify_gpu.py -x -q > gpurun_out/pytest_verify.log 2>&1
timeout 300 python -m paper_2603_18016_b200.verify_bench --quick --json gpurun_out/verify_quick2.json > gpurun_out/verify_quick2.log 2>&1
echo done
