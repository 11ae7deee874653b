cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_pair_gpu.py -q -x > gpurun_out/q_pytest_pair.log 2>&1
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/q_pytest.log 2>&1
timeout 900 python bench.py > gpurun_out/q_bench.log 2>&1
echo done
