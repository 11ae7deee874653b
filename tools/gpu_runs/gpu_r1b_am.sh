cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/am_pytest.log 2>&1
timeout 900 python bench.py > gpurun_out/am_bench.log 2>&1
echo done
