cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/ay_pytest.log 2>&1
timeout 300 python tools/kbench.py --only norm > gpurun_out/ay_norm.log 2>&1
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/ay_bench.log 2>&1
echo done
