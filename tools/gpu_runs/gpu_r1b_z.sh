cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/z_pytest.log 2>&1
timeout 300 python tools/prof_step.py 48 0 1 > gpurun_out/z_single.log 2>&1
timeout 300 python tools/prof_step.py 48 1 1 > gpurun_out/z_dual.log 2>&1
timeout 900 python bench.py > gpurun_out/z_bench.log 2>&1
echo done
