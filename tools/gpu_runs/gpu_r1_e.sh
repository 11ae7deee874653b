cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_psd_gpu.py -x -q > gpurun_out/pytest_psd.log 2>&1
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench2.log 2>&1
echo done
