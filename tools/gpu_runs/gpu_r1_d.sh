cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_psd_gpu.py -x -q > gpurun_out/pytest_psd.log 2>&1
timeout 600 python tools/calibrate_beta.py 4,5,6,7,8,10 > gpurun_out/calib.log 2>&1
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench1.log 2>&1
echo done
