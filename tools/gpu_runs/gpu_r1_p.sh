cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_psd_gpu.py -x -q > gpurun_out/pytest_p.log 2>&1
echo done
