cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 400 python -m pytest tests/test_pair_gpu.py -q -x > gpurun_out/ba_pytest.log 2>&1
echo done
