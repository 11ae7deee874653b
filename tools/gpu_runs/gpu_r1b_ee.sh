cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_verify_gpu.py -q -x > gpurun_out/ee_pytest.log 2>&1
timeout 300 python tools/kbench.py --only k1 > gpurun_out/ee_kbench.log 2>&1
echo done
