cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_tp_gpu.py -q -x > gpurun_out/v_pytest_tp.log 2>&1
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/v_pytest.log 2>&1
echo done
