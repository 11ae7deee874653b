cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_psd_gpu.py -q -x -k fused > gpurun_out/n_pytest.log 2>&1
timeout 300 python tools/mk_trace.py 32 5 > gpurun_out/n_trace.log 2>&1
echo done
