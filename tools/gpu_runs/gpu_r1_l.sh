cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_layers_gpu.py -q > gpurun_out/pytest_layers.log 2>&1
echo done
