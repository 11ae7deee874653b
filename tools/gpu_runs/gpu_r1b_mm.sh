cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python tools/sk_trace.py > gpurun_out/mm_trace.log 2>&1
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/mm_pytest.log 2>&1
timeout 900 python bench.py > gpurun_out/mm_bench.log 2>&1
echo done
