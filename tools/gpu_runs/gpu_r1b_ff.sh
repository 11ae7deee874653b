cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/ff_pytest.log 2>&1
timeout 1200 python bench.py --ktune --no-cpu-baseline > gpurun_out/ff_bench_ktune.log 2>&1
echo done
