cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/av_pytest.log 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/av_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/av_bench.log 2>&1
timeout 600 python bench.py --impl reference > gpurun_out/av_bench_ref.log 2>&1
echo done
