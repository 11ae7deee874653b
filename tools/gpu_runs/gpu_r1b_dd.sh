cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/dd_pytest.log 2>&1
timeout 300 python tools/kbench.py --only gemmnt > gpurun_out/dd_kb_nt.log 2>&1
timeout 900 python bench.py > gpurun_out/dd_bench.log 2>&1
timeout 1200 python bench.py --layout tp --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/dd_bench_cfg4.log 2>&1
echo done
