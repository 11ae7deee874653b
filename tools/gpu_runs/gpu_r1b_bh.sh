cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python bench.py --layout tp --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/bh_bench_cfg4.log 2>&1
timeout 900 python bench.py > gpurun_out/bh_bench.log 2>&1
echo done
