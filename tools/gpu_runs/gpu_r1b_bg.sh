cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python bench.py --workload cfg3 --no-cpu-baseline --steps 2 --warmup 3 > gpurun_out/bg_bench_cfg3.log 2>&1
timeout 1500 python bench.py --layout tp --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/bg_bench_cfg4.log 2>&1
echo done
