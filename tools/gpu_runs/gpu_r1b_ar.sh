cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --launch-skip 150000 -c 6000 --log-file gpurun_out/ar_bench_launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ar_bench_under_ncu.log 2>&1
echo done
