cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python bench.py --workload cfg3 --no-cpu-baseline --steps 2 --warmup 3 > gpurun_out/bj_cfg3.log 2>&1
echo done
