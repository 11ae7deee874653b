cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/at_bench.log 2>&1
echo done
