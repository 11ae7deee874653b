cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in 88 96 92; do PSD_VERIFY_CTAS=$v timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bk_bench_$v.log 2>&1; done
echo done
