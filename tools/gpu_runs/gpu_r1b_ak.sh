cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in 116 100 84 0; do
PSD_VERIFY_CTAS=$v timeout 900 python bench.py --no-cpu-baseline > gpurun_out/ak_bench_$v.log 2>&1
done
echo done
