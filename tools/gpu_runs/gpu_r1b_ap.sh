cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
PSD_FUSED_ROPE_MAXQ=16 timeout 900 python bench.py --no-cpu-baseline > gpurun_out/ap_bench_fused16.log 2>&1
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/ap_bench_default.log 2>&1
echo done
