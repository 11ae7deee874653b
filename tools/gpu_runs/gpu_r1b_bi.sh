cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
PSD_VERIFY_CTAS=0 timeout 1200 python bench.py --workload cfg3 --no-cpu-baseline --steps 2 --warmup 3 > gpurun_out/bi_cfg3_nocap.log 2>&1
PSD_VERIFY_CTAS=104 timeout 1200 python bench.py --workload cfg3 --no-cpu-baseline --steps 2 --warmup 3 > gpurun_out/bi_cfg3_104.log 2>&1
timeout 1200 python bench.py --workload cfg3 --no-cpu-baseline --steps 2 --warmup 3 > gpurun_out/bi_cfg3_default.log 2>&1
echo done
