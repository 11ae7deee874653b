cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
PSD_STREAM_PRIO=draft timeout 900 python bench.py --no-cpu-baseline > gpurun_out/as_bench_prio_draft.log 2>&1
PSD_STREAM_PRIO=draft PSD_VERIFY_CTAS=116 timeout 900 python bench.py --no-cpu-baseline > gpurun_out/as_bench_prio_draft_116.log 2>&1
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/as_bench_default.log 2>&1
echo done
