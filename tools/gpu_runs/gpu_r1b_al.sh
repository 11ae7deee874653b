cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in 116:0 92:0 84:0 84:64 116:32 92:0; do
  vc=${v%%:*}; dc=${v##*:}
  PSD_VERIFY_CTAS=$vc PSD_DRAFT_CTAS=$dc timeout 900 python bench.py --no-cpu-baseline >> gpurun_out/al_bench_${vc}_${dc}.log 2>&1
done
echo done
