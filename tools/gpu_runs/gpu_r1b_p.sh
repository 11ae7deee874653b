cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for c in 0 132 116 100; do
  PSD_GEMM_PAIR=0 PSD_VERIFY_CTAS=$c timeout 300 python tools/prof_step.py 48 1 1 > gpurun_out/p_dual_$c.log 2>&1
done
echo done
