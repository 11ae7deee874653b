cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for pr in none draft target; do
  PSD_STREAM_PRIO=$pr timeout 300 python tools/prof_step.py 48 1 1 > gpurun_out/j_dual_$pr.log 2>&1
done
echo done
