cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python tools/kbench.py --only gemmskp > gpurun_out/aq_kbench.log 2>&1
echo done
