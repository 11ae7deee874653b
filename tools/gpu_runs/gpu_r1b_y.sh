cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python tools/kbench.py --only gemmsp > gpurun_out/y_kb_sp.log 2>&1
echo done
