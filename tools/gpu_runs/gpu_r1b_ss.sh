cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python tools/sk_trace.py > gpurun_out/ss_trace.log 2>&1
echo done
