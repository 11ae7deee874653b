cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python tools/mk_trace.py 32 5 > gpurun_out/l_trace.log 2>&1
timeout 300 python tools/mk_trace.py 32 1 > gpurun_out/l_trace1.log 2>&1
echo done
