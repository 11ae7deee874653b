cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
PSD_DEBUG_LAUNCH=1 timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/ab_debug.log 2>&1
echo done
