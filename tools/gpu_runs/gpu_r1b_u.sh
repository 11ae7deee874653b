cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/u_pytest.log 2>&1
timeout 300 python tools/prof_step.py 48 0 1 > gpurun_out/u_single.log 2>&1
timeout 300 python tools/prof_step.py 48 1 1 > gpurun_out/u_dual.log 2>&1
PSD_FUSED_ROPE=0 timeout 300 python tools/prof_step.py 48 0 1 > gpurun_out/u_single_nofuse.log 2>&1
echo done
