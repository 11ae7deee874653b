cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q > gpurun_out/pytest_q.log 2>&1
timeout 300 python tools/kbench.py --only gemm,gemmx > gpurun_out/kbench7.log 2>&1
timeout 300 python tools/prof_step.py 48 0 1 > gpurun_out/prof_step_single7.log 2>&1
timeout 300 python tools/prof_step.py 48 1 1 > gpurun_out/prof_step_dual7.log 2>&1
echo done
