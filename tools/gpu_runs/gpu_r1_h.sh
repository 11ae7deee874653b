cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_all.log 2>&1
timeout 300 python tools/prof_step.py 48 1 1 > gpurun_out/prof_step_dual3.log 2>&1
timeout 300 python tools/prof_step.py 48 0 1 > gpurun_out/prof_step_single3.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 20000 -c 4000 --csv --log-file gpurun_out/step_launches3.csv python tools/prof_step.py 16 0 1 > gpurun_out/ncu_step3.log 2>&1
echo done
