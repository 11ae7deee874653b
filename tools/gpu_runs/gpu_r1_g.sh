cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_attention_gpu.py tests/test_psd_gpu.py -x -q > gpurun_out/pytest_attn.log 2>&1
timeout 300 python tools/prof_step.py 48 1 1 > gpurun_out/prof_step_dual2.log 2>&1
timeout 300 python tools/prof_step.py 48 0 1 > gpurun_out/prof_step_single2.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 20000 -c 4000 --csv --log-file gpurun_out/step_launches2.csv python tools/prof_step.py 16 0 1 > gpurun_out/ncu_step2.log 2>&1
echo done
