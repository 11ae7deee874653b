cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_w.log 2>&1
timeout 300 python tools/prof_step.py 48 0 1 > gpurun_out/prof_step_single9.log 2>&1
PSD_PDL=0 timeout 300 python tools/prof_step.py 48 0 1 > gpurun_out/prof_step_single9_nopdl.log 2>&1
timeout 300 python tools/kbench.py --only gemm > gpurun_out/kbench11.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attention_kernel -s 3 -c 1 -o gpurun_out/attn_prof python tools/kbench.py --only attn > /dev/null 2>&1
echo done
