cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/g_pytest.log 2>&1
timeout 300 python tools/kbench.py --only k1,attn > gpurun_out/g_kbench.log 2>&1
timeout 300 python tools/prof_step.py 48 0 1 > gpurun_out/g_prof_single.log 2>&1
timeout 300 python tools/prof_step.py 48 1 1 > gpurun_out/g_prof_dual.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:verify -c 6 -o gpurun_out/g_verify python tools/prof_verify.py > /dev/null 2>&1
echo done
