cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_verify_gpu.py -q -x > gpurun_out/t_pytest.log 2>&1
timeout 300 python tools/kbench.py --only k1 > gpurun_out/t_kbench.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:verify_stats -s 4 -c 1 -o gpurun_out/t_vstats python tools/prof_verify.py > /dev/null 2>&1
echo done
