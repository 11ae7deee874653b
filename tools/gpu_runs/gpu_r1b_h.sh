cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/h_pytest.log 2>&1
timeout 300 python tools/kbench.py --only k1 > gpurun_out/h_kbench.log 2>&1
PSD_K1_TWO_PASS=1 timeout 300 python tools/kbench.py --only k1 > gpurun_out/h_kbench_2p.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:verify -c 6 -o gpurun_out/h_verify python tools/prof_verify.py > /dev/null 2>&1
echo done
