cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_verify_gpu.py -q -x > gpurun_out/f_pytest.log 2>&1
timeout 300 python tools/kbench.py --only k1 > gpurun_out/f_kbench.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:verify -c 6 -o gpurun_out/f_verify python tools/prof_verify.py > /dev/null 2>&1
PSD_GEMM_PREFETCH=4 timeout 200 python -X faulthandler tools/kbench.py --only gemmpf > gpurun_out/f_pf4.log 2> gpurun_out/f_pf4.err; echo "rc=$?" >> gpurun_out/f_pf4.err
echo done
