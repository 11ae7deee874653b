cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_verify_gpu.py -q -x > gpurun_out/c_pytest.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/c_smoke.log 2>&1
timeout 300 python tools/kbench.py --only k1,norm > gpurun_out/c_kbench_new.log 2>&1
PSD_K1_LEGACY=1 timeout 300 python tools/kbench.py --only k1 > gpurun_out/c_kbench_legacy.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:verify -c 12 -o gpurun_out/c_verify python tools/prof_verify.py > gpurun_out/c_ncu_verify.log 2>&1
echo done
