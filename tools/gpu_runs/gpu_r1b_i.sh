cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_verify_gpu.py tests/test_psd_gpu.py -q -x > gpurun_out/i_pytest.log 2>&1
timeout 300 python tools/kbench.py --only k1 > gpurun_out/i_kbench.log 2>&1
for pf in 0 1; do
  PSD_L2_PREFETCH=$pf timeout 300 python tools/prof_step.py 48 0 1 > gpurun_out/i_single_pf$pf.log 2>&1
  PSD_L2_PREFETCH=$pf timeout 300 python tools/prof_step.py 48 1 1 > gpurun_out/i_dual_pf$pf.log 2>&1
done
echo done
