cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
cat gpurun_out/j_dual_none.log > /dev/null 2>&1
timeout 300 python -m pytest tests/test_psd_gpu.py -q -x -k fused > gpurun_out/k_pytest_fused.log 2>&1
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/k_pytest.log 2>&1
PSD_FUSED_DRAFT=1 timeout 300 python tools/prof_step.py 48 0 1 > gpurun_out/k_single_mk.log 2>&1
PSD_FUSED_DRAFT=1 timeout 300 python tools/prof_step.py 48 1 1 > gpurun_out/k_dual_mk.log 2>&1
PSD_FUSED_DRAFT=1 PSD_MK_GRID=74 timeout 300 python tools/prof_step.py 48 1 1 > gpurun_out/k_dual_mk74.log 2>&1
PSD_FUSED_DRAFT=1 PSD_MK_GRID=100 timeout 300 python tools/prof_step.py 48 1 1 > gpurun_out/k_dual_mk100.log 2>&1
echo done
