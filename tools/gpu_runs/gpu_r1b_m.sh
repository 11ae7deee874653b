cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_psd_gpu.py -q -x -k fused > gpurun_out/m_pytest.log 2>&1
for pf in 0 1 2; do
PSD_MK_PF=$pf timeout 300 python tools/mk_trace.py 32 5 > gpurun_out/m_trace_pf$pf.log 2>&1
done
echo done
