cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gemm_gpu.py -q -x > gpurun_out/cc_pytest_gemm.log 2>&1
PSD_GEMM_NT2=0 timeout 300 python tools/kbench.py --only gemmnt > gpurun_out/cc_kb_nt1.log 2>&1
PSD_GEMM_NT2=1 timeout 300 python tools/kbench.py --only gemmnt > gpurun_out/cc_kb_nt2.log 2>&1
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/cc_pytest.log 2>&1
echo done
