cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
PSD_LIB=variants/lib_head.so timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/yy_head.log 2>&1
PSD_GEMM_SK_DP=0 timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/yy_nodp.log 2>&1
timeout 900 python -m pytest tests/test_pair_gpu.py -m gpu -q -x > gpurun_out/yy_pairfile.log 2>&1
echo done
