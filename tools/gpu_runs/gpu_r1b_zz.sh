cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "not strided" > gpurun_out/zz_nostrided.log 2>&1
timeout 900 python -m pytest tests/test_gemm_gpu.py tests/test_pair_gpu.py -m gpu -q -x > gpurun_out/zz_gemm_pair.log 2>&1
timeout 900 python -m pytest tests/test_gemm_gpu.py tests/test_pair_gpu.py -m gpu -q -x -k "strided or pair" > gpurun_out/zz_strided_pair.log 2>&1
echo done
