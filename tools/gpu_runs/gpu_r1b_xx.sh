cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/xx_default.log 2>&1
PSD_GEMM_TMA_STORE=0 timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/xx_notma.log 2>&1
echo done
