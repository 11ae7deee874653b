cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=tests/test_pair_gpu.py::test_pair_gpu_sampling_ships_q_rows
timeout 300 python -m pytest $T -q -x > gpurun_out/ww_default.log 2>&1
PSD_GEMM_TMA_STORE=0 timeout 300 python -m pytest $T -q -x > gpurun_out/ww_notma.log 2>&1
PSD_GEMM_SK_DP=0 timeout 300 python -m pytest $T -q -x > gpurun_out/ww_nodp.log 2>&1
timeout 300 python -m pytest tests/test_psd_gpu.py::test_tiny_forward_matches_oracle -q -x > gpurun_out/ww_tiny.log 2>&1
echo done
