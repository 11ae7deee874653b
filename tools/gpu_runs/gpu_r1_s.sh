cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_attention_gpu.py tests/test_layers_gpu.py tests/test_gemm_gpu.py -q > gpurun_out/pytest_s.log 2>&1
timeout 300 python -m pytest tests/test_psd_gpu.py -q >> gpurun_out/pytest_s.log 2>&1
timeout 300 python tools/kbench.py --only attn,gemmx > gpurun_out/kbench8.log 2>&1
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench4.log 2>&1
echo done
