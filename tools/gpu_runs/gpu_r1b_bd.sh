cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_attention_gpu.py tests/test_psd_gpu.py tests/test_layers_gpu.py -q -x > gpurun_out/bd_pytest.log 2>&1
for i in 1 2; do timeout 300 python tools/kbench.py --only attnrope >> gpurun_out/bd_attn.log 2>&1; done
echo done
