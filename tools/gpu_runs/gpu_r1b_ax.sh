cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_attention_gpu.py -q -x > gpurun_out/ax_pytest.log 2>&1
for s in 2 4 8; do echo "== max splits $s" >> gpurun_out/ax_attn.log; PSD_ATT_MAX_SPLITS=$s timeout 300 python tools/kbench.py --only attn >> gpurun_out/ax_attn.log 2>&1; done
echo done
