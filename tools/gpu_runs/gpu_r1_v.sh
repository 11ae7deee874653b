cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_attention_gpu.py tests/test_psd_gpu.py -q > gpurun_out/pytest_v.log 2>&1
timeout 200 python tools/kbench.py --only attn > gpurun_out/kbench10.log 2>&1
timeout 300 python tools/prof_step.py 48 0 1 > gpurun_out/prof_step_single8.log 2>&1
echo done
