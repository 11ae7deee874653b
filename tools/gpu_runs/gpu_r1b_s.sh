cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_attention_gpu.py tests/test_psd_gpu.py -q -x > gpurun_out/s_pytest.log 2>&1
timeout 300 python tools/kbench.py --only attn > gpurun_out/s_kbench.log 2>&1
timeout 300 python tools/prof_step.py 48 0 1 > gpurun_out/s_single.log 2>&1
timeout 300 python tools/prof_step.py 48 1 1 > gpurun_out/s_dual.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attention_kernel -s 6 -c 1 -o gpurun_out/s_attn_verify python tools/kbench.py --only attn8b > /dev/null 2>&1
echo done
