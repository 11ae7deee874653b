cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gemm_gpu.py -q -x > gpurun_out/an_pytest.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:attention_kernel --launch-skip 10 -c 1 -o gpurun_out/an_attn_draft python tools/kbench.py --only attn1b > gpurun_out/an_ncu.log 2>&1
echo done
