# A/B of the attention kernels (kbench attn / attnrope) + the GPU tests that cover them
timeout 900 python -m pytest tests/test_attention_gpu.py tests/test_psd_gpu.py -x -q -m gpu > gpurun_out/r02e_attn_tests.log 2>&1; echo tests=$?; tail -3 gpurun_out/r02e_attn_tests.log
for cfg in "PSD_ATT_TMA=0" "PSD_ATT_TMA=1"; do
  echo "== $cfg"; env $cfg timeout 120 python tools/kbench.py --only attn,attnrope 2>&1 | grep -v "verify  \|draft  "
done > gpurun_out/r02e_attn_ab.txt 2>&1
cat gpurun_out/r02e_attn_ab.txt
