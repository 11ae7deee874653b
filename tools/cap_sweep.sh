# PSD tok/s at cfg2 vs the verify GEMM CTA cap (PSD_VERIFY_CTAS; 0 = all SMs)
for v in 0 74 92 104 120 136; do
  echo "== PSD_VERIFY_CTAS=$v"
  PSD_VERIFY_CTAS=$v timeout 300 python tools/prof_step.py 256 1 1 2>&1 | head -1
done
