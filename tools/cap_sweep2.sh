# cfg2 PSD tok/s vs the verify GEMM CTA cap beside the draft stream
# (PSD_VERIFY_CTAS; 0 = all SMs); prints cap, PSD, SD(2m), hidden fraction
for v in "$@"; do
  PSD_VERIFY_CTAS=$v timeout 600 python bench.py --no-sweep --no-cpu-baseline > gpurun_out/cap_$v.log 2>&1
  tail -1 gpurun_out/cap_$v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print($v, d['value'], d['sd']['value'], d['draft_hiding']['draft_hidden_frac'], d['clocks']['sm_mhz'])"
done
