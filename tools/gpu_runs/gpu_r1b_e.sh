cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_verify_gpu.py -q -x > gpurun_out/e_pytest.log 2>&1
timeout 300 python tools/kbench.py --only k1 > gpurun_out/e_kbench.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:verify_sample -c 2 -o gpurun_out/e_vsample python tools/prof_verify.py > /dev/null 2>&1
for pf in 0 4 8 16; do
  echo "== PSD_GEMM_PREFETCH=$pf"
  PSD_GEMM_PREFETCH=$pf timeout 200 python tools/kbench.py --only gemmpf
done > gpurun_out/e_prefetch.log 2>&1
echo done
