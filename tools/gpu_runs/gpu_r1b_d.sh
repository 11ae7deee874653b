cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for pf in 0 2 4 8 16; do
  echo "== PSD_GEMM_PREFETCH=$pf"
  PSD_GEMM_PREFETCH=$pf timeout 200 python tools/kbench.py --only gemmpf
done > gpurun_out/d_prefetch.log 2>&1
echo done
