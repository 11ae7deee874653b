cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for kb in 200 160 120; do
  echo "== smem $kb" >> gpurun_out/jj_kbench.log
  PSD_GEMM_SK_SMEM_KB=$kb timeout 300 python tools/kbench.py --only gemmgu,gemmpf >> gpurun_out/jj_kbench.log 2>&1
done
echo done
