cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python tools/kbench.py --json gpurun_out/kbench2.json > gpurun_out/kbench2.log 2>&1
for pf in 4 8 16; do
  PSD_GEMM_PREFETCH=$pf timeout 200 python tools/kbench.py --only gemm > gpurun_out/kbench_pf$pf.log 2>&1
done
echo done
