cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python tools/kbench.py --only gemmx > gpurun_out/kbench6.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_sk_kernel -s 8 -c 1 -o gpurun_out/gemm_sk_prof python tools/kbench.py --only gemmx > /dev/null 2>&1
echo done
