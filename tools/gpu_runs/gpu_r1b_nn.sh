cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python tools/sk_trace.py > gpurun_out/nn_trace.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gemm_sk_kernel --launch-skip 6 -c 1 -o gpurun_out/nn_sk_gu python tools/kbench.py --only gemmgu > gpurun_out/nn_ncu.log 2>&1
echo done
