cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python tools/kbench.py > gpurun_out/b_kbench.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:verify -c 4 -o gpurun_out/b_verify python tools/prof_verify.py > gpurun_out/b_ncu_verify.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm -s 20 -c 6 -o gpurun_out/b_gemm_draft python tools/kbench.py --only gemm1b > gpurun_out/b_ncu_gemm1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_sk -s 10 -c 2 -o gpurun_out/b_gemm_gu python tools/kbench.py --only gemmgu > gpurun_out/b_ncu_gemm2.log 2>&1
echo done
