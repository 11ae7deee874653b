cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/ad_bench.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gemm_sk_kernel --launch-skip 6 -c 1 -o gpurun_out/ad_sk_gu python tools/kbench.py --only gemmgu > gpurun_out/ad_ncu.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ad_launches.csv python tools/prof_step.py 24 1 1 > /dev/null 2>&1
echo done
