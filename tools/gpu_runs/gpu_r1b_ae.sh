cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for i in 1 2; do
echo "== default" >> gpurun_out/ae_kbench.log
timeout 300 python tools/kbench.py --only gemmpf >> gpurun_out/ae_kbench.log 2>&1
echo "== f32 per-thread stores, no staging smem" >> gpurun_out/ae_kbench.log
PSD_LIB=variants/lib_f32off.so timeout 300 python tools/kbench.py --only gemmpf >> gpurun_out/ae_kbench.log 2>&1
done
echo done
