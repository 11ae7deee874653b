cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for i in 1 2; do
for v in default noearly ll; do
echo "== $v" >> gpurun_out/af_kbench.log
if [ $v = default ]; then timeout 300 python tools/kbench.py --only gemmgu,gemmpf >> gpurun_out/af_kbench.log 2>&1
else PSD_LIB=variants/lib_$v.so timeout 300 python tools/kbench.py --only gemmgu,gemmpf >> gpurun_out/af_kbench.log 2>&1; fi
done; done
echo done
