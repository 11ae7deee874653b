cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in nost nobar nosts; do echo "== $v" >> gpurun_out/tt_trace.log; PSD_LIB=variants/lib_$v.so timeout 300 python tools/sk_trace.py >> gpurun_out/tt_trace.log 2>&1; done
echo done
