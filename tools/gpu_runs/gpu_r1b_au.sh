cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
PSD_LIB=variants/lib_fround.so timeout 300 python tools/sk_trace.py > gpurun_out/au_trace_fround.log 2>&1
timeout 300 python tools/sk_trace.py > gpurun_out/au_trace_default.log 2>&1
echo done
