cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for s in 2 4 8; do echo "== max splits $s" >> gpurun_out/aw_attn.log; PSD_ATT_MAX_SPLITS=$s timeout 300 python tools/kbench.py --only attn >> gpurun_out/aw_attn.log 2>&1; done
echo done
