cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python tools/kbench.py --only gemmpart > gpurun_out/aa_kb_part.log 2>&1
timeout 300 python tools/kbench.py --only norm,attn > gpurun_out/aa_kb_norm.log 2>&1
echo done
