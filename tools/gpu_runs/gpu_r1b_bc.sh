cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python tools/kbench.py --only attnrope,attn1b > gpurun_out/bc_attn.log 2>&1
echo done
