cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attention_kernel -s 6 -c 1 -o gpurun_out/r_attn_draft python tools/kbench.py --only attn1b > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attention_kernel -s 6 -c 1 -o gpurun_out/r_attn_verify python tools/kbench.py --only attn8b > /dev/null 2>&1
echo done
