cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k "regex:attention_kernel<.int.64, .int.32, .int.2, .bool.1>" --launch-skip 300 -c 1 -o gpurun_out/az_attn_draft_rope python tools/prof_step.py 24 1 1 > gpurun_out/az_ncu1.log 2>&1
KB_AUTO_ONLY=1 timeout 600 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k "regex:gemm_kernel<.int.32, .int.4" --launch-skip 60 -c 1 -o gpurun_out/az_gemm_1b_part python tools/kbench.py --only gemmpart > gpurun_out/az_ncu2.log 2>&1
echo done
