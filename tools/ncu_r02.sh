# ncu --set full captures of the kernels changed in round 2 (session 3), one launch each
set -x
ncu --set full --clock-control none --import-source on -k regex:attention_tma -s 5 -c 1 -o gpurun_out/r02m_attn_tma python tools/kbench.py --only attn8b > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:attn_dec -s 20 -c 1 -o gpurun_out/r02m_attn_dec python tools/draft_breakdown.py llama-3.2-1b 32 300 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:gemm_sk_kernel -s 5 -c 1 -o gpurun_out/r02m_lm_argmax python tools/kbench.py --only lmargmax > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:add_rmsnorm -s 20 -c 1 -o gpurun_out/r02m_norm python tools/draft_breakdown.py llama-3.2-1b 32 300 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02m_draft_step_launches.csv python tools/draft_breakdown.py llama-3.2-1b 32 300 > /dev/null 2>&1
ls gpurun_out | grep r02m
