cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python tools/prof_step.py 48 1 1 > gpurun_out/prof_step_dual.log 2>&1
timeout 300 python tools/prof_step.py 48 0 1 > gpurun_out/prof_step_single.log 2>&1
timeout 300 python tools/prof_step.py 48 0 0 > gpurun_out/prof_step_nograph.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 20000 -c 4000 --csv --log-file gpurun_out/step_launches.csv python tools/prof_step.py 16 0 1 > gpurun_out/ncu_step.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 5 -c 2 -o gpurun_out/gemm_prof python -c "
import sys; sys.path.insert(0,'.')
import torch
from paper_2603_18016_b200 import ops, native
x=torch.randn(192,4096,device='cuda').to(torch.bfloat16)
ws=[(torch.randn(28672,4096,device='cuda')*0.02).to(torch.bfloat16) for _ in range(4)]
out=torch.empty(192,14336,dtype=torch.bfloat16,device='cuda')
for i in range(8): ops.gemm(x, ws[i%4], out=out, epi=native.EPI_SILU)
torch.cuda.synchronize()
" > gpurun_out/ncu_gemm.log 2>&1
echo done
