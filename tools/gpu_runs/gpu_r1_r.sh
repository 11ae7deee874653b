cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
cat > /tmp/gu.py <<'PY'
import sys; sys.path.insert(0,'.')
import torch
from paper_2603_18016_b200 import ops, native
x=torch.randn(192,4096,device='cuda').to(torch.bfloat16)
ws=[(torch.randn(28672,4096,device='cuda')*0.02).to(torch.bfloat16) for _ in range(3)]
wsp=torch.zeros(64<<20,dtype=torch.uint8,device='cuda')
o1=torch.empty(192,14336,dtype=torch.bfloat16,device='cuda')
o2=torch.empty(192,28672,dtype=torch.bfloat16,device='cuda')
for i in range(6):
    ops.gemm(x, ws[i%3], out=o1, epi=native.EPI_SILU, workspace=wsp)
    ops.gemm(x, ws[i%3], out=o2, epi=native.EPI_BF16, workspace=wsp)
torch.cuda.synchronize()
PY
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_sk_kernel -s 4 -c 2 -o gpurun_out/gu_prof python /tmp/gu.py > gpurun_out/ncu_gu.log 2>&1
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench3.log 2>&1
echo done
