import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch, ctypes
from paper_2603_18016_b200 import native
lib = native.load()
dev = torch.device("cuda:0")
torch.manual_seed(0)
for (M, N, K) in [(135, 6144, 4096), (135, 4096, 14336), (24, 4096, 4096)]:
    x = (torch.randn(M, K, device=dev)).to(torch.bfloat16)
    w = (torch.rand(N, K, device=dev) - 0.5).mul(0.0693).to(torch.bfloat16)
    ref = x.double() @ w.double().T
    outs = {}
    for S in (1, 2, 3, 4, 0):
        P = torch.zeros(8 * M * N, device=dev)
        su = ctypes.c_int()
        rc = lib.psd_gemm_partials(x.data_ptr(), K, M, K, w.data_ptr(), K, N, P.data_ptr(), P.numel() * 4,
                                   S, ctypes.byref(su), torch.cuda.current_stream().cuda_stream)
        assert rc == 0
        torch.cuda.synchronize()
        y = P[:su.value * M * N].view(su.value, M, N).sum(0).double()
        outs[S] = (su.value, y)
        rel = ((y - ref).abs() / ref.abs().clamp_min(1e-3)).median().item()
        print(M, N, K, "S", S, "->", su.value, "max|y-ref|", (y - ref).abs().max().item(), "ref rms", ref.pow(2).mean().sqrt().item(), "median rel", rel)
    print("  S1 vs S3 max diff", (outs[1][1] - outs[3][1]).abs().max().item())
