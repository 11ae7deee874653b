"""70B verify GEMM times at M = 320 (PSD) and 640 (SD(2m)) through the same
calls the forward makes (stream-K for gate/up and the LM head, grid split-K
partials for QKV / O / down), in a CUDA graph, inputs > L2.  Run with
PSD_LIB=<another build> to A/B two builds."""
import ctypes
import sys
sys.path.insert(0, ".")
import torch
from paper_2603_18016_b200 import native, ops

dev = torch.device("cuda:0")
lib = native.load()
g = torch.Generator(device=dev).manual_seed(0)
shapes = [("qkv part", 10240, 8192, "part"), ("o part", 8192, 8192, "part"),
          ("gate/up silu", 57344, 8192, "silu"), ("down part", 8192, 28672, "part"),
          ("lm_head f32", 128256, 8192, "f32")]
for M in (320, 640):
    for name, N, K, kind in shapes:
        nw = max(1, int(3e9 // (N * K * 2)))  # rotate weights: > L2
        ws = [(torch.randn(N, K, device=dev, generator=g) * 0.02).to(torch.bfloat16)
              for _ in range(min(nw, 4))]
        x = torch.randn(M, K, device=dev, generator=g).to(torch.bfloat16)
        part = torch.empty(8 * M * N, device=dev)
        y = torch.empty(M, N // 2 if kind == "silu" else N,
                        dtype=torch.float32 if kind == "f32" else torch.bfloat16, device=dev)
        need = ops.gemm_plan(M, N, K, {"silu": native.EPI_SILU, "f32": native.EPI_F32,
                                       "part": native.EPI_PARTIAL}[kind], 0)[1]
        wsp = torch.zeros(max(need, 16), dtype=torch.uint8, device=dev)
        sp = ctypes.c_int()

        def run():
            st = torch.cuda.current_stream().cuda_stream
            for w in ws:
                if kind == "part":
                    native.check(lib.psd_gemm_partials(x.data_ptr(), K, M, K, w.data_ptr(), K, N,
                                                       part.data_ptr(), part.numel() * 4, 0,
                                                       ctypes.byref(sp), st), name)
                else:
                    e = native.EPI_SILU if kind == "silu" else native.EPI_F32
                    native.check(lib.psd_gemm_bf16(x.data_ptr(), K, M, K, w.data_ptr(), K, N,
                                                   y.data_ptr(), y.shape[1], e, None, 0, 0,
                                                   wsp.data_ptr(), wsp.numel(), st), name)
        run()
        torch.cuda.synchronize()
        gr = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            with torch.cuda.graph(gr, stream=s):
                for _ in range(4):
                    run()
        torch.cuda.current_stream().wait_stream(s)
        gr.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            gr.replay()
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / (5 * 4 * len(ws))
        gbps = N * K * 2 / (us * 1e-6) / 1e9
        print(f"M={M:4d} {name:14s} N={N:6d} K={K:5d} splits={sp.value if kind == 'part' else '-'} "
              f"{us:8.1f} us  {gbps:6.0f} GB/s (weights)")
