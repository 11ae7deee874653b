import sys, os, dataclasses
sys.path.insert(0, os.getcwd())
import torch
from paper_2603_18016_b200 import SimConfig, make_requests, run
from paper_2603_18016_b200.gpu import GpuBackend
from paper_2603_18016_b200.model import PRESETS
dev = torch.device("cuda:0")
def outs(tgt, drf, mode, N=4, k=5, mb=4, OUT=16):
    gb = GpuBackend(tgt, drf, max_requests=N, max_batch=mb, k_max=k, max_seq_len=128 + OUT + 16,
                    seed=0, beta_target=7.0, beta_draft=16.0, device=dev)
    cfg = (SimConfig(mode="psd", m=N // 2, k=k) if mode == "psd" else
           SimConfig(mode="standard-sd", m=N // 2, k=k, sd_batch_factor=2))
    st, rep = run(cfg, make_requests([OUT] * N, prompt_len=128), backend=gb)
    o = [r.output_ids for r in st.request_list()]
    del gb; torch.cuda.empty_cache()
    return o
base_t, base_d = PRESETS["llama-3.1-8b"], PRESETS["llama-3.2-1b"]
for L in (1, 2, 4, 8, 16, 32):
    PRESETS[f"t{L}"] = dataclasses.replace(base_t, name=f"t{L}", layers=L)
    a = outs(f"t{L}", "llama-3.2-1b", "psd"); b = outs(f"t{L}", "llama-3.2-1b", "sd")
    print("target layers", L, "psd==sd", a == b, [(i, next(j for j in range(16) if a[i][j] != b[i][j])) for i in range(4) if a[i] != b[i]], flush=True)
for L in (1, 2, 4, 16):
    PRESETS[f"d{L}"] = dataclasses.replace(base_d, name=f"d{L}", layers=L)
    a = outs("llama-3.1-8b", f"d{L}", "psd"); b = outs("llama-3.1-8b", f"d{L}", "sd")
    print("draft layers", L, "psd==sd", a == b, [(i, next(j for j in range(16) if a[i][j] != b[i][j])) for i in range(4) if a[i] != b[i]], flush=True)
