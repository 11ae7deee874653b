import sys, os
sys.path.insert(0, os.getcwd())
import torch
from paper_2603_18016_b200 import SimConfig, make_requests, run
from paper_2603_18016_b200.gpu import GpuBackend
dev = torch.device("cuda:0")
def outs(tgt, drf, mode, k, N=4, OUT=12, mb=4, bt=7.0, bd=16.0, prompt=128, **kw):
    gb = GpuBackend(tgt, drf, max_requests=N, max_batch=mb, k_max=k, max_seq_len=prompt + OUT + 16,
                    seed=0, beta_target=bt, beta_draft=bd, device=dev, **kw)
    cfg = (SimConfig(mode="psd", m=N // 2, k=k) if mode == "psd" else
           SimConfig(mode="standard-sd", m=N // 2, k=k, sd_batch_factor=2))
    st, rep = run(cfg, make_requests([OUT] * N, prompt_len=prompt), backend=gb)
    return [r.output_ids for r in st.request_list()]
for tgt, drf, bt, bd in [("tiny-target", "tiny-draft", 3.0, 12.0), ("llama-3.1-8b", "tiny-draft", 7.0, 12.0),
                         ("tiny-target", "llama-3.2-1b", 3.0, 16.0), ("llama-3.2-1b", "llama-3.2-1b", 7.0, 16.0)]:
    if tgt.startswith("tiny") and drf.startswith("llama"):
        continue  # vocab mismatch
    for prompt in (128, 16):
        a = outs(tgt, drf, "psd", 5, bt=bt, bd=bd, prompt=prompt)
        b = outs(tgt, drf, "sd", 5, bt=bt, bd=bd, prompt=prompt)
        c = outs(tgt, drf, "sd", 1, bt=bt, bd=bd, prompt=prompt)
        print(tgt, drf, prompt, "psd==sd5", a == b, "psd==sd1", a == c, "sd1==sd5", b == c,
              [i for i in range(4) if a[i] != b[i]], flush=True)
