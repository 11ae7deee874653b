"""Bisect the cfg2-shape SD(k=5) divergence: graphs / streams / order."""
import sys, os
sys.path.insert(0, os.getcwd())
import torch
from paper_2603_18016_b200 import SimConfig, make_requests, run
from paper_2603_18016_b200.gpu import GpuBackend

REF0 = [55289, 18730, 79584, 12206, 38020, 93923, 73264, 52550, 54219, 60826, 21654, 12808]
N, OUT, K = 4, 12, 5
dev = torch.device("cuda:0")
tgt = os.environ.get("T", "llama-3.1-8b")
drf = os.environ.get("D", "llama-3.2-1b")
def go(tag, modes, **kw):
    base = dict(max_requests=N, max_batch=4, k_max=K, max_seq_len=128 + OUT + 16, seed=0,
                beta_target=7.0, beta_draft=16.0, device=dev)
    base.update(kw)
    gb = GpuBackend(tgt, drf, **base)
    for mode, k in modes:
        cfg = (SimConfig(mode="psd", m=N // 2, k=k) if mode == "psd" else
               SimConfig(mode="standard-sd", m=N // 2, k=k, sd_batch_factor=2))
        st, rep = run(cfg, make_requests([OUT] * N, prompt_len=128), backend=gb)
        o = [r.output_ids for r in st.request_list()]
        print(tag, mode, k, "req0 ok" if o[0] == REF0 else f"req0 BAD {o[0]}", "acc", rep.total_accepted,
              "steps", rep.total_steps, flush=True)
    del gb
    torch.cuda.empty_cache()
go("graphs", [("sd", 5), ("sd", 5), ("psd", 5)])
go("nographs", [("sd", 5)], use_graphs=False)
go("onestream", [("sd", 5)], dual_stream=False)
go("onestream-nographs", [("sd", 5)], dual_stream=False, use_graphs=False)
for k in (2, 3, 4):
    go(f"k{k}", [("sd", k)], k_max=k)
go("mb8", [("sd", 5)], max_batch=8)
