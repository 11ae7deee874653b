import sys, os
sys.path.insert(0, os.getcwd())
import torch
from paper_2603_18016_b200 import SimConfig, make_requests, run
from paper_2603_18016_b200.gpu import GpuBackend
dev = torch.device("cuda:0")
mode = sys.argv[1]; k = int(sys.argv[2]); N = int(sys.argv[3]); mb = int(sys.argv[4])
OUT = 12
gb = GpuBackend("llama-3.1-8b", "llama-3.2-1b", max_requests=N, max_batch=mb, k_max=k,
                max_seq_len=128 + OUT + 16, seed=0, beta_target=7.0, beta_draft=16.0,
                device=dev, use_graphs=os.environ.get("G", "0") == "1")
cfg = (SimConfig(mode="psd", m=N // 2, k=k) if mode == "psd" else
       SimConfig(mode="standard-sd", m=N // 2, k=k, sd_batch_factor=2))
st, rep = run(cfg, make_requests([OUT] * N, prompt_len=128), backend=gb)
for r in st.request_list()[:4]:
    print(mode, k, N, mb, r.output_ids)
