import sys, os
sys.path.insert(0, os.getcwd())
import torch
from paper_2603_18016_b200 import SimConfig, make_requests, run
from paper_2603_18016_b200.gpu import GpuBackend
dev = torch.device("cuda:0")
mode = sys.argv[1]; k = int(sys.argv[2]); prompt = int(sys.argv[3])
N, OUT = 4, 12
gb = GpuBackend("tiny-target", "tiny-draft", max_requests=N, max_batch=4, k_max=k,
                max_seq_len=prompt + OUT + 16, seed=0, beta_target=3.0, beta_draft=12.0,
                device=dev, use_graphs=os.environ.get("G", "0") == "1")
cfg = (SimConfig(mode="psd", m=N // 2, k=k) if mode == "psd" else
       SimConfig(mode="standard-sd", m=N // 2, k=k, sd_batch_factor=2))
st, rep = run(cfg, make_requests([OUT] * N, prompt_len=prompt), backend=gb)
print(mode, k, prompt, [r.output_ids for r in st.request_list()][0])
