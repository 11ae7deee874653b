import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2603_18016_b200 import SimConfig, make_requests, run
from paper_2603_18016_b200.gpu import GpuBackend
from paper_2603_18016_b200.model import successor_table
succ = successor_table(128256, 128256, 0)
N, OUT, K = 4, 12, 5
dev = torch.device("cuda:0")
gb = GpuBackend(os.environ.get("T", "llama-3.1-8b"), os.environ.get("D", "llama-3.2-1b"),
                max_requests=N, max_batch=4, k_max=K,
                max_seq_len=128 + OUT + 16, seed=0, beta_target=7.0, beta_draft=16.0, device=dev,
                use_graphs=False)
gb.capture_verify = []
orig = gb._verify_launch_inner
toks_log = []
def wrapped(nb, kmax):
    orig(nb, kmax)
    torch.cuda.synchronize()
    M = nb * (kmax + 1)
    toks_log.append((gb.tfwd.view("tokens")[:M].cpu().numpy().copy(),
                     gb.tfwd.view("positions")[:M].cpu().numpy().copy(),
                     gb.tfwd.view("slots")[:M].cpu().numpy().copy(),
                     gb.slot_tok.cpu().numpy().copy(), gb.block_table.cpu().numpy()[:, :12].copy()))
gb._verify_launch_inner = wrapped
mode = os.environ.get("MODE", "sd")
cfg = (SimConfig(mode="standard-sd", m=N // 2, k=K, sd_batch_factor=2) if mode == "sd"
       else SimConfig(mode="psd", m=N // 2, k=K))
st, rep = run(cfg, make_requests([OUT] * N, prompt_len=128), backend=gb)
for i, (rec, tl) in enumerate(zip(gb.capture_verify[:4], toks_log)):
    print("verify", i, "len", rec["len"].tolist(), "acc", rec["acc"].tolist())
    t, pos, sl, stok, bt = tl
    print("  tokens", t.tolist()); print("  pos", pos.tolist()); print("  slots", sl.tolist())
    print("  ids", rec["ids"].tolist())
    am = rec["target"].argmax(axis=2)
    print("  argmax", am.tolist())
    print("  succ(tokens)", [int(succ[x]) for x in t])
    print("  out", rec["out"].tolist())
    print("  bt", bt.tolist())
