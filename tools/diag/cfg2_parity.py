"""Diagnose PSD vs SD vs oracle at cfg2 shapes (prints per-request details)."""
import sys, os, time
sys.path.insert(0, os.getcwd())
import numpy as np
import torch
from paper_2603_18016_b200 import SimConfig, make_requests, run
from paper_2603_18016_b200.gpu import GpuBackend
from tests._parity import oracle_rows, gpu_logits

N, OUT, K = 4, 16, 5
mb = int(sys.argv[1]) if len(sys.argv) > 1 else 4
use_graphs = os.environ.get("G", "1") == "1"
dev = torch.device("cuda:0")
kw = dict(max_requests=N, max_batch=mb, k_max=K, max_seq_len=128 + OUT + 16, seed=0,
          beta_target=7.0, beta_draft=16.0, device=dev, use_graphs=use_graphs)
gb = GpuBackend("llama-3.1-8b", "llama-3.2-1b", **kw)
res = {}
for mode, cfg in [("psd", SimConfig(mode="psd", m=N // 2, k=K)),
                  ("sd", SimConfig(mode="standard-sd", m=N // 2, k=K, sd_batch_factor=2)),
                  ("sd1", SimConfig(mode="standard-sd", m=N // 2, k=1, sd_batch_factor=2)),
                  ("sdk0", SimConfig(mode="standard-sd", m=N // 2, k=0, sd_batch_factor=2))]:
    try:
        st, rep = run(cfg, make_requests([OUT] * N, prompt_len=128), backend=gb)
    except Exception as e:
        print(mode, "ERR", e); continue
    res[mode] = st
    print(mode, "acc", rep.total_accepted, "drafted", rep.total_drafted, "steps", rep.total_steps)
    for r in st.request_list():
        print("  ", r.id, r.output_ids)
from oracle.model import OracleModel
from paper_2603_18016_b200.model import PRESETS, successor_table
t0 = time.time()
om = OracleModel(PRESETS["llama-3.1-8b"], 1)
succ = successor_table(128256, 128256, 0)
print("oracle init", time.time() - t0)
st = res["psd"]
for r in st.request_list():
    ref = oracle_rows(om, succ, 7.0, r.prompt_ids, r.output_ids)
    got = gpu_logits(gb, r.prompt_ids, r.output_ids)
    am = ref.argmax(axis=1)
    print("req", r.id, "oracle argmax", am.tolist())
    print("     gpu prefill argmax", got.argmax(axis=1).tolist())
    print("     max abs err", float(np.abs(got - ref).max()), "succ of prev", [int(succ[t]) for t in ([r.prompt_ids[-1]] + r.output_ids[:-1])])
