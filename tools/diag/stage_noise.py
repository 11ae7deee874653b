import sys, os, dataclasses
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2603_18016_b200.model import PRESETS, Transformer, Forward
dev = torch.device("cuda:0")
base = PRESETS["llama-3.1-8b"]
sh = dataclasses.replace(base, name="L1", layers=1)
rng = np.random.default_rng(0)
n = 135
seq = rng.integers(0, base.vocab, n).tolist()
m = Transformer(sh, dev, 1, 16, 16, 16)
def run(hint):
    bt = torch.zeros(1, 16, dtype=torch.int32, device=dev)
    bt[0, :9] = torch.arange(1, 10, dtype=torch.int32)
    os.environ["PSD_SPLITS_HINT"] = str(hint)
    fwd = Forward(m, n, 4, 6, bt)
    fwd.begin()
    fwd.stage(0, {"tokens": np.asarray(seq, np.int32), "positions": np.arange(n, dtype=np.int32),
                  "slots": np.asarray([(1 + i // 16) * 16 + i % 16 for i in range(n)], np.int32),
                  "seq_slot": np.zeros(1, np.int32), "q_start": np.zeros(1, np.int32),
                  "q_len": np.asarray([n], np.int32), "q_pos0": np.zeros(1, np.int32),
                  "kv_len": np.asarray([n], np.int32), "logit_rows": np.arange(n - 6, n, dtype=np.int32)})
    fwd.upload(1)
    lg = torch.empty(6, sh.vocab, device=dev)
    fwd.run(n, 1, n, 6, lg, sh.vocab)
    torch.cuda.synchronize()
    return {"kv": m.kv[0, :, 16:16 + n].float().clone(), "attn": fwd.attn[:n].float().clone(),
            "x": fwd.x[:n].float().clone(), "act": fwd.act[:n].float().clone(),
            "xf": fwd.xf[:6].float().clone(), "lg": lg.clone()}
a = run(0); b = run(1)
for k in a:
    d = (a[k] - b[k]).abs()
    print(k, "max diff", d.max().item(), "rms", a[k].pow(2).mean().sqrt().item(), "frac elems differing", (d > 0).float().mean().item())
