"""Snapshot req 0's target KV right after SD verify #1 and compare with a
clean prefill of the same tokens (per layer, per position)."""
import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2603_18016_b200 import SimConfig, make_requests, run
from paper_2603_18016_b200.gpu import GpuBackend
from paper_2603_18016_b200.model import Forward
N, OUT, K = 4, 12, 5
dev = torch.device("cuda:0")
gb = GpuBackend("llama-3.1-8b", "llama-3.2-1b", max_requests=N, max_batch=4, k_max=K,
                max_seq_len=128 + OUT + 16, seed=0, beta_target=7.0, beta_draft=16.0, device=dev,
                use_graphs=False)
orig = gb._verify_launch_inner
snap = {}
cnt = [0]
def wrapped(nb, kmax):
    orig(nb, kmax)
    cnt[0] += 1
    if cnt[0] == 2:
        torch.cuda.synchronize()
        M = nb * (kmax + 1)
        toks = gb.tfwd.view("tokens")[:M].cpu().numpy().copy()
        pos = gb.tfwd.view("positions")[:M].cpu().numpy().copy()
        bt = gb.block_table[0].cpu().numpy().copy()
        L1 = int(pos[kmax])  # last position of req 0 in this pass
        slots = np.asarray([bt[p // 16] * 16 + p % 16 for p in range(L1 + 1)])
        snap["kv"] = gb.target.kv[:, :, torch.as_tensor(slots, device=dev)].float().cpu().numpy()
        snap["toks"] = toks[:kmax + 1]; snap["pos"] = pos[:kmax + 1]
        snap["logits"] = gb.tlogits[:kmax + 1].cpu().numpy().copy()
gb._verify_launch_inner = wrapped
reqs = make_requests([OUT] * N, prompt_len=128)
st, rep = run(SimConfig(mode="standard-sd", m=N // 2, k=K, sd_batch_factor=2), reqs, backend=gb)
r0 = st.request_list()[0]
print("out0", r0.output_ids)
p0 = int(snap["pos"][0])
seq = list(r0.prompt_ids) + r0.output_ids[:p0 - 128]  # committed up to p0-1
assert len(seq) == p0
seq = seq + list(snap["toks"])  # tokens at positions p0 .. p0+k
print("verify#1 tokens", snap["toks"].tolist(), "positions", snap["pos"].tolist())
n = len(seq)
m = gb.target
bt = torch.zeros(1, 16, dtype=torch.int32, device=dev)
nb = (n + 15) // 16
base = 36
bt[0, :nb] = torch.arange(base, base + nb, dtype=torch.int32)
fwd = Forward(m, n, 4, 6, bt)
fwd.begin()
fwd.stage(0, {"tokens": np.asarray(seq, np.int32), "positions": np.arange(n, dtype=np.int32),
              "slots": np.asarray([(base + i // 16) * 16 + i % 16 for i in range(n)], np.int32),
              "seq_slot": np.zeros(1, np.int32), "q_start": np.zeros(1, np.int32),
              "q_len": np.asarray([n], np.int32), "q_pos0": np.zeros(1, np.int32),
              "kv_len": np.asarray([n], np.int32), "logit_rows": np.arange(n - 6, n, dtype=np.int32)})
fwd.upload(1)
lg = torch.empty(6, 128256, device=dev)
fwd.run(n, 1, n, 6, lg, 128256, bigram=(gb.succ_t, 7.0))
torch.cuda.synchronize()
slots = torch.as_tensor([(base + i // 16) * 16 + i % 16 for i in range(n)], device=dev)
ref = m.kv[:, :, slots].float().cpu().numpy()
got = snap["kv"]
print("shapes", ref.shape, got.shape)
for li in range(ref.shape[0]):
    for kv in (0, 1):
        d = np.abs(ref[li, kv] - got[li, kv]).max(axis=(1, 2))  # per position
        sc = np.abs(ref[li, kv]).max(axis=(1, 2)) + 1e-6
        bad = np.where(d / sc > 0.05)[0]
        if len(bad):
            print("layer", li, "KV"[kv], "bad positions", bad.tolist()[:20], "rel", np.round((d / sc)[bad][:8], 3).tolist())
lg = lg.cpu().numpy()
print("prefill argmax", lg.argmax(1).tolist(), "verify argmax", snap["logits"].argmax(1).tolist())
print("row max abs diff", np.abs(lg - snap["logits"]).max(1).tolist())
for r in range(6):
    row = lg[r]
    srt = np.sort(row)
    print("row", r, "std", float(row.std()), "max", float(srt[-1]), "2nd", float(srt[-2]), "margin", float(srt[-1]-srt[-2]),
          "verify row margin(12206 vs 93183)" if r == 1 else "", float(row[12206] - row[93183]) if r == 1 else "")
