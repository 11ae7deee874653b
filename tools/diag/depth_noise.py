"""GPU vs oracle logits error as a function of depth (8B shapes truncated to L
layers), next to the GPU's own reordering floor (same forward, other split-K)."""
import sys, os, dataclasses
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2603_18016_b200.model import PRESETS, Transformer, Forward, successor_table
from oracle.model import OracleModel
dev = torch.device("cuda:0")
name = sys.argv[1] if len(sys.argv) > 1 else "llama-3.1-8b"
base = PRESETS[name]
rng = np.random.default_rng(0)
n = 135
seq = rng.integers(0, base.vocab, n).tolist()
def gpu(shape, hint):
    m = Transformer(shape, dev, 1, 16, 16, 16)
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
    lg = torch.empty(6, shape.vocab, device=dev)
    fwd.run(n, 1, n, 6, lg, shape.vocab)
    torch.cuda.synchronize()
    out = lg.cpu().numpy()
    del m, fwd; torch.cuda.empty_cache()
    return out
for L in [1, 2, 4, 8, 16, base.layers]:
    sh = dataclasses.replace(base, name=f"{name}-L{L}", layers=L)
    a = gpu(sh, 0); b = gpu(sh, 1)
    om = OracleModel(sh, 1)
    h = om.forward([(seq, 0)], [om.new_cache(n + 1)])
    ref = om.logits(h[-6:], None)
    rms = np.sqrt((ref ** 2).mean())
    e_or = np.abs(a - ref).max(); e_gg = np.abs(a - b).max()
    rel = (np.abs(a - ref) / (np.abs(ref) + 1e-2 * rms)).max()
    print(f"L={L:3d} rms={rms:.3f} |gpu-oracle|max={e_or:.4f} ({e_or/rms:.4f} rms)  |gpu-gpu(split1)|max={e_gg:.4f}  max |d|/(|ref|+0.01rms)={rel:.4f}", flush=True)
