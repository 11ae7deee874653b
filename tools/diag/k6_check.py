"""K6 debug: one decode step of a tiny / 1B draft through Forward.run with the
argmax epilogue vs the stored-logits path (+ bigram bias + torch argmax)."""
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
from paper_2603_18016_b200.model import PRESETS, Forward, Transformer, successor_table

preset = sys.argv[1] if len(sys.argv) > 1 else "tiny-draft"
graphs = len(sys.argv) > 2 and sys.argv[2] == "graph"
shape = PRESETS[preset]
dev = torch.device("cuda:0")
m = Transformer(shape, dev, seed=21, num_blocks=64, block_size=16, max_blocks_per_seq=8)
nseq = 4
bt = torch.zeros(nseq, 8, dtype=torch.int32, device=dev)
for s_ in range(nseq):
    bt[s_, :4] = torch.arange(1 + 4 * s_, 5 + 4 * s_)
fwd = Forward(m, 128, 8, 64, bt)
rng = np.random.default_rng(3)
lens = [19, 33, 7, 12]
toks = [rng.integers(0, shape.vocab, n).tolist() for n in lens]
succ = torch.as_tensor(rng.integers(0, shape.vocab, shape.vocab), dtype=torch.int32, device=dev)


def stage(seq_toks, p0s, rows):
    flat = np.concatenate(seq_toks).astype(np.int32)
    pos = np.concatenate([np.arange(p0, p0 + len(t)) for t, p0 in zip(seq_toks, p0s)])
    slots = np.concatenate([[bt[s_, (p0 + i) // 16].item() * 16 + (p0 + i) % 16
                             for i in range(len(t))] for s_, (t, p0) in enumerate(zip(seq_toks, p0s))])
    qs = np.cumsum([0] + [len(t) for t in seq_toks])[:-1]
    fwd.begin()
    fwd.stage(0, {"tokens": flat, "positions": pos.astype(np.int32), "slots": slots.astype(np.int32),
                  "seq_slot": np.arange(len(seq_toks), dtype=np.int32),
                  "q_start": qs.astype(np.int32),
                  "q_len": np.asarray([len(t) for t in seq_toks], np.int32),
                  "q_pos0": np.asarray(p0s, np.int32),
                  "kv_len": np.asarray([p0 + len(t) for t, p0 in zip(seq_toks, p0s)], np.int32),
                  "logit_rows": np.asarray(rows, np.int32),
                  "scatter_dst": np.arange(len(rows), dtype=np.int32) * 2})
    fwd.upload(1)
    return len(flat)


M = stage(toks, [0] * nseq, [0])
fwd.run(M, nseq, max(lens), 0, None, shape.vocab)
nxt = [[int(rng.integers(0, shape.vocab))] for _ in range(nseq)]
for beta in (0.0, 16.0):
    M = stage(nxt, lens, list(range(nseq)))
    logits = torch.empty(nseq, shape.vocab, device=dev)
    fwd.run(M, nseq, 1, nseq, logits, shape.vocab, bigram=(succ, beta))
    ref = logits.argmax(1).to(torch.int32)
    out = torch.full((nseq,), -1, dtype=torch.int32, device=dev)
    dst = torch.full((2 * nseq,), -1, dtype=torch.int32, device=dev)

    def launch():
        fwd.run(M, nseq, 1, nseq, None, shape.vocab, bigram=(succ, beta),
                argmax_into=(out, dst, fwd.view("scatter_dst", 0)))
    if graphs:
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            launch()
        g.replay()
    else:
        launch()
    torch.cuda.synchronize()
    print(preset, "beta", beta, "ref", ref.tolist(), "k6", out.tolist(), "dst", dst.tolist(),
          "bias cols", [int(succ[t[0]]) for t in nxt])
