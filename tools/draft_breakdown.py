"""Marginal in-graph cost of each kernel family in one draft decode step
(or, with qlen > 2, one verify pass: qlen query tokens per sequence, fp32
logits for every row as the target's verification needs them).

    python tools/draft_breakdown.py [preset] [nseq] [ctx] [qlen]

Builds the 1B draft (random init), prefills nseq sequences of ctx tokens,
captures one decode step (1 token per sequence, K6 greedy LM head) in a CUDA
graph and times it; then, for each kernel family, replaces its C-ABI entry
with a no-op, re-captures and re-times: the difference is what that family
costs inside the real kernel chain (launch gaps and PDL overlap included),
which isolated microbenchmarks do not show.  The no-op runs produce garbage
values; only timing is read.
"""
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2603_18016_b200 import native  # noqa: E402
from paper_2603_18016_b200.model import PRESETS, Forward, Transformer  # noqa: E402

preset = sys.argv[1] if len(sys.argv) > 1 else "llama-3.2-1b"
nseq = int(sys.argv[2]) if len(sys.argv) > 2 else 32
ctx = int(sys.argv[3]) if len(sys.argv) > 3 else 300
qlen = int(sys.argv[4]) if len(sys.argv) > 4 else 1
shape = PRESETS[preset]
dev = torch.device("cuda:0")
bs = 16
mb = (ctx + 16) // bs + 2
m = Transformer(shape, dev, seed=1, num_blocks=nseq * mb + 1, block_size=bs,
                max_blocks_per_seq=mb)
bt = torch.arange(1, 1 + nseq * mb, dtype=torch.int32, device=dev).view(nseq, mb)
fwd = Forward(m, max(nseq * 64, 256), nseq, nseq * max(1, int(sys.argv[4]) if len(sys.argv) > 4
                                                         else 1), bt, sets=1)
rng = np.random.default_rng(0)
lib = native.load()


def slot(s_, p):
    return int(bt[s_, p // bs]) * bs + p % bs


# prefill in chunks of 4 sequences x ctx tokens
for c0 in range(0, nseq, 4):
    seqs = list(range(c0, min(nseq, c0 + 4)))
    toks = rng.integers(0, shape.vocab, len(seqs) * ctx).astype(np.int32)
    fwd.begin()
    fwd.stage(0, {"tokens": toks, "positions": np.tile(np.arange(ctx), len(seqs)).astype(np.int32),
                  "slots": np.asarray([slot(s_, p) for s_ in seqs for p in range(ctx)], np.int32),
                  "seq_slot": np.asarray(seqs, np.int32),
                  "q_start": (np.arange(len(seqs)) * ctx).astype(np.int32),
                  "q_len": np.full(len(seqs), ctx, np.int32), "q_pos0": np.zeros(len(seqs), np.int32),
                  "kv_len": np.full(len(seqs), ctx, np.int32),
                  "logit_rows": np.zeros(1, np.int32)})
    fwd.upload(1)
    fwd.run(len(seqs) * ctx, len(seqs), ctx, 0, None, shape.vocab)
torch.cuda.synchronize()
# the decode step's metadata
M = nseq * qlen
fwd.begin()
fwd.stage(0, {"tokens": rng.integers(0, shape.vocab, M).astype(np.int32),
              "positions": np.tile(ctx + np.arange(qlen), nseq).astype(np.int32),
              "slots": np.asarray([slot(s_, ctx + t) for s_ in range(nseq) for t in range(qlen)],
                                  np.int32),
              "seq_slot": np.arange(nseq, dtype=np.int32),
              "q_start": (np.arange(nseq) * qlen).astype(np.int32),
              "q_len": np.full(nseq, qlen, np.int32),
              "q_pos0": np.full(nseq, ctx, np.int32),
              "kv_len": np.full(nseq, ctx + qlen, np.int32),
              "logit_rows": np.arange(min(M, nseq * qlen), dtype=np.int32),
              "scatter_dst": np.arange(nseq, dtype=np.int32)})
fwd.upload(1)
succ = torch.as_tensor(rng.integers(0, shape.vocab, shape.vocab), dtype=torch.int32, device=dev)
out = torch.empty(nseq, dtype=torch.int32, device=dev)
dst = torch.empty(nseq, dtype=torch.int32, device=dev)


logits = torch.empty(M, shape.vocab, device=dev) if qlen > 2 else None


def step():
    if qlen > 2:  # verify pass: fp32 logits of every row
        fwd.run(M, nseq, qlen, M, logits, shape.vocab)
    else:
        fwd.run(M, nseq, qlen, nseq, None, shape.vocab, bigram=(succ, 16.0),
                argmax_into=(out, dst, fwd.view("scatter_dst", 0)))


def timed(reps=20):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        step()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(reps):
            step()
    g.replay()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e3 / reps)
    return best


base = timed()
print(f"{preset} nseq={nseq} ctx={ctx} qlen={qlen}: step {base:8.1f} us")
families = {
    "attention+rope": ["psd_attention_rope"],
    "rope_kv": ["psd_rope_kv_partials"],
    "attention": ["psd_attention"],
    "add_rmsnorm": ["psd_add_rmsnorm"],
    "split-K GEMMs (qkv, o, down)": ["psd_gemm_partials"],
    "stream-K GEMMs (gate/up; LM head when qlen > 2)": ["psd_gemm_bf16"],
    "LM head + argmax (K6)": ["psd_gemm_argmax", "psd_argmax_fold"],
    "embed": ["psd_embed"],
}
def noop_partials(*a, **k):
    # report one split: the consumers then read a single (garbage) slice
    # instead of a stale count left by the previous real GEMM
    a[10]._obj.value = 1
    return 0


orig = {}
for name, fns in families.items():
    for f in fns:
        orig[f] = getattr(lib, f)
        setattr(lib, f, noop_partials if f == "psd_gemm_partials" else (lambda *a, **k: 0))
    t = timed()
    for f in fns:
        setattr(lib, f, orig[f])
    print(f"  without {name:32s} {t:8.1f} us   -> costs {base - t:7.1f} us "
          f"({100 * (base - t) / base:4.1f} %)")
