"""Greedy-parity helpers shared by the GPU end-to-end tests.

``teacher_forced`` re-runs the oracle target (oracle/model.py) over a
request's prompt + the GPU's output and checks EVERY emitted token, not just
the first divergence: each one must be the oracle's greedy choice
(argmax, lowest id on ties), or -- where the oracle's top-2 logits are closer
than ``tie_tol`` -- one of a documented near-tie that bf16-vs-fp32 summation
order can flip.  ``gpu_logits`` produces the device forward's logits for the
same rows (a prefill pass of the backend's own target model), so logits can
be compared elementwise.
"""

from __future__ import annotations

import numpy as np


def oracle_rows(om, succ, beta, prompt, out):
    """Oracle logits of the rows that emitted ``out`` (row i predicts out[i])."""
    seq = list(prompt) + list(out)
    cache = om.new_cache(len(seq) + 1)
    h = om.forward([(seq[:-1], 0)], [cache])
    p = len(prompt)
    return om.logits(h[p - 1:], np.asarray(seq[p - 1:-1], np.int64), succ, beta)


def teacher_forced(lg: np.ndarray, out, tie_tol: float = 0.05):
    """(#exact, [(position, margin)] near-ties) -- raises on a real mismatch."""
    exact, ties = 0, []
    for i, tok in enumerate(out):
        row = lg[i]
        top = int(np.argmax(row))
        if tok == top:
            exact += 1
            continue
        margin = float(row[top] - row[tok])
        assert margin < tie_tol, (i, tok, top, margin)
        ties.append((i, margin))
    return exact, ties


def gpu_logits(backend, prompt, out):
    """The device target forward's fp32 logits (bigram bias included) of the
    rows that emitted ``out``: one prefill pass over prompt + out[:-1] with
    its own block-table row (uses blocks 1.. of the backend's KV cache, which
    are free once a run has finished)."""
    import torch

    from paper_2603_18016_b200.model import Forward
    m = backend.target
    dev = backend.device
    seq = list(prompt) + list(out)
    n = len(seq) - 1
    bs = m.block_size
    nblk = (n + bs - 1) // bs
    bt = torch.zeros(1, max(nblk, 1), dtype=torch.int32, device=dev)
    bt[0, :nblk] = torch.arange(1, nblk + 1, dtype=torch.int32)
    p = len(prompt)
    rows = np.arange(p - 1, n, dtype=np.int32)
    fwd = Forward(m, n, 4, len(rows), bt)
    fwd.begin()
    fwd.stage(0, {"tokens": np.asarray(seq[:n], np.int32),
                  "positions": np.arange(n, dtype=np.int32),
                  "slots": np.asarray([(1 + i // bs) * bs + i % bs for i in range(n)], np.int32),
                  "seq_slot": np.zeros(1, np.int32), "q_start": np.zeros(1, np.int32),
                  "q_len": np.asarray([n], np.int32), "q_pos0": np.zeros(1, np.int32),
                  "kv_len": np.asarray([n], np.int32), "logit_rows": rows})
    fwd.upload(1)
    V = backend.tshape.vocab
    logits = torch.empty(len(rows), V, dtype=torch.float32, device=dev)
    fwd.run(n, 1, n, len(rows), logits, V, bigram=(backend.succ_t, backend.beta_target))
    torch.cuda.synchronize()
    return logits.cpu().numpy()


def elementwise_ok(got: np.ndarray, ref: np.ndarray, rtol: float = 1e-2,
                   atol_frac: float = 1e-2):
    """|got - ref| <= rtol * |ref| + atol elementwise, atol = atol_frac x the
    RMS of the reference row (logits near zero carry only absolute error);
    returns (ok, worst ratio of error to bound)."""
    atol = atol_frac * np.sqrt((ref.astype(np.float64) ** 2).mean(axis=-1, keepdims=True))
    bound = rtol * np.abs(ref) + atol
    ratio = np.abs(got.astype(np.float64) - ref) / bound
    return bool((ratio <= 1.0).all()), float(ratio.max())
