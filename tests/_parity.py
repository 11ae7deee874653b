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


def gpu_logits(backend, prompt, out, splits_hint: int = 0):
    """The device target forward's fp32 logits (bigram bias included) of the
    rows that emitted ``out``: one prefill pass over prompt + out[:-1] with
    its own block-table row (uses blocks 1.. of the backend's KV cache, which
    are free once a run has finished).  ``splits_hint`` > 0 forces that
    split-K count on the QKV / O / down GEMMs: an equally valid summation order,
    whose distance to the default is the forward's own noise floor."""
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
    fwd.splits_hint = splits_hint
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


def noise_floor_ok(got: np.ndarray, ref: np.ndarray, alt: np.ndarray, factor: float = 1.5,
                   atol_frac: float = 1e-2):
    """The device logits are as close to the oracle's as two valid device
    summation orders are to each other: max |got - ref| <= factor x max |got -
    alt| + atol_frac x rms(ref), and the same for the RMS error.  bf16 storage
    of every activation turns any reordering into a half-ulp noise on most
    elements, which the 32-layer random-init stack accumulates (~sqrt(depth):
    profiles/r02_forward_noise_floor.txt), so a fixed rtol cannot hold at depth
    while this bound does."""
    rms = float(np.sqrt((ref.astype(np.float64) ** 2).mean()))
    e_max, f_max = float(np.abs(got - ref).max()), float(np.abs(got - alt).max())
    e_rms = float(np.sqrt(((got.astype(np.float64) - ref) ** 2).mean()))
    f_rms = float(np.sqrt(((got.astype(np.float64) - alt) ** 2).mean()))
    ok = e_max <= factor * f_max + atol_frac * rms and e_rms <= factor * f_rms + atol_frac * rms
    return ok, {"err_max": e_max, "floor_max": f_max, "err_rms": e_rms, "floor_rms": f_rms,
                "rms": rms}


def elementwise_ok(got: np.ndarray, ref: np.ndarray, rtol: float = 1e-2,
                   atol_frac: float = 1e-2):
    """|got - ref| <= rtol * |ref| + atol elementwise, atol = atol_frac x the
    RMS of the reference row (logits near zero carry only absolute error);
    returns (ok, worst ratio of error to bound)."""
    atol = atol_frac * np.sqrt((ref.astype(np.float64) ** 2).mean(axis=-1, keepdims=True))
    bound = rtol * np.abs(ref) + atol
    ratio = np.abs(got.astype(np.float64) - ref) / bound
    return bool((ratio <= 1.0).all()), float(ratio.max())
