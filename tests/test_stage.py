"""psd_stage_draft / psd_stage_verify (host code in libpsd.so, no GPU needed)
against a numpy statement of the same metadata: the draft loop's k decode
sets and the verify pass's K1-token rows, with padding rows, ragged k,
replay-mode rows past the allocation and the overrun / capacity errors."""

import ctypes

import numpy as np
import pytest

from paper_2603_18016_b200 import native
from paper_2603_18016_b200.model import META_FIELDS

BS = 16
LDT = 7  # k_max + 2


def _lib():
    try:
        return native.load()
    except Exception as exc:  # pragma: no cover - build missing
        pytest.skip(f"libpsd.so not loadable: {exc}")


def _layout(T, S, R):
    sizes = {"tokens": T, "positions": T, "slots": T, "seq_slot": S, "q_start": S, "q_len": S,
             "q_pos0": S, "kv_len": S, "logit_rows": R, "gather_src": T, "scatter_dst": R}
    off, o = {}, 0
    for name in META_FIELDS:
        off[name] = (o, sizes[name])
        o += sizes[name]
    return off, o


def _slots_at(bt, nblk, replay, s, pos):
    bi = pos // BS
    beyond = bi >= nblk[s]
    if beyond.any() and not replay:
        raise OverflowError
    bi = np.where(beyond, 0, bi)
    return np.where(beyond, -1, bt[s, bi] * BS + pos % BS)


def _draft_ref(bt, nblk, replay, scratch, sl_r, L_r, k_r, nb):
    n = len(sl_r)
    sl = np.full(nb, scratch, np.int64)
    L = np.full(nb, 2, np.int64)
    k = np.zeros(nb, np.int64)
    sl[:n], L[:n], k[:n] = sl_r, L_r, k_r
    kmax = int(k.max())
    real = np.arange(nb) < n
    pos = np.stack([L - 2, L - 1], axis=1).reshape(-1)
    srow = np.repeat(sl, 2)
    real2 = np.repeat(real, 2)
    sets = [{
        "gather_src": srow * LDT + np.tile([0, 1], nb),
        "positions": np.where(real2, pos, 0),
        "slots": np.where(real2, _slots_at(bt, nblk, replay, srow, np.maximum(pos, 0)), -1),
        "seq_slot": sl, "q_start": np.arange(0, 2 * nb, 2), "q_len": np.full(nb, 2),
        "q_pos0": np.where(real, L - 2, 0), "kv_len": np.where(real, L, 1),
        "logit_rows": np.arange(1, 2 * nb, 2), "scatter_dst": np.where(real, sl * LDT + 2, -1)}]
    for i in range(1, kmax):
        act = real & (i < k)
        p = np.where(act, L - 1 + i, 0)
        sets.append({
            "gather_src": sl * LDT + 1 + i, "positions": p,
            "slots": np.where(act, _slots_at(bt, nblk, replay, sl, p), -1),
            "seq_slot": sl, "q_start": np.arange(nb), "q_len": np.ones(nb),
            "q_pos0": p, "kv_len": np.where(act, L + i, 1), "logit_rows": np.arange(nb),
            "scatter_dst": np.where(act, sl * LDT + 2 + i, -1)})
    return sets


def _verify_ref(bt, nblk, replay, scratch, sl_r, L_r, k_r, nb, kmax):
    n = len(sl_r)
    K1 = kmax + 1
    sl = np.full(nb, scratch, np.int64)
    L = np.full(nb, 1, np.int64)
    k = np.zeros(nb, np.int64)
    sl[:n], L[:n], k[:n] = sl_r, L_r, k_r
    real = np.arange(nb) < n
    j = np.arange(K1)[None, :]
    src = np.where((j == 0) | (j > k[:, None]), 1, 1 + j)
    pos = (L - 1)[:, None] + j
    wr = real[:, None] & (j <= k[:, None])
    slots = np.where(wr, _slots_at(bt, nblk, replay, np.repeat(sl, K1).reshape(nb, K1),
                                   np.where(wr, pos, 0)), -1)
    return {"gather_src": (sl[:, None] * LDT + src).reshape(-1),
            "positions": np.where(real[:, None], pos, 0).reshape(-1),
            "slots": slots.reshape(-1), "seq_slot": sl,
            "q_start": np.arange(0, nb * K1, K1), "q_len": np.full(nb, K1),
            "q_pos0": np.where(real, L - 1, 0), "kv_len": np.where(real, L + k, 1),
            "logit_rows": np.arange(nb * K1)}


def _table(rng, nslot, max_blocks, scratch):
    bt = np.zeros((nslot, max_blocks), np.int32)
    nblk = np.zeros(nslot, np.int32)
    free = list(rng.permutation(np.arange(1, nslot * max_blocks)))
    for s in range(nslot):
        if s == scratch:
            nblk[s] = 1
            continue
        nb_ = int(rng.integers(1, max_blocks + 1))
        bt[s, :nb_] = [free.pop() for _ in range(nb_)]
        nblk[s] = nb_
    return bt, nblk


def _rows(rng, nblk, scratch, n, kmax_budget, ensure_fit):
    slots = rng.choice([s for s in range(len(nblk)) if s != scratch], n, replace=False)
    L, k = [], []
    for s in slots:
        cap = int(nblk[s]) * BS
        kk = int(rng.integers(0, kmax_budget + 1))
        hi = cap - kk if ensure_fit else cap + 3
        L.append(int(rng.integers(2, max(3, hi + 1))))
        k.append(kk)
    return slots.astype(np.int32), np.array(L, np.int32), np.array(k, np.int32)


def _call_draft(lib, off, size, sets, bt, nblk, replay, scratch, sl, L, k, nb):
    n = len(sl)
    kmax = int(k.max()) if n else 1
    buf = np.full((max(kmax, 1), size), 12345, np.int32)
    fields = np.array([v for nm in META_FIELDS for v in off[nm]], np.int32)
    a = np.zeros((3, nb), np.int32)
    a[0, :n], a[1, :n], a[2, :n] = sl, L, k
    rc = lib.psd_stage_draft(buf.ctypes.data, size, fields.ctypes.data, bt.ctypes.data,
                             bt.shape[1], nblk.ctypes.data, BS, int(replay), LDT, scratch,
                             a[0].ctypes.data, a[1].ctypes.data, a[2].ctypes.data, n, nb, kmax)
    return rc, buf


def _check_set(buf_row, off, want):
    for name, arr in want.items():
        o, _ = off[name]
        got = buf_row[o:o + len(arr)]
        np.testing.assert_array_equal(got, np.asarray(arr, np.int64).astype(np.int32),
                                      err_msg=name)


@pytest.mark.parametrize("seed", range(12))
@pytest.mark.parametrize("replay", [False, True])
def test_stage_draft_matches_numpy(seed, replay):
    lib = _lib()
    rng = np.random.default_rng(seed)
    nslot, max_blocks, scratch = 24, 6, 23
    bt, nblk = _table(rng, nslot, max_blocks, scratch)
    n = int(rng.integers(1, 17))
    nb = (n + 7) // 8 * 8
    sl, L, k = _rows(rng, nblk, scratch, n, 5, ensure_fit=not replay)
    k[0] = max(k[0], 1)
    off, size = _layout(2 * 32, 32, 32)
    rc, buf = _call_draft(lib, off, size, None, bt, nblk, replay, scratch, sl, L, k, nb)
    try:
        want = _draft_ref(bt, nblk, replay, scratch, sl, L, k, nb)
    except OverflowError:
        assert rc == native.STAGE_KV_OVERRUN
        return
    assert rc == 0
    for i, w in enumerate(want):
        _check_set(buf[i], off, w)


@pytest.mark.parametrize("seed", range(12))
@pytest.mark.parametrize("replay", [False, True])
def test_stage_verify_matches_numpy(seed, replay):
    lib = _lib()
    rng = np.random.default_rng(100 + seed)
    nslot, max_blocks, scratch, kmax = 24, 6, 23, 5
    bt, nblk = _table(rng, nslot, max_blocks, scratch)
    n = int(rng.integers(0, 17))
    nb = max(8, (n + 7) // 8 * 8)
    sl, L, k = _rows(rng, nblk, scratch, n, kmax, ensure_fit=not replay)
    off, size = _layout(32 * (kmax + 1), 32, 32 * (kmax + 1))
    buf = np.full(size, 12345, np.int32)
    fields = np.array([v for nm in META_FIELDS for v in off[nm]], np.int32)
    a = np.zeros((3, nb), np.int32)
    a[0, :n], a[1, :n], a[2, :n] = sl, L, k
    rc = lib.psd_stage_verify(buf.ctypes.data, fields.ctypes.data, bt.ctypes.data, max_blocks,
                              nblk.ctypes.data, BS, int(replay), LDT, scratch, a[0].ctypes.data,
                              a[1].ctypes.data, a[2].ctypes.data, n, nb, kmax)
    try:
        want = _verify_ref(bt, nblk, replay, scratch, sl, L, k, nb, kmax)
    except OverflowError:
        assert rc == native.STAGE_KV_OVERRUN
        return
    assert rc == 0
    _check_set(buf, off, want)


def test_stage_overrun_and_capacity_errors():
    lib = _lib()
    nslot, scratch = 4, 3
    bt = np.arange(nslot * 2, dtype=np.int32).reshape(nslot, 2)
    nblk = np.array([1, 2, 1, 1], np.int32)
    off, size = _layout(64, 32, 32)
    # slot 0 holds one block (16 tokens): a verify of 4 drafts from L = 15 overruns
    sl, L, k = np.array([0], np.int32), np.array([15], np.int32), np.array([4], np.int32)
    rc, _ = _call_draft(lib, off, size, None, bt, nblk, False, scratch, sl, L, k, 8)
    assert rc == native.STAGE_KV_OVERRUN
    rc, buf = _call_draft(lib, off, size, None, bt, nblk, True, scratch, sl, L, k, 8)
    assert rc == 0
    o, _ = off["slots"]
    assert buf[2][o] == -1  # step 2 writes position 16: past the grant, nowhere
    # capacity: 40 rows do not fit a 32-sequence layout
    sl40 = np.zeros(40, np.int32)
    rc, _ = _call_draft(lib, off, size, None, bt, nblk, True, scratch, sl40,
                        np.full(40, 3, np.int32), np.ones(40, np.int32), 40)
    assert rc == native.STAGE_CAPACITY
    assert lib.psd_stage_draft(None, 0, None, None, 0, None, 0, 0, 0, 0, None, None, None,
                               2, 1, 1) == native.STAGE_BAD_ARGS
    assert ctypes.sizeof(ctypes.c_int) == 4
