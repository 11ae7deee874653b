"""K3 paged multi-query attention vs a torch fp32 reference of the same op.

Covers head dims 32 / 64 / 128, GQA groups 4 / 7 / 8, the verify window
(q_len = k+1 at q_pos0 = L-1), draft steps (q_len 1-2), prefill chunks
(q_len > 64 / G), padded rows with kv_len clamping, non-contiguous blocks.
"""

import math

import pytest
import torch

from paper_2603_18016_b200 import native

pytestmark = pytest.mark.gpu


def _case(dev, D, Hq, Hkv, seqs, bs=16, nblocks=200, seed=0, maxb=40):
    g = torch.Generator(device=dev).manual_seed(seed)
    M = sum(ql for ql, _, _ in seqs)
    q = torch.randn(M, Hq, D, device=dev, generator=g).to(torch.bfloat16)
    kc = torch.randn(nblocks * bs, Hkv, D, device=dev, generator=g).to(torch.bfloat16)
    vc = torch.randn(nblocks * bs, Hkv, D, device=dev, generator=g).to(torch.bfloat16)
    bt = torch.zeros(len(seqs), maxb, dtype=torch.int32, device=dev)
    perm = torch.randperm(nblocks - 1, generator=torch.Generator().manual_seed(seed)) + 1
    used = 0
    q_start, q_len, q_pos0, kv_len = [], [], [], []
    o = 0
    for i, (ql, p0, kvl) in enumerate(seqs):
        nb = (max(kvl, p0 + ql) + bs - 1) // bs
        bt[i, :nb] = perm[used:used + nb].to(torch.int32)
        used += nb
        q_start.append(o)
        q_len.append(ql)
        q_pos0.append(p0)
        kv_len.append(kvl)
        o += ql
    t = lambda x: torch.tensor(x, dtype=torch.int32, device=dev)  # noqa: E731
    meta = dict(seq_slot=t(list(range(len(seqs)))), q_start=t(q_start), q_len=t(q_len),
                q_pos0=t(q_pos0), kv_len=t(kv_len))
    return q, kc, vc, bt, meta


def _ref(q, kc, vc, bt, meta, seqs, Hq, Hkv, D, bs=16):
    G = Hq // Hkv
    out = torch.zeros_like(q, dtype=torch.float32)
    o = 0
    for i, (ql, p0, kvl) in enumerate(seqs):
        keys = torch.arange(kvl, device=q.device)
        slots = bt[i, keys // bs].long() * bs + keys % bs
        K = kc[slots].float()  # [kvl, Hkv, D]
        V = vc[slots].float()
        for t in range(ql):
            lim = min(p0 + t, kvl - 1)
            for h in range(Hq):
                qq = q[o + t, h].float()
                s = (K[:lim + 1, h // G] @ qq) / math.sqrt(D)
                p = torch.softmax(s, 0)
                out[o + t, h] = p @ V[:lim + 1, h // G]
        o += ql
    return out


@pytest.mark.parametrize("D,Hq,Hkv", [(128, 32, 8), (64, 32, 8), (32, 8, 2), (128, 28, 4),
                                      (128, 64, 8), (64, 14, 2)])
def test_attention_matches_torch(cuda_device, D, Hq, Hkv):
    # (q_len, q_pos0, kv_len): verify windows, a draft 2-token step, a 1-token
    # step, a prefill chunk, and a padded row (kv_len clamps the window)
    seqs = [(6, 140, 146), (6, 7, 10), (2, 30, 32), (1, 63, 64), (40, 0, 40), (6, 0, 1),
            (5, 300, 305)]
    q, kc, vc, bt, meta = _case(cuda_device, D, Hq, Hkv, seqs)
    lib = native.load()
    st = torch.cuda.current_stream().cuda_stream
    ref = _ref(q, kc, vc, bt, meta, seqs, Hq, Hkv, D)
    maxq = max(s[0] for s in seqs)
    maxkv = max(max(kv, p0 + ql) for ql, p0, kv in seqs)
    ws = torch.zeros(lib.psd_attention_workspace_bytes(len(seqs), Hkv, maxq, Hq, D, 1024) +
                     16384, dtype=torch.uint8, device=cuda_device)
    for kvhint in (0, maxkv, 1024):  # no split, split-KV, more splits
        out = torch.full_like(q, float("nan"))
        for _ in range(2):  # tickets are self-resetting
            rc = lib.psd_attention(q.data_ptr(), kc.data_ptr(), vc.data_ptr(), bt.data_ptr(),
                                   bt.shape[1], meta["seq_slot"].data_ptr(),
                                   meta["q_start"].data_ptr(), meta["q_len"].data_ptr(),
                                   meta["q_pos0"].data_ptr(), meta["kv_len"].data_ptr(),
                                   len(seqs), maxq, Hq, Hkv, D, 16, 1.0 / math.sqrt(D),
                                   out.data_ptr(), kvhint, ws.data_ptr(), ws.numel(), st)
            assert rc == 0
        torch.cuda.synchronize()
        err = (out.float() - ref).abs().max().item()
        assert err < 2e-2, (kvhint, err)


@pytest.mark.parametrize("D,Hq,Hkv", [(128, 32, 8), (64, 32, 8), (32, 8, 2), (128, 28, 4),
                                      (128, 64, 8), (64, 14, 2)])
@pytest.mark.parametrize("maxb", [2, 8, 40, 200])
def test_decode_attention_matches_torch(cuda_device, D, Hq, Hkv, maxb):
    """Decode widths (q_len * G <= 16) take attn_dec_kernel: one CTA per
    (sequence, kv head) with every key tile in flight; the tiles per round come
    from the block-table width (maxb 2 / 8 / 40: one round; 200: 3200 keys,
    several rounds at D = 128)."""
    kmax = maxb * 16
    seqs = [(6, 140, 146), (6, 7, 10), (2, 30, 32), (1, 63, 64), (6, 0, 1), (5, 300, 305),
            (1, 600, 601), (6, 3000, 3006), (2, 1, 3)]
    seqs = [s for s in seqs if max(s[2], s[1] + s[0]) <= kmax]
    G = Hq // Hkv
    seqs = [(min(ql, 16 // G), p0, kv) for ql, p0, kv in seqs]
    need = sum((max(kv, p0 + ql) + 15) // 16 for ql, p0, kv in seqs)
    q, kc, vc, bt, meta = _case(cuda_device, D, Hq, Hkv, seqs, nblocks=need + 8, maxb=maxb)
    lib = native.load()
    st = torch.cuda.current_stream().cuda_stream
    ref = _ref(q, kc, vc, bt, meta, seqs, Hq, Hkv, D)
    maxq = max(s[0] for s in seqs)
    out = torch.full_like(q, float("nan"))
    for _ in range(2):
        rc = lib.psd_attention(q.data_ptr(), kc.data_ptr(), vc.data_ptr(), bt.data_ptr(),
                               bt.shape[1], meta["seq_slot"].data_ptr(),
                               meta["q_start"].data_ptr(), meta["q_len"].data_ptr(),
                               meta["q_pos0"].data_ptr(), meta["kv_len"].data_ptr(),
                               len(seqs), maxq, Hq, Hkv, D, 16, 1.0 / math.sqrt(D),
                               out.data_ptr(), 0, None, 0, st)
        assert rc == 0
    torch.cuda.synchronize()
    err = (out.float() - ref).abs().max().item()
    assert err < 2e-2, err
