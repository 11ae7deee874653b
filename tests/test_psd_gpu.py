"""End-to-end PSD on the GPU vs the CPU oracle (tiny BASELINE config 1).

* forward parity: the tcgen05/paged-attention forward of the tiny target
  matches the numpy oracle's logits within rtol 1e-2 (north-star tolerance);
* greedy end-to-end identity: every request's output tokens from GPU PSD
  equal the CPU oracle PSD's, and equal GPU sequential SD's (greedy output is
  schedule independent);
* scheduler invariants on the GPU path: KV blocks at finish == ceil(total /
  block), one bonus per verified row, every request finishes.
"""

import numpy as np
import pytest
import torch

from oracle.model import OracleModel
from oracle.psd_cpu import CpuBackend
from paper_2603_18016_b200 import SimConfig, blocks_needed, make_requests, run
from paper_2603_18016_b200.gpu import GpuBackend
from paper_2603_18016_b200.model import PRESETS, Forward, Transformer

pytestmark = pytest.mark.gpu


def test_tiny_forward_matches_oracle(cuda_device):
    shape = PRESETS["tiny-target"]
    dev = cuda_device
    m = Transformer(shape, dev, seed=11, num_blocks=16, block_size=16, max_blocks_per_seq=8)
    bt = torch.zeros(4, 8, dtype=torch.int32, device=dev)
    bt[0, :4] = torch.tensor([1, 2, 3, 4])
    bt[1, :4] = torch.tensor([5, 6, 7, 8])
    fwd = Forward(m, 128, 8, 64, bt)
    rng = np.random.default_rng(0)
    lens = [23, 40]
    toks = [rng.integers(0, shape.vocab, n).tolist() for n in lens]
    flat = np.concatenate(toks).astype(np.int32)
    pos = np.concatenate([np.arange(n) for n in lens]).astype(np.int32)
    slots = np.concatenate([
        np.asarray([bt[s, p // 16].item() * 16 + p % 16 for p in range(n)])
        for s, n in enumerate(lens)]).astype(np.int32)
    fwd.begin()
    fwd.stage(0, {"tokens": flat, "positions": pos, "slots": slots,
                  "seq_slot": np.asarray([0, 1], np.int32),
                  "q_start": np.asarray([0, lens[0]], np.int32),
                  "q_len": np.asarray(lens, np.int32), "q_pos0": np.zeros(2, np.int32),
                  "kv_len": np.asarray(lens, np.int32),
                  "logit_rows": np.arange(sum(lens), dtype=np.int32)})
    fwd.upload(1)
    logits = torch.empty(sum(lens), shape.vocab, dtype=torch.float32, device=dev)
    fwd.run(sum(lens), 2, max(lens), sum(lens), logits, shape.vocab)
    torch.cuda.synchronize()
    om = OracleModel(shape, 11)
    caches = [om.new_cache(64), om.new_cache(64)]
    h = om.forward([(toks[0], 0), (toks[1], 0)], caches)
    ref = om.logits(h, flat.astype(np.int64))
    got = logits.cpu().numpy()
    err = np.abs(got - ref).max()
    assert err <= 1e-2 * np.abs(ref).max(), err
    # and the KV the GPU wrote matches the oracle's cache (layer 0 keys)
    kc = m.kv[0, 0].float().cpu().numpy()
    for s, n in enumerate(lens):
        for p in range(n):
            slot = slots[sum(lens[:s]) + p]
            np.testing.assert_allclose(kc[slot], caches[s][0][0][p], rtol=2e-2, atol=2e-2)


def _tiny_run(mode, backend, n=16, out_len=32, prompt=16, k=4):
    cfg = SimConfig(mode=mode, m=8, k=k, sd_batch_factor=2 if mode == "standard-sd" else 1)
    reqs = make_requests([out_len] * n, prompt_len=prompt)
    return run(cfg, reqs, backend=backend)


def _near_tie_ok(cb, req, gpu_out, cpu_out, tol=0.05):
    """Sequences may only diverge where the oracle's top-2 target logits are
    within ``tol`` (a near-tie that bf16 vs fp32 summation order can flip)."""
    i = next(j for j, (a, b) in enumerate(zip(gpu_out, cpu_out)) if a != b)
    prefix = list(req.prompt_ids) + list(gpu_out[:i])
    cache = cb.t.new_cache(len(prefix) + 1)
    h = cb.t.forward([(prefix, 0)], [cache])
    lg = cb.t.logits(h[-1:], np.asarray([prefix[-1]]), cb.succ, cb.beta_t)[0]
    top = np.argsort(-lg)[:2]
    margin = float(lg[top[0]] - lg[top[1]])
    assert gpu_out[i] in top and cpu_out[i] in top, (i, top, gpu_out[i], cpu_out[i])
    assert margin < tol, margin
    return i, margin


@pytest.mark.parametrize("beta", [3.0, 1.0])
def test_greedy_psd_identical_to_cpu_oracle(cuda_device, beta):
    gb = GpuBackend("tiny-target", "tiny-draft", max_requests=16, max_batch=16, k_max=4,
                    max_seq_len=128, seed=0, beta_target=beta, beta_draft=12.0,
                    prefill_chunk_tokens=512)
    gs, grep = _tiny_run("psd", gb)
    cb = CpuBackend("tiny-target", "tiny-draft", seed=0, beta_target=beta, beta_draft=12.0)
    cs, crep = _tiny_run("psd", cb)
    g = [r.output_ids for r in gs.request_list()]
    c = [r.output_ids for r in cs.request_list()]
    assert grep.finished == 16 and all(len(x) == 32 for x in g)
    for snap in gs.finish_log:
        assert snap.blocks_at_finish == blocks_needed(snap.total_len, 16)
    if beta >= 3.0:
        # clear margins: identical token sequences and identical step logs
        assert g == c
        assert [(s.drafted_tokens, s.accepted_tokens, s.bonus_tokens) for s in gs.step_log] == \
            [(s.drafted_tokens, s.accepted_tokens, s.bonus_tokens) for s in cs.step_log]
    else:
        # weak synthetic-language bias: logits of random-init models have
        # near-ties.  Every token of every GPU sequence (not just the first
        # divergence) must be the oracle target's greedy choice given the GPU's
        # own prefix, or a documented near-tie (tests/_parity.py)
        from tests._parity import oracle_rows, teacher_forced
        exact, ties = 0, []
        for req, a in zip(gs.request_list(), g):
            lg = oracle_rows(cb.t, cb.succ, cb.beta_t, req.prompt_ids, a)
            e, t = teacher_forced(lg, a)
            exact += e
            ties += t
        assert exact >= 0.97 * sum(len(a) for a in g), ties
        # sequences that agree with the oracle PSD up to a divergence diverge
        # only at one of those near-ties
        for req, a, b in zip(gs.request_list(), g, c):
            if a != b:
                _near_tie_ok(cb, req, a, b)


def test_greedy_psd_equals_sd_on_gpu(cuda_device):
    gb = GpuBackend("tiny-target", "tiny-draft", max_requests=16, max_batch=16, k_max=4,
                    max_seq_len=128, seed=0, beta_target=3.0, beta_draft=12.0,
                    prefill_chunk_tokens=512)
    ps, _ = _tiny_run("psd", gb)
    gb2 = GpuBackend("tiny-target", "tiny-draft", max_requests=16, max_batch=16, k_max=4,
                     max_seq_len=128, seed=0, beta_target=3.0, beta_draft=12.0,
                     prefill_chunk_tokens=512)
    ss, _ = _tiny_run("standard-sd", gb2)
    assert [r.output_ids for r in ps.request_list()] == [r.output_ids for r in ss.request_list()]


@pytest.mark.parametrize("temperature", [1.0, 0.7])
def test_sampling_psd_k1_bit_exact_on_real_logits(cuda_device, temperature):
    """Sampling mode end to end: every verification K1 ran inside the PSD loop
    is replayed through the CPU oracle on the same (GPU-produced) logits and
    uniforms -> identical accepted lengths and tokens."""
    from oracle import verify as ov
    gb = GpuBackend("tiny-target", "tiny-draft", max_requests=16, max_batch=16, k_max=4,
                    max_seq_len=128, seed=3, beta_target=1.0, beta_draft=1.0,
                    mode="sample", temperature=temperature, prefill_chunk_tokens=512)
    gb.capture_verify = []
    st, rep = _tiny_run("psd", gb)
    assert rep.finished == 16 and all(len(r.output_ids) == 32 for r in st.request_list())
    assert len(gb.capture_verify) >= 5
    for rec in gb.capture_verify:
        acc, out = ov.verify_sample(rec["target"], rec["draft"], rec["ids"], rec["len"],
                                    rec["uniforms"], temperature)
        np.testing.assert_array_equal(acc, rec["acc"])
        np.testing.assert_array_equal(out, rec["out"])
    assert 0 < rep.total_accepted < rep.total_drafted


def test_continuous_batching_preemption_and_k_overrides_on_gpu(cuda_device):
    """SURVEY §8(f) ranks 1-2 on the GPU path: poisson arrivals (admission while
    other requests decode), preemption of decoding requests, per-request draft
    depth; greedy tokens still equal the CPU oracle's for every request."""
    from paper_2603_18016_b200 import (LengthSpec, Preemption, WorkloadSpec, generate_requests)

    spec = WorkloadSpec(arrival="poisson", rate=0.02, count=12,
                        prompt_len=LengthSpec("uniform", lo=4, hi=20),
                        output_len=LengthSpec("uniform", lo=8, hi=40))
    cfg = SimConfig(mode="psd", m=4, k=4, k_overrides=(1, 2, 3, 4, 4, 3, 2, 1))
    pre = [Preemption(0, 0.0)]  # request 0 arrives first: evicted at its first sync point

    def go(backend):
        reqs = generate_requests(spec, 11)
        return run(cfg, reqs, pre, backend=backend)

    gb = GpuBackend("tiny-target", "tiny-draft", max_requests=16, max_batch=8, k_max=4,
                    max_seq_len=128, seed=0, beta_target=3.0, beta_draft=12.0,
                    prefill_chunk_tokens=512)
    gs, grep = go(gb)
    cs, crep = go(CpuBackend("tiny-target", "tiny-draft", seed=0, beta_target=3.0,
                             beta_draft=12.0))
    assert grep.preempted == crep.preempted == 1
    assert grep.finished == crep.finished == 11
    for a, b in zip(gs.request_list(), cs.request_list()):
        assert a.state == b.state
        if a.state.value == "finished":  # greedy output is schedule independent
            assert a.output_ids == b.output_ids and len(a.output_ids) == a.target_output_len


@pytest.mark.parametrize("draft", ["llama-3.2-1b", "tiny-draft"])
def test_fused_draft_decode_matches_per_kernel_forward(cuda_device, draft):
    from paper_2603_18016_b200 import native
    if not native.has("psd_mk_create"):
        pytest.skip("experimental build only (PSD_EXPERIMENTAL=1)")
    """The fused k-step draft decode (csrc/decode_mk.cu, one persistent kernel)
    proposes the same draft tokens as the per-kernel forward: identical
    drafted / accepted counts in every step and identical outputs."""
    target = "llama-3.2-1b" if draft == "llama-3.2-1b" else "tiny-target"
    kw = dict(max_requests=16, max_batch=16, k_max=4, max_seq_len=128, seed=5,
              beta_target=6.0, beta_draft=12.0, prefill_chunk_tokens=512)
    fused = GpuBackend(target, draft, fused_draft=True, **kw)
    assert fused.mk is not None
    plain = GpuBackend(target, draft, fused_draft=False, **kw)
    assert plain.mk is None
    fs, frep = _tiny_run("psd", fused)
    ps, prep = _tiny_run("psd", plain)
    assert [r.output_ids for r in fs.request_list()] == [r.output_ids for r in ps.request_list()]
    assert [(s.drafted_tokens, s.accepted_tokens) for s in fs.step_log] == \
        [(s.drafted_tokens, s.accepted_tokens) for s in ps.step_log]
    assert frep.total_accepted > 0
    fused.close()


def test_online_k_tuner_on_gpu_keeps_greedy_tokens(cuda_device):
    """the online draft-depth tuner (ktune.KTuner) on
    measured CUDA-event durations.  Greedy output does not depend on the
    draft depth, so tokens must equal the fixed-k run's; the tuner must have
    estimated acceptance and timings and changed depth within [1, k]."""
    from paper_2603_18016_b200 import KTuner
    kw = dict(max_requests=16, max_batch=16, k_max=4, max_seq_len=128, seed=0, beta_target=3.0,
              beta_draft=12.0, prefill_chunk_tokens=512)
    ref, _ = _tiny_run("psd", GpuBackend("tiny-target", "tiny-draft", **kw))
    tuner = KTuner(k_max=4, mode="psd", warmup=2)
    cfg = SimConfig(mode="psd", m=8, k=4)
    st, rep = run(cfg, make_requests([32] * 16, prompt_len=16),
                  backend=GpuBackend("tiny-target", "tiny-draft", **kw), k_tuner=tuner)
    assert [r.output_ids for r in st.request_list()] == [r.output_ids for r in ref.request_list()]
    assert tuner.p is not None and tuner.d and tuner.v
    assert all(1 <= h[1] <= 4 for h in tuner.history)


@pytest.mark.parametrize("preset", ["tiny-qwen", "tiny-draft", "tiny-target"])
def test_decode_step_matches_oracle(cuda_device, preset):
    """Decode passes (1-2 query tokens per sequence) take the fused RoPE + KV
    write + attention kernel (psd_attention_rope), incl. the Qwen2 qkv bias;
    their logits match the numpy oracle within rtol 1e-2 after a prefill."""
    shape = PRESETS[preset]
    dev = cuda_device
    m = Transformer(shape, dev, seed=21, num_blocks=16, block_size=16, max_blocks_per_seq=8)
    bt = torch.zeros(4, 8, dtype=torch.int32, device=dev)
    bt[0, :4] = torch.tensor([1, 2, 3, 4])
    bt[1, :4] = torch.tensor([5, 6, 7, 8])
    fwd = Forward(m, 128, 8, 64, bt)
    rng = np.random.default_rng(3)
    lens = [19, 33]
    toks = [rng.integers(0, shape.vocab, n).tolist() for n in lens]
    nxt = [rng.integers(0, shape.vocab, q).tolist() for q in (1, 2)]

    def slot(s, p):
        return bt[s, p // 16].item() * 16 + p % 16

    def stage_run(seq_toks, p0s, logits_rows):
        flat = np.concatenate(seq_toks).astype(np.int32)
        pos = np.concatenate([np.arange(p0, p0 + len(t)) for t, p0 in zip(seq_toks, p0s)])
        slots = np.concatenate([[slot(s, p0 + i) for i in range(len(t))]
                                for s, (t, p0) in enumerate(zip(seq_toks, p0s))])
        qs = np.cumsum([0] + [len(t) for t in seq_toks])[:-1]
        fwd.begin()
        fwd.stage(0, {"tokens": flat, "positions": pos.astype(np.int32),
                      "slots": slots.astype(np.int32), "seq_slot": np.asarray([0, 1], np.int32),
                      "q_start": qs.astype(np.int32),
                      "q_len": np.asarray([len(t) for t in seq_toks], np.int32),
                      "q_pos0": np.asarray(p0s, np.int32),
                      "kv_len": np.asarray([p0 + len(t) for t, p0 in zip(seq_toks, p0s)],
                                           np.int32),
                      "logit_rows": np.asarray(logits_rows, np.int32)})
        fwd.upload(1)
        out = torch.empty(len(logits_rows), shape.vocab, dtype=torch.float32, device=dev)
        fwd.run(len(flat), 2, max(len(t) for t in seq_toks), len(logits_rows), out, shape.vocab)
        torch.cuda.synchronize()
        return out.cpu().numpy()

    stage_run(toks, [0, 0], [0])                     # prefill (unfused RoPE path)
    got = stage_run(nxt, lens, [0, 1, 2])            # decode: fused RoPE + attention
    om = OracleModel(shape, 21)
    caches = [om.new_cache(64), om.new_cache(64)]
    om.forward([(toks[0], 0), (toks[1], 0)], caches)
    h = om.forward([(nxt[0], lens[0]), (nxt[1], lens[1])], caches)
    ref = om.logits(h, np.concatenate(nxt))
    err = np.abs(got - ref).max()
    assert err <= 1e-2 * np.abs(ref).max(), err
