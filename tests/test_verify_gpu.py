"""K1 on the GPU vs the CPU oracle: bit-exact accepted lengths and tokens.

Sweep subset of BASELINE config 5 (batch x k x vocab, greedy and sampling),
ragged draft lengths incl. idle rows, draft vocab < target vocab, ties,
temperature, workspace reuse across launches, the golden vectors.
"""

import json
import os

import numpy as np
import pytest
import torch

from oracle import verify as ov
from paper_2603_18016_b200 import ops
from tests import _gen

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "verify_golden.json")


def _run_gpu(t, d, ids, ln, u, greedy, temperature=1.0):
    dev = torch.device("cuda:0")
    tt = torch.from_numpy(t).to(dev)
    ii = torch.from_numpy(np.ascontiguousarray(ids)).to(dev)
    ll = torch.from_numpy(ln).to(dev)
    if greedy:
        acc, out = ops.verify_greedy(tt, ii, ll)
    else:
        dd = torch.from_numpy(d).to(dev)
        uu = torch.from_numpy(u).to(dev)
        acc, out = ops.verify_sample(tt, dd, ii, ll, uu, temperature)
    torch.cuda.synchronize()
    return acc.cpu().numpy(), out.cpu().numpy()


CASES = [
    # (B, K, V, Vd, tau)
    (1, 1, 32000, 32000, 0.5),
    (3, 4, 65536, 65536, 0.3),
    (32, 5, 128256, 128256, 0.5),
    (8, 8, 152064, 151936, 0.7),
    (64, 4, 32000, 32000, 1.0),
    (2, 0, 4096, 4096, 0.5),
    (5, 16, 8192, 8192, 0.4),
]


@pytest.mark.parametrize("greedy", [True, False])
@pytest.mark.parametrize("B,K,V,Vd,tau", CASES)
def test_gpu_matches_oracle(cuda_device, B, K, V, Vd, tau, greedy):
    seed = B * 1000 + K * 10 + (V % 97)
    t, d, ids, ln, u = _gen.verify_case(seed, B, K, V, Vd, tau, greedy=greedy)
    if greedy:
        ea, eo = ov.verify_greedy(t, ids, ln)
    else:
        ea, eo = ov.verify_sample(t, d, ids, ln, u)
    for _ in range(2):  # second launch reuses the self-cleaning workspace
        ga, go = _run_gpu(t, d, ids, ln, u, greedy)
        np.testing.assert_array_equal(ga, ea)
        np.testing.assert_array_equal(go, eo)


def test_gpu_greedy_ties_lowest_index(cuda_device):
    t, d, ids, ln, u = _gen.verify_case(9, 4, 2, 40000, greedy=True)
    t[:, :, 123] = 100.0
    t[:, :, 35000] = 100.0
    ids[:] = 123
    ln[:] = 2
    ga, go = _run_gpu(t, d, ids, ln, u, True)
    assert (ga == 2).all() and (go == 123).all()


def test_gpu_temperature(cuda_device):
    t, d, ids, ln, u = _gen.verify_case(21, 6, 3, 50000, tau=0.6)
    ea, eo = ov.verify_sample(t, d, ids, ln, u, 0.6)
    ga, go = _run_gpu(t, d, ids, ln, u, False, 0.6)
    np.testing.assert_array_equal(ga, ea)
    np.testing.assert_array_equal(go, eo)


def test_gpu_golden_vectors(cuda_device):
    with open(GOLDEN) as fh:
        cases = json.load(fh)
    for c in cases:
        t, d, ids, ln, u = _gen.verify_case(c["seed"], c["B"], c["K"], c["V"], c["Vd"],
                                            c["tau"], greedy=c["greedy"])
        ga, go = _run_gpu(t, d, ids, ln, u, c["greedy"], c["temperature"])
        assert ga.tolist() == c["accepted_len"], c["name"]
        assert go.tolist() == c["out_tokens"], c["name"]


@pytest.mark.parametrize("B,K,V,Vd,temperature", [(32, 5, 128256, 128256, 1.0),
                                                  (8, 8, 152064, 151936, 0.7),
                                                  (5, 3, 8192, 8192, 1.3)])
def test_cached_draft_stats_bit_exact(cuda_device, B, K, V, Vd, temperature):
    """psd_verify_sample_ext: the draft sampler's pass (K = 0 over the draft
    rows) publishes each row's canonical (max, sum); K1 given those cached
    statistics skips re-reading the draft rows and still matches the oracle
    (and the uncached kernel) bit for bit."""
    t, d, ids, ln, u = _gen.verify_case(B * 7 + K, B, K, V, tau=0.6, greedy=False, Vd=Vd)
    dev = cuda_device
    dd = torch.from_numpy(d).to(dev)
    rows = dd.reshape(B * K, 1, Vd)
    stats = torch.full((B, K, 2), float("nan"), device=dev)
    zeros = torch.zeros(B * K, dtype=torch.int32, device=dev)
    ops.verify_sample(rows, rows[:, :0], torch.zeros(B * K, 0, dtype=torch.int32, device=dev),
                      zeros, torch.rand(B * K, 1, device=dev), temperature,
                      t_stats_out=stats.view(B * K, 2),
                      t_stats_rows=torch.arange(B * K, dtype=torch.int32, device=dev))
    tt = torch.from_numpy(t).to(dev)
    ii = torch.from_numpy(np.ascontiguousarray(ids)).to(dev)
    ll = torch.from_numpy(ln).to(dev)
    uu = torch.from_numpy(u).to(dev)
    acc, out = ops.verify_sample(tt, dd, ii, ll, uu, temperature, d_stats=stats)
    acc0, out0 = ops.verify_sample(tt, dd, ii, ll, uu, temperature)
    torch.cuda.synchronize()
    ea, eo = ov.verify_sample(t, d, ids, ln, u, temperature)
    np.testing.assert_array_equal(acc.cpu().numpy(), ea)
    np.testing.assert_array_equal(out.cpu().numpy(), eo)
    np.testing.assert_array_equal(acc0.cpu().numpy(), ea)
    np.testing.assert_array_equal(out0.cpu().numpy(), eo)
