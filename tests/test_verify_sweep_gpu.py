"""K1 at the corners of BASELINE config 5 (verification sweep): batch 128-512,
k 1 and 8, vocabulary 32000 and 262144 (= PSD_MAX_SLICES x 8192, the largest
the kernel takes), greedy and sampling, ragged draft lengths.

The inputs live on the GPU (up to 9 GB of fp32 logits at B 512, k 8, V 262144);
K1 runs over the whole batch.  Verification rows are independent (each request's
decision reads only its own logit rows: acceptance_model.py:82-97 is per row),
so the CPU oracle re-decides a seeded sample of 24 requests -- always including
the first and last -- and the GPU's accepted lengths and tokens must match it
bit for bit.  A second launch over the same workspace must reproduce the first.
"""

import numpy as np
import pytest
import torch

from oracle import verify as ov
from paper_2603_18016_b200 import ops

pytestmark = pytest.mark.gpu

N_CHECK = 24


def _inputs(B, K, V, Vd, greedy, temperature, seed, dev):
    g = torch.Generator(device=dev).manual_seed(seed)
    t = torch.randn(B, K + 1, V, device=dev, generator=g).mul_(2.0)
    d = None
    if K:
        d = t[:, :K, :Vd] + 0.5 * torch.randn(B, K, Vd, device=dev, generator=g)
    if greedy:
        ids = (d.argmax(dim=2).to(torch.int32) if K
               else torch.zeros(B, 0, dtype=torch.int32, device=dev))
    else:
        # Gumbel-max draw from q = softmax(d / T), chunked to bound scratch memory
        ids = torch.empty(B, K, dtype=torch.int32, device=dev)
        for b0 in range(0, B, 32):
            dd = d[b0:b0 + 32]
            gum = -torch.log(-torch.log(torch.rand(dd.shape, device=dev, generator=g)
                                        .clamp_(1e-12, 1 - 1e-7)))
            ids[b0:b0 + 32] = (dd / temperature + gum).argmax(dim=2).to(torch.int32)
            del gum
    ln = torch.randint(0, K + 1, (B,), device=dev, generator=g, dtype=torch.int32)
    ln[0] = K
    u = torch.rand(B, K + 1, device=dev, generator=g)
    return t, d, ids.contiguous(), ln, u


@pytest.mark.parametrize("greedy", [True, False], ids=["greedy", "sample"])
@pytest.mark.parametrize("V,Vd", [(32000, 32000), (262144, 262144), (262144, 256000)])
@pytest.mark.parametrize("K", [1, 8])
@pytest.mark.parametrize("B", [128, 256, 512])
def test_sweep_corner_matches_oracle(cuda_device, B, K, V, Vd, greedy):
    if greedy and Vd != V:
        pytest.skip("draft vocabulary only matters for sampling")
    dev = cuda_device
    temperature = 1.0 if (B + K) % 2 else 0.8
    seed = B * 131 + K * 17 + V % 1009 + int(greedy)
    t, d, ids, ln, u = _inputs(B, K, V, Vd, greedy, temperature, seed, dev)
    if d is None:
        d = t[:, :0, :Vd]
    runs = []
    for _ in range(2):
        if greedy:
            acc, out = ops.verify_greedy(t, ids, ln)
        else:
            acc, out = ops.verify_sample(t, d, ids, ln, u, temperature)
        torch.cuda.synchronize()
        runs.append((acc.cpu().numpy().copy(), out.cpu().numpy().copy()))
    np.testing.assert_array_equal(runs[0][0], runs[1][0])
    np.testing.assert_array_equal(runs[0][1], runs[1][1])
    ga, go = runs[0]
    assert ((ga >= 0) & (ga <= ln.cpu().numpy())).all()

    rng = np.random.default_rng(seed)
    rows = np.unique(np.concatenate([[0, B - 1], rng.choice(B, N_CHECK - 2, replace=False)]))
    ri = torch.from_numpy(rows).to(dev)
    t_s = t.index_select(0, ri).cpu().numpy()
    ids_s = ids.index_select(0, ri).cpu().numpy()
    ln_s = ln.index_select(0, ri).cpu().numpy()
    if greedy:
        ea, eo = ov.verify_greedy(t_s, ids_s, ln_s)
    else:
        d_s = d.index_select(0, ri).cpu().numpy()
        u_s = u.index_select(0, ri).cpu().numpy()
        ea, eo = ov.verify_sample(t_s, d_s, ids_s, ln_s, u_s, temperature)
    np.testing.assert_array_equal(ga[rows], ea)
    np.testing.assert_array_equal(go[rows], eo)
    if K and not greedy:
        # the sample exercises both outcomes: some rejections and some acceptances
        assert 0 < int(ga.sum()) < int(ln.sum().item())
