"""Launch K1 at the cfg2 shape a few times (target for ncu captures)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2603_18016_b200 import ops  # noqa: E402
from paper_2603_18016_b200.verify_bench import make_inputs  # noqa: E402

B, K, V = (int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (32, 5, 128256)))
dev = torch.device("cuda:0")
for sampling in (False, True):
    t, d, ids, ln, u = make_inputs(B, K, V, sampling, dev)
    for _ in range(4):
        if sampling:
            ops.verify_sample(t, d, ids, ln, u)
        else:
            ops.verify_greedy(t, ids, ln)
    torch.cuda.synchronize()
print("done")
