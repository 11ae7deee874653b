"""Regression vectors for the verification oracle (and the GPU kernel).

    python tests/golden/make_verify_golden.py

Inputs are regenerated from seeds by tests/_gen.py (splitmix64, numpy-version
independent); only seeds, shapes and the oracle's outputs are stored.  The
oracle itself is pinned by tests/test_verify_oracle.py (float64 evaluation,
distributional identity); these vectors freeze its exact outputs so the GPU
kernel (tests/test_verify_gpu.py) and future oracle edits are held to them.
"""

import json
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))

from oracle import verify as ov  # noqa: E402
from tests import _gen  # noqa: E402

CASES = [
    dict(name="greedy-small", seed=101, B=8, K=4, V=1024, Vd=1024, tau=0.3, greedy=True,
         temperature=1.0),
    dict(name="greedy-3slice", seed=102, B=3, K=5, V=20000, Vd=20000, tau=0.2, greedy=True,
         temperature=1.0),
    dict(name="sample-small", seed=103, B=8, K=4, V=1024, Vd=1024, tau=0.6, greedy=False,
         temperature=1.0),
    dict(name="sample-3slice", seed=104, B=3, K=5, V=20000, Vd=19996, tau=0.5, greedy=False,
         temperature=1.0),
    dict(name="sample-temp0.7", seed=105, B=4, K=3, V=4100, Vd=4100, tau=0.8, greedy=False,
         temperature=0.7),
    dict(name="sample-k1", seed=106, B=5, K=1, V=9000, Vd=8800, tau=1.0, greedy=False,
         temperature=1.3),
]


def main():
    out = []
    for c in CASES:
        t, d, ids, ln, u = _gen.verify_case(c["seed"], c["B"], c["K"], c["V"], c["Vd"],
                                            c["tau"], greedy=c["greedy"])
        if c["greedy"]:
            acc, tok = ov.verify_greedy(t, ids, ln)
        else:
            acc, tok = ov.verify_sample(t, d, ids, ln, u, c["temperature"])
        out.append(dict(c, accepted_len=acc.tolist(), out_tokens=tok.tolist()))
    path = os.path.join(os.path.dirname(__file__), "verify_golden.json")
    with open(path, "w") as fh:
        json.dump(out, fh, indent=1)
    print("wrote", path)


if __name__ == "__main__":
    main()
