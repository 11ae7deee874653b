"""Per-op timeline of the fused draft decode kernel (csrc/decode_mk.cu).

    python tools/mk_trace.py [nb] [steps] [grid]

Runs a short PSD pass to build the (nb, steps) program, then one traced
launch: every CTA stamps %globaltimer at each op's entry, inputs-ready and
done.  Prints, per op type, the time between consecutive op completions (the
critical path) summed over layers, and the first layer's ops in order.
"""
import collections
import os
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2603_18016_b200 import SimConfig, make_requests, native, run  # noqa: E402
from paper_2603_18016_b200.gpu import GpuBackend  # noqa: E402

nb = int(sys.argv[1]) if len(sys.argv) > 1 else 32
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
grid = int(sys.argv[3]) if len(sys.argv) > 3 else 0
be = GpuBackend("llama-3.2-1b", "llama-3.2-1b", max_requests=64, max_batch=64, k_max=steps,
                max_seq_len=128 + 64 + 16, seed=0, beta_target=7.0, beta_draft=16.0,
                fused_draft=True, mk_grid=grid, dual_stream=False)
cfg = SimConfig(mode="psd", m=nb, k=steps)
run(cfg, make_requests([40] * (2 * nb), prompt_len=128), backend=be)
torch.cuda.synchronize()
lib = native.load()
n_ops = lib.psd_mk_n_ops(be.mk, nb, steps)
G = lib.psd_mk_grid(be.mk)
assert n_ops > 0, "program not built"
tr = torch.zeros(G * n_ops * 3, dtype=torch.int64, device=be.device)
st = torch.cuda.current_stream().cuda_stream
for _ in range(3):
    native.check(lib.psd_mk_launch_traced(be.mk, nb, steps, tr.data_ptr(), st), "traced")
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
native.check(lib.psd_mk_launch(be.mk, nb, steps, st), "mk")
e1.record()
torch.cuda.synchronize()
print(f"untraced launch: {e0.elapsed_time(e1):.3f} ms for {steps} steps, nb={nb}, grid={G}")
t = tr.view(G, n_ops, 3).cpu().numpy().astype(np.float64)
t0 = t[:, 0, 0].min()
end = t[:, :, 2].max(axis=0) - t0
ready = t[:, :, 1].max(axis=0) - t0
L = be.dshape.layers
names = ["embed+norm"] + ["qkv", "rope+attn", "o", "add+norm", "gate/up", "down", "add+norm2"] * L \
    + ["lm_head+argmax", "argmax"]
per_step = len(names)
assert per_step * steps == n_ops, (per_step, steps, n_ops)
tot = collections.defaultdict(float)
prev = 0.0
for j in range(n_ops):
    d = end[j] - prev
    tot[names[j % per_step]] += d
    prev = end[j]
print(f"traced total {end[-1] / 1e3:.1f} us")
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"  {k:16s} {v / 1e3:9.1f} us  {v / end[-1] * 100:5.1f}%")
print("first layer of step 1 (us): op, inputs-ready(max over CTAs), done(max)")
base = per_step * min(1, steps - 1)
for j in range(base, base + 9):
    print(f"  {names[j % per_step]:14s} ready {ready[j] / 1e3:9.1f}  done {end[j] / 1e3:9.1f}")
be.close()
