"""Where does greedy SD(m) diverge from PSD at the bench's cfg2 workload?

For every request whose tokens differ, print the first differing position and
the GPU target's top-2 logit margin there (teacher-forced prefill of prompt +
PSD output), plus the admission / prefill pattern of both runs."""
import sys

import numpy as np

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2603_18016_b200 import run  # noqa: E402
from paper_2603_18016_b200.gpu import GpuBackend  # noqa: E402
from tests._parity import gpu_logits  # noqa: E402

C = bench.CFG
be = GpuBackend(C["target"], C["draft"], max_requests=C["n_requests"], max_batch=C["n_requests"],
                k_max=C["k"], max_seq_len=C["prompt"] + C["output"] + 16, seed=0,
                beta_target=bench.BETA_TARGET, beta_draft=bench.BETA_DRAFT)
outs = {}
for mode in ("psd", "sd-m", "standard-sd"):
    st, rep = run(bench._config(mode), bench._workload(0), backend=be)
    outs[mode] = st
    print(mode, "steps", len(st.step_log), "prefill steps",
          sum(1 for r in st.step_log if r.prefill_duration > 0))
p = outs["psd"].request_list()
for other in ("sd-m", "standard-sd"):
    o = outs[other].request_list()
    bad = [(a, b) for a, b in zip(p, o) if a.output_ids != b.output_ids]
    print(f"{other}: {len(bad)} of {len(p)} requests differ")
    for a, b in bad[:8]:
        i = next(j for j, (x, y) in enumerate(zip(a.output_ids, b.output_ids)) if x != y)
        lg = gpu_logits(be, a.prompt_ids, a.output_ids[:i + 1])[i]
        top = np.sort(lg)[-2:]
        print(f"  req {a.id}: first diff at {i}: psd {a.output_ids[i]} vs {b.output_ids[i]}, "
              f"logit[psd]={lg[a.output_ids[i]]:.4f} logit[other]={lg[b.output_ids[i]]:.4f} "
              f"top2 margin {top[1] - top[0]:.4f}")
