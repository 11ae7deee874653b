"""Is the SD(m) divergence history-dependent (slot / KV block reuse) or
composition-dependent?  Runs on fresh backends: (a) PSD, all 64 requests;
(b) SD(m), all 64; (c) SD(m) of requests 32..63 alone; (d) PSD, all 64, on a
backend that first ran SD(m) (reused slots / blocks)."""
import sys

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2603_18016_b200 import make_requests, run  # noqa: E402
from paper_2603_18016_b200.gpu import GpuBackend  # noqa: E402

C = bench.CFG


def backend():
    return GpuBackend(C["target"], C["draft"], max_requests=C["n_requests"],
                      max_batch=C["n_requests"], k_max=C["k"],
                      max_seq_len=C["prompt"] + C["output"] + 16, seed=0,
                      beta_target=bench.BETA_TARGET, beta_draft=bench.BETA_DRAFT)


def outs(st):
    return {r.id: r.output_ids for r in st.request_list()}


be = backend()
a = outs(run(bench._config("psd"), bench._workload(0), backend=be)[0])
b = outs(run(bench._config("sd-m"), bench._workload(0), backend=be)[0])
d = outs(run(bench._config("psd"), bench._workload(0), backend=be)[0])
reqs = [r for r in make_requests([C["output"]] * C["n_requests"], prompt_len=C["prompt"])
        if r.id >= 32]
c = outs(run(bench._config("sd-m"), reqs, backend=backend())[0])
hi = range(32, 64)
print("psd vs sd-m (32..63) differ:", sum(a[i] != b[i] for i in hi))
print("psd vs sd-m alone (32..63) differ:", sum(a[i] != c[i] for i in hi))
print("sd-m vs sd-m alone (32..63) differ:", sum(b[i] != c[i] for i in hi))
print("psd vs psd after sd-m (all) differ:", sum(a[i] != d[i] for i in range(64)))
