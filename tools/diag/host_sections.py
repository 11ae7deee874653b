"""Host wall time of the sections of GpuBackend.execute before the draft
graph launch (cfg2 PSD), without a profiler's overhead."""
import sys
import time
import collections
sys.path.insert(0, ".")
import torch
from paper_2603_18016_b200 import SimConfig, make_requests, run
from paper_2603_18016_b200.gpu import GpuBackend

be = GpuBackend("llama-3.1-8b", "llama-3.2-1b", max_requests=64, max_batch=64, k_max=5,
                max_seq_len=128 + 256 + 16, seed=0, beta_target=7.0, beta_draft=16.0)
cfg = SimConfig(mode="psd", m=32, k=5)
for _ in range(2):
    run(cfg, make_requests([256] * 64, prompt_len=128), backend=be)
torch.cuda.synchronize()
acc = collections.defaultdict(float)
cnt = collections.Counter()


def wrap(name):
    f = getattr(be, name)

    def g(*a, **k):
        t0 = time.perf_counter()
        r = f(*a, **k)
        acc[name] += time.perf_counter() - t0
        cnt[name] += 1
        return r
    setattr(be, name, g)


for n in ("_upload_block_table", "_draft_loop", "_draft_rows", "_run_graph", "_verify",
          "_admit", "_prefill"):
    wrap(n)
# host time from entering execute to the first draft-graph replay of the step
t_in = [0.0]
f_exec, f_graph = be.execute, be._run_graph


def ex(*a, **k):
    t_in[0] = time.perf_counter()
    t0 = time.perf_counter()
    r = f_exec(*a, **k)
    acc["execute"] += time.perf_counter() - t0
    cnt["execute"] += 1
    return r


def rg(key, launch):
    if key[0] == "draft" and t_in[0]:
        acc["execute -> draft replay"] += time.perf_counter() - t_in[0]
        cnt["execute -> draft replay"] += 1
        t_in[0] = 0.0
    return f_graph(key, launch)


be.execute, be._run_graph = ex, rg
fwd = be.dfwd
for n in ("stage", "stage_many", "upload", "begin"):
    f = getattr(fwd, n)

    def g(*a, _f=f, _n=n, **k):
        t0 = time.perf_counter()
        r = _f(*a, **k)
        acc["dfwd." + _n] += time.perf_counter() - t0
        cnt["dfwd." + _n] += 1
        return r
    setattr(fwd, n, g)
t0 = time.perf_counter()
st, rep = run(cfg, make_requests([256] * 64, prompt_len=128), backend=be)
torch.cuda.synchronize()
wall = time.perf_counter() - t0
steps = len(st.step_log)
print(f"wall {wall * 1e3:.1f} ms, {steps} steps")
for k, v in sorted(acc.items(), key=lambda x: -x[1]):
    print(f"  {k:24s} {v * 1e3 / steps:8.3f} ms/step  ({cnt[k]} calls)")
