"""GPU idle at the start of a PSD step: from the step's first event (after
the host synchronised on the previous step) to the draft graph's start on
the draft stream, i.e. the host building the step's metadata (cfg2)."""
import sys
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
orig_exec, orig_graph = be.execute, be._run_graph
marks = []


ds_marks = []
import time
host = []


def execute(state, plan, rows):
    torch.cuda.synchronize()
    host.append([time.perf_counter(), None])
    e = torch.cuda.Event(enable_timing=True)
    e.record(be.s_target)
    e2 = torch.cuda.Event(enable_timing=True)
    e2.record(be.s_draft)
    ds_marks.append(e2)
    marks.append([e, None])
    return orig_exec(state, plan, rows)


def run_graph(key, launch):
    if key[0] == "draft" and marks and marks[-1][1] is None:
        host[-1][1] = time.perf_counter()
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        marks[-1][1] = e
    orig_graph(key, launch)


up_marks = []
orig_up = be.dfwd.upload


def upload(n_sets=1):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    orig_up(n_sets)
    e1.record()
    up_marks.append((len(marks), e0, e1))


be.dfwd.upload = upload
be.execute, be._run_graph = execute, run_graph
st, rep = run(cfg, make_requests([256] * 64, prompt_len=128), backend=be)
torch.cuda.synchronize()
gaps = [a.elapsed_time(b) for a, b in marks if b is not None]
hg = [b - a for a, b in host if b is not None]
print(f"host: execute entry -> draft replay {sum(hg) / len(hg) * 1e6:.0f} us")
dsg = [a.elapsed_time(b) for a, (_, b) in zip(ds_marks, marks) if b is not None]
print(f"draft-stream mark -> draft graph {sum(dsg) / len(dsg) * 1e3:.0f} us; target-stream mark -> "
      f"draft-stream mark {sum(m[0].elapsed_time(d) for m, d in zip(marks, ds_marks)) / len(ds_marks) * 1e3:.0f} us")
# per step: step start -> upload issued on the GPU, upload duration
pre, dur = [], []
for idx, e0, e1 in up_marks:
    if 0 < idx <= len(marks):
        pre.append(marks[idx - 1][0].elapsed_time(e0))
        dur.append(e0.elapsed_time(e1))
if pre:
    print(f"step start -> metadata upload begins {sum(pre) / len(pre) * 1e3:.0f} us, upload "
          f"{sum(dur) / len(dur) * 1e3:.0f} us (GPU time)")
steps = sum(r.step_duration for r in st.step_log)
print(f"{len(gaps)} steps: step-start -> draft graph {sum(gaps) / len(gaps) * 1e3:.0f} us mean, "
      f"{sum(gaps):.1f} ms of {steps:.1f} ms device step time ({100 * sum(gaps) / steps:.1f} %)")
