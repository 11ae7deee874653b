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


def execute(state, plan, rows):
    torch.cuda.synchronize()
    e = torch.cuda.Event(enable_timing=True)
    e.record(be.s_target)
    marks.append([e, None])
    return orig_exec(state, plan, rows)


def run_graph(key, launch):
    if key[0] == "draft" and marks and marks[-1][1] is None:
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        marks[-1][1] = e
    orig_graph(key, launch)


be.execute, be._run_graph = execute, run_graph
st, rep = run(cfg, make_requests([256] * 64, prompt_len=128), backend=be)
torch.cuda.synchronize()
gaps = [a.elapsed_time(b) for a, b in marks if b is not None]
steps = sum(r.step_duration for r in st.step_log)
print(f"{len(gaps)} steps: step-start -> draft graph {sum(gaps) / len(gaps) * 1e3:.0f} us mean, "
      f"{sum(gaps):.1f} ms of {steps:.1f} ms device step time ({100 * sum(gaps) / steps:.1f} %)")
