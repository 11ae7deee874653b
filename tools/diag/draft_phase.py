"""Time the real draft phase (GpuBackend's captured k-step draft graph) at
cfg2 shapes: an SD(m) run (draft then verify, nothing concurrent) with the
per-phase CUDA-event times the backend records."""
import sys
sys.path.insert(0, ".")
import torch
from paper_2603_18016_b200 import SimConfig, make_requests, run
from paper_2603_18016_b200.gpu import GpuBackend

be = GpuBackend("llama-3.1-8b", "llama-3.2-1b", max_requests=64, max_batch=64, k_max=5,
                max_seq_len=128 + 256 + 16, seed=0, beta_target=7.0, beta_draft=16.0)
cfg = SimConfig(mode="standard-sd", m=32, k=5, sd_batch_factor=1)
for _ in range(2):
    run(cfg, make_requests([256] * 64, prompt_len=128), backend=be)
torch.cuda.synchronize()
be.stats = {"draft_ms": 0.0, "verify_ms": 0.0, "prefill_ms": 0.0, "steps": 0}
st, rep = run(cfg, make_requests([256] * 64, prompt_len=128), backend=be)
torch.cuda.synchronize()
n = be.stats["steps"]
print(f"SD(m) steps {n}: draft {be.stats['draft_ms'] / n:.3f} ms/step, verify "
      f"{be.stats['verify_ms'] / n:.3f} ms/step, launches {be.launches}")

# pure device time of the captured draft graphs (events right around each
# replay) vs the phase time the backend records (from the phase's first event,
# i.e. including the host building that phase's metadata)
orig = be._run_graph
evs = []


def timed_graph(key, launch):
    if key[0] == "draft":
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        orig(key, launch)
        e1.record()
        evs.append((e0, e1))
    else:
        orig(key, launch)


be._run_graph = timed_graph
be.stats = {"draft_ms": 0.0, "verify_ms": 0.0, "prefill_ms": 0.0, "steps": 0}
st, rep = run(cfg, make_requests([256] * 64, prompt_len=128), backend=be)
torch.cuda.synchronize()
n = be.stats["steps"]
g = sum(a.elapsed_time(b) for a, b in evs)
print(f"draft phase {be.stats['draft_ms'] / n:.3f} ms/step; draft graphs alone {g / n:.3f} ms/step "
      f"({len(evs)} replays)")
