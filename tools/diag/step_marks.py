"""Where the GPU falls behind the host at the start of a PSD step (cfg2):
events on the draft stream at points inside GpuBackend.execute, each paired
with the host clock when it was enqueued.  Prints, per mark, the mean host
time and mean GPU time since the step's first mark -- a GPU time well above
the host time means the device (not Python) delays that point."""
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

steps = []  # per step: list of (name, host_t, event)


def mark(name, stream=None):
    e = torch.cuda.Event(enable_timing=True)
    e.record(stream if stream is not None else torch.cuda.current_stream())
    steps[-1].append((name, time.perf_counter(), e))


orig = {}


def wrap(obj, name, before=None, after=None):
    f = getattr(obj, name)

    def g(*a, **k):
        if before:
            mark(before)
        r = f(*a, **k)
        if after:
            mark(after)
        return r
    setattr(obj, name, g)


def execute(state, plan, rows):
    torch.cuda.synchronize()
    steps.append([])
    mark("entry(ds)", be.s_draft)
    return orig["execute"](state, plan, rows)


orig["execute"] = be.execute
be.execute = execute
wrap(be, "_upload_block_table", "bt.before", "bt.after")
wrap(be.dfwd, "begin", "dfwd.begin", None)
wrap(be.dfwd, "upload", "dfwd.upload.before", "dfwd.upload.after")
wrap(be.tfwd, "upload", "tfwd.upload.before", "tfwd.upload.after")
og = be._run_graph


def run_graph(key, launch):
    mark(f"{key[0]}.replay.before")
    og(key, launch)
    mark(f"{key[0]}.replay.after")


be._run_graph = run_graph
st, rep = run(cfg, make_requests([256] * 64, prompt_len=128), backend=be)
torch.cuda.synchronize()
host = collections.defaultdict(list)
gpu = collections.defaultdict(list)
order = []
for marks in steps[1:]:
    if not any(n == "draft.replay.before" for n, _, _ in marks):
        continue
    _, h0, e0 = marks[0]
    seen = set()
    for n, h, e in marks:
        if n in seen:
            continue
        seen.add(n)
        if n not in order:
            order.append(n)
        host[n].append((h - h0) * 1e6)
        gpu[n].append(e0.elapsed_time(e) * 1e3)
print(f"{len(host['entry(ds)'])} steps; mean us since the step's first mark (first occurrence)")
print(f"  {'mark':24s} {'host':>8s} {'gpu':>8s} {'gpu-host':>9s}")
for n in order:
    hh = sum(host[n]) / len(host[n])
    gg = sum(gpu[n]) / len(gpu[n])
    print(f"  {n:24s} {hh:8.0f} {gg:8.0f} {gg - hh:9.0f}")
