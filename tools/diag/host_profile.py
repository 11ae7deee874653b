"""Host-side (Python) cost of a cfg2 PSD run: cProfile of the scheduler +
GpuBackend while the GPU runs, top functions by own time."""
import cProfile
import pstats
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
pr = cProfile.Profile()
pr.enable()
st, rep = run(cfg, make_requests([256] * 64, prompt_len=128), backend=be)
torch.cuda.synchronize()
pr.disable()
ps = pstats.Stats(pr).sort_stats("tottime")
ps.print_stats(25)
ps.sort_stats("cumulative").print_stats("gpu.py|model.py|scheduler.py|ops.py|native.py", 30)
ps.print_callees("_draft_rows|_verify$")
