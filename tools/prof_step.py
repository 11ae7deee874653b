"""A short cfg2-shaped PSD run (target for ncu launch lists).

    python tools/prof_step.py [out_len] [dual]
"""
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2603_18016_b200 import SimConfig, make_requests, mean_accepted_length, run  # noqa: E402
from paper_2603_18016_b200.gpu import GpuBackend  # noqa: E402

out_len = int(sys.argv[1]) if len(sys.argv) > 1 else 24
dual = (sys.argv[2] != "0") if len(sys.argv) > 2 else True
graphs = (sys.argv[3] != "0") if len(sys.argv) > 3 else True
be = GpuBackend("llama-3.1-8b", "llama-3.2-1b", max_requests=64, max_batch=64, k_max=5,
                max_seq_len=128 + 256 + 16, seed=0, beta_target=7.0, beta_draft=16.0,
                dual_stream=dual, use_graphs=graphs)
cfg = SimConfig(mode="psd", m=32, k=5)
for _ in range(2):
    st, rep = run(cfg, make_requests([out_len] * 64, prompt_len=128), backend=be)
torch.cuda.synchronize()
be.stats = {"draft_ms": 0.0, "verify_ms": 0.0, "prefill_ms": 0.0, "steps": 0}
t0 = time.perf_counter()
st, rep = run(cfg, make_requests([out_len] * 64, prompt_len=128), backend=be)
torch.cuda.synchronize()
dt = time.perf_counter() - t0
print(f"dual={dual} graphs={graphs} out_len={out_len} wall={dt*1e3:.1f}ms "
      f"tok/s={rep.total_generated/dt:.0f} steps={rep.total_steps} "
      f"mean_acc={mean_accepted_length(rep):.2f} stats={be.stats}")
for s in st.step_log[:12]:
    print(s.step_index, s.target_batch, s.drafted_tokens, s.accepted_tokens, s.bonus_tokens,
          f"draft={s.draft_duration:.2f} verify={s.verify_duration:.2f} "
          f"prefill={s.prefill_duration:.2f} step={s.step_duration:.2f}")
