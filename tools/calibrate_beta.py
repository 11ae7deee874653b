"""Mean accepted length vs the target's synthetic-language bias (cfg2 shapes)."""
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2603_18016_b200 import SimConfig, make_requests, mean_accepted_length, run  # noqa: E402
from paper_2603_18016_b200.gpu import GpuBackend  # noqa: E402

bt = [float(x) for x in sys.argv[1].split(",")] if len(sys.argv) > 1 else [5, 6, 7, 8, 9]
bd = float(sys.argv[2]) if len(sys.argv) > 2 else 16.0
be = GpuBackend("llama-3.1-8b", "llama-3.2-1b", max_requests=64, max_batch=64, k_max=5,
                max_seq_len=128 + 256 + 16, seed=0, beta_target=bt[0], beta_draft=bd)
for b in bt:
    be.beta_target = b
    t0 = time.time()
    st, rep = run(SimConfig(mode="psd", m=32, k=5), make_requests([48] * 64, prompt_len=128),
                  backend=be)
    torch.cuda.synchronize()
    print(f"beta_t={b} beta_d={bd} mean_acc_len={mean_accepted_length(rep):.3f} "
          f"vsr={rep.vsr:.3f} steps={rep.total_steps} wall={time.time() - t0:.2f}s "
          f"draft_ms={be.stats['draft_ms']:.0f} verify_ms={be.stats['verify_ms']:.0f}",
          flush=True)
