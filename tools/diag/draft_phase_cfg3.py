"""cfg3 draft phase (Qwen2.5-0.5B, k = 4, 32 sequences): device time of the
captured k-step draft graph in sampling mode (LM head -> q rows -> Philox ->
K1 k = 0 -> scatter per step) vs greedy mode (K6: argmax in the LM-head
epilogue) -- the difference is what drafting by sampling costs."""
import sys
sys.path.insert(0, ".")
import torch
from paper_2603_18016_b200 import SimConfig, make_requests, run
from paper_2603_18016_b200.gpu import GpuBackend

for mode in ("sample", "greedy"):
    be = GpuBackend("qwen2.5-7b", "qwen2.5-0.5b", max_requests=64, max_batch=64, k_max=4,
                    max_seq_len=128 + 256 + 16, seed=0, beta_target=14.0, beta_draft=14.0,
                    mode=mode, temperature=1.0)
    cfg = SimConfig(mode="standard-sd", m=32, k=4, sd_batch_factor=1)
    run(cfg, make_requests([64] * 64, prompt_len=128), backend=be)
    torch.cuda.synchronize()
    orig = be._run_graph
    evs = []

    def timed(key, launch, orig=orig, evs=evs):
        if key[0] == "draft":
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            orig(key, launch)
            e1.record()
            evs.append((key, e0, e1))
        else:
            orig(key, launch)
    be._run_graph = timed
    be.stats = {"draft_ms": 0.0, "verify_ms": 0.0, "prefill_ms": 0.0, "steps": 0}
    run(cfg, make_requests([128] * 64, prompt_len=128), backend=be)
    torch.cuda.synchronize()
    ts = [a.elapsed_time(b) for k, a, b in evs if k[2] == 4]
    n = be.stats["steps"]
    print(f"{mode:6s}: draft graph (k=4, 32 seqs) {sum(ts) / len(ts) * 1e3:7.1f} us over {len(ts)} "
          f"replays; SD(m) draft phase {be.stats['draft_ms'] / n:.3f} ms/step, verify "
          f"{be.stats['verify_ms'] / n:.3f} ms/step")
    be.close()
    del be
    torch.cuda.empty_cache()
