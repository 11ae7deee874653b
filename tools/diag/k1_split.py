import sys
sys.path.insert(0, ".")
import torch
from paper_2603_18016_b200.verify_bench import time_verify
for cached in (False, True):
    r = time_verify(32, 5, 128256, True, iters=10, cached=cached)
    print(cached, r["us"])
