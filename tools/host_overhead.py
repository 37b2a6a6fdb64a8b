"""Wall-clock per call of the public pieces (host overhead check)."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2210_15748_b200 as d  # noqa: E402
from paper_2210_15748_b200 import engine  # noqa: E402

dev = torch.device("cuda")
fam = d.sample_srp_family(128, 7, 32, 0)
for n, dt in ((8192, torch.float16), (32, torch.float16), (32, torch.float64)):
    X = torch.randn(n, 128, device=dev, dtype=dt)
    mode = d.lsh.default_mode(X.dtype, 128, 7, n)
    for check in (False, True):
        for _ in range(5):
            d.lsh.hash_device(fam, X, want_codes=False, check_zero=check)
        torch.cuda.synchronize()
        t = time.perf_counter()
        for _ in range(200):
            d.lsh.hash_device(fam, X, want_codes=False, check_zero=check)
        torch.cuda.synchronize()
        print(f"hash n={n} {dt} mode={mode} check_zero={check}: {1e6 * (time.perf_counter() - t) / 200:.1f} us/call")
s = torch.rand(256, 4096, device=dev, dtype=torch.float64)
for _ in range(5):
    engine.topk(s, 100)
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(200):
    engine.topk(s, 100)
torch.cuda.synchronize()
print(f"topk 256x4096 k=100: {1e6 * (time.perf_counter() - t) / 200:.1f} us/call")
