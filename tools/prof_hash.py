"""Time the K1 hash kernel alone on cfg2-shaped bf16/fp16 vectors (CUDA events).

  python tools/prof_hash.py [--n 10000000] [--mode 2] [--dtype bf16] [--reps 10]
DSRT_LIB selects an alternate library build (timing experiments)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2210_15748_b200 as d  # noqa: E402
from paper_2210_15748_b200 import engine, workloads  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=10_000_000)
ap.add_argument("--mode", type=int, default=2)
ap.add_argument("--dtype", default="bf16")
ap.add_argument("--L", type=int, default=64)
ap.add_argument("--C", type=int, default=7)
ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--no-codes", action="store_true", help="records only (no u8 codes output)")
a = ap.parse_args()
dev = torch.device("cuda", 0)
dt = torch.bfloat16 if a.dtype == "bf16" else torch.float16
X, _ = workloads.gpu_mixture(a.n, 4096, 128, 0.05, seed=601, dtype=dt, device=dev)
fam = d.sample_srp_family(128, a.C, a.L, 0)
planes = fam.device_planes(a.mode, dev)
for _ in range(3):
    engine.hash_vectors(X, planes, a.mode, a.L, a.C, want_codes=not a.no_codes, check_zero=False)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(a.reps):
    engine.hash_vectors(X, planes, a.mode, a.L, a.C, want_codes=not a.no_codes, check_zero=False)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / a.reps
fl = 2.0 * 128 * a.L * a.C * a.n
print(f"lib={os.environ.get('DSRT_LIB', 'default')} mode={a.mode} dtype={a.dtype} n={a.n} codes={not a.no_codes} "
      f"ms={ms:.3f} alg_TFLOPs={fl / ms / 1e9:.1f}")
