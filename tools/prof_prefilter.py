"""Isolated prefilter timing / ncu driver: rows = qsets*32 query vectors vs k_c centroids."""
import argparse
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2210_15748_b200 import prefilter as pf  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--qsets", type=int, default=256)
ap.add_argument("--kc", type=int, default=65536)
ap.add_argument("--docs", type=int, default=1_000_000)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--tc", type=int, default=1)
a = ap.parse_args()
dev = torch.device("cuda")
g = torch.Generator(device=dev).manual_seed(0)
C = torch.randn(a.kc, 128, generator=g, device=dev, dtype=torch.float64)
C = C / C.norm(dim=1, keepdim=True)
cents = pf.Centroids(k=a.kc, seed=0, vectors=C.cpu().numpy())
# synthetic postings: each doc in ~4 random postings
n_post = a.docs * 4
cent_of = torch.randint(0, a.kc, (n_post,), generator=g, device=dev).to(torch.int32)
set_off = torch.arange(0, n_post + 1, 4, device=dev, dtype=torch.int64)
from paper_2210_15748_b200 import engine  # noqa: E402
off, docs = engine.postings_from_assign(cent_of, set_off, a.docs, a.kc)
cindex = pf.CentroidIndex(n_docs=a.docs, post_off=off, post_docs=docs)
Q = torch.randn(a.qsets * 32, 128, generator=g, device=dev, dtype=torch.float64)
torch.cuda.synchronize()
for _ in range(a.reps):
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    cand, n = pf.filter_candidates_device(cindex, cents, Q, 32, 4, 4096, use_tc=bool(a.tc))
    e1.record()
    torch.cuda.synchronize()
    print(f"prefilter tc={a.tc} qsets={a.qsets} ms={e0.elapsed_time(e1):.3f}")
