"""Batch-1 query latency split on a cfg3-shaped index: the captured graph alone vs the whole query() call."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2210_15748_b200 as d  # noqa: E402
from paper_2210_15748_b200 import prefilter, workloads  # noqa: E402

dev = torch.device("cuda")
n_sets = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
sizes = workloads.set_sizes(n_sets, 70, 20, seed=500)
off = workloads.offsets(sizes)
X, cents = workloads.gpu_mixture(int(off[-1]), 65536, 128, 0.05, seed=501, dtype=torch.float16, device=dev)
cfg = d.IndexConfig(d=128, C=7, L=32, seed=0,
                    filter=d.FilterConfig(enabled=True, centroids=65536, probe=4, k_filter=4096))
idx = d.build_from_vectors(X, sizes, np.arange(n_sets), cfg)
cvec = cents.double()
cvec = cvec / cvec.norm(dim=1, keepdim=True)
centroids = d.Centroids(k=65536, seed=0, vectors=cvec.cpu().numpy())
idx.filter = (centroids, prefilter.build_centroid_index(X, centroids, set_off=idx.set_off, n_docs=n_sets))
Q = workloads.gpu_queries(X, off, 64, 32, seed=502).cpu()
del X


def pct(v):
    v = np.sort(np.asarray(v)) * 1e3
    return f"p50 {v[len(v) // 2]:.1f} us  p99 {v[int(len(v) * 0.99)]:.1f} us"


for i in range(20):
    d.query(idx, Q[i % 64], 100)
t = []
for i in range(1000):
    t0 = time.perf_counter()
    d.query(idx, Q[i % 64], 100)
    t.append((time.perf_counter() - t0) * 1e3)
print("query()            ", pct(t))
g = next(iter(idx._graphs.values()))
torch.cuda.synchronize()
t = []
for i in range(1000):
    t0 = time.perf_counter()
    g.graph.replay()
    torch.cuda.synchronize()
    t.append((time.perf_counter() - t0) * 1e3)
print("graph replay + sync", pct(t))
ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(200)]
for a, b in ev:
    a.record()
    g.graph.replay()
    b.record()
torch.cuda.synchronize()
print("graph device time  ", pct([a.elapsed_time(b) for a, b in ev][20:]))
