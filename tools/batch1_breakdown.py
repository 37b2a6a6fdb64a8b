"""Kernel launch list of batch-1 queries on a cfg3-shaped index (run under ncu
--metrics gpu__time_duration.sum)."""
import os
import sys

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
Q = workloads.gpu_queries(X, off, 8, 32, seed=502).cpu()
del X
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
for i in range(8):
    d.query(idx, Q[i], 100)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
