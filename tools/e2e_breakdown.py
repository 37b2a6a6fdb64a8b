"""Host-side breakdown of query_batch on a cfg3-shaped index (stages synchronised)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2210_15748_b200 as d  # noqa: E402
from paper_2210_15748_b200 import index as I, prefilter, workloads  # noqa: E402
from paper_2210_15748_b200.lsh import hash_device, to_device_matrix  # noqa: E402

dev = torch.device("cuda")
n_sets = int(sys.argv[1]) if len(sys.argv) > 1 else 200_000
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
Q = workloads.gpu_queries(X, off, 256, 32, seed=502).cpu().pin_memory()
del X


def sync():
    torch.cuda.synchronize()
    return time.perf_counter()


for it in range(12):
    t0 = sync()
    Qd = Q.to(dev, non_blocking=True)
    t1 = sync()
    t = to_device_matrix(Qd.reshape(-1, 128), 128, dev)
    _, qrecs = hash_device(idx.family, t, want_codes=False)
    t2 = sync()
    cand, n_cand = I._candidates(idx, t, 32, None, None)
    t3 = sync()
    s, i = I.rank_records(idx, qrecs, 32, 100, cand, n_cand)
    t4 = sync()
    hs, hi = s.cpu(), i.cpu()
    t5 = sync()
    if it >= 2:
        print(f"h2d {1e3*(t1-t0):.3f} hash {1e3*(t2-t1):.3f} filter {1e3*(t3-t2):.3f} "
              f"rank {1e3*(t4-t3):.3f} d2h {1e3*(t5-t4):.3f} total {1e3*(t5-t0):.3f} ms")
