"""Where query_batch's host-side time goes on a cfg1-shaped index (eager path: not graphed)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2210_15748_b200 as d  # noqa: E402
from paper_2210_15748_b200 import engine, workloads  # noqa: E402
from paper_2210_15748_b200 import index as I  # noqa: E402
from paper_2210_15748_b200 import lsh  # noqa: E402

dev = torch.device("cuda")
n_sets, n_q, m_q, L, C, top_k = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000, 1000, 32, 64, 7, 100
sizes = workloads.set_sizes(n_sets, 70, 20, seed=100)
off = workloads.offsets(sizes)
X, _ = workloads.gpu_mixture(int(off[-1]), 4096, 128, 0.05, seed=200, dtype=torch.float16, device=dev)
Qv = workloads.gpu_queries(X, off, n_q, m_q, seed=300)
cfg = d.IndexConfig(d=128, C=C, L=L, seed=0, filter=d.FilterConfig(enabled=False))
_, recs = d.lsh.hash_device(d.sample_srp_family(128, C, L, 0), X, want_codes=False)
del X
idx = d.build_from_records(recs, sizes, np.arange(n_sets), cfg)
Qh = Qv.cpu().pin_memory()


def t(fn, n=5):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        r = fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n * 1e3, r


Q2 = Qv.reshape(n_q * m_q, 128).contiguous()
mode = lsh.default_mode(Q2.dtype, 128, C, Q2.shape[0], L)
planes = idx.family.device_planes(mode, dev)
ms, (_, qrecs, _) = t(lambda: engine.hash_vectors(Q2, planes, mode, L, C, want_codes=False, check_zero=False))
print(f"engine.hash_vectors            {ms:8.3f} ms")
ms, _ = t(lambda: engine.search_all(idx.records, idx.set_off, idx.doc_ids_dev, qrecs, m_q, L, C, idx.lut_dev, top_k, mode=0))
print(f"engine.search_all              {ms:8.3f} ms")
ms, _ = t(lambda: lsh.hash_device(idx.family, Q2, want_codes=False))
print(f"lsh.hash_device (check_zero)   {ms:8.3f} ms")
ms, _ = t(lambda: I.rank_records(idx, qrecs, m_q, top_k))
print(f"index.rank_records             {ms:8.3f} ms")
ms, _ = t(lambda: d.query_batch(idx, Qv, top_k, return_tensors=True))
print(f"query_batch (device in/out)    {ms:8.3f} ms")
ms, _ = t(lambda: [x.cpu() for x in d.query_batch(idx, Qh.to(dev, non_blocking=True), top_k, return_tensors=True)])
print(f"query_batch (host in/out)      {ms:8.3f} ms")
