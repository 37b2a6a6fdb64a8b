"""cfg3 batch-256 step: one graph replayed back to back vs two graphs (own buffers) on two streams."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2210_15748_b200 as d  # noqa: E402
from paper_2210_15748_b200 import engine, prefilter, workloads  # noqa: E402

dev = torch.device("cuda")
n_sets, m_q, L, C, top_k, probe, k_filter, n_cent = 1_000_000, 32, 32, 7, 100, 4, 4096, 65536
sizes = workloads.set_sizes(n_sets, 70, 20, seed=500)
off = workloads.offsets(sizes)
X, cents = workloads.gpu_mixture(int(off[-1]), n_cent, 128, 0.05, seed=501, dtype=torch.float16, device=dev)
cfg = d.IndexConfig(d=128, C=C, L=L, seed=0,
                    filter=d.FilterConfig(enabled=True, centroids=n_cent, probe=probe, k_filter=k_filter))
idx = d.build_from_vectors(X, sizes, np.arange(n_sets), cfg, keep_codes=False)
cvec = cents.double()
cvec = cvec / cvec.norm(dim=1, keepdim=True)
centroids = prefilter.Centroids(k=n_cent, seed=0, vectors=cvec.cpu().numpy())
cindex = prefilter.build_centroid_index(X, centroids, set_off=idx.set_off, n_docs=n_sets)
idx.filter = (centroids, cindex)
Qall = workloads.gpu_queries(X, off, 512, m_q, seed=502)
del X
torch.cuda.synchronize()


def make_step(Qb):
    def step():
        Q2 = Qb.reshape(-1, 128)
        _, qrecs = d.lsh.hash_device(idx.family, Q2, want_codes=False, check_zero=False)
        cand, n_cand = prefilter.filter_candidates_device(cindex, centroids, Q2, m_q, probe, k_filter)
        scores, _ = engine.score_candidates(idx.records, idx.set_off, qrecs, m_q, L, C, idx.lut_dev,
                                            cand=cand, n_cand=n_cand)
        return engine.topk(scores, top_k, ids=idx.doc_ids_dev, n_valid=n_cand, id_index=cand)
    return step


steps = [make_step(Qall[:256]), make_step(Qall[256:512])]
for s in steps:
    for _ in range(3):
        s()
torch.cuda.synchronize()
graphs, outs = [], []
for s in steps:
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        outs.append(s())
    graphs.append(g)
torch.cuda.synchronize()
K = 40
main = torch.cuda.current_stream()


def timed(fn):
    for _ in range(5):
        fn(0), fn(1)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(main)
    fn("run")
    e1.record(main)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / K


def serial(arg):
    if arg == "run":
        for t in range(K):
            graphs[t & 1].replay()
    else:
        graphs[arg].replay()


ss = [torch.cuda.Stream(), torch.cuda.Stream()]


def overlapped(arg):
    if arg != "run":
        graphs[arg].replay()
        return
    start = torch.cuda.Event()
    start.record(main)
    for s in ss:
        s.wait_event(start)
    for t in range(K):
        with torch.cuda.stream(ss[t & 1]):
            graphs[t & 1].replay()
    for s in ss:
        e = torch.cuda.Event()
        e.record(s)
        main.wait_event(e)


a = timed(serial)
ref = [o.clone() for g in outs for o in g[:2]]
b = timed(overlapped)
assert all(torch.equal(x, y) for x, y in zip(ref, [o for g in outs for o in g[:2]]))
print(f"serial {a:.4f} ms/step ({256 / a * 1e3:.0f} query sets/s)   two streams {b:.4f} ms/step ({256 / b * 1e3:.0f} query sets/s)")
