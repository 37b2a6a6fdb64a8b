"""Time the general aggregation kernel (K3g, dsrt_score_agg) against the
sigma=max fast path on a cfg1-shaped index (L=64, C=7, m_q=32).

    python tools/bench_agg.py [--sets 100000] [--qsets 64]
"""

import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2210_15748_b200 as d  # noqa: E402
from paper_2210_15748_b200 import engine, workloads  # noqa: E402
from paper_2210_15748_b200.index import score_plan  # noqa: E402


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sets", type=int, default=100_000)
    ap.add_argument("--qsets", type=int, default=64)
    args = ap.parse_args()
    dev = torch.device("cuda")
    L, C, m_q = 64, 7, 32
    sizes = workloads.set_sizes(args.sets, 70, 20, seed=100)
    off = workloads.offsets(sizes)
    X, _ = workloads.gpu_mixture(int(off[-1]), 4096, 128, 0.05, seed=200, dtype=torch.float16,
                                 device=dev)
    cfg = d.IndexConfig(d=128, C=C, L=L, seed=0, filter=d.FilterConfig(enabled=False))
    idx = d.build_from_vectors(X, sizes, np.arange(args.sets), cfg)
    Qv = workloads.gpu_queries(X, off, args.qsets, m_q, seed=300)
    del X
    _, qrecs = d.lsh.hash_device(idx.family, Qv.reshape(-1, 128).contiguous())
    pairs = args.qsets * args.sets
    out = {"sets": args.sets, "qsets": args.qsets}
    ms = timed(lambda: engine.score_all(idx.records, idx.set_off, qrecs, m_q, L, C, idx.lut_dev))
    out["max_fast"] = {"ms": ms, "set_pairs_per_s": pairs / ms * 1e3}
    w = np.random.default_rng(0).uniform(0, 1, m_q)
    for name, sc in [("max_weights", d.Scorer(d.max_aggregation(), w)),
                     ("avg_identity", d.Scorer(d.avg_phi_aggregation("identity"))),
                     ("avg_sigmoid_w", d.Scorer(d.avg_phi_aggregation("debiased-sigmoid"), w))]:
        plan = score_plan(idx, sc, m_q)
        f = lambda: engine.score_agg(idx.records, idx.set_off, qrecs, m_q, L, C, plan.table,  # noqa
                                     plan.kind, weights=plan.weights, m_cap=plan.m_cap,
                                     n_qsets=args.qsets, cand_ld=args.sets)
        ms = timed(f)
        out[name] = {"ms": ms, "set_pairs_per_s": pairs / ms * 1e3}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
