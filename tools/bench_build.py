"""Timing of the index-build "next" rows on one B200, with CPU estimates.

* K7 train_centroids: n samples (cfg-1 mixture, d=128) x k centroids x iters,
  next to one numpy Lloyd iteration on a subsample (oracle restatement),
  extrapolated per (sample, centroid) pair.
* .dsri save_index / load_index of a cfg-1-shaped index (L=64, C=7), next to
  TinyTable construction + serialisation of a set subsample on the host
  (oracle build_tiny_table), extrapolated per set.

    python tools/bench_build.py [--samples 1048576] [--k 1024] [--sets 100000]
"""

import argparse
import json
import os
import sys
import tempfile
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2210_15748_b200 as d  # noqa: E402
from oracle import dessert_oracle as O  # noqa: E402
from paper_2210_15748_b200 import engine, workloads  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--samples", type=int, default=1 << 20)
    ap.add_argument("--k", type=int, default=1024)
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--sets", type=int, default=100_000)
    args = ap.parse_args()
    dev = torch.device("cuda")
    out = {}

    # ---- K7
    X, _ = workloads.gpu_mixture(args.samples, 4096, 128, 0.05, seed=11, dtype=torch.float16,
                                 device=dev)
    S = X.double().contiguous()
    del X
    init = np.random.default_rng(0).choice(args.samples, size=args.k, replace=False)
    engine.train_centroids(S[:65536].contiguous(), 64, 1, init[init < 65536][:64]
                           if (init < 65536).sum() >= 64 else np.arange(64))  # warm-up
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    C = engine.train_centroids(S, args.k, args.iters, init)
    torch.cuda.synchronize()
    t_gpu = time.perf_counter() - t0
    pairs = args.samples * args.k * args.iters
    sub = S[:32768].cpu().numpy()
    Cn = C.cpu().numpy()
    t0 = time.perf_counter()
    Xu = sub / np.linalg.norm(sub, axis=1, keepdims=True)
    sims = Xu @ Cn.T
    a = np.argmax(sims, axis=1)
    sums = np.zeros_like(Cn)
    np.add.at(sums, a, Xu)
    t_cpu = time.perf_counter() - t0
    cpu_rate = sub.shape[0] * args.k / t_cpu
    out["train_centroids"] = {
        "samples": args.samples, "k": args.k, "iters": args.iters, "d": 128,
        "seconds": t_gpu, "pairs_per_s": pairs / t_gpu,
        "cpu_numpy_pairs_per_s": cpu_rate, "cpu_threads": os.cpu_count(),
        "cpu_sample": f"one Lloyd iteration, {sub.shape[0]} samples x {args.k} centroids"}
    del S

    # ---- .dsri
    sizes = workloads.set_sizes(args.sets, 70, 20, seed=100)
    off = workloads.offsets(sizes)
    X, _ = workloads.gpu_mixture(int(off[-1]), 4096, 128, 0.05, seed=200, dtype=torch.float16,
                                 device=dev)
    cfg = d.IndexConfig(d=128, C=7, L=64, seed=0, filter=d.FilterConfig(enabled=False))
    idx = d.build_from_vectors(X, sizes, np.arange(args.sets), cfg, keep_codes=True)
    del X
    with tempfile.TemporaryDirectory() as tmp:
        path = os.path.join(tmp, "i.dsri")
        d.save_index(path, idx)  # warm-up
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        d.save_index(path, idx)
        t_save = time.perf_counter() - t0
        nbytes = os.path.getsize(path)
        d.load_index(path)  # warm-up
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        back = d.load_index(path)
        torch.cuda.synchronize()
        t_load = time.perf_counter() - t0
        same = bool(torch.equal(back.records, idx.records))
    # host reference work for the sets section: build_tiny_table + bytes per set
    codes = idx.codes[: int(off[2000])].cpu().numpy()
    t0 = time.perf_counter()
    for i in range(2000):
        tt = O.build_tiny_table(codes[off[i]:off[i + 1]], 64, 128)
        tt.offsets.tobytes()
        tt.ids.tobytes()
    t_cpu = time.perf_counter() - t0
    out["dsri"] = {
        "sets": args.sets, "bytes": nbytes, "save_s": t_save, "load_s": t_load,
        "save_sets_per_s": args.sets / t_save, "load_sets_per_s": args.sets / t_load,
        "save_GBps": nbytes / t_save / 1e9, "load_GBps": nbytes / t_load / 1e9,
        "round_trip_records_equal": same,
        "cpu_tinytable_sets_per_s": 2000 / t_cpu,
        "cpu_sample": "oracle build_tiny_table + tobytes, 2000 sets, 1 thread"}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
