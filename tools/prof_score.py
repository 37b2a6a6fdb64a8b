"""Small driver for ncu captures of the scoring / top-k / hash kernels.

  python tools/prof_score.py --sets 100000 --qsets 1000 --L 64 --C 7 --reps 2
"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2210_15748_b200 as d  # noqa: E402
from paper_2210_15748_b200 import engine, workloads  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--sets", type=int, default=100_000)
ap.add_argument("--qsets", type=int, default=1000)
ap.add_argument("--L", type=int, default=64)
ap.add_argument("--C", type=int, default=7)
ap.add_argument("--mq", type=int, default=32)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--topk", type=int, default=100)
ap.add_argument("--mode", default="all", choices=["all", "cand"])
ap.add_argument("--cand", type=int, default=0, help="random candidate lists of this length (cfg3-like)")
a = ap.parse_args()
dev = torch.device("cuda")
sizes = workloads.set_sizes(a.sets, 70, 20, seed=1)
off = workloads.offsets(sizes)
g = torch.Generator(device=dev)
g.manual_seed(0)
codes = torch.randint(0, 1 << a.C, (int(off[-1]), a.L), generator=g, device=dev,
                      dtype=torch.int32).to(torch.uint8 if a.C <= 8 else torch.int32)
cfg = d.IndexConfig(d=128, C=a.C, L=a.L, filter=d.FilterConfig(enabled=False))
idx = d.build_from_codes(codes, sizes, np.arange(a.sets), cfg, keep_codes=False)
q = torch.randint(0, 1 << a.C, (a.qsets * a.mq, a.L), generator=g, device=dev, dtype=torch.int32)
qrecs, _ = engine.codes_to_records(q, a.L, a.C)
cand = (torch.randint(0, a.sets, (a.qsets, a.cand), generator=g, device=dev)
        if a.cand else None)
torch.cuda.synchronize()
ev = []
for _ in range(a.reps):
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    if a.mode == "all":
        s, _ = engine.score_all(idx.records, idx.set_off, qrecs, a.mq, a.L, a.C, idx.lut_dev)
    elif a.cand:
        s, _ = engine.score_candidates(idx.records, idx.set_off, qrecs, a.mq, a.L, a.C,
                                       idx.lut_dev, cand=cand)
    else:
        s, _ = engine.score_candidates(idx.records, idx.set_off, qrecs, a.mq, a.L, a.C,
                                       idx.lut_dev, cand_ld=a.sets, n_qsets=a.qsets)
    e1.record()
    ev.append((e0, e1))
    engine.topk(s, a.topk, ids=idx.doc_ids_dev)
torch.cuda.synchronize()
ms = [x.elapsed_time(y) for x, y in ev]
if a.cand:  # compares of the candidate lists actually scored
    sz = torch.from_numpy(np.asarray(sizes)).to(dev)
    comp = a.mq * a.L * int(sz[cand].sum().item())
else:
    comp = a.qsets * a.mq * a.L * int(off[-1])
best = min(ms)
print(f"ok L={a.L} C={a.C} sets={a.sets} qsets={a.qsets} mode={a.mode} QS={os.environ.get('DSRT_QS','auto')} "
      f"ms={best:.3f} Gcmp/s={comp / best / 1e6:.0f} frac={comp / best / 1e6 / 74100:.3f}")
