import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2210_15748_b200 as d
from paper_2210_15748_b200 import index as I, engine
from oracle import c_oracle, dessert_oracle as O
rng = np.random.default_rng(31)
L, C, N = 16, 3, 6000
sizes = rng.integers(1, 6, size=N)
codes = rng.integers(0, 8, size=(int(sizes.sum()), L)).astype(np.int32)
off = np.concatenate([[0], np.cumsum(sizes)])
ids = rng.permutation(100_000)[:N]
cfg = d.IndexConfig(d=4, C=C, L=L, filter=d.FilterConfig(enabled=False))
idx = d.build_from_codes(torch.from_numpy(codes).to("cuda"), sizes, ids, cfg)
qc = rng.integers(0, 8, size=(2, 5, L))
scores = c_oracle.score(codes.astype(np.int64), off, qc, idx.lookup.table)
qrecs, _ = engine.codes_to_records(torch.from_numpy(qc.reshape(-1, L).astype(np.int32)).cuda(), L, C)
for k in (4097, 5000, 6000, 100, 3000):
    want = [O.rank_topk(scores[r], ids, k) for r in range(2)]
    for buf in (4 << 30, 8 * 2 * 2500, 8 * 2 * 1000):
        s, i, _ = engine.search_all(idx.records, idx.set_off, idx.doc_ids_dev, qrecs, 5, L, C, idx.lut_dev, k, mode=1, score_buffer_bytes=buf)
        got = I._results(s, i)
        for r in range(2):
            if got[r] != want[r]:
                g, w = got[r], want[r]
                bad = [j for j in range(min(len(g), len(w))) if g[j] != w[j]]
                print("k", k, "buf", buf, "row", r, "len", len(g), len(w), "first bad", bad[:5], [g[j] for j in bad[:3]], [w[j] for j in bad[:3]])
            else:
                print("k", k, "buf", buf, "row", r, "ok")
