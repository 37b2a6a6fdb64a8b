"""Generate golden vectors by running the REAL reference package.

Run in the build container (where /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Outputs small .npz fixtures next to this script.  They pin the oracle
(oracle/dessert_oracle.py) and the CUDA path; nothing at test time reads
/root/reference.  Only the public reference API plus its private scoring
helpers (index.py:_score_chunk, sketch.py:accumulate_collisions_batch) are
called; no reference source is copied.
"""

from __future__ import annotations

import importlib.util
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))

import dessert  # noqa: E402  (the reference, via PYTHONPATH)
from dessert import index as ref_index  # noqa: E402
from dessert import prefilter as ref_prefilter  # noqa: E402
from dessert import sketch as ref_sketch  # noqa: E402


def _load_workloads():
    spec = importlib.util.spec_from_file_location(
        "workloads", os.path.join(REPO, "paper_2210_15748_b200", "workloads.py"))
    mod = importlib.util.module_from_spec(spec)
    sys.modules["workloads"] = mod
    spec.loader.exec_module(mod)
    return mod


def no_filter(**kw):
    return dessert.IndexConfig(filter=dessert.FilterConfig(enabled=False), **kw)


def ref_scores(index, qcodes):
    """Reference scores of every set for one code matrix (index.py:250-261)."""
    scorer = index.config.scorer()
    weights = ref_index._resolve_weights(scorer, qcodes.shape[0])
    return np.array(ref_index._score_chunk(index, np.arange(index.n_docs), qcodes, scorer,
                                           weights), dtype=np.float64)


def ref_maxcounts(index, qcodes):
    return np.stack([ref_sketch.accumulate_collisions_batch(t, qcodes).max(axis=1)
                     for t in index.sketches], axis=0)  # (N, m_q)


def make_cfg0():
    wl = _load_workloads()
    sizes, X, Q = wl.cfg0_data(0)
    off = wl.offsets(sizes)
    docs = [(i, X[off[i]:off[i + 1]]) for i in range(len(sizes))]
    index = dessert.build_index(docs, no_filter(d=128, C=6, L=32, seed=0))
    codes = np.concatenate([dessert.hash_matrix(index.family, X[off[i]:off[i + 1]])
                            for i in range(len(sizes))]).astype(np.uint8)
    qcodes = np.stack([dessert.hash_matrix(index.family, q) for q in Q]).astype(np.uint8)
    scores = np.stack([ref_scores(index, qc.astype(np.int64)) for qc in qcodes])
    maxc = np.stack([ref_maxcounts(index, qc.astype(np.int64)) for qc in qcodes]).astype(np.uint8)
    top_ids = np.zeros((len(Q), 10), dtype=np.int64)
    top_sc = np.zeros((len(Q), 10), dtype=np.float64)
    for i, q in enumerate(Q):
        res = dessert.query(index, q, top_k=10)
        top_ids[i] = [d for d, _ in res]
        top_sc[i] = [s for _, s in res]
    np.savez_compressed(os.path.join(HERE, "cfg0.npz"), sizes=sizes, codes=codes, qcodes=qcodes,
                        scores=scores, maxcounts=maxc, top_ids=top_ids, top_scores=top_sc,
                        lut=index.lookup.table, planes_head=index.family.planes[:8])


SMALL_SHAPES = [  # (L, C, m_q, n_sets, m_max)
    (32, 6, 32, 40, 120), (64, 7, 32, 40, 180), (32, 8, 32, 40, 100), (32, 7, 32, 30, 70),
    (16, 3, 5, 30, 40), (8, 2, 200, 20, 30), (64, 7, 1, 20, 50), (24, 4, 7, 25, 60),
    (40, 5, 129, 15, 40), (96, 3, 33, 15, 20), (20, 12, 17, 15, 30), (128, 1, 64, 10, 12),
    (32, 7, 300, 6, 300), (33, 9, 31, 12, 260),
]


def make_small():
    rng = np.random.default_rng(1234)
    out = {}
    for n, (L, C, m_q, n_sets, m_max) in enumerate(SMALL_SHAPES):
        r = 1 << C
        sizes = rng.integers(1, m_max + 1, size=n_sets)
        # bias codes toward a few values so collisions (and ties) are common
        hot = rng.integers(0, r, size=(L,))
        codes = rng.integers(0, r, size=(int(sizes.sum()), L))
        mask = rng.random(codes.shape) < 0.5
        codes[mask] = np.broadcast_to(hot, codes.shape)[mask]
        off = np.concatenate([[0], np.cumsum(sizes)])
        tables = [dessert.build_tiny_table(codes[off[i]:off[i + 1]], L, r) for i in range(n_sets)]
        fam = dessert.sample_srp_family(4, C, L, 0)
        index = ref_index.DessertIndex(config=no_filter(d=4, C=C, L=L), family=fam,
                                       lookup=dessert.build_sim_lookup(C, L), sketches=tables,
                                       doc_ids=rng.permutation(10 * n_sets)[:n_sets].astype(np.uint64),
                                       sizes=sizes.astype(np.int64), filter=None)
        qcodes = rng.integers(0, r, size=(3, m_q, L))
        qm = rng.random(qcodes.shape) < 0.5
        qcodes[qm] = np.broadcast_to(hot, qcodes.shape)[qm]
        scores = np.stack([ref_scores(index, qc) for qc in qcodes])
        maxc = np.stack([ref_maxcounts(index, qc) for qc in qcodes])
        out[f"s{n}_shape"] = np.array([L, C, m_q])
        out[f"s{n}_sizes"] = sizes
        out[f"s{n}_codes"] = codes.astype(np.int32)
        out[f"s{n}_qcodes"] = qcodes.astype(np.int32)
        out[f"s{n}_doc_ids"] = index.doc_ids
        out[f"s{n}_scores"] = scores
        out[f"s{n}_maxcounts"] = maxc.astype(np.int32)
        out[f"s{n}_lut"] = index.lookup.table
        # TinyTables of the first 3 sets (for layout export parity)
        for i in range(3):
            out[f"s{n}_tt{i}_offsets"] = tables[i].offsets
            out[f"s{n}_tt{i}_ids"] = tables[i].ids
    out["n_shapes"] = np.array(len(SMALL_SHAPES))
    np.savez_compressed(os.path.join(HERE, "small.npz"), **out)


def make_end_to_end():
    """Vectors -> build_index -> query, small enough to store the vectors."""
    rng = np.random.default_rng(77)
    out = {}
    cases = [(16, 3, 16, 5, 40, 8, 10), (32, 6, 32, 6, 60, 32, 10), (64, 7, 128, 7, 30, 32, 5),
             (8, 2, 8, 4, 25, 3, 25), (48, 5, 24, 9, 35, 40, 7)]
    for n, (d, C, L, seed, n_sets, m_q, top_k) in enumerate(cases):
        sizes = rng.integers(1, 24, size=n_sets)
        X = rng.standard_normal((int(sizes.sum()), d))
        off = np.concatenate([[0], np.cumsum(sizes)])
        ids = rng.permutation(1000)[:n_sets]
        docs = [(int(ids[i]), X[off[i]:off[i + 1]]) for i in range(n_sets)]
        index = dessert.build_index(docs, no_filter(d=d, C=C, L=L, seed=seed))
        Q = rng.standard_normal((2, m_q, d))
        res = [dessert.query(index, q, top_k=top_k) for q in Q]
        out[f"e{n}_shape"] = np.array([d, C, L, seed, top_k])
        out[f"e{n}_sizes"] = sizes
        out[f"e{n}_X"] = X
        out[f"e{n}_ids"] = ids
        out[f"e{n}_Q"] = Q
        out[f"e{n}_codes"] = dessert.hash_matrix(index.family, X)
        out[f"e{n}_top_ids"] = np.array([[d_ for d_, _ in r] for r in res])
        out[f"e{n}_top_scores"] = np.array([[s for _, s in r] for r in res])
    out["n_cases"] = np.array(len(cases))
    np.savez_compressed(os.path.join(HERE, "end_to_end.npz"), **out)


def make_lsh():
    rng = np.random.default_rng(5)
    fam = dessert.sample_srp_family(128, 6, 32, 0)
    X = rng.standard_normal((256, 128))
    X[:4] = 0.0
    X[0, 0] = 1.0          # axis vectors give exact-zero projections on no plane
    X[1, :] = 1e-3
    X[2, 5] = -2.0
    X[3, 7] = 1e-30        # tiny but non-zero
    luts = {f"lut_{C}_{L}": dessert.build_sim_lookup(C, L).table
            for C in (1, 2, 3, 6, 7, 8, 12, 24) for L in (1, 4, 8, 16, 32, 33, 64, 128)}
    np.savez_compressed(os.path.join(HERE, "lsh.npz"), planes=fam.planes, X=X,
                        codes=dessert.hash_matrix(fam, X),
                        fam2_planes=dessert.sample_srp_family(16, 3, 5, 9).planes, **luts)


def make_prefilter():
    rng = np.random.default_rng(31)
    d, k = 16, 24
    docs = [rng.standard_normal((int(rng.integers(1, 9)), d)) for _ in range(300)]
    cents = ref_prefilter.train_centroids(np.concatenate(docs), k=k, iters=5, seed=3)
    vecs = cents.vectors.copy()
    vecs[5] = vecs[4]      # duplicate centroid: ties must go to the lower id
    cents = ref_prefilter.Centroids(k=k, seed=3, vectors=vecs)
    cindex = ref_prefilter.build_centroid_index(docs, cents)
    out = {"centroids": vecs, "n_docs": np.array(len(docs)),
           "doc_sizes": np.array([len(x) for x in docs]), "docs": np.concatenate(docs)}
    post_off = np.concatenate([[0], np.cumsum([len(p) for p in cindex.postings])])
    out["post_off"] = post_off
    out["post_docs"] = np.concatenate(cindex.postings).astype(np.int64)
    cases = []
    for t in range(24):
        m_q = int(rng.integers(1, 40))
        Q = rng.standard_normal((m_q, d))
        if t % 5 == 0:
            Q[0] = vecs[4] * 3.0   # exact tie between centroid 4 and 5
        probe = int(rng.integers(1, 7))
        k_filter = int(rng.choice([1, 5, 17, 64, 1000]))
        got = ref_prefilter.filter_candidates(cindex, cents, Q, probe, k_filter)
        out[f"q{t}"] = Q
        out[f"r{t}"] = got
        cases.append((probe, k_filter))
    out["cases"] = np.array(cases)
    np.savez_compressed(os.path.join(HERE, "prefilter.npz"), **out)


AGG_SHAPES = [  # (L, C, m_q, n_sets, m_max)
    (32, 6, 32, 20, 120), (64, 7, 40, 16, 300), (16, 3, 5, 20, 200), (8, 2, 70, 12, 260),
    (128, 4, 9, 10, 40), (33, 9, 33, 12, 60),
]


def _agg_scorers(m_q, rng):
    """(name, Scorer) pairs covering every inner kind, with and without weights."""
    from dessert.scoring import Scorer, avg_phi_aggregation, max_aggregation
    w = rng.uniform(0.0, 1.0, size=m_q)
    w[rng.random(m_q) < 0.2] = 0.0
    out = [("max_w", Scorer(inner=max_aggregation(), weights=w))]
    for phi in ("identity", "exp-minus-one", "debiased-sigmoid"):
        out.append((f"{phi}", Scorer(inner=avg_phi_aggregation(phi), weights=None)))
        out.append((f"{phi}_w", Scorer(inner=avg_phi_aggregation(phi), weights=w)))
    return out, w


def make_agg():
    """Scores for every Scorer kind (index.py:183-216) on code-level cases, plus
    query() end to end with avg-phi configs -- row f3."""
    rng = np.random.default_rng(4321)
    out = {}
    for n, (L, C, m_q, n_sets, m_max) in enumerate(AGG_SHAPES):
        r = 1 << C
        sizes = rng.integers(1, m_max + 1, size=n_sets)
        sizes[0] = m_max  # long rows: > 128 non-zero counts for the recursive pairwise split
        hot = rng.integers(0, r, size=(L,))
        codes = rng.integers(0, r, size=(int(sizes.sum()), L))
        mask = rng.random(codes.shape) < 0.6
        codes[mask] = np.broadcast_to(hot, codes.shape)[mask]
        off = np.concatenate([[0], np.cumsum(sizes)])
        tables = [dessert.build_tiny_table(codes[off[i]:off[i + 1]], L, r) for i in range(n_sets)]
        fam = dessert.sample_srp_family(4, C, L, 0)
        index = ref_index.DessertIndex(config=no_filter(d=4, C=C, L=L), family=fam,
                                       lookup=dessert.build_sim_lookup(C, L), sketches=tables,
                                       doc_ids=np.arange(n_sets, dtype=np.uint64),
                                       sizes=sizes.astype(np.int64), filter=None)
        qcodes = rng.integers(0, r, size=(2, m_q, L))
        qm = rng.random(qcodes.shape) < 0.6
        qcodes[qm] = np.broadcast_to(hot, qcodes.shape)[qm]
        scorers, w = _agg_scorers(m_q, rng)
        out[f"a{n}_shape"] = np.array([L, C, m_q])
        out[f"a{n}_sizes"] = sizes
        out[f"a{n}_codes"] = codes.astype(np.int32)
        out[f"a{n}_qcodes"] = qcodes.astype(np.int32)
        out[f"a{n}_weights"] = w
        out[f"a{n}_lut"] = index.lookup.table
        for name, sc in scorers:
            weights = ref_index._resolve_weights(sc, m_q)
            out[f"a{n}_{name}"] = np.stack([
                np.array(ref_index._score_chunk(index, np.arange(n_sets), qc, sc, weights))
                for qc in qcodes])
    out["n_shapes"] = np.array(len(AGG_SHAPES))
    out["scorers"] = np.array([name for name, _ in _agg_scorers(4, rng)[0]])
    # end to end: vectors -> build_index(avg-phi config) -> query
    cases = [(16, 4, 32, 3, 30, 16, 10, "identity"), (32, 6, 32, 5, 40, 20, 8, "exp-minus-one"),
             (24, 5, 64, 7, 25, 33, 6, "debiased-sigmoid")]
    for n, (d, C, L, seed, n_sets, m_q, top_k, phi) in enumerate(cases):
        sizes = rng.integers(1, 30, size=n_sets)
        X = rng.standard_normal((int(sizes.sum()), d))
        off = np.concatenate([[0], np.cumsum(sizes)])
        ids = rng.permutation(500)[:n_sets]
        docs = [(int(ids[i]), X[off[i]:off[i + 1]]) for i in range(n_sets)]
        cfg = dessert.IndexConfig(d=d, C=C, L=L, seed=seed, inner_kind="avg-phi", phi=phi,
                                  filter=dessert.FilterConfig(enabled=False))
        index = dessert.build_index(docs, cfg)
        Q = rng.standard_normal((2, m_q, d))
        res = [dessert.query(index, q, top_k=top_k) for q in Q]
        out[f"e{n}_shape"] = np.array([d, C, L, seed, top_k])
        out[f"e{n}_phi"] = np.array(phi)
        out[f"e{n}_sizes"] = sizes
        out[f"e{n}_X"] = X
        out[f"e{n}_ids"] = ids
        out[f"e{n}_Q"] = Q
        out[f"e{n}_top_ids"] = np.array([[d_ for d_, _ in r_] for r_ in res])
        out[f"e{n}_top_scores"] = np.array([[s_ for _, s_ in r_] for r_ in res])
    out["n_e2e"] = np.array(len(cases))
    np.savez_compressed(os.path.join(HERE, "agg.npz"), **out)


def make_kmeans():
    """train_centroids (prefilter.py:47-82) and a filter-enabled build_index +
    query end to end (index.py:147-157) -- row f4.  Inputs: kmeans_inputs.py."""
    sys.path.insert(0, HERE)
    import kmeans_inputs as KI
    out = {}
    for c, (n, d, k, iters, seed, _) in enumerate(KI.SPECS):
        out[f"k{c}_C"] = ref_prefilter.train_centroids(KI.samples(c), k=k, iters=iters,
                                                       seed=seed).vectors
    sizes, X, ids, Q = KI.e2e_docs()
    off = np.concatenate([[0], np.cumsum(sizes)])
    docs = [(int(ids[i]), X[off[i]:off[i + 1]]) for i in range(len(sizes))]
    cfg = dessert.IndexConfig(d=128, C=6, L=32, seed=11,
                              filter=dessert.FilterConfig(enabled=True, iters=4, probe=3,
                                                          k_filter=40))
    index = dessert.build_index(docs, cfg)
    centroids, cindex = index.filter
    out["e_centroids"] = centroids.vectors
    out["e_post_off"] = np.concatenate([[0], np.cumsum([len(p) for p in cindex.postings])])
    out["e_post_docs"] = np.concatenate(cindex.postings).astype(np.int64)
    res = [dessert.query(index, q, top_k=10) for q in Q]
    out["e_top_ids"] = np.array([[d_ for d_, _ in r_] for r_ in res])
    out["e_top_scores"] = np.array([[s_ for _, s_ in r_] for r_ in res])
    np.savez_compressed(os.path.join(HERE, "kmeans.npz"), **out)


def make_storage():
    """.dsri files written by the reference's save_index (storage.py:130-173) and
    query results of the same indexes -- row f2.  Inputs: storage_inputs.py."""
    import tempfile
    sys.path.insert(0, HERE)
    import storage_inputs as SI
    from dessert import storage as ref_storage
    out = {}
    for name, (d, C, L, seed, inner, phi, fkw, _) in SI.CASES.items():
        filt = dessert.FilterConfig(enabled=fkw is not None, **(fkw or {}))
        cfg = dessert.IndexConfig(d=d, C=C, L=L, seed=seed, inner_kind=inner, phi=phi, filter=filt)
        index = dessert.build_index(SI.docs(name), cfg)
        with tempfile.TemporaryDirectory() as tmp:
            path = os.path.join(tmp, "x.dsri")
            ref_storage.save_index(path, index)
            raw = open(path, "rb").read()
        out[f"{name}_file"] = np.frombuffer(raw, dtype=np.uint8)
        for q, Q in enumerate(SI.queries(name)):
            res = dessert.query(index, Q, top_k=5)
            out[f"{name}_q{q}_ids"] = np.array([x for x, _ in res], dtype=np.int64)
            out[f"{name}_q{q}_scores"] = np.array([v for _, v in res], dtype=np.float64)
    np.savez_compressed(os.path.join(HERE, "storage.npz"), **out)


ENVELOPE_SHAPES = [  # (L, C, m_q, n_sets, m_max): outside the register-blocked kernels
    (32, 20, 32, 12, 40), (160, 5, 16, 10, 30), (40, 24, 8, 10, 25), (256, 3, 33, 8, 20),
    (129, 17, 5, 9, 12)]


def make_envelope():
    """Shapes the reference accepts beyond the fast kernels' register envelope
    (C up to 24, L > 128; lsh.py:17, 54-66), and the prefilter with probe > 32 and
    k_filter > 16384 (prefilter.py:111-144)."""
    rng = np.random.default_rng(4321)
    out = {}
    for n, (L, C, m_q, n_sets, m_max) in enumerate(ENVELOPE_SHAPES):
        r = 1 << C
        sizes = rng.integers(1, m_max + 1, size=n_sets)
        hot = rng.integers(0, r, size=(L,))
        codes = rng.integers(0, r, size=(int(sizes.sum()), L))
        mask = rng.random(codes.shape) < 0.6
        codes[mask] = np.broadcast_to(hot, codes.shape)[mask]
        off = np.concatenate([[0], np.cumsum(sizes)])
        tables = [dessert.build_tiny_table(codes[off[i]:off[i + 1]], L, r) for i in range(n_sets)]
        index = ref_index.DessertIndex(config=no_filter(d=4, C=C, L=L),
                                       family=dessert.sample_srp_family(4, C, L, 0),
                                       lookup=dessert.build_sim_lookup(C, L), sketches=tables,
                                       doc_ids=rng.permutation(10 * n_sets)[:n_sets].astype(np.uint64),
                                       sizes=sizes.astype(np.int64), filter=None)
        qcodes = rng.integers(0, r, size=(3, m_q, L))
        qm = rng.random(qcodes.shape) < 0.6
        qcodes[qm] = np.broadcast_to(hot, qcodes.shape)[qm]
        out[f"s{n}_shape"] = np.array([L, C, m_q])
        out[f"s{n}_sizes"] = sizes
        out[f"s{n}_codes"] = codes.astype(np.int32)
        out[f"s{n}_qcodes"] = qcodes.astype(np.int32)
        out[f"s{n}_doc_ids"] = index.doc_ids
        out[f"s{n}_scores"] = np.stack([ref_scores(index, qc) for qc in qcodes])
    out["n_shapes"] = np.array(len(ENVELOPE_SHAPES))
    # vectors -> build_index -> query at such shapes
    for n, (d, C, L, seed, n_sets, m_q, top_k) in enumerate([(16, 18, 20, 3, 25, 12, 6),
                                                             (24, 4, 200, 5, 20, 20, 8)]):
        sizes = rng.integers(1, 16, size=n_sets)
        X = rng.standard_normal((int(sizes.sum()), d))
        off = np.concatenate([[0], np.cumsum(sizes)])
        ids = rng.permutation(500)[:n_sets]
        index = dessert.build_index([(int(ids[i]), X[off[i]:off[i + 1]]) for i in range(n_sets)],
                                    no_filter(d=d, C=C, L=L, seed=seed))
        Q = rng.standard_normal((2, m_q, d))
        res = [dessert.query(index, q, top_k=top_k) for q in Q]
        out[f"e{n}_shape"] = np.array([d, C, L, seed, top_k])
        out[f"e{n}_sizes"] = sizes
        out[f"e{n}_X"] = X
        out[f"e{n}_ids"] = ids
        out[f"e{n}_Q"] = Q
        out[f"e{n}_top_ids"] = np.array([[d_ for d_, _ in r] for r in res])
        out[f"e{n}_top_scores"] = np.array([[s for _, s in r] for r in res])
    # prefilter: probe > 32 and k_filter > 16384 over 20,000 documents
    d, k = 16, 96
    docs = [rng.standard_normal((int(rng.integers(1, 6)), d)) for _ in range(20000)]
    cents = ref_prefilter.train_centroids(np.concatenate(docs), k=k, iters=3, seed=5)
    cindex = ref_prefilter.build_centroid_index(docs, cents)
    out["pf_centroids"] = cents.vectors
    out["pf_n_docs"] = np.array(len(docs))
    out["pf_post_off"] = np.concatenate([[0], np.cumsum([len(p) for p in cindex.postings])])
    out["pf_post_docs"] = np.concatenate(cindex.postings).astype(np.int64)
    cases = []
    for t, (m_q, probe, k_filter) in enumerate([(32, 40, 20000), (8, 96, 17000), (40, 33, 300),
                                                (32, 4, 18000), (3, 200, 16385)]):
        Q = rng.standard_normal((m_q, d))
        out[f"pf_q{t}"] = Q
        out[f"pf_r{t}"] = ref_prefilter.filter_candidates(cindex, cents, Q, probe, k_filter)
        cases.append((probe, k_filter))
    out["pf_cases"] = np.array(cases)
    np.savez_compressed(os.path.join(HERE, "envelope.npz"), **out)


if __name__ == "__main__":
    assert "reference" in dessert.__file__, dessert.__file__
    makers = {"lsh": make_lsh, "agg": make_agg, "small": make_small, "end_to_end": make_end_to_end,
              "prefilter": make_prefilter, "cfg0": make_cfg0, "kmeans": make_kmeans,
              "storage": make_storage, "envelope": make_envelope}
    for name in (sys.argv[1:] or list(makers)):  # e.g. `make_golden.py agg` for one fixture
        makers[name]()
    print("golden vectors written to", HERE)
    for f in sorted(os.listdir(HERE)):
        print(f, os.path.getsize(os.path.join(HERE, f)))
    sys.exit(0)
